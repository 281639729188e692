// Generator-row-sharded single-shot engine: run_single_shot<uint64_t>
// (reference simulator.hpp:46-76) over `world` shards of the tableau, bit-identical to the
// unsharded engine for every world size.
//
// Sharding. Shard r holds generator-words [j0, j0+kg) of both halves (k*r/world ..
// k*(r+1)/world), i.e. destabilizers AND stabilizers g = 64*j0 .. 64*(j0+kg)-1, for all n
// qubits; contiguous blocks, so shard order = generator order. Gate rules act per
// generator-word (gates.hpp:173-194) and S[j] only receives j's contributions, so gate windows
// and both transposes are shard-local: zero communication for ~all of the bytes.
//
// Measurement window (measure.hpp:381-442), per process:
//   flags      local find_probabilistic (CM) -> max-all-reduce (u8 per measurement); the host
//              reads them once per window.
//   collapses  batches of <= 32 flagged measurements (k_batch.cu), enqueued two ahead with no
//              host round trip inside a batch. The reference's pivot is the smallest stabilizer
//              with X at q. Each shard ORs its stabilizers' batch-start bits into a 32-bit mask
//              (all-gather, 4 B per shard); every shard then computes the same plan on the
//              device (k_shard_plan): the leader L = the first shard with bit 0 set holds the
//              global pivot of collapse 0, and a shard d < L has no stabilizer with X at q_m for
//              m < ctz(mask_d), so its rows can neither be pivots nor change before that: L alone
//              computes pivots, pivot rows and coins for m < lim = min(b, min_{d<L} ctz(mask_d)),
//              stopping earlier if it has no candidate. The batch block (V rows + vinfo) then
//              moves by a root-free max-all-reduce: every other shard's block is zero, so no
//              host needs to know L. Every shard absorbs it into its own rows in one pass.
//              No shard with bit 0 => the measurement is deterministic now (measure.hpp:417-421).
//              The host reads each batch's plan one batch behind (pinned copy + event): a batch
//              that ended early makes the speculative one behind it a no-op (device position),
//              and the loop re-plans from there.
//   deterministic  each shard folds its ordered partial product (k_det_partial), the partials of
//              up to 16 measurements are all-gathered together, and every shard folds them in
//              shard order (associativity of the ordered product).
//   record     the leader writes collapse entries; a max-all-reduce of the window's record
//              (zero-initialised everywhere) gives every shard the whole record.
// Coins: the coin index advances only on collapses, in window order, on every shard alike
// (k_batch_member), so each batch's leader draws from the same position.
#include <algorithm>
#include <chrono>
#include <cstring>

#include "abi.hpp"
#include "engine.hpp"
#include "exchange.hpp"

using namespace qsr;

namespace {

void shard_range(uint64_t n, int world, int rank, uint64_t &j0, uint64_t &kg) {
    if (n == 0) fail(QSR_INVALID_ARGUMENT, "shard_range: n must be >= 1");
    const uint64_t k = (n + 63) / 64;
    if (world < 1 || uint64_t(world) > k)
        fail(QSR_INVALID_ARGUMENT, "shard_range: world must be in [1, ceil(n/64)]");
    if (rank < 0 || rank >= world) fail(QSR_INVALID_ARGUMENT, "shard_range: rank out of range");
    j0 = k * uint64_t(rank) / uint64_t(world);
    kg = k * uint64_t(rank + 1) / uint64_t(world) - j0;
}

struct Shard {
    std::unique_ptr<DeviceTableau> t;
    uint64_t j0 = 0;
    qsr_record_entry *d_rec = nullptr;   // whole record (every shard)
    uint32_t *d_masks = nullptr;         // [world] gathered stabilizer OR-masks
    uint32_t *d_plan = nullptr;          // [4] batch plan (k_shard_plan)
    uint64_t *det_send = nullptr;        // [kDetChunk][det_slot_words]
    uint64_t *det_recv = nullptr;        // [world][kDetChunk][det_slot_words]
};

constexpr uint32_t kDetChunk = 16; // deterministic outcomes whose partials share one all-gather

} // namespace

struct qsr_sharded {
    uint64_t n = 0, k = 0;
    uint64_t measure_count = 0;
    int world = 1;
    int device = 0;
    std::vector<Shard> sh;                 // local shards, ascending global rank
    std::unique_ptr<Exchange> ex;
    std::unique_ptr<DeviceSchedule> ds;    // one copy per process (all local shards share a device)
    RunTimes last;
    uint64_t launches = 0;
    uint32_t *h_ctl = nullptr;             // pinned [2][8]: shard 0's plan + block control per slot
    cudaEvent_t bev[2] = {nullptr, nullptr};
    ~qsr_sharded() {
        cudaSetDevice(device);
        for (auto &s : sh) {
            if (s.t) s.t->sync();
            for (void *p : {(void *)s.d_rec, (void *)s.d_masks, (void *)s.d_plan, (void *)s.det_send,
                            (void *)s.det_recv})
                if (p) cudaFree(p);
        }
        if (h_ctl) cudaFreeHost(h_ctl);
        for (auto e : bev)
            if (e) cudaEventDestroy(e);
    }

    // Deterministic outcomes of qubits qs[i] into entries idx[i] of every shard's window record
    // (measure.hpp:343-376): each shard folds its ordered partial product per measurement, one
    // all-gather moves up to kDetChunk of them, and every shard folds the world's partials in
    // shard order (the ordered product is associative).
    void deterministic(const uint32_t *qs, const uint32_t *idx, size_t cnt) {
        const uint64_t sw = det_slot_words(*sh[0].t);
        for (size_t c0 = 0; c0 < cnt; c0 += kDetChunk) {
            const uint32_t c = uint32_t(std::min<size_t>(kDetChunk, cnt - c0));
            std::vector<const void *> send;
            std::vector<void *> recv;
            for (auto &s : sh) {
                for (uint32_t i = 0; i < c; ++i) det_local_partial(*s.t, qs[c0 + i], s.det_send + i * sw);
                send.push_back(s.det_send);
                recv.push_back(s.det_recv);
            }
            ex->allgather(send, recv, c * sw * 8);
            for (auto &s : sh)
                for (uint32_t i = 0; i < c; ++i)
                    det_combine(*s.t, qs[c0 + i], s.det_recv + i * sw, uint32_t(world), s.t->ms.out + idx[c0 + i],
                                c * sw);
        }
    }

    // One batch of <= kMaxBatch flagged measurements starting at `start` (speculatively: it is a
    // no-op unless every shard's device position equals `start` when it runs), with no host
    // round trip: column bits and stabilizer masks -> all-gather -> the plan on every shard ->
    // the leader's pivots -> a root-free max-all-reduce of the batch block (the others' blocks
    // are zero) -> every shard absorbs. Shard 0's plan and block control are copied to pinned
    // slot `slot` for the host, which reads them one batch behind.
    void enqueue_batch(size_t start, uint32_t b, uint64_t seed, int slot) {
        std::vector<const void *> msend;
        std::vector<void *> mrecv, blocks;
        for (auto &s : sh) {
            batch_colbits(*s.t, s.t->ms.fq + start, b, /*zero_block=*/true);
            msend.push_back(s.t->ms.bctl + 2);
            mrecv.push_back(s.d_masks);
            blocks.push_back(s.t->ms.batch_block);
        }
        ex->allgather(msend, mrecv, 4);
        for (size_t i = 0; i < sh.size(); ++i) {
            DeviceTableau &t = *sh[i].t;
            shard_plan(t, sh[i].d_masks, world, ex->ranks[i], b, uint32_t(start), sh[i].d_plan);
            batch_pivots(t, t.ms.fq + start, t.ms.fidx + start, b, seed, nullptr, 0, sh[i].d_plan);
        }
        ex->allreduce_max_u64(blocks, sh[0].t->ms.batch_block_bytes / 8);
        for (auto &s : sh) batch_apply(*s.t);
        DeviceTableau &t0 = *sh[0].t;
        QSR_CUDA(cudaMemcpyAsync(h_ctl + 8 * slot, sh[0].d_plan, 16, cudaMemcpyDeviceToHost, t0.stream));
        QSR_CUDA(cudaMemcpyAsync(h_ctl + 8 * slot + 4, t0.ms.bctl, 16, cudaMemcpyDeviceToHost, t0.stream));
        QSR_CUDA(cudaEventRecord(bev[slot], t0.stream));
    }

    void set_position(uint32_t pos) {
        for (auto &s : sh) set_device_u32(s.t->ms.d_pos, pos, s.t->stream);
    }

    void measure_window(const std::vector<uint32_t> &mq, uint64_t seed, RunTimes &rt) {
        const uint64_t m = mq.size();
        DeviceTableau &t0 = *sh[0].t;
        cudaEvent_t ev[4];
        for (auto &e : ev) QSR_CUDA(cudaEventCreate(&e));
        std::vector<void *> flag_bufs, out_bufs;
        for (auto &s : sh) {
            DeviceTableau &t = *s.t;
            t.ensure_window_cap(m);
            QSR_CUDA(cudaMemcpyAsync(t.ms.mqubits, mq.data(), m * 4, cudaMemcpyHostToDevice, t.stream));
            QSR_CUDA(cudaMemsetAsync(t.ms.out, 0, m * sizeof(qsr_record_entry), t.stream));
            flags_cm(t, m);
            flag_bufs.push_back(t.ms.flags);
            out_bufs.push_back(t.ms.out);
        }
        ex->allreduce_max_u8(flag_bufs, m);
        std::vector<uint8_t> flags(m);
        QSR_CUDA(cudaMemcpyAsync(flags.data(), t0.ms.flags, m, cudaMemcpyDeviceToHost, t0.stream));
        QSR_CUDA(cudaEventRecord(ev[0], t0.stream));
        for (auto &s : sh) transpose_to_rm(*s.t);
        QSR_CUDA(cudaEventRecord(ev[1], t0.stream));
        QSR_CUDA(cudaStreamSynchronize(t0.stream)); // flags (once per window)

        std::vector<uint32_t> fq, fidx;
        for (uint64_t i = 0; i < m; ++i)
            if (flags[i]) { fq.push_back(mq[i]); fidx.push_back(uint32_t(i)); }
        if (!fq.empty())
            for (auto &s : sh) {
                DeviceTableau &t = *s.t;
                QSR_CUDA(cudaMemcpyAsync(t.ms.fq, fq.data(), fq.size() * 4, cudaMemcpyHostToDevice, t.stream));
                QSR_CUDA(cudaMemcpyAsync(t.ms.fidx, fidx.data(), fidx.size() * 4, cudaMemcpyHostToDevice,
                                         t.stream));
            }
        // Collapses in window order (measure.hpp:409-431), two batches in flight: batch k + 1 is
        // enqueued (assuming batch k collapses all its measurements) before the host looks at
        // batch k, so the devices never wait for the host.
        struct Pending { size_t start; uint32_t b; int slot; };
        Pending queue[2];
        int qhead = 0, qsize = 0, slot = 0;
        size_t pos = 0, spec = 0;
        set_position(0);
        auto drain = [&] {
            while (qsize) {
                QSR_CUDA(cudaEventSynchronize(bev[queue[qhead].slot]));
                qhead = (qhead + 1) % 2;
                --qsize;
            }
        };
        while (pos < fq.size()) {
            while (qsize < 2 && spec < fq.size()) {
                const uint32_t b = uint32_t(std::min<size_t>(kMaxBatch, fq.size() - spec));
                enqueue_batch(spec, b, seed, slot);
                queue[(qhead + qsize) % 2] = Pending{spec, b, slot};
                ++qsize;
                slot ^= 1;
                spec += b;
            }
            const Pending p = queue[qhead];
            qhead = (qhead + 1) % 2;
            --qsize;
            QSR_CUDA(cudaEventSynchronize(bev[p.slot]));
            const uint32_t *plan = h_ctl + 8 * p.slot, *bctl = plan + 4;
            if (plan[3]) continue; // skipped: behind a batch that ended early
            if (plan[2]) {         // no stabilizer anywhere anticommutes with Z_q: deterministic now
                drain();           // (measure.hpp:417-421)
                deterministic(&fq[p.start], &fidx[p.start], 1);
                pos = p.start + 1;
                set_position(uint32_t(pos));
                spec = pos;
                continue;
            }
            const uint32_t len = bctl[0];
            if (len == 0) fail(QSR_INTERNAL, "sharded measure: leader found no pivot");
            pos = p.start + len;
            if (len < p.b) { // ended early (another shard holds a later pivot): re-plan from pos
                drain();
                spec = pos;
            }
        }
        drain();
        // Deterministic outcomes of the unflagged measurements (measure.hpp:432-438), batched.
        std::vector<uint32_t> dq, didx;
        for (uint64_t i = 0; i < m; ++i)
            if (!flags[i]) { dq.push_back(mq[i]); didx.push_back(uint32_t(i)); }
        if (!dq.empty()) deterministic(dq.data(), didx.data(), dq.size());
        ex->allreduce_max_u8(out_bufs, m * sizeof(qsr_record_entry));
        QSR_CUDA(cudaEventRecord(ev[2], t0.stream));
        for (auto &s : sh) transpose_to_cm(*s.t);
        QSR_CUDA(cudaEventRecord(ev[3], t0.stream));
        QSR_CUDA(cudaEventSynchronize(ev[3]));
        float a = 0, b2 = 0, c = 0;
        QSR_CUDA(cudaEventElapsedTime(&a, ev[0], ev[1]));
        QSR_CUDA(cudaEventElapsedTime(&b2, ev[1], ev[2]));
        QSR_CUDA(cudaEventElapsedTime(&c, ev[2], ev[3]));
        rt.t_ms += a + c;
        rt.ge_ms += b2;
        for (auto &e : ev) cudaEventDestroy(e);
    }

    void run(uint64_t seed) {
        QSR_CUDA(cudaSetDevice(device));
        RunTimes rt;
        DeviceTableau &t0 = *sh[0].t;
        cudaEvent_t e_start, e_end, a, b;
        for (auto *e : {&e_start, &e_end, &a, &b}) QSR_CUDA(cudaEventCreate(e));
        for (auto &s : sh) {
            s.t->sync();
            launch_zero_state(*s.t, nullptr);
        }
        for (auto &s : sh) QSR_CUDA(cudaMemsetAsync(s.t->ms.coin_index, 0, 8, s.t->stream));
        QSR_CUDA(cudaEventRecord(e_start, t0.stream));
        uint64_t rec_off = 0;
        const uint64_t W = ds->is_meas.size();
        uint64_t w = 0;
        while (w < W) {
            if (!ds->is_meas[w]) {
                QSR_CUDA(cudaEventRecord(a, t0.stream));
                const uint64_t w0 = w;
                while (w < W && !ds->is_meas[w]) ++w;
                for (auto &s : sh) rt.gate_launches += run_unitary_windows(*s.t, *ds, w0, w, &rt.gate_bytes);
                // Shard 0's stream waits for the others so the event pair brackets all shards.
                for (size_t i = 1; i < sh.size(); ++i) {
                    QSR_CUDA(cudaEventRecord(b, sh[i].t->stream));
                    QSR_CUDA(cudaStreamWaitEvent(t0.stream, b, 0));
                }
                QSR_CUDA(cudaEventRecord(b, t0.stream));
                QSR_CUDA(cudaEventSynchronize(b));
                float ms = 0;
                QSR_CUDA(cudaEventElapsedTime(&ms, a, b));
                rt.to_ms += ms;
                continue;
            }
            if (const uint32_t *perm = ds->perm_before(w))
                for (auto &s : sh) launch_unpermute_rows(*s.t, perm);
            const auto &mq = ds->mqubits[w];
            measure_window(mq, seed, rt);
            for (auto &s : sh)
                QSR_CUDA(cudaMemcpyAsync(s.d_rec + rec_off, s.t->ms.out, mq.size() * sizeof(qsr_record_entry),
                                         cudaMemcpyDeviceToDevice, s.t->stream));
            rec_off += mq.size();
            ++w;
        }
        // Gate fusion (fuse.hpp): rows back to logical order.
        if (const uint32_t *perm = ds->perm_before(W))
            for (auto &s : sh) launch_unpermute_rows(*s.t, perm);
        for (size_t i = 1; i < sh.size(); ++i) {
            QSR_CUDA(cudaEventRecord(b, sh[i].t->stream));
            QSR_CUDA(cudaStreamWaitEvent(t0.stream, b, 0));
        }
        QSR_CUDA(cudaEventRecord(e_end, t0.stream));
        QSR_CUDA(cudaEventSynchronize(e_end));
        float total = 0;
        QSR_CUDA(cudaEventElapsedTime(&total, e_start, e_end));
        rt.total_ms = total;
        for (auto e : {e_start, e_end, a, b}) cudaEventDestroy(e);
        for (auto &s : sh)
            if (read_error_flag(*s.t))
                fail(QSR_LOGIC_ERROR, "product of anti-commuting rows (corrupted tableau)");
        last = rt;
    }
};

extern "C" {

qsr_status qsr_shard_range(uint64_t n, int world, int rank, uint64_t *j0, uint64_t *kg) {
    return guard([&] {
        REQUIRE_PTR(j0);
        REQUIRE_PTR(kg);
        shard_range(n, world, rank, *j0, *kg);
    });
}

qsr_status qsr_nccl_unique_id(uint8_t out[128]) {
    return guard([&] {
        REQUIRE_PTR(out);
        nccl_unique_id(out);
    });
}

} // extern "C"

namespace {
// Shards of this process + the exchange; with `circ` set, also the device-resident (fused)
// schedule of the resident engine.
std::unique_ptr<qsr_sharded> make_sharded(const Circuit &circ, const qsr_schedule *s, const qsr_shard_config *cfg,
                                          bool resident) {
    auto e = std::make_unique<qsr_sharded>();
    e->n = circ.num_qubits;
    e->world = cfg->world;
    e->device = cfg->device;
    if (e->n == 0) fail(QSR_INVALID_ARGUMENT, "Tableau: n must be >= 1");
    e->k = (e->n + 63) / 64;
    if (cfg->world < 1 || uint64_t(cfg->world) > e->k)
        fail(QSR_INVALID_ARGUMENT, "sharded: world must be in [1, ceil(n/64)]");
    std::vector<int> my_ranks;
    if (cfg->exchange == QSR_EXCHANGE_LOCAL) {
        for (int r = 0; r < cfg->world; ++r) my_ranks.push_back(r);
    } else if (cfg->exchange == QSR_EXCHANGE_NCCL) {
        REQUIRE_PTR(cfg->nccl_id);
        my_ranks.push_back(cfg->rank);
    } else {
        fail(QSR_INVALID_ARGUMENT, "sharded: unknown exchange");
    }
    QSR_CUDA(cudaSetDevice(cfg->device));
    std::vector<cudaStream_t> streams;
    for (int r : my_ranks) {
        uint64_t j0 = 0, kg = 0;
        shard_range(e->n, cfg->world, r, j0, kg);
        Shard sd;
        sd.j0 = j0;
        sd.t = std::make_unique<DeviceTableau>(e->n, cfg->device, j0, kg);
        streams.push_back(sd.t->stream);
        e->sh.push_back(std::move(sd));
    }
    e->measure_count = circ.measure_count();
    if (resident) {
        e->ds = s ? upload_schedule(e->n, *s, cfg->device, e->sh[0].t->stream, true)
                  : upload_circuit(circ, cfg->device, e->sh[0].t->stream, true);
        if (e->ds->measure_count != e->measure_count)
            fail(QSR_INVALID_ARGUMENT, "schedule does not match the circuit's measurement count");
    }
    const uint64_t nm = std::max<uint64_t>(e->measure_count, 1);
    for (auto &sd : e->sh) {
        const uint64_t sw = det_slot_words(*sd.t);
        QSR_CUDA(cudaMalloc(&sd.d_rec, nm * sizeof(qsr_record_entry)));
        QSR_CUDA(cudaMalloc(&sd.d_masks, 4 * size_t(cfg->world)));
        QSR_CUDA(cudaMalloc(&sd.d_plan, 16));
        QSR_CUDA(cudaMalloc(&sd.det_send, kDetChunk * sw * 8));
        QSR_CUDA(cudaMemset(sd.det_send, 0, kDetChunk * sw * 8));
        QSR_CUDA(cudaMalloc(&sd.det_recv, kDetChunk * sw * 8 * size_t(cfg->world)));
    }
    QSR_CUDA(cudaMallocHost(&e->h_ctl, 2 * 8 * sizeof(uint32_t)));
    for (auto &ev : e->bev) QSR_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    if (cfg->exchange == QSR_EXCHANGE_LOCAL)
        e->ex = make_local_exchange(cfg->world, streams);
    else
        e->ex = make_nccl_exchange(cfg->world, cfg->rank, streams[0], cfg->nccl_id);
    QSR_CUDA(cudaDeviceSynchronize());
    return e;
}

// The streamed driver (stream.cpp) on this process's one shard, with the sharded protocol for
// every measurement window.
struct ShardMeasure final : MeasureHook {
    qsr_sharded &e;
    explicit ShardMeasure(qsr_sharded &ee) : e(ee) {}
    void measure(const std::vector<uint32_t> &qubits, uint64_t seed, RunTimes &rt) override {
        e.measure_window(qubits, seed, rt);
    }
};
} // namespace

extern "C" {

qsr_status qsr_sharded_create(const qsr_circuit *c, const qsr_schedule *s,
                              const qsr_shard_config *cfg, qsr_sharded **out) {
    return guard([&] {
        REQUIRE_PTR(c);
        REQUIRE_PTR(cfg);
        REQUIRE_PTR(out);
        *out = make_sharded(*c, s, cfg, /*resident=*/true).release();
    });
}

qsr_status qsr_sharded_run_circuit(const qsr_circuit *c, const qsr_shard_config *cfg, uint64_t seed,
                                   qsr_record_entry *record, qsr_sharded **out, double *device_ms) {
    return guard([&] {
        REQUIRE_PTR(c);
        REQUIRE_PTR(cfg);
        REQUIRE_PTR(out);
        const Circuit &circ = *c;
        auto e = make_sharded(circ, nullptr, cfg, /*resident=*/false);
        if (e->sh.size() != 1)
            fail(QSR_INVALID_ARGUMENT, "sharded streamed run: one shard per process (NCCL exchange, or world 1)");
        Shard &sd = e->sh[0];
        RunTimes rt;
        StreamCounts sc;
        ShardMeasure hook(*e);
        run_circuit_streaming(*sd.t, circ, seed, sd.d_rec, rt, sc, nullptr, &hook);
        e->last = rt;
        if (e->measure_count) {
            REQUIRE_PTR(record);
            QSR_CUDA(cudaMemcpyAsync(record, sd.d_rec, e->measure_count * sizeof(qsr_record_entry),
                                     cudaMemcpyDeviceToHost, sd.t->stream));
        }
        sd.t->sync();
        if (device_ms) *device_ms = rt.total_ms;
        *out = e.release();
    });
}

qsr_status qsr_sharded_run(qsr_sharded *e, uint64_t seed, double *device_ms) {
    return guard([&] {
        REQUIRE_PTR(e);
        if (!e->ds) fail(QSR_INVALID_ARGUMENT, "sharded: no resident schedule (object of qsr_sharded_run_circuit)");
        const uint64_t l0 = g_launches;
        e->run(seed);
        e->launches = g_launches - l0;
        if (device_ms) *device_ms = e->last.total_ms;
    });
}

qsr_status qsr_sharded_stats(const qsr_sharded *e, double *gate_ms, uint64_t *gate_launches,
                             double *transpose_ms, double *measure_ms, uint64_t *launches) {
    return guard([&] {
        REQUIRE_PTR(e);
        if (gate_ms) *gate_ms = e->last.to_ms;
        if (gate_launches) *gate_launches = e->last.gate_launches;
        if (transpose_ms) *transpose_ms = e->last.t_ms;
        if (measure_ms) *measure_ms = e->last.ge_ms + e->last.cmp_ms;
        if (launches) *launches = e->launches;
    });
}

qsr_status qsr_sharded_gate_bytes(const qsr_sharded *e, double *bytes) {
    return guard([&] {
        REQUIRE_PTR(e);
        REQUIRE_PTR(bytes);
        *bytes = e->last.gate_bytes;
    });
}

qsr_status qsr_sharded_record(const qsr_sharded *e, qsr_record_entry *record) {
    return guard([&] {
        REQUIRE_PTR(e);
        const uint64_t nm = e->measure_count;
        if (!nm) return;
        REQUIRE_PTR(record);
        QSR_CUDA(cudaSetDevice(e->device));
        const Shard &s = e->sh[0];
        QSR_CUDA(cudaMemcpyAsync(record, s.d_rec, nm * sizeof(qsr_record_entry), cudaMemcpyDeviceToHost,
                                 s.t->stream));
        s.t->sync();
    });
}

qsr_status qsr_sharded_tableau_local(const qsr_sharded *e, uint64_t *x, uint64_t *z, uint64_t *s) {
    return guard([&] {
        REQUIRE_PTR(e);
        QSR_CUDA(cudaSetDevice(e->device));
        const uint64_t n_pad = 64 * e->k;
        uint64_t xo = 0, so = 0;
        for (const Shard &sd : e->sh) {
            DeviceTableau &t = *sd.t;
            if (t.layout != QSR_COLUMN_MAJOR) fail(QSR_INTERNAL, "sharded tableau not ColumnMajor");
            const uint64_t w = 2 * t.kg; // destabilizer words then stabilizer words of this shard
            if (x) QSR_CUDA(cudaMemcpy2DAsync(x + xo, w * 8, t.x, t.cm_pitch * 8, w * 8, n_pad,
                                              cudaMemcpyDeviceToHost, t.stream));
            if (z) QSR_CUDA(cudaMemcpy2DAsync(z + xo, w * 8, t.z, t.cm_pitch * 8, w * 8, n_pad,
                                              cudaMemcpyDeviceToHost, t.stream));
            if (s) QSR_CUDA(cudaMemcpyAsync(s + so, t.s, w * 8, cudaMemcpyDeviceToHost, t.stream));
            xo += n_pad * w;
            so += w;
            t.sync();
        }
    });
}

qsr_status qsr_sharded_tableau(const qsr_sharded *e, uint64_t *x, uint64_t *z, uint64_t *s) {
    return guard([&] {
        REQUIRE_PTR(e);
        QSR_CUDA(cudaSetDevice(e->device));
        const uint64_t k = e->k, n_pad = 64 * k;
        for (const Shard &sd : e->sh) {
            DeviceTableau &t = *sd.t;
            if (t.layout != QSR_COLUMN_MAJOR) fail(QSR_INTERNAL, "sharded tableau not ColumnMajor");
            // Destabilizer words j0.. and stabilizer words k+j0.. of every qubit row.
            for (int plane = 0; plane < 2; ++plane) {
                uint64_t *dst = plane ? z : x;
                const uint64_t *src = plane ? t.z : t.x;
                if (!dst) continue;
                QSR_CUDA(cudaMemcpy2DAsync(dst + sd.j0, 2 * k * 8, src, t.cm_pitch * 8, t.kg * 8, n_pad,
                                           cudaMemcpyDeviceToHost, t.stream));
                QSR_CUDA(cudaMemcpy2DAsync(dst + k + sd.j0, 2 * k * 8, src + t.kg, t.cm_pitch * 8,
                                           t.kg * 8, n_pad, cudaMemcpyDeviceToHost, t.stream));
            }
            if (s) {
                QSR_CUDA(cudaMemcpyAsync(s + sd.j0, t.s, t.kg * 8, cudaMemcpyDeviceToHost, t.stream));
                QSR_CUDA(cudaMemcpyAsync(s + k + sd.j0, t.s + t.kg, t.kg * 8, cudaMemcpyDeviceToHost,
                                         t.stream));
            }
            t.sync();
        }
    });
}

void qsr_sharded_destroy(qsr_sharded *e) { delete e; }

} // extern "C"
