// Streaming single-shot driver: run_single_shot (reference simulator.hpp:46-76) on a Circuit with
// the window scheduler (schedule.hpp:51-137, one-pass closed form of host_circuit.cpp) running on
// the host WHILE the device executes the windows that are already final.
//
// Why windows become final early. The scheduler assigns key = 2*round + is_measure with
//   round(U) = 1 + max round(previous gate on its wires),  round(M) = max(1, round(prev on wire)),
// and emits windows in key order. After the first i gates, let R = min over all wires of the
// round of the wire's last gate. Every later unitary gate has round >= R + 1 (key >= 2R + 2) and
// every later measurement round >= R (key >= 2R + 1), so all windows with key < 2R + 1 already
// hold every gate they will ever hold, in circuit index order. The driver plans the circuit in
// chunks, and after each chunk uploads and launches the newly final windows, so planning (a
// serial pass of ~6 ns/gate on the host) hides behind the gate kernels.
//
// The result is identical to scheduling first and running after: same windows, same order, same
// coin sequence. Errors the reference raises while scheduling (check_valid, a measurement chained
// behind another in one window, measure.hpp:394-395) are raised when the offending gate is
// planned; the tableau being built is then discarded, so no caller-visible state was mutated.
#include <algorithm>
#include <thread>
#include <map>
#include <mutex>
#include <exception>
#include <condition_variable>
#include <array>
#include <chrono>
#include <cstring>

#include "engine.hpp"
#include "fuse.hpp"
#include "stream_plan.hpp"

namespace qsr {

namespace {

constexpr uint64_t kPlanChunk = uint64_t(1) << 22;  // gates planned between emissions
constexpr uint64_t kRingGates = uint64_t(1) << 21;  // pinned staging per slot (16 MB)

struct PinnedRing {
    uint64_t *buf[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    bool used[2] = {false, false};
    int cur = 0;
    uint64_t fill = 0;
    PinnedRing() {
        for (int i = 0; i < 2; ++i) {
            QSR_CUDA(cudaMallocHost(&buf[i], kRingGates * 8));
            QSR_CUDA(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
        }
    }
    void reset() { // the previous call's copies have completed; start from slot 0, empty
        for (int i = 0; i < 2; ++i) {
            if (used[i]) QSR_CUDA(cudaEventSynchronize(done[i]));
            used[i] = false;
        }
        cur = 0;
        fill = 0;
    }
    ~PinnedRing() {
        for (int i = 0; i < 2; ++i) {
            if (done[i]) cudaEventSynchronize(done[i]), cudaEventDestroy(done[i]);
            if (buf[i]) cudaFreeHost(buf[i]);
        }
    }
};

} // namespace

void run_circuit_streaming(DeviceTableau &t, const Circuit &c, uint64_t seed,
                           qsr_record_entry *d_record, RunTimes &rt, StreamCounts &counts,
                           FramesSink *frames, MeasureHook *measure_hook) {
    const uint64_t G = c.gates.size();
    const uint32_t n = c.num_qubits;
    t.ensure_gate_buf(std::max<uint64_t>(G, 1));
    uint64_t *d_gates = t.gate_buf;
    // One ring per (host thread, device): its events belong to the device whose stream records
    // them, and every call starts from an empty ring.
    static thread_local std::map<int, std::unique_ptr<PinnedRing>> rings;
    std::unique_ptr<PinnedRing> &ring_store = rings[t.device];
    if (!ring_store) {
        QSR_CUDA(cudaSetDevice(t.device));
        ring_store = std::make_unique<PinnedRing>();
    }
    PinnedRing &ring = *ring_store;
    ring.reset();
    using clk = std::chrono::steady_clock;
    auto since = [](clk::time_point a) { return std::chrono::duration<double, std::milli>(clk::now() - a).count(); };

    cudaEvent_t e_start, e_end;
    QSR_CUDA(cudaEventCreate(&e_start));
    QSR_CUDA(cudaEventCreate(&e_end));
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> to_events; // unitary runs (TO bucket)
    QSR_CUDA(cudaEventRecord(e_start, t.stream));
    launch_zero_state(t, nullptr);
    QSR_CUDA(cudaMemsetAsync(t.ms.coin_index, 0, 8, t.stream));

    // Keys are 2*round + is_measure with round <= gates on the wire + 1 <= G + 1.
    BucketDir buckets(2 * G + 4);
    std::mutex pool_mu;
    std::vector<std::vector<uint64_t>> pool; // emptied buckets keep their capacity
    auto fresh_bucket = [&](std::vector<uint64_t> &b) {
        {
            std::lock_guard<std::mutex> g(pool_mu);
            if (!pool.empty()) {
                b.swap(pool.back());
                pool.pop_back();
                return;
            }
        }
        b.reserve(size_t(n) * 3 / 4 + 16);
    };

    // ---- emitter: fuse, stage and launch every final window, in key order ------------------
    std::mutex mu;
    std::condition_variable cv;
    uint64_t limit = 2;       // keys below are final (guarded by mu)
    bool done = false;        // the planner has published its last limit (guarded by mu)
    bool stop = false;        // planner failed: emitter quits
    std::exception_ptr emit_error;
    double t_fuse = 0, t_stage = 0, t_ringwait = 0, t_meas = 0, t_plan = 0;

    auto emitter = [&] {
        try {
            QSR_CUDA(cudaSetDevice(t.device));
            const bool fuse = fusion_enabled();
            Fuser fuser(fuse ? n : 0);
            WordVec dev; // device gates of the window being emitted
            std::vector<uint8_t> flags;
            std::vector<uint32_t> mq;
            uint64_t next_key = 2, dev_off = 0, rec_off = 0;
            uint32_t *d_perm = nullptr;
            cudaEvent_t ra = nullptr, rb = nullptr;
            bool in_run = false;
            auto open_run = [&] {
                if (in_run) return;
                QSR_CUDA(cudaEventCreate(&ra));
                QSR_CUDA(cudaEventCreate(&rb));
                QSR_CUDA(cudaEventRecord(ra, t.stream));
                in_run = true;
            };
            auto close_run = [&] {
                if (!in_run) return;
                QSR_CUDA(cudaEventRecord(rb, t.stream));
                to_events.emplace_back(ra, rb);
                in_run = false;
            };
            // Stage one device window through the pinned ring (async H2D) and launch it. The device
            // gate buffer is used as a ring too: copies and kernels share t.stream, so a copy
            // into a recycled region runs after every kernel that read it.
            auto launch_staged = [&](const uint64_t *src, uint64_t cnt) {
                const auto ts = clk::now();
                open_run();
                if (dev_off + cnt > t.gate_buf_cap) dev_off = 0;
                for (uint64_t i = 0; i < cnt;) {
                    if (ring.fill == kRingGates) {
                        QSR_CUDA(cudaEventRecord(ring.done[ring.cur], t.stream));
                        ring.used[ring.cur] = true;
                        ring.cur ^= 1;
                        ring.fill = 0;
                        if (ring.used[ring.cur]) {
                            const auto tw = clk::now();
                            QSR_CUDA(cudaEventSynchronize(ring.done[ring.cur]));
                            t_ringwait += since(tw);
                        }
                    }
                    const uint64_t take = std::min(cnt - i, kRingGates - ring.fill);
                    uint64_t *dst = ring.buf[ring.cur] + ring.fill;
                    std::memcpy(dst, src + i, take * 8);
                    QSR_CUDA(cudaMemcpyAsync(d_gates + dev_off + i, dst, take * 8, cudaMemcpyHostToDevice,
                                             t.stream));
                    ring.fill += take;
                    i += take;
                }
                launch_gate_window(t, d_gates + dev_off, cnt);
                if (frames) frames->unitary(d_gates + dev_off, cnt, t.stream);
                ++rt.gate_launches;
                dev_off += cnt;
                t_stage += since(ts);
            };
            auto unitary_window = [&](WordVec &w) {
                if (!w.empty()) launch_staged(w.data(), w.size());
            };
            // CM rows back to logical order (before a measurement window and at the end).
            auto unpermute = [&] {
                if (!fuse || fuser.identity_permutation()) return;
                if (!d_perm) QSR_CUDA(cudaMalloc(&d_perm, uint64_t(n) * 4));
                const std::vector<uint32_t> pm = fuser.permutation();
                QSR_CUDA(cudaMemcpyAsync(d_perm, pm.data(), uint64_t(n) * 4, cudaMemcpyHostToDevice, t.stream));
                QSR_CUDA(cudaStreamSynchronize(t.stream)); // pm is about to go away
                launch_unpermute_rows(t, d_perm);
                if (frames) frames->unpermute(d_perm, t.stream);
                fuser.reset_permutation();
            };
            for (;;) {
                uint64_t lim;
                bool last;
                {
                    std::unique_lock<std::mutex> lk(mu);
                    cv.wait(lk, [&] { return stop || done || limit > next_key; });
                    if (stop) break;
                    lim = limit;
                    last = done;
                }
                for (; next_key < lim; ++next_key) {
                    std::vector<uint64_t> *bp = buckets.find(next_key);
                    if (!bp || bp->empty()) continue;
                    std::vector<uint64_t> &b = *bp;
                    const uint64_t cnt = b.size();
                    ++counts.windows;
                    if ((next_key & 1) == 0) {
                        counts.unitary += cnt;
                        if (fuse) {
                            const auto tf = clk::now();
                            dev.clear();
                            fuser.unitary(b.data(), cnt, dev);
                            t_fuse += since(tf);
                            unitary_window(dev);
                        } else {
                            launch_staged(b.data(), cnt);
                        }
                    } else {
                        if (fuse) {
                            dev.clear();
                            fuser.flush(dev);
                            unitary_window(dev);
                            close_run();
                            unpermute();
                        }
                        close_run();
                        mq.resize(cnt);
                        for (uint64_t i = 0; i < cnt; ++i) mq[i] = packed_q0(b[i]);
                        t.ensure_window_cap(cnt);
                        const auto tm = clk::now();
                        QSR_CUDA(cudaMemcpyAsync(t.ms.mqubits, mq.data(), cnt * 4, cudaMemcpyHostToDevice, t.stream));
                        if (measure_hook)
                            measure_hook->measure(mq, seed, rt);
                        else
                            measure_window_device(t, cnt, seed, mq, flags, true, &rt.t_ms, &rt.ge_ms, &rt.cmp_ms);
                        t_meas += since(tm);
                        if (frames) frames->measure(mq.data(), cnt, t.stream);
                        QSR_CUDA(cudaMemcpyAsync(d_record + rec_off, t.ms.out, cnt * sizeof(qsr_record_entry),
                                                 cudaMemcpyDeviceToDevice, t.stream));
                        rec_off += cnt;
                        counts.measures += cnt;
                    }
                    b.clear();
                    {
                        std::lock_guard<std::mutex> g(pool_mu);
                        if (pool.size() < 64) pool.push_back(std::move(b));
                    }
                    std::vector<uint64_t>().swap(b);
                }
                if (last) break; // the planner is done and everything is out
            }
            close_run();
            if (!stop && fuse) {
                dev.clear();
                fuser.flush(dev);
                unitary_window(dev);
                close_run();
                unpermute();
                QSR_CUDA(cudaStreamSynchronize(t.stream));
            }
            if (d_perm) cudaFree(d_perm);
        } catch (...) {
            emit_error = std::current_exception();
            std::lock_guard<std::mutex> lk(mu);
            stop = true;
        }
    };

    // ---- planner (this thread): the one-pass round closed form, chunk by chunk -------------
    std::thread emit_thread(emitter);
    auto publish = [&](uint64_t lim, bool final) {
        {
            std::lock_guard<std::mutex> lk(mu);
            limit = std::max(limit, lim);
            done = final;
        }
        cv.notify_one();
    };
    auto halt = [&] {
        {
            std::lock_guard<std::mutex> lk(mu);
            stop = true;
        }
        cv.notify_one();
        emit_thread.join();
    };
    ChunkPlanner<decltype(fresh_bucket)> planner(n, buckets, fresh_bucket);
    try {
        const qsr_gate *gates = c.gates.data();
        // Small chunks first (the device starts after ~a layer), then kPlanChunk.
        uint64_t chunk = uint64_t(1) << 17;
        for (uint64_t i0 = 0; i0 < G; i0 += chunk, chunk = std::min(chunk * 2, kPlanChunk)) {
            const uint64_t i1 = std::min(G, i0 + chunk);
            const auto tp = clk::now();
            planner.plan(gates, i0, i1);
            t_plan += since(tp);
            {
                std::lock_guard<std::mutex> lk(mu);
                if (stop) break; // the emitter failed
            }
            if (i1 == G) break;
            publish(2 * uint64_t(planner.min_round()) + 1, false);
        }
    } catch (...) {
        halt();
        throw;
    }
    const uint64_t max_key = planner.max_key();
    publish(max_key + 1, true);
    emit_thread.join();
    if (emit_error) std::rethrow_exception(emit_error);

    if (trace_on()) {
        trace("  stream: plan (thread 1)", t_plan);
        trace("  stream: fuse (thread 2)", t_fuse);
        trace("  stream: stage+launch", t_stage);
        trace("  stream: (ring waits)", t_ringwait);
        trace("  stream: measure windows", t_meas);
    }
    QSR_CUDA(cudaEventRecord(e_end, t.stream));
    QSR_CUDA(cudaEventSynchronize(e_end));
    float total = 0;
    QSR_CUDA(cudaEventElapsedTime(&total, e_start, e_end));
    rt.total_ms = total;
    for (auto &pr : to_events) {
        float ms = 0;
        QSR_CUDA(cudaEventElapsedTime(&ms, pr.first, pr.second));
        rt.to_ms += ms;
        cudaEventDestroy(pr.first);
        cudaEventDestroy(pr.second);
    }
    cudaEventDestroy(e_start);
    cudaEventDestroy(e_end);
    if (read_error_flag(t))
        fail(QSR_LOGIC_ERROR, "product of anti-commuting rows (corrupted tableau)");
}

} // namespace qsr
