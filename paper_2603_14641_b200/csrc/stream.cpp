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
#include <cstring>

#include "engine.hpp"
#include "fuse.hpp"

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
    ~PinnedRing() {
        for (int i = 0; i < 2; ++i) {
            if (done[i]) cudaEventSynchronize(done[i]), cudaEventDestroy(done[i]);
            if (buf[i]) cudaFreeHost(buf[i]);
        }
    }
};

} // namespace

void run_circuit_streaming(DeviceTableau &t, const Circuit &c, uint64_t seed,
                           qsr_record_entry *d_record, RunTimes &rt, StreamCounts &counts) {
    const uint64_t G = c.gates.size();
    const uint32_t n = c.num_qubits;
    t.ensure_gate_buf(std::max<uint64_t>(G, 1));
    uint64_t *d_gates = t.gate_buf;
    static thread_local std::unique_ptr<PinnedRing> ring_store;
    if (!ring_store) ring_store = std::make_unique<PinnedRing>();
    PinnedRing &ring = *ring_store;

    cudaEvent_t e_start, e_end;
    QSR_CUDA(cudaEventCreate(&e_start));
    QSR_CUDA(cudaEventCreate(&e_end));
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> to_events; // unitary runs (TO bucket)
    QSR_CUDA(cudaEventRecord(e_start, t.stream));
    launch_zero_state(t, nullptr);
    QSR_CUDA(cudaMemsetAsync(t.ms.coin_index, 0, 8, t.stream));

    const bool fuse = fusion_enabled();
    Fuser fuser(fuse ? n : 0);
    std::vector<uint64_t> dev;            // device gates of the window being emitted
    std::vector<uint32_t> wire(n, 0); // round << 1 | last gate was a MEASURE
    std::vector<std::vector<uint64_t>> buckets(2);
    uint64_t next_key = 2, dev_off = 0, rec_off = 0;
    std::vector<uint8_t> flags;
    std::vector<uint32_t> mq;

    // Stage one device window through the pinned ring (async H2D) and launch it.
    // (No per-gate byte accounting here: the host is on the critical path of this pipeline; the
    // resident engines report gate bytes.)
    auto launch_staged = [&](const uint64_t *src, uint64_t cnt) {
        for (uint64_t i = 0; i < cnt;) {
            if (ring.fill == kRingGates) {
                QSR_CUDA(cudaEventRecord(ring.done[ring.cur], t.stream));
                ring.used[ring.cur] = true;
                ring.cur ^= 1;
                ring.fill = 0;
                if (ring.used[ring.cur]) QSR_CUDA(cudaEventSynchronize(ring.done[ring.cur]));
            }
            const uint64_t take = std::min(cnt - i, kRingGates - ring.fill);
            uint64_t *dst = ring.buf[ring.cur] + ring.fill;
            std::memcpy(dst, src + i, take * 8);
            QSR_CUDA(cudaMemcpyAsync(d_gates + dev_off + i, dst, take * 8, cudaMemcpyHostToDevice, t.stream));
            ring.fill += take;
            i += take;
        }
        launch_gate_window(t, d_gates + dev_off, cnt);
        ++rt.gate_launches;
        dev_off += cnt;
    };

    // CM rows back to logical order (before a measurement window and at the end).
    uint32_t *d_perm = nullptr;
    auto unpermute = [&] {
        if (fuser.identity_permutation()) return;
        if (!d_perm) QSR_CUDA(cudaMalloc(&d_perm, uint64_t(n) * 4));
        QSR_CUDA(cudaMemcpyAsync(d_perm, fuser.permutation().data(), uint64_t(n) * 4, cudaMemcpyHostToDevice,
                                 t.stream));
        QSR_CUDA(cudaStreamSynchronize(t.stream)); // the host map is reset right after
        launch_unpermute_rows(t, d_perm);
        fuser.reset_permutation();
    };

    // Upload + launch every window with key in [next_key, limit).
    auto emit = [&](uint64_t limit) {
        limit = std::min<uint64_t>(limit, buckets.size());
        bool in_run = false;
        cudaEvent_t ra = nullptr, rb = nullptr;
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
        for (; next_key < limit; ++next_key) {
            std::vector<uint64_t> &b = buckets[next_key];
            if (b.empty()) continue;
            const uint64_t cnt = b.size();
            ++counts.windows;
            if ((next_key & 1) == 0) {
                counts.unitary += cnt;
                const uint64_t *src = b.data();
                uint64_t ng = cnt;
                if (fuse) {
                    dev.clear();
                    fuser.unitary(b.data(), cnt, dev);
                    src = dev.data();
                    ng = dev.size();
                }
                if (ng) {
                    open_run();
                    launch_staged(src, ng);
                }
            } else {
                if (fuse) {
                    dev.clear();
                    fuser.flush(dev);
                    if (!dev.empty()) {
                        open_run();
                        launch_staged(dev.data(), dev.size());
                    }
                    close_run();
                    unpermute();
                }
                close_run();
                mq.resize(cnt);
                for (uint64_t i = 0; i < cnt; ++i) mq[i] = packed_q0(b[i]);
                t.ensure_window_cap(cnt);
                QSR_CUDA(cudaMemcpyAsync(t.ms.mqubits, mq.data(), cnt * 4, cudaMemcpyHostToDevice, t.stream));
                measure_window_device(t, cnt, seed, mq, flags, true, &rt.t_ms, &rt.ge_ms, &rt.cmp_ms);
                QSR_CUDA(cudaMemcpyAsync(d_record + rec_off, t.ms.out, cnt * sizeof(qsr_record_entry),
                                         cudaMemcpyDeviceToDevice, t.stream));
                rec_off += cnt;
                counts.measures += cnt;
            }
            std::vector<uint64_t>().swap(b);
        }
        close_run();
    };

    const qsr_gate *gates = c.gates.data();
    for (uint64_t i0 = 0; i0 < G; i0 += kPlanChunk) {
        const uint64_t i1 = std::min(G, i0 + kPlanChunk);
        for (uint64_t i = i0; i < i1; ++i) {
            const qsr_gate g = gates[i];
            const uint32_t kind = g.kind;
            if (kind > QSR_MEASURE) fail(QSR_INVALID_ARGUMENT, "unknown gate kind");
            const bool two = kind >= QSR_CX && kind <= QSR_ISWAP;
            const uint32_t q0 = g.q0, q1 = two ? g.q1 : g.q0;
            if (q0 >= n || q1 >= n) fail(QSR_OUT_OF_RANGE, "gate operand out of range");
            if (two && q0 == q1) fail(QSR_INVALID_ARGUMENT, "two-qubit gate with equal operands");
            const uint32_t w0 = wire[q0], w1 = wire[q1];
            const uint32_t r0 = w0 >> 1, r1 = w1 >> 1;
            const uint32_t meas = kind == QSR_MEASURE;
            const uint32_t r = meas ? (r0 > 1 ? r0 : 1) : 1 + (r0 > r1 ? r0 : r1);
            if (meas & w0 & 1u) fail(QSR_INVALID_ARGUMENT, "measure_window: qubit measured twice");
            wire[q0] = (r << 1) | meas;
            wire[q1] = (r << 1) | meas;
            const uint64_t key = 2 * uint64_t(r) + meas;
            if (key >= buckets.size()) buckets.resize(key + 1);
            buckets[key].push_back(pack_gate(g));
        }
        if (i1 == G) break;
        uint32_t rmin = 0xFFFFFFFFu;
        for (uint32_t q = 0; q < n; ++q) rmin = std::min(rmin, wire[q] >> 1);
        emit(2 * uint64_t(rmin) + 1);
    }
    emit(~uint64_t(0));
    if (fuse) {
        dev.clear();
        fuser.flush(dev);
        if (!dev.empty()) {
            cudaEvent_t ra, rb;
            QSR_CUDA(cudaEventCreate(&ra));
            QSR_CUDA(cudaEventCreate(&rb));
            QSR_CUDA(cudaEventRecord(ra, t.stream));
            launch_staged(dev.data(), dev.size());
            QSR_CUDA(cudaEventRecord(rb, t.stream));
            to_events.emplace_back(ra, rb);
        }
        unpermute();
        QSR_CUDA(cudaStreamSynchronize(t.stream));
    }
    if (d_perm) cudaFree(d_perm);

    QSR_CUDA(cudaEventRecord(e_end, t.stream));
    QSR_CUDA(cudaEventSynchronize(e_end));
    float total = 0;
    QSR_CUDA(cudaEventElapsedTime(&total, e_start, e_end));
    rt.total_ms = total;
    for (auto &p : to_events) {
        float ms = 0;
        QSR_CUDA(cudaEventElapsedTime(&ms, p.first, p.second));
        rt.to_ms += ms;
        cudaEventDestroy(p.first);
        cudaEventDestroy(p.second);
    }
    cudaEventDestroy(e_start);
    cudaEventDestroy(e_end);
    if (read_error_flag(t))
        fail(QSR_LOGIC_ERROR, "product of anti-commuting rows (corrupted tableau)");
}

} // namespace qsr
