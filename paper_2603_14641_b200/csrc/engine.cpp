// Device-resident schedules, the single-shot driver and layout conversion (engine.hpp).
#include "engine.hpp"
#include "fuse.hpp"

#include <cstring>
#include <algorithm>
#include <thread>

namespace qsr {

void upload_packed(DeviceSchedule &ds, uint32_t n, const uint64_t *packed, uint64_t G, int device,
                   cudaStream_t st, bool fuse);

std::unique_ptr<DeviceSchedule> upload_schedule(uint64_t n, const Schedule &s, int device,
                                                cudaStream_t st, bool fuse) {
    // Validate every window first (apply_window / measure_window checks, gates.hpp:149-165,
    // measure.hpp:385-398) so no device state is touched by a schedule that would throw.
    std::vector<uint32_t> stamp(n, 0);
    const uint64_t W = s.num_windows();
    for (uint64_t w = 0; w < W; ++w)
        validate_window(n, s.gates.data() + s.offsets[w], s.offsets[w + 1] - s.offsets[w],
                        s.is_meas[w] != 0, stamp, uint32_t(w + 1));
    auto ds = std::make_unique<DeviceSchedule>();
    ds->device = device;
    ds->offsets = s.offsets;
    ds->is_meas = s.is_meas;
    ds->mqubits.resize(W);
    for (uint64_t w = 0; w < W; ++w) {
        if (!s.is_meas[w]) {
            ds->unitary_count += s.offsets[w + 1] - s.offsets[w];
            continue;
        }
        for (uint64_t i = s.offsets[w]; i < s.offsets[w + 1]; ++i)
            ds->mqubits[w].push_back(s.gates[i].q0);
        ds->measure_count += ds->mqubits[w].size();
    }
    const uint64_t G = s.gates.size();
    std::unique_ptr<uint64_t[]> packed(new uint64_t[std::max<uint64_t>(G, 1)]);
    for (uint64_t i = 0; i < G; ++i) packed[i] = pack_gate(s.gates[i]);
    upload_packed(*ds, uint32_t(n), packed.get(), G, device, st, fuse);
    return ds;
}

// Rewrites a planned schedule with the gate fusion of fuse.hpp: unitary windows go through the
// Fuser, pending single-qubit operations are flushed in a window of their own before every
// measurement window and at the end, and the rows return to logical order before every
// measurement window (perm_at). Windows that end up empty are dropped.
void fuse_into(DeviceSchedule &ds, uint32_t n, const uint64_t *packed, WordVec &out,
               std::vector<uint32_t> &perms) {
    Fuser f(n);
    const std::vector<uint64_t> offsets = ds.offsets;
    const std::vector<uint8_t> is_meas = ds.is_meas;
    ds.offsets.assign(1, 0);
    ds.is_meas.clear();
    ds.mqubits.clear();
    ds.wwords.clear();
    ds.fwords.clear();
    constexpr uint32_t kDeferredWords = ~0u; // gate-window words, computed after fusion in parallel
    auto gate_words = [](const uint64_t *g, size_t cnt) {
        uint32_t words = 0;
        for (size_t i = 0; i < cnt; ++i)
            words += uint32_t(__builtin_popcount(packed_reads(g[i])) + __builtin_popcount(packed_writes(g[i])));
        return words;
    };
    auto push_window = [&](uint64_t words) {
        ds.offsets.push_back(out.size());
        ds.is_meas.push_back(0);
        ds.mqubits.emplace_back();
        ds.wwords.push_back(uint32_t(words));
        ds.fwords.push_back(kDeferredWords);
    };
    auto close_unitary = [&](size_t s0) {
        if (out.size() != s0) push_window(kDeferredWords);
    };
    for (size_t w = 0; w + 1 < offsets.size(); ++w) {
        const uint64_t b = offsets[w], e = offsets[w + 1];
        size_t s0 = out.size();
        if (!is_meas[w]) {
            f.unitary(packed + b, e - b, out);
            close_unitary(s0);
            continue;
        }
        f.flush(out);
        close_unitary(s0);
        auto unpermute_here = [&] {
            ds.perm_at.resize(ds.is_meas.size() + 1, -1);
            if (f.identity_permutation()) return;
            ds.perm_at[ds.is_meas.size()] = int64_t(perms.size());
            const std::vector<uint32_t> pm = f.permutation();
            perms.insert(perms.end(), pm.begin(), pm.end());
            f.reset_permutation();
        };
        unpermute_here();
        std::vector<uint32_t> qs;
        for (uint64_t i = b; i < e; ++i) {
            qs.push_back(packed_q0(packed[i]));
            out.push_back(packed[i]);
        }
        ds.offsets.push_back(out.size());
        ds.is_meas.push_back(1);
        ds.mqubits.push_back(std::move(qs));
        ds.wwords.push_back(0);
        ds.fwords.push_back(0);
    }
    const size_t s0 = out.size();
    f.flush(out);
    close_unitary(s0);
    ds.perm_at.resize(ds.is_meas.size() + 1, -1);
    if (!f.identity_permutation()) {
        ds.perm_at[ds.is_meas.size()] = int64_t(perms.size());
        const std::vector<uint32_t> pm = f.permutation();
        perms.insert(perms.end(), pm.begin(), pm.end());
    }
    // Bytes accounting of the gate windows, off the sequential fusion pass.
    const uint64_t W = ds.wwords.size();
    parallel_chunks(W, std::max(1u, std::min<unsigned>(host_threads(), unsigned(W / 8) + 1)),
                    [&](unsigned, uint64_t b, uint64_t e) {
                        for (uint64_t w = b; w < e; ++w)
                            if (ds.wwords[w] == kDeferredWords) {
                                const uint64_t *g = out.data() + ds.offsets[w];
                                const size_t cnt = ds.offsets[w + 1] - ds.offsets[w];
                                ds.wwords[w] = gate_words(g, cnt);
                                uint32_t fw = 0;
                                for (size_t i = 0; i < cnt; ++i)
                                    fw += uint32_t(__builtin_popcount(packed_reads_frames(g[i])) +
                                                   __builtin_popcount(packed_writes(g[i])));
                                ds.fwords[w] = fw;
                            }
                    });
}

// Packed gates of a planned / validated schedule -> device (optionally through the gate fusion).
void upload_packed(DeviceSchedule &ds, uint32_t n, const uint64_t *packed, uint64_t G, int device,
                   cudaStream_t st, bool fuse) {
    QSR_CUDA(cudaSetDevice(device));
    const uint64_t *dev_gates = packed;
    uint64_t DG = G;
    WordVec fused;
    if (fuse && fusion_enabled()) {
        TraceScope tr("  fuse");
        std::vector<uint32_t> perms;
        // First-touch the output pages on all host threads (the fusion pass itself is sequential
        // and would otherwise take every page fault of a G-word buffer on one core).
        fused.resize(G);
        parallel_chunks(G, std::max(1u, std::min<unsigned>(host_threads(), unsigned(G >> 16) + 1)),
                        [&](unsigned, uint64_t b, uint64_t e) {
                            if (e > b) memset(fused.data() + b, 0, (e - b) * 8);
                        });
        fused.resize(0);
        fuse_into(ds, n, packed, fused, perms);
        dev_gates = fused.data();
        DG = fused.size();
        if (!perms.empty()) {
            ds.d_perms_bytes = perms.size() * 4;
            ds.d_perms = static_cast<uint32_t *>(cache_acquire(device, ds.d_perms_bytes));
            QSR_CUDA(cudaMemcpyAsync(ds.d_perms, perms.data(), perms.size() * 4, cudaMemcpyHostToDevice, st));
        }
    } else {
        for (size_t w = 0; w + 1 < ds.offsets.size(); ++w) {
            uint32_t words = 0, fw = 0;
            if (!ds.is_meas[w])
                for (uint64_t i = ds.offsets[w]; i < ds.offsets[w + 1]; ++i) {
                    words += uint32_t(__builtin_popcount(packed_reads(packed[i])) +
                                      __builtin_popcount(packed_writes(packed[i])));
                    fw += uint32_t(__builtin_popcount(packed_reads_frames(packed[i])) +
                                   __builtin_popcount(packed_writes(packed[i])));
                }
            ds.wwords.push_back(words);
            ds.fwords.push_back(fw);
        }
    }
    ds.d_gates_bytes = std::max<uint64_t>(DG, 1) * 8;
    ds.d_gates = static_cast<uint64_t *>(cache_acquire(device, ds.d_gates_bytes));
    if (DG) {
        TraceScope tr("  gates H2D");
        QSR_CUDA(cudaMemcpyAsync(ds.d_gates, dev_gates, DG * 8, cudaMemcpyHostToDevice, st));
    }
    QSR_CUDA(cudaStreamSynchronize(st));
}

// Circuit -> device schedule without materialising the API Schedule: the O(G) plan, then a
// parallel stable scatter straight into packed device words, then one upload. Windows built
// by the plan are operand-disjoint by construction; the only error the reference would raise
// later is the duplicate-qubit measurement window (measure.hpp:394-395), checked up front.
std::unique_ptr<DeviceSchedule> upload_circuit(const Circuit &c, int device, cudaStream_t st, bool fuse) {
    TraceScope tr_all("upload_circuit");
    WindowPlan p = [&] {
        TraceScope tr("  plan_windows");
        return plan_windows(c);
    }();
    if (p.duplicate_measure)
        fail(QSR_INVALID_ARGUMENT, "measure_window: qubit measured twice");
    const uint64_t G = c.gates.size();
    std::unique_ptr<uint64_t[]> packed(new uint64_t[std::max<uint64_t>(G, 1)]);
    {
        TraceScope tr("  scatter_windows");
        scatter_windows(c, p, packed.get(), [](const qsr_gate &g) { return pack_gate(g); });
    }

    auto ds = std::make_unique<DeviceSchedule>();
    ds->device = device;
    ds->offsets = std::move(p.offsets);
    ds->is_meas = std::move(p.is_meas);
    const uint64_t W = ds->is_meas.size();
    ds->mqubits.resize(W);
    for (uint64_t w = 0; w < W; ++w) {
        const uint64_t b = ds->offsets[w], e = ds->offsets[w + 1];
        if (!ds->is_meas[w]) {
            ds->unitary_count += e - b;
            continue;
        }
        for (uint64_t i = b; i < e; ++i) ds->mqubits[w].push_back(packed_q0(packed[i]));
        ds->measure_count += e - b;
    }
    upload_packed(*ds, c.num_qubits, packed.get(), G, device, st, fuse);
    return ds;
}

namespace {
uint64_t launch_unitary_windows(DeviceTableau &t, const DeviceSchedule &ds, uint64_t w0, uint64_t w1) {
    for (uint64_t w = w0; w < w1; ++w)
        launch_gate_window(t, ds.d_gates + ds.offsets[w], ds.offsets[w + 1] - ds.offsets[w]);
    return w1 - w0;
}
} // namespace

uint64_t run_unitary_windows(DeviceTableau &t, const DeviceSchedule &ds, uint64_t w0, uint64_t w1,
                             double *bytes) {
    if (w1 <= w0) return 0;
    if (bytes && ds.wwords.size() >= w1)
        for (uint64_t w = w0; w < w1; ++w) *bytes += (8.0 * ds.wwords[w] + 16.0) * 2.0 * double(t.kg);
    if (!ds.use_graphs || ds.runs == 0 || w1 - w0 < 2) return launch_unitary_windows(t, ds, w0, w1);
    for (const auto &g : ds.graphs)
        if (g.w0 == w0 && g.w1 == w1 && g.x == t.x && g.z == t.z) {
            QSR_CUDA(cudaGraphLaunch(g.exec, t.stream));
            count_launch(g.kernels);
            return w1 - w0;
        }
    // Capture (kernels are recorded, not run), instantiate, then replay.
    const uint64_t l0 = g_launches;
    cudaGraph_t graph = nullptr;
    QSR_CUDA(cudaStreamBeginCapture(t.stream, cudaStreamCaptureModeThreadLocal));
    try {
        launch_unitary_windows(t, ds, w0, w1);
    } catch (...) {
        cudaStreamEndCapture(t.stream, &graph);
        if (graph) cudaGraphDestroy(graph);
        throw;
    }
    QSR_CUDA(cudaStreamEndCapture(t.stream, &graph));
    const uint64_t kernels = g_launches - l0;
    g_launches = l0;
    cudaGraphExec_t exec = nullptr;
    QSR_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    QSR_CUDA(cudaGraphDestroy(graph));
    ds.graphs.push_back({w0, w1, t.x, t.z, exec, kernels});
    QSR_CUDA(cudaGraphLaunch(exec, t.stream));
    count_launch(kernels);
    return w1 - w0;
}

// The single-shot driver on device-resident inputs (simulator.hpp:46-70). `record` is a
// device array of measure_count entries.
void run_device(DeviceTableau &t, const DeviceSchedule &ds, uint64_t seed,
                qsr_record_entry *d_record, RunTimes &rt, FramesSink *frames) {
    cudaEvent_t e_start, e_end, a, b;
    QSR_CUDA(cudaEventCreate(&e_start));
    QSR_CUDA(cudaEventCreate(&e_end));
    QSR_CUDA(cudaEventCreate(&a));
    QSR_CUDA(cudaEventCreate(&b));
    QSR_CUDA(cudaEventRecord(e_start, t.stream));
    launch_zero_state(t, nullptr);
    QSR_CUDA(cudaMemsetAsync(t.ms.coin_index, 0, 8, t.stream));
    const uint64_t W = ds.is_meas.size();
    uint64_t rec_off = 0;
    std::vector<uint8_t> flags;
    uint64_t w = 0;
    while (w < W) {
        if (!ds.is_meas[w]) {
            // A maximal run of unitary windows, bracketed by one event pair (TO bucket).
            QSR_CUDA(cudaEventRecord(a, t.stream));
            uint64_t w1 = w;
            while (w1 < W && !ds.is_meas[w1]) ++w1;
            if (!frames) {
                rt.gate_launches += run_unitary_windows(t, ds, w, w1, &rt.gate_bytes);
            } else {
                const cudaStream_t fs = frames->own ? frames->own : t.stream;
                cudaEvent_t fa = nullptr, fb = nullptr;
                const bool delayed = frames->own != nullptr;
                if (delayed) {
                    // The reference shot's windows first, alone on the GPU; the frames' windows of
                    // this run follow on their own stream (beside the shot's next measurement
                    // window, which only needs these windows' tableau).
                    for (uint64_t v = w; v < w1; ++v)
                        launch_gate_window(t, ds.d_gates + ds.offsets[v], ds.offsets[v + 1] - ds.offsets[v]);
                    cudaEvent_t done;
                    QSR_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
                    QSR_CUDA(cudaEventRecord(done, t.stream));
                    QSR_CUDA(cudaStreamWaitEvent(fs, done, 0));
                    QSR_CUDA(cudaEventDestroy(done));
                }
                if (frames->own) {
                    QSR_CUDA(cudaEventCreate(&fa));
                    QSR_CUDA(cudaEventCreate(&fb));
                    QSR_CUDA(cudaEventRecord(fa, fs));
                }
                for (uint64_t v = w; v < w1; ++v) {
                    const uint64_t *g = ds.d_gates + ds.offsets[v];
                    const uint64_t cnt = ds.offsets[v + 1] - ds.offsets[v];
                    if (!delayed) launch_gate_window(t, g, cnt);
                    frames->unitary(g, cnt, fs);
                    if (v < ds.wwords.size()) {
                        rt.gate_bytes += (8.0 * ds.wwords[v] + 16.0) * 2.0 * double(t.kg);
                        rt.frames_bytes += 8.0 * ds.fwords[v] * double(frames->row_words);
                    }
                }
                rt.gate_launches += 2 * (w1 - w);
                if (frames->own) {
                    QSR_CUDA(cudaEventRecord(fb, fs));
                    frames->runs.emplace_back(fa, fb);
                }
            }
            w = w1;
            QSR_CUDA(cudaEventRecord(b, t.stream));
            QSR_CUDA(cudaEventSynchronize(b));
            float ms = 0;
            QSR_CUDA(cudaEventElapsedTime(&ms, a, b));
            rt.to_ms += ms;
            continue;
        }
        if (const uint32_t *perm = ds.perm_before(w)) {
            launch_unpermute_rows(t, perm);
            if (frames) frames->unpermute(perm, frames->own ? frames->own : t.stream);
        }
        const auto &mq = ds.mqubits[w];
        const uint64_t m = mq.size();
        t.ensure_window_cap(m);
        QSR_CUDA(cudaMemcpyAsync(t.ms.mqubits, mq.data(), m * 4, cudaMemcpyHostToDevice, t.stream));
        measure_window_device(t, m, seed, mq, flags, true, &rt.t_ms, &rt.ge_ms, &rt.cmp_ms);
        if (frames) frames->measure(mq.data(), m, frames->own ? frames->own : t.stream);
        QSR_CUDA(cudaMemcpyAsync(d_record + rec_off, t.ms.out, m * sizeof(qsr_record_entry),
                                 cudaMemcpyDeviceToDevice, t.stream));
        rec_off += m;
        ++w;
    }
    if (const uint32_t *perm = ds.perm_before(W)) {
        launch_unpermute_rows(t, perm);
        if (frames) frames->unpermute(perm, frames->own ? frames->own : t.stream);
    }
    QSR_CUDA(cudaEventRecord(e_end, t.stream));
    QSR_CUDA(cudaEventSynchronize(e_end));
    float total = 0;
    QSR_CUDA(cudaEventElapsedTime(&total, e_start, e_end));
    rt.total_ms = total;
    for (auto e : {e_start, e_end, a, b}) cudaEventDestroy(e);
    if (read_error_flag(t))
        fail(QSR_LOGIC_ERROR, "product of anti-commuting rows (corrupted tableau)");
    ++const_cast<DeviceSchedule &>(ds).runs;
}

void fill_report(qsr_run_report *rep, const RunTimes &rt, const DeviceSchedule &ds,
                 const std::vector<qsr_record_entry> &record, double total_s) {
    if (!rep) return;
    rep->timers.to_seconds = rt.to_ms * 1e-3;
    rep->timers.t_seconds = rt.t_ms * 1e-3;
    rep->timers.cmp_seconds = rt.cmp_ms * 1e-3;
    rep->timers.ge_seconds = rt.ge_ms * 1e-3;
    rep->gate_count = ds.unitary_count;
    rep->measure_count = ds.measure_count;
    rep->window_count = ds.is_meas.size();
    rep->probabilistic_count = 0;
    for (const auto &e : record) rep->probabilistic_count += e.deterministic ? 0 : 1;
    rep->total_seconds = total_s;
}

// Host reference-layout <-> device layout conversion.
void upload_planes(DeviceTableau &t, const uint64_t *x, const uint64_t *z, int layout) {
    if (layout == QSR_COLUMN_MAJOR) {
        if (t.layout != QSR_COLUMN_MAJOR) { std::swap(t.x, t.x2); std::swap(t.z, t.z2); }
        QSR_CUDA(cudaMemcpy2DAsync(t.x, t.cm_pitch * 8, x, 2 * t.k * 8, 2 * t.k * 8, t.n_pad,
                                   cudaMemcpyHostToDevice, t.stream));
        QSR_CUDA(cudaMemcpy2DAsync(t.z, t.cm_pitch * 8, z, 2 * t.k * 8, 2 * t.k * 8, t.n_pad,
                                   cudaMemcpyHostToDevice, t.stream));
        t.layout = QSR_COLUMN_MAJOR;
    } else {
        if (t.layout != QSR_ROW_MAJOR) { std::swap(t.x, t.x2); std::swap(t.z, t.z2); }
        // Reference RM: word (i, col) at i*2n_pad + col  ->  internal row col, word i.
        const uint64_t R = 2 * t.n_pad, K = t.k;
        std::vector<uint64_t> tmp(R * K);
        for (int plane = 0; plane < 2; ++plane) {
            const uint64_t *src = plane ? z : x;
            for (uint64_t i = 0; i < K; ++i)
                for (uint64_t c = 0; c < R; ++c) tmp[c * K + i] = src[i * R + c];
            QSR_CUDA(cudaMemcpy2DAsync(plane ? t.z : t.x, t.rm_pitch * 8, tmp.data(), K * 8, K * 8,
                                       R, cudaMemcpyHostToDevice, t.stream));
            QSR_CUDA(cudaStreamSynchronize(t.stream));
        }
        t.layout = QSR_ROW_MAJOR;
    }
}

void download_planes(DeviceTableau &t, uint64_t *x, uint64_t *z) {
    TraceScope tr("download_planes");
    if (t.layout == QSR_COLUMN_MAJOR) {
        if (x) download_2d(x, 2 * t.kg * 8, t.x, t.cm_pitch * 8, 2 * t.kg * 8, t.n_pad, t.stream);
        if (z) download_2d(z, 2 * t.kg * 8, t.z, t.cm_pitch * 8, 2 * t.kg * 8, t.n_pad, t.stream);
        t.sync();
        return;
    }
    const uint64_t R = 2 * t.n_pad, K = t.k;
    std::vector<uint64_t> tmp(R * K);
    for (int plane = 0; plane < 2; ++plane) {
        uint64_t *dst = plane ? z : x;
        if (!dst) continue;
        QSR_CUDA(cudaMemcpy2DAsync(tmp.data(), K * 8, plane ? t.z : t.x, t.rm_pitch * 8, K * 8, R,
                                   cudaMemcpyDeviceToHost, t.stream));
        t.sync();
        for (uint64_t c = 0; c < R; ++c)
            for (uint64_t i = 0; i < K; ++i) dst[i * R + c] = tmp[c * K + i];
    }
}

std::vector<uint64_t> download_signs(DeviceTableau &t) {
    std::vector<uint64_t> s(2 * t.kg);
    QSR_CUDA(cudaMemcpyAsync(s.data(), t.s, 2 * t.kg * 8, cudaMemcpyDeviceToHost, t.stream));
    t.sync();
    return s;
}


} // namespace qsr
