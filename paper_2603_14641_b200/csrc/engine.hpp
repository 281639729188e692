// Device-resident schedules and the single-shot driver (reference simulator.hpp:46-76) on one
// DeviceTableau, plus host <-> device layout conversion. Shared by the C ABI (capi.cpp) and the
// generator-row-sharded engine (shard.cpp).
#pragma once

#include <memory>
#include <vector>

#include "device.hpp"

namespace qsr {

// Device-resident schedule: packed gates + per-window measured qubits.
struct DeviceSchedule {
    int device = 0;
    uint64_t *d_gates = nullptr;
    std::vector<uint64_t> offsets;
    std::vector<uint8_t> is_meas;
    std::vector<std::vector<uint32_t>> mqubits; // per window (empty for unitary windows)
    uint64_t measure_count = 0, unitary_count = 0; // of the circuit (before fusion)
    // Gate fusion (fuse.hpp): per-window device words moved per generator-word (reads + writes,
    // for the bytes accounting) and where the CM rows return to logical order.
    std::vector<uint32_t> wwords;
    std::vector<uint32_t> fwords; // the same for the Pauli frames (no sign words)
    // perm_at[w] >= 0: before window w (w == num_windows: after the last one) un-permute the CM
    // rows with the logical -> physical map at d_perms + perm_at[w].
    std::vector<int64_t> perm_at;
    uint32_t *d_perms = nullptr;
    // Resident engines replay each maximal unitary run as a CUDA graph (captured on the second
    // run, when every lazily sized buffer exists). Keyed by the run and the plane pointers the
    // kernels were captured with (x / x2 trade places across runs with an odd swap count).
    bool use_graphs = false;
    uint64_t runs = 0;
    struct Graph {
        uint64_t w0, w1;
        const uint64_t *x, *z;
        cudaGraphExec_t exec;
        uint64_t kernels;
    };
    mutable std::vector<Graph> graphs;
    uint64_t d_gates_bytes = 0, d_perms_bytes = 0; // cached blocks
    ~DeviceSchedule() {
        cudaSetDevice(device);
        cudaDeviceSynchronize(); // kernels reading d_gates may still be queued on the owner's stream
        for (auto &g : graphs) cudaGraphExecDestroy(g.exec);
        cache_release(device, d_gates_bytes, d_gates);
        cache_release(device, d_perms_bytes, d_perms);
    }
    const uint32_t *perm_before(uint64_t w) const {
        return (w < perm_at.size() && perm_at[w] >= 0) ? d_perms + perm_at[w] : nullptr;
    }
};

// Validates every window (apply_window / measure_window checks) and uploads the packed gates.
std::unique_ptr<DeviceSchedule> upload_schedule(uint64_t n, const Schedule &s, int device,
                                                cudaStream_t st, bool fuse = false);
// Circuit -> device schedule through the O(G) plan (no API Schedule materialised); with `fuse`
// (and QSR_FUSE != 0) the windows are rewritten by the gate fusion of fuse.hpp.
std::unique_ptr<DeviceSchedule> upload_circuit(const Circuit &c, int device, cudaStream_t st,
                                               bool fuse = false);

struct RunTimes {
    double to_ms = 0, t_ms = 0, ge_ms = 0, cmp_ms = 0, total_ms = 0;
    double gate_bytes = 0; // algorithmic bytes of the gate-window launches (device gates)
    uint64_t gate_launches = 0; // gate-window kernel launches
    double frames_bytes = 0;    // algorithmic bytes of the frames' window launches (sampling)
};

// Windows [w0, w1) (all unitary) on t: one launch per window (replayed as one CUDA graph from a
// resident engine's second run on). Returns launches.
uint64_t run_unitary_windows(DeviceTableau &t, const DeviceSchedule &ds, uint64_t w0, uint64_t w1,
                             double *bytes = nullptr);

// Optional passenger of the stream: sample()'s Pauli frames ride the same (fused) device windows,
// measurement windows and row un-permutes, on the tableau's stream (capi.cpp).
struct FramesSink {
    uint64_t row_words = 0; // shot-words per frames row (bytes accounting)
    // Resident engines only: the frames' own stream. Frames never read the tableau, so their
    // windows run concurrently with the reference shot's (the caller joins the streams); each
    // unitary run is bracketed by an event pair on it (frames-window device time).
    cudaStream_t own = nullptr;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> runs;
    virtual ~FramesSink() = default;
    virtual void unitary(const uint64_t *d_gates, uint64_t cnt, cudaStream_t st) = 0;
    virtual void unpermute(const uint32_t *d_perm, cudaStream_t st) = 0;
    virtual void measure(const uint32_t *qubits, uint64_t m, cudaStream_t st) = 0;
};

// The single-shot driver on device-resident inputs; `d_record` has measure_count entries. With
// `frames`, the Pauli frames ride every window, on t.stream or on frames->own (sample() on a
// resident schedule; the unitary runs are then launched window by window, not as graphs).
void run_device(DeviceTableau &t, const DeviceSchedule &ds, uint64_t seed,
                qsr_record_entry *d_record, RunTimes &rt, FramesSink *frames = nullptr);
void fill_report(qsr_run_report *rep, const RunTimes &rt, const DeviceSchedule &ds,
                 const std::vector<qsr_record_entry> &record, double total_s);

// run_single_shot straight from a Circuit with the scheduler overlapped with the device
// (stream.cpp): windows are uploaded and launched as soon as they are final.
struct StreamCounts {
    uint64_t unitary = 0, measures = 0, windows = 0;
};
// Optional replacement of the measurement-window step (the generator-row-sharded engine's
// protocol, shard.cpp): it must leave the window's record in t.ms.out.
struct MeasureHook {
    virtual ~MeasureHook() = default;
    virtual void measure(const std::vector<uint32_t> &qubits, uint64_t seed, RunTimes &rt) = 0;
};
void run_circuit_streaming(DeviceTableau &t, const Circuit &c, uint64_t seed,
                           qsr_record_entry *d_record, RunTimes &rt, StreamCounts &counts,
                           FramesSink *frames = nullptr, MeasureHook *measure_hook = nullptr);
// Host reference-layout <-> device layout (CM: [n_pad][2kg] words; RM: reference i-major).
void upload_planes(DeviceTableau &t, const uint64_t *x, const uint64_t *z, int layout);
void download_planes(DeviceTableau &t, uint64_t *x, uint64_t *z);
std::vector<uint64_t> download_signs(DeviceTableau &t);

} // namespace qsr
