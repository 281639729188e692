// Host-side runtime of libqsr: circuits, the O(G) window scheduler, error plumbing and
// the device object model. Kernel launchers are declared in device.hpp.
#pragma once

#include <chrono>
#include <memory>
#include <utility>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/qsr.h"

namespace qsr {

// Allocator that default-initialises: a gate vector of 100 M+ entries is always written before
// it is read, and value-initialising it (a per-element zero fill + single-threaded first touch)
// cost ~2 s at c5.
template <typename T>
struct NoInitAlloc : std::allocator<T> {
    template <typename U>
    struct rebind { using other = NoInitAlloc<U>; };
    NoInitAlloc() = default;
    template <typename U>
    NoInitAlloc(const NoInitAlloc<U> &) noexcept {}
    template <typename U>
    void construct(U *p) noexcept { ::new (static_cast<void *>(p)) U; }
    template <typename U, typename... A>
    void construct(U *p, A &&...a) { ::new (static_cast<void *>(p)) U(std::forward<A>(a)...); }
};
using GateVec = std::vector<qsr_gate, NoInitAlloc<qsr_gate>>;
using WordVec = std::vector<uint64_t, NoInitAlloc<uint64_t>>; // packed device gate words

// Host-side phase trace: QSR_TRACE=1 prints "[qsr] phase ms" lines to stderr (wall clock of the
// calling thread; device work inside a phase is synchronised by the phase itself).
bool trace_on();
void trace(const char *phase, double ms);
struct TraceScope {
    const char *phase;
    std::chrono::steady_clock::time_point t0;
    explicit TraceScope(const char *p) : phase(p), t0(std::chrono::steady_clock::now()) {}
    ~TraceScope() {
        if (trace_on())
            trace(phase, std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
};

// Error carrying a qsr_status; thrown inside the library, converted at the C boundary.
struct Error : std::runtime_error {
    qsr_status status;
    Error(qsr_status s, const std::string &m) : std::runtime_error(m), status(s) {}
};
[[noreturn]] inline void fail(qsr_status s, const std::string &m) { throw Error(s, m); }

inline int gate_arity(uint8_t kind) {
    return (kind == QSR_CX || kind == QSR_CY || kind == QSR_CZ || kind == QSR_SWAP ||
            kind == QSR_ISWAP)
               ? 2
               : 1;
}

// Packed device gate word (8 bytes per gate, a whole c5 schedule is ~1 GB of HBM):
//   bits [0,24) q0 | [24,28) kind | [28,33) pre0 | [33,38) pre1 | [38,62) q1
// pre0 / pre1 = single-qubit Clifford (index into the 24-element group, fuse.hpp; 0 = identity)
// applied to operand 0 / 1 before the gate's own rule (gate fusion, fuse.cpp). Device-only kinds
// beyond the reference's: kDevC1 (pre0 alone on q0) and kDevIswapR (ISWAP after its SWAP part
// has been absorbed into the qubit relabelling).
constexpr uint32_t kDevC1 = 11, kDevIswapR = 12;
inline uint64_t pack_dev(uint32_t kind, uint32_t q0, uint32_t q1, uint32_t pre0 = 0, uint32_t pre1 = 0) {
    return uint64_t(q0 & 0xFFFFFFu) | (uint64_t(kind & 0xF) << 24) | (uint64_t(pre0 & 31) << 28) |
           (uint64_t(pre1 & 31) << 33) | (uint64_t(q1 & 0xFFFFFFu) << 38);
}
inline uint64_t pack_gate(const qsr_gate &g) { return pack_dev(g.kind, g.q0, g.q1); }
inline uint32_t packed_q0(uint64_t w) { return uint32_t(w & 0xFFFFFFu); }
inline uint32_t packed_kind(uint64_t w) { return uint32_t(w >> 24) & 0xF; }
inline uint32_t packed_q1(uint64_t w) { return uint32_t(w >> 38) & 0xFFFFFFu; }
constexpr uint64_t kMaxQubits = (uint64_t(1) << 24) - 1; // 16.7 M qubits (a 2.2 PB tableau)

// Host worker threads for the parallel host passes (scheduler scatter, QASM parse / emit):
// qsr_set_num_threads(t) (t = 0 restores the hardware default), like the reference's
// set_num_threads (parallel.hpp).
unsigned host_threads();
void set_host_threads(unsigned t);
// f(t, begin, end) over T contiguous chunks of [0, n) on T threads (the caller runs chunk 0).
template <typename F>
void parallel_chunks(uint64_t n, unsigned T, F &&f) {
    if (T <= 1 || n < 2) { f(0u, uint64_t(0), n); return; }
    std::vector<std::thread> th;
    for (unsigned t = 1; t < T; ++t) th.emplace_back([&, t] { f(t, n * t / T, n * (t + 1) / T); });
    f(0u, uint64_t(0), n / T);
    for (auto &x : th) x.join();
}

// Philox-4x32-10 (reference rng.hpp:28-55), host side.
void philox_block(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
uint64_t philox_word(uint64_t seed, uint32_t stream, uint32_t ctx, uint64_t index);

struct Circuit {
    uint32_t num_qubits = 0;
    GateVec gates;
    uint32_t num_clbits = 0; // classical bits named in the source (labels only, circuit.hpp:103-105)
    uint64_t measure_count() const; // cached (keyed by the gate vector's size and storage)
    void check_valid() const; // circuit.hpp:108-115

  private:
    mutable uint64_t cached_measures_ = 0, cached_measures_for_ = ~uint64_t(0);
    mutable const qsr_gate *cached_data_ = nullptr;
};

// generate_random (circuit.hpp:132-173): same Philox stream, same draw order.
Circuit generate_random(uint32_t n, uint32_t depth, uint64_t seed, double measure_prob);

struct Schedule {
    int mode = QSR_SINGLE_SHOT;
    GateVec gates;                   // flattened, schedule order
    std::vector<uint64_t> offsets;   // nwindows + 1
    std::vector<uint8_t> is_meas;    // nwindows
    uint64_t num_windows() const { return is_meas.size(); }
};

// Window plan of the O(G) scheduler: key = 2*round + is_measure per gate, the window
// boundaries, and per-thread stable scatter offsets (see host_circuit.cpp).
struct WindowPlan {
    std::vector<uint32_t, NoInitAlloc<uint32_t>> key;
    uint64_t nkeys = 0;
    unsigned threads = 1;
    std::vector<uint64_t> chunk_offsets; // [threads][nkeys]
    std::vector<uint64_t> offsets;       // nwindows + 1
    std::vector<uint8_t> is_meas;        // nwindows
    bool duplicate_measure = false;      // some measurement window repeats a qubit
};
WindowPlan plan_windows(const Circuit &c);

// Stable parallel scatter of the circuit's gates into schedule order, converted per gate
// (qsr_gate for the API Schedule, packed device words for the engine).
template <typename T, typename F>
void scatter_windows(const Circuit &c, WindowPlan &p, T *out, F convert) {
    const uint64_t G = c.gates.size();
    const unsigned nt = p.threads;
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t)
        th.emplace_back([&, t] {
            uint64_t *off = p.chunk_offsets.data() + uint64_t(t) * p.nkeys;
            for (uint64_t i = G * t / nt; i < G * (t + 1) / nt; ++i)
                out[off[p.key[i]]++] = convert(c.gates[i]);
        });
    for (auto &x : th) x.join();
}

// schedule_windows (schedule.hpp:51-137) via the one-pass round closed form.
Schedule schedule_windows(const Circuit &c, int mode);

// Validates a schedule window by window exactly as apply_window / measure_window do
// (gates.hpp:149-165, measure.hpp:385-398), before anything touches the device.
void validate_window(uint64_t n, const qsr_gate *gates, uint64_t ngates, bool is_measurement,
                     std::vector<uint32_t> &stamp, uint32_t stamp_id);

// OpenQASM 2.0 subset (qasm.hpp:29-271) and schedule text / validation (schedule.hpp:143-249).
struct QasmFailure : std::runtime_error {
    int line, column;
    std::string reason;
    QasmFailure(const std::string &r, int l, int c)
        : std::runtime_error("qasm:" + std::to_string(l) + ":" + std::to_string(c) + ": " + r),
          line(l), column(c), reason(r) {}
};
Circuit parse_qasm(const char *text, uint64_t len);         // throws QasmFailure
uint64_t emit_qasm(const Circuit &c, char *out);             // out = NULL: size only
uint64_t schedule_text(const Schedule &s, char *out);        // out = NULL: size only
std::string validate_schedule(const Circuit &c, const Schedule &s);

} // namespace qsr
