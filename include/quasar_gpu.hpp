// quasar_gpu.hpp — header-only C++ drop-in for the reference's hot-path API
// (proj/include/quasar) on the B200 engine (libqsr.so, C ABI in qsr.h).
//
// A reference user keeps their types (quasar::Circuit, Schedule, Window, Tableau<uint64_t>,
// MeasurementRecord, RandomStream, ShotRecord<uint64_t>, RunReport) and swaps the namespace:
//
//     #include "quasar/simulator.hpp"     // reference headers (types)
//     #include "quasar_gpu.hpp"           // this file
//     auto r = quasar::gpu::run_single_shot<uint64_t>(circuit, seed);   // was quasar::
//
// Signatures, results (bit-exact) and exception types are the reference's: the C ABI status
// is rethrown as std::invalid_argument / std::out_of_range / std::logic_error, parse errors as
// quasar::QasmError with the reference's line / column. Every word type W of the reference is
// accepted: the engine computes on 64-bit words and Tableau<W> / ShotRecord<W> are exact
// repackings of the same bits (ColumnMajor tableaux). Host tableaux are uploaded, processed on
// the GPU and downloaded in the reference's own storage layout.
#ifndef QUASAR_GPU_HPP_
#define QUASAR_GPU_HPP_

#include <algorithm>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "qsr.h"
#include "quasar/frames.hpp"
#include "quasar/measure.hpp"
#include "quasar/qasm.hpp"
#include "quasar/simulator.hpp"

namespace quasar::gpu {

static_assert(sizeof(Gate) == sizeof(qsr_gate), "quasar::Gate must match qsr_gate (12 bytes)");
static_assert(sizeof(MeasurementRecord::Entry) == sizeof(qsr_record_entry),
              "MeasurementRecord::Entry must match qsr_record_entry (8 bytes)");

inline void check(qsr_status st) {
    switch (st) {
    case QSR_OK: return;
    case QSR_INVALID_ARGUMENT: throw std::invalid_argument(qsr_last_error());
    case QSR_OUT_OF_RANGE: throw std::out_of_range(qsr_last_error());
    case QSR_LOGIC_ERROR: throw std::logic_error(qsr_last_error());
    default: throw std::runtime_error(std::string("libqsr: ") + qsr_last_error());
    }
}

inline int& device() { // CUDA device used by the free functions below
    static int d = 0;
    return d;
}

namespace detail {
struct CircuitDel { void operator()(qsr_circuit *c) const { qsr_circuit_destroy(c); } };
struct ScheduleDel { void operator()(qsr_schedule *s) const { qsr_schedule_destroy(s); } };
struct TableauDel { void operator()(qsr_tableau *t) const { qsr_tableau_destroy(t); } };
struct FramesDel { void operator()(qsr_frames *f) const { qsr_frames_destroy(f); } };
using CircuitPtr = std::unique_ptr<qsr_circuit, CircuitDel>;
using SchedulePtr = std::unique_ptr<qsr_schedule, ScheduleDel>;
using TableauPtr = std::unique_ptr<qsr_tableau, TableauDel>;
using FramesPtr = std::unique_ptr<qsr_frames, FramesDel>;

inline const qsr_gate *gates(const std::vector<Gate> &g) {
    return reinterpret_cast<const qsr_gate *>(g.data());
}

inline CircuitPtr circuit(const Circuit &c) {
    qsr_circuit *h = nullptr;
    check(qsr_circuit_create(c.num_qubits, gates(c.gates), c.gates.size(), &h));
    return CircuitPtr(h);
}

inline SchedulePtr schedule(const Schedule &s) {
    std::vector<Gate> flat;
    std::vector<uint64_t> off{0};
    std::vector<uint8_t> meas;
    for (const Window &w : s.windows) {
        flat.insert(flat.end(), w.gates.begin(), w.gates.end());
        off.push_back(flat.size());
        meas.push_back(w.is_measurement ? 1 : 0);
    }
    qsr_schedule *h = nullptr;
    check(qsr_schedule_create(gates(flat), off.data(), meas.data(), meas.size(),
                              s.mode == ScheduleMode::sampling ? QSR_SAMPLING : QSR_SINGLE_SHOT, &h));
    return SchedulePtr(h);
}

inline TableauPtr upload(const Tableau<uint64_t> &t) {
    qsr_tableau *h = nullptr;
    check(qsr_tableau_create(t.num_qubits(), device(), &h));
    TableauPtr p(h);
    check(qsr_tableau_upload(h, t.x_plane().data(), t.z_plane().data(), t.signs().data(),
                             t.layout() == Layout::RowMajor ? QSR_ROW_MAJOR : QSR_COLUMN_MAJOR));
    return p;
}

// Download into a reference Tableau of the same layout (the device converts its internal
// generator-major RowMajor back to the reference's i-major storage, tableau.hpp:91-94).
inline void download(qsr_tableau *h, Tableau<uint64_t> &t) {
    int layout = 0;
    check(qsr_tableau_info(h, nullptr, nullptr, nullptr, &layout));
    if ((layout == QSR_ROW_MAJOR) != (t.layout() == Layout::RowMajor))
        throw std::logic_error("quasar::gpu: host and device layouts differ");
    check(qsr_tableau_download(h, t.x_plane().data(), t.z_plane().data(), t.signs().data()));
}

// A zero Tableau<W> in `layout`. tableau.hpp has no layout setter: the only way to a RowMajor
// object is its own transpose_in_place, run here on zeros (a flag flip, no user data).
template <Word W>
Tableau<W> blank(size_t n, Layout layout) {
    Tableau<W> t(n);
    if (layout == Layout::RowMajor) t.transpose_in_place();
    return t;
}

// Logical-bit copy between word types (same n, same layout): x / z bit of every (generator,
// qubit) and every sign, through the reference's own accessors (tableau.hpp:98-114).
template <Word A, Word B>
void copy_bits(const Tableau<A> &a, Tableau<B> &b) {
    const size_t n = a.num_qubits();
    for (size_t g = 0; g < 2 * n; ++g) {
        for (size_t q = 0; q < n; ++q) {
            b.set_x_bit(g, q, a.x_bit(g, q));
            b.set_z_bit(g, q, a.z_bit(g, q));
        }
        b.set_sign_bit(g, a.sign_bit(g));
    }
}

// Runs `op(qsr_tableau *)` on the device copy of t and writes the result back into t (in the
// layout the device ends in). Every W: other word types go through a 64-bit image.
template <Word W, typename Op>
void on_device(Tableau<W> &t, Op op) {
    if constexpr (std::is_same_v<W, uint64_t>) {
        auto h = upload(t);
        op(h.get());
        int layout = 0;
        check(qsr_tableau_info(h.get(), nullptr, nullptr, nullptr, &layout));
        const Layout lay = layout == QSR_ROW_MAJOR ? Layout::RowMajor : Layout::ColumnMajor;
        if (lay != t.layout()) t = blank<uint64_t>(t.num_qubits(), lay);
        download(h.get(), t);
    } else {
        Tableau<uint64_t> t64 = blank<uint64_t>(t.num_qubits(), t.layout());
        copy_bits(t, t64);
        on_device(t64, op);
        Tableau<W> out = blank<W>(t.num_qubits(), t64.layout());
        copy_bits(t64, out);
        t = std::move(out);
    }
}

// Read-only device query on t (every W).
template <Word W, typename Op>
void query_device(const Tableau<W> &t, Op op) {
    if constexpr (std::is_same_v<W, uint64_t>) {
        auto h = upload(t);
        op(h.get());
    } else {
        Tableau<uint64_t> t64 = blank<uint64_t>(t.num_qubits(), t.layout());
        copy_bits(t, t64);
        query_device(t64, op);
    }
}

// Tableau<W> <-> Tableau<uint64_t>, ColumnMajor (tableau.hpp:51-61): the generator bits of every
// qubit row are the same bit string in either word size, so W-words are the 64-bit words' W-bit
// pieces (little-endian order); rows and words past n stay zero padding in both.
template <Word W>
Tableau<W> from64(const Tableau<uint64_t> &a) {
    if (a.layout() != Layout::ColumnMajor) throw std::logic_error("quasar::gpu: ColumnMajor expected");
    const size_t n = a.num_qubits(), k64 = a.num_words();
    Tableau<W> b(n);
    const size_t kw = b.num_words();
    constexpr size_t bits = 8 * sizeof(W), per = 64 / bits;
    auto piece = [&](const std::vector<uint64_t> &v, size_t base, size_t jw) {
        return static_cast<W>(v[base + jw / per] >> (bits * (jw % per)));
    };
    for (size_t q = 0; q < n; ++q)
        for (size_t h = 0; h < 2; ++h)
            for (size_t jw = 0; jw < kw; ++jw) {
                b.x_plane()[q * 2 * kw + h * kw + jw] = piece(a.x_plane(), q * 2 * k64 + h * k64, jw);
                b.z_plane()[q * 2 * kw + h * kw + jw] = piece(a.z_plane(), q * 2 * k64 + h * k64, jw);
            }
    for (size_t h = 0; h < 2; ++h)
        for (size_t jw = 0; jw < kw; ++jw) b.signs()[h * kw + jw] = piece(a.signs(), h * k64, jw);
    return b;
}

template <Word W>
Tableau<uint64_t> to64(const Tableau<W> &b) {
    if (b.layout() != Layout::ColumnMajor) throw std::invalid_argument("tableau must be ColumnMajor");
    const size_t n = b.num_qubits(), kw = b.num_words();
    Tableau<uint64_t> a(n);
    const size_t k64 = a.num_words();
    constexpr size_t bits = 8 * sizeof(W), per = 64 / bits;
    auto put = [&](std::vector<uint64_t> &v, size_t base, size_t jw, W w) {
        v[base + jw / per] |= uint64_t(w) << (bits * (jw % per));
    };
    std::fill(a.x_plane().begin(), a.x_plane().end(), 0);
    std::fill(a.z_plane().begin(), a.z_plane().end(), 0);
    std::fill(a.signs().begin(), a.signs().end(), 0);
    for (size_t q = 0; q < b.padded_qubits() && q < a.padded_qubits(); ++q)
        for (size_t h = 0; h < 2; ++h)
            for (size_t jw = 0; jw < kw; ++jw) {
                put(a.x_plane(), q * 2 * k64 + h * k64, jw, b.x_plane()[q * 2 * kw + h * kw + jw]);
                put(a.z_plane(), q * 2 * k64 + h * k64, jw, b.z_plane()[q * 2 * kw + h * kw + jw]);
            }
    for (size_t h = 0; h < 2; ++h)
        for (size_t jw = 0; jw < kw; ++jw) put(a.signs(), h * k64, jw, b.signs()[h * kw + jw]);
    return a;
}

inline RunReport report(const qsr_run_report &r) {
    RunReport o;
    o.timers.to_seconds = r.timers.to_seconds;
    o.timers.t_seconds = r.timers.t_seconds;
    o.timers.cmp_seconds = r.timers.cmp_seconds;
    o.timers.ge_seconds = r.timers.ge_seconds;
    o.gate_count = r.gate_count;
    o.measure_count = r.measure_count;
    o.probabilistic_count = r.probabilistic_count;
    o.window_count = r.window_count;
    o.total_seconds = r.total_seconds;
    return o;
}

inline SingleShotResult<uint64_t> run(const Circuit &c, const Schedule *s, uint64_t seed) {
    auto ch = circuit(c);
    SchedulePtr sh;
    if (s) sh = schedule(*s);
    std::vector<MeasurementRecord::Entry> rec(c.measure_count());
    qsr_run_report rep{};
    qsr_tableau *th = nullptr;
    check(qsr_run_single_shot(ch.get(), sh.get(), seed, device(), &th,
                              reinterpret_cast<qsr_record_entry *>(rec.data()), &rep));
    TableauPtr tp(th);
    SingleShotResult<uint64_t> out{Tableau<uint64_t>(c.num_qubits), {}, {}};
    download(th, out.tableau);
    out.record.entries = std::move(rec);
    out.report = report(rep);
    return out;
}
} // namespace detail

// run_single_shot<W>(circuit, schedule, seed)   (simulator.hpp:46-70), every W: the engine runs
// on 64-bit words; other word types get the same tableau bits repacked (records are word-size
// independent, test_measure.cpp:315-335).
template <Word W>
SingleShotResult<W> run_single_shot(const Circuit &circuit, const Schedule &schedule,
                                    uint64_t seed) {
    if constexpr (std::is_same_v<W, uint64_t>) {
        return detail::run(circuit, &schedule, seed);
    } else {
        auto r = detail::run(circuit, &schedule, seed);
        return {detail::from64<W>(r.tableau), std::move(r.record), r.report};
    }
}

// run_single_shot<W>(circuit, seed)   (simulator.hpp:72-76)
template <Word W>
SingleShotResult<W> run_single_shot(const Circuit &circuit, uint64_t seed) {
    if constexpr (std::is_same_v<W, uint64_t>) {
        return detail::run(circuit, nullptr, seed);
    } else {
        auto r = detail::run(circuit, nullptr, seed);
        return {detail::from64<W>(r.tableau), std::move(r.record), r.report};
    }
}

// schedule_windows(circuit, mode)   (schedule.hpp:51-137)
inline Schedule schedule_windows(const Circuit &circuit, ScheduleMode mode) {
    auto ch = detail::circuit(circuit);
    qsr_schedule *sh = nullptr;
    check(qsr_schedule_windows(ch.get(), mode == ScheduleMode::sampling ? QSR_SAMPLING : QSR_SINGLE_SHOT, &sh));
    detail::SchedulePtr sp(sh);
    uint64_t nwin = 0, ng = 0;
    check(qsr_schedule_info(sh, &nwin, &ng, nullptr));
    const qsr_gate *g = qsr_schedule_gates(sh);
    const uint64_t *off = qsr_schedule_offsets(sh);
    const uint8_t *meas = qsr_schedule_is_measurement(sh);
    Schedule s;
    s.mode = mode;
    s.windows.resize(nwin);
    for (uint64_t w = 0; w < nwin; ++w) {
        s.windows[w].is_measurement = meas[w] != 0;
        const Gate *b = reinterpret_cast<const Gate *>(g + off[w]);
        s.windows[w].gates.assign(b, b + (off[w + 1] - off[w]));
    }
    return s;
}

// generate_random(n, depth, seed, measure_prob)   (circuit.hpp:132-173)
inline Circuit generate_random(uint32_t n, uint32_t depth, uint64_t seed, double measure_prob) {
    qsr_circuit *h = nullptr;
    check(qsr_generate_random(n, depth, seed, measure_prob, &h));
    detail::CircuitPtr p(h);
    uint32_t nq = 0;
    uint64_t ng = 0;
    check(qsr_circuit_info(h, &nq, &ng, nullptr));
    Circuit c;
    c.num_qubits = nq;
    c.num_clbits = nq;
    const Gate *g = reinterpret_cast<const Gate *>(qsr_circuit_gates(h));
    c.gates.assign(g, g + ng);
    return c;
}

// apply_window(tableau, window)   (gates.hpp:147-197)
inline void apply_window(Tableau<uint64_t> &t, const Window &window);
template <Word W, typename = std::enable_if_t<!std::is_same_v<W, uint64_t>>>
void apply_window(Tableau<W> &t, const Window &window) {
    if (window.is_measurement) throw std::invalid_argument("apply_window: window contains measurements");
    auto t64 = detail::to64(t);
    apply_window(t64, window);
    t = detail::from64<W>(t64);
}
inline void apply_window(Tableau<uint64_t> &t, const Window &window) {
    if (window.is_measurement)
        throw std::invalid_argument("apply_window: window contains measurements");
    if (t.layout() != Layout::ColumnMajor)
        throw std::invalid_argument("apply_window: tableau must be ColumnMajor");
    auto h = detail::upload(t);
    check(qsr_apply_window(h.get(), detail::gates(window.gates), window.gates.size()));
    detail::download(h.get(), t);
}

// measure_window(t, window, rng, record, scratch, timers)   (measure.hpp:381-442). The coins
// are drawn from the caller's RandomStream (any stream/context) and it is advanced by exactly
// the number of probabilistic collapses, as in the reference.
inline void measure_window(Tableau<uint64_t> &t, const Window &window, RandomStream &rng,
                           MeasurementRecord &record, MeasureScratch<uint64_t> &,
                           PhaseTimers *timers = nullptr);
template <Word W, typename = std::enable_if_t<!std::is_same_v<W, uint64_t>>>
void measure_window(Tableau<W> &t, const Window &window, RandomStream &rng, MeasurementRecord &record,
                    MeasureScratch<W> &, PhaseTimers *timers = nullptr) {
    if (!window.is_measurement) throw std::invalid_argument("measure_window: not a measurement window");
    auto t64 = detail::to64(t);
    MeasureScratch<uint64_t> scratch;
    measure_window(t64, window, rng, record, scratch, timers);
    t = detail::from64<W>(t64);
}
inline void measure_window(Tableau<uint64_t> &t, const Window &window, RandomStream &rng,
                           MeasurementRecord &record, MeasureScratch<uint64_t> &,
                           PhaseTimers *timers) {
    if (t.layout() != Layout::ColumnMajor)
        throw std::invalid_argument("measure_window: tableau must be ColumnMajor");
    if (!window.is_measurement)
        throw std::invalid_argument("measure_window: not a measurement window");
    RandomStream peek = rng;
    std::vector<uint8_t> coins(window.gates.size());
    for (auto &c : coins) c = uint8_t(peek.next_word() & 1);
    auto h = detail::upload(t);
    std::vector<MeasurementRecord::Entry> out(window.gates.size());
    uint64_t used = 0;
    qsr_phase_timers pt{};
    check(qsr_measure_window_coins(h.get(), detail::gates(window.gates), window.gates.size(),
                                   coins.data(), coins.size(), &used,
                                   reinterpret_cast<qsr_record_entry *>(out.data()), &pt));
    for (uint64_t i = 0; i < used; ++i) rng.next_word();
    detail::download(h.get(), t);
    record.entries.insert(record.entries.end(), out.begin(), out.end());
    if (timers) {
        timers->t_seconds += pt.t_seconds;
        timers->cmp_seconds += pt.cmp_seconds;
        timers->ge_seconds += pt.ge_seconds;
    }
}

// sample<W>(circuit, shots, seed, report)   (frames.hpp:163-204), every W of the reference. The
// engine keeps 64-bit shot words and draws the Z frames as sample<W> does; the little-endian bytes
// of a row are the W-words of the reference's row.
template <Word W>
ShotRecord<W> sample(const Circuit &circuit, size_t shots, uint64_t seed, RunReport *report = nullptr) {
    auto ch = detail::circuit(circuit);
    qsr_frames *fh = nullptr;
    qsr_run_report rep{};
    check(qsr_sample_word(ch.get(), shots, seed, unsigned(8 * sizeof(W)), device(), &fh, &rep));
    detail::FramesPtr fp(fh);
    uint64_t nrows = 0, kf64 = 0;
    check(qsr_frames_record(fh, &nrows, nullptr, nullptr));
    check(qsr_frames_info(fh, nullptr, nullptr, &kf64));
    std::vector<uint64_t> words(nrows * kf64);
    ShotRecord<W> r;
    r.shots = shots;
    r.kf = (shots + 8 * sizeof(W) - 1) / (8 * sizeof(W));
    r.measured.resize(nrows);
    check(qsr_frames_record(fh, &nrows, r.measured.data(), words.data()));
    r.words.resize(nrows * r.kf);
    constexpr size_t per = 64 / (8 * sizeof(W));
    for (uint64_t row = 0; row < nrows; ++row)
        for (size_t j = 0; j < r.kf; ++j)
            r.words[row * r.kf + j] =
                static_cast<W>(words[row * kf64 + j / per] >> (8 * sizeof(W) * (j % per)));
    if (report) *report = detail::report(rep);
    return r;
}

// ---- measurement kernels of measure_window, one at a time (measure.hpp:104-376) -----------
// Same preconditions and exceptions as the reference (RowMajor tableaux, invalid_argument on an
// empty pivot list, a block size of 0 or a swap precondition; logic_error on an odd phase).

// find_probabilistic(t, window)   (measure.hpp:104-126)
template <Word W>
std::vector<int64_t> find_probabilistic(const Tableau<W> &t, const Window &window) {
    if (t.layout() != Layout::RowMajor) throw std::invalid_argument("find_probabilistic: tableau must be RowMajor");
    std::vector<int64_t> out(window.gates.size(), -1);
    detail::query_device(t, [&](qsr_tableau *h) {
        check(qsr_find_probabilistic(h, detail::gates(window.gates), window.gates.size(), out.data()));
    });
    return out;
}

// find_and_compact_pivots(t, q, scratch)   (measure.hpp:130-150)
template <Word W>
PivotList find_and_compact_pivots(const Tableau<W> &t, size_t q, MeasureScratch<W> &) {
    if (t.layout() != Layout::RowMajor)
        throw std::invalid_argument("find_and_compact_pivots: tableau must be RowMajor");
    PivotList p;
    p.entries.assign(t.num_qubits(), -1);
    uint64_t count = 0;
    detail::query_device(t, [&](qsr_tableau *h) { check(qsr_find_and_compact_pivots(h, q, p.entries.data(), &count)); });
    p.count = count;
    return p;
}

// parallel_ge(t, pivots, scratch, block_targets)   (measure.hpp:161-273); the block size never
// changes bits (test_measure.cpp:112-145) and is validated like the reference's.
template <Word W>
void parallel_ge(Tableau<W> &t, const PivotList &pivots, MeasureScratch<W> &, size_t block_targets = kGeBlockTargets) {
    if (t.layout() != Layout::RowMajor) throw std::invalid_argument("parallel_ge: tableau must be RowMajor");
    if (pivots.count == 0) throw std::invalid_argument("parallel_ge: empty pivot list");
    if (block_targets < 1) throw std::invalid_argument("parallel_ge: block size must be >= 1");
    detail::on_device(t, [&](qsr_tableau *h) {
        check(qsr_parallel_ge(h, pivots.entries.data(), pivots.count, block_targets));
    });
}

// swap_anti_commuting(t, p, q, scratch)   (measure.hpp:279-332)
template <Word W>
void swap_anti_commuting(Tableau<W> &t, size_t p, size_t q, MeasureScratch<W> &) {
    if (t.layout() != Layout::RowMajor) throw std::invalid_argument("swap_anti_commuting: tableau must be RowMajor");
    detail::on_device(t, [&](qsr_tableau *h) { check(qsr_swap_anti_commuting(h, p, q)); });
}

// inject_x(t, p)   (measure.hpp:335-338)
template <Word W>
void inject_x(Tableau<W> &t, size_t p) {
    detail::on_device(t, [&](qsr_tableau *h) { check(qsr_inject_x(h, p)); });
}

// deterministic_outcome(t, q, scratch)   (measure.hpp:343-376)
template <Word W>
bool deterministic_outcome(const Tableau<W> &t, size_t q, MeasureScratch<W> &) {
    if (t.layout() != Layout::RowMajor)
        throw std::invalid_argument("deterministic_outcome: tableau must be RowMajor");
    uint8_t o = 0;
    detail::query_device(t, [&](qsr_tableau *h) { check(qsr_deterministic_outcome(h, q, &o)); });
    return o != 0;
}

// Tableau::transpose_in_place()   (tableau.hpp:166-176) as a free function (a member cannot
// be replaced from outside the class): the device's one-pass TMA transpose, every W.
template <Word W>
void transpose_in_place(Tableau<W> &t) {
    detail::on_device(t, [&](qsr_tableau *h) { check(qsr_transpose_in_place(h)); });
}

// ---- Pauli frames one step at a time (frames.hpp:46-158), every W ---------------------------
namespace detail {
template <Word W>
FramesPtr frames_upload(const FrameTableau<W> &f) {
    qsr_frames *h = nullptr;
    check(qsr_init_frames_word(f.n, f.shots, 0, unsigned(8 * sizeof(W)), device(), &h));
    FramesPtr p(h);
    uint64_t kf64 = 0;
    check(qsr_frames_info(h, nullptr, nullptr, &kf64));
    std::vector<uint64_t> x(f.n * kf64, 0), z(f.n * kf64, 0);
    constexpr size_t bits = 8 * sizeof(W), per = 64 / bits;
    for (size_t q = 0; q < f.n; ++q)
        for (size_t j = 0; j < f.kf; ++j) {
            x[q * kf64 + j / per] |= uint64_t(f.xf[q * f.kf + j]) << (bits * (j % per));
            z[q * kf64 + j / per] |= uint64_t(f.zf[q * f.kf + j]) << (bits * (j % per));
        }
    check(qsr_frames_upload(h, x.data(), z.data()));
    return p;
}
template <Word W>
void frames_download(qsr_frames *h, FrameTableau<W> &f) {
    uint64_t kf64 = 0;
    check(qsr_frames_info(h, nullptr, nullptr, &kf64));
    std::vector<uint64_t> x(f.n * kf64), z(f.n * kf64);
    check(qsr_frames_download(h, x.data(), z.data()));
    constexpr size_t bits = 8 * sizeof(W), per = 64 / bits;
    for (size_t q = 0; q < f.n; ++q)
        for (size_t j = 0; j < f.kf; ++j) {
            f.xf[q * f.kf + j] = static_cast<W>(x[q * kf64 + j / per] >> (bits * (j % per)));
            f.zf[q * f.kf + j] = static_cast<W>(z[q * kf64 + j / per] >> (bits * (j % per)));
        }
}
} // namespace detail

// init_frames<W>(n, shots, seed)   (frames.hpp:46-72): Z frames drawn on the device with
// sample<W>'s keys (Philox(seed, 1, 0, (q << 24) | j) per W-word j).
template <Word W>
FrameTableau<W> init_frames(size_t n, size_t shots, uint64_t seed) {
    if (shots < 1) throw std::invalid_argument("init_frames: shots must be >= 1");
    qsr_frames *h = nullptr;
    check(qsr_init_frames_word(n, shots, seed, unsigned(8 * sizeof(W)), device(), &h));
    detail::FramesPtr p(h);
    FrameTableau<W> f;
    f.n = n;
    f.shots = shots;
    f.kf = words_for<W>(shots);
    f.xf.assign(n * f.kf, W{0});
    f.zf.assign(n * f.kf, W{0});
    detail::frames_download(h, f);
    return f;
}

// apply_window_frames(f, window)   (frames.hpp:76-94)
template <Word W>
void apply_window_frames(FrameTableau<W> &f, const Window &window) {
    if (window.is_measurement) throw std::invalid_argument("apply_window_frames: measurement window");
    auto h = detail::frames_upload(f);
    check(qsr_apply_window_frames(h.get(), detail::gates(window.gates), window.gates.size(), 0));
    detail::frames_download(h.get(), f);
}

// measure_sample(f, window, record, seed, epoch)   (frames.hpp:111-158): the device records the
// window's X frames and redraws their Z frames; rows merge into `record` with the reference's
// row reuse for qubits measured before.
template <Word W>
void measure_sample(FrameTableau<W> &f, const Window &window, ShotRecord<W> &record, uint64_t seed, uint32_t epoch) {
    if (!window.is_measurement) throw std::invalid_argument("measure_sample: not a measurement window");
    auto h = detail::frames_upload(f);
    check(qsr_measure_sample(h.get(), detail::gates(window.gates), window.gates.size(), 1, seed, epoch));
    uint64_t nrows = 0, kf64 = 0;
    check(qsr_frames_record(h.get(), &nrows, nullptr, nullptr));
    check(qsr_frames_info(h.get(), nullptr, nullptr, &kf64));
    std::vector<uint32_t> measured(nrows);
    std::vector<uint64_t> words(nrows * kf64);
    if (nrows) check(qsr_frames_record(h.get(), &nrows, measured.data(), words.data()));
    detail::frames_download(h.get(), f);
    constexpr size_t bits = 8 * sizeof(W), per = 64 / bits;
    for (size_t m = 0; m < measured.size(); ++m) {
        const uint32_t q = measured[m];
        size_t row = record.measured.size();
        for (size_t r = 0; r < record.measured.size(); ++r)
            if (record.measured[r] == q) { row = r; break; }
        if (row == record.measured.size()) {
            record.measured.push_back(q);
            record.words.resize(record.measured.size() * f.kf, W{0});
        }
        for (size_t j = 0; j < f.kf; ++j)
            record.words[row * f.kf + j] = static_cast<W>(words[m * kf64 + j / per] >> (bits * (j % per)));
    }
}

// parse_qasm(text)   (qasm.hpp:159-252): same Circuit, same QasmError (line, column, reason);
// large bodies are parsed on all host threads.
inline Circuit parse_qasm(std::string_view text) {
    qsr_circuit *h = nullptr;
    qsr_qasm_error err{};
    const qsr_status st = qsr_parse_qasm(text.data(), text.size(), &h, &err);
    if (st == QSR_PARSE_ERROR) {
        std::string what = qsr_last_error(); // "qasm:L:C: reason"
        size_t p = what.find(": ");
        throw QasmError(p == std::string::npos ? what : what.substr(p + 2), err.line, err.column);
    }
    check(st);
    detail::CircuitPtr cp(h);
    uint32_t nq = 0, ncl = 0;
    uint64_t ng = 0;
    check(qsr_circuit_info(h, &nq, &ng, nullptr));
    check(qsr_circuit_clbits(h, &ncl));
    Circuit c;
    c.num_qubits = nq;
    c.num_clbits = ncl;
    const Gate *g = reinterpret_cast<const Gate *>(qsr_circuit_gates(h));
    c.gates.assign(g, g + ng);
    return c;
}

// emit_qasm(circuit)   (qasm.hpp:254-271)
inline std::string emit_qasm(const Circuit &circuit) {
    auto ch = detail::circuit(circuit);
    uint64_t len = 0;
    check(qsr_emit_qasm(ch.get(), nullptr, 0, &len));
    std::string out(len, '\0');
    check(qsr_emit_qasm(ch.get(), out.data(), len, &len));
    return out;
}

// Tableau::check_group_validity()   (tableau.hpp:184-213) on the device, every W.
template <Word W>
std::string check_group_validity(const Tableau<W> &tw) {
    if constexpr (!std::is_same_v<W, uint64_t>) {
        return check_group_validity(detail::to64(tw));
    } else {
    const Tableau<uint64_t> &t = tw;
    auto h = detail::upload(t);
    uint64_t len = 0;
    check(qsr_tableau_check_validity(h.get(), nullptr, 0, &len));
    std::string out(len, '\0');
    check(qsr_tableau_check_validity(h.get(), out.data(), len, &len));
    return out;
    }
}

} // namespace quasar::gpu

#endif // QUASAR_GPU_HPP_
