// TEST INFRASTRUCTURE ONLY — the reference implementation behind orc.h.
//
// Compiles the reference headers (/root/reference/proj/include/quasar, unmodified, not
// copied) into oracle/_ref/libquasar_ref.so so that tests and bench.py's reference arm can
// call the reference's own run_single_shot / measure_window / sample on the same inputs as
// the CUDA engine. Build recipe: oracle/Makefile (target `ref`).
#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>

#include "orc.h"
#include "quasar/frames.hpp"
#include "quasar/measure.hpp"
#include "quasar/qasm.hpp"
#include "quasar/simulator.hpp"

using namespace quasar;
using T64 = Tableau<uint64_t>;

static_assert(sizeof(Gate) == sizeof(orc_gate), "Gate layout");
static_assert(sizeof(MeasurementRecord::Entry) == sizeof(orc_entry), "Entry layout");

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F &&f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument &e) {
        g_err = e.what();
        return 1;
    } catch (const std::out_of_range &e) {
        g_err = e.what();
        return 2;
    } catch (const std::logic_error &e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception &e) {
        g_err = e.what();
        return 7;
    }
}

T64 load(uint64_t n, int layout, const uint64_t *x, const uint64_t *z, const uint64_t *s) {
    T64 t(n);
    if (layout == 1) t.transpose_in_place(); // layout tag only; storage overwritten below
    std::memcpy(t.x_plane().data(), x, t.plane_words() * 8);
    std::memcpy(t.z_plane().data(), z, t.plane_words() * 8);
    if (s) std::memcpy(t.signs().data(), s, t.signs().size() * 8);
    return t;
}

void store(const T64 &t, uint64_t *x, uint64_t *z, uint64_t *s) {
    if (x) std::memcpy(x, t.x_plane().data(), t.plane_words() * 8);
    if (z) std::memcpy(z, t.z_plane().data(), t.plane_words() * 8);
    if (s) std::memcpy(s, t.signs().data(), t.signs().size() * 8);
}

Window window_of(const orc_gate *g, uint64_t ng, bool meas) {
    Window w;
    w.is_measurement = meas;
    w.gates.resize(ng);
    if (ng) std::memcpy(w.gates.data(), g, ng * sizeof(Gate));
    return w;
}

Circuit circuit_of(uint64_t n, const orc_gate *g, uint64_t ng) {
    Circuit c;
    c.num_qubits = uint32_t(n);
    c.gates.resize(ng);
    if (ng) std::memcpy(c.gates.data(), g, ng * sizeof(Gate));
    c.num_clbits = uint32_t(n);
    return c;
}

Schedule schedule_of(const orc_gate *sg, const uint64_t *off, const uint8_t *is_meas,
                     uint64_t nwin) {
    Schedule s;
    for (uint64_t w = 0; w < nwin; ++w)
        s.windows.push_back(window_of(sg + off[w], off[w + 1] - off[w], is_meas[w] != 0));
    return s;
}

void report_of(const RunReport &r, orc_report *rep) {
    if (!rep) return;
    rep->to_s = r.timers.to_seconds;
    rep->t_s = r.timers.t_seconds;
    rep->cmp_s = r.timers.cmp_seconds;
    rep->ge_s = r.timers.ge_seconds;
    rep->gate_count = r.gate_count;
    rep->measure_count = r.measure_count;
    rep->probabilistic_count = r.probabilistic_count;
    rep->window_count = r.window_count;
    rep->total_s = r.total_seconds;
}
} // namespace

extern "C" {

const char *orc_last_error(void) { return g_err.c_str(); }
const char *orc_name(void) { return "reference"; }
void orc_set_threads(unsigned threads) { set_num_threads(threads); }

void orc_philox_block(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    auto o = Philox::block({ctr[0], ctr[1], ctr[2], ctr[3]}, {key[0], key[1]});
    for (int i = 0; i < 4; ++i) out[i] = o[i];
}
uint64_t orc_philox_word(uint64_t seed, uint32_t stream, uint32_t ctx, uint64_t index) {
    return Philox::word_at(seed, stream, ctx, index);
}

int orc_generate_random(uint32_t n, uint32_t depth, uint64_t seed, double p, orc_gate *out,
                        uint64_t cap, uint64_t *count) {
    return guard([&] {
        Circuit c = generate_random(n, depth, seed, p);
        *count = c.gates.size();
        if (out) std::memcpy(out, c.gates.data(), std::min<uint64_t>(cap, c.gates.size()) * sizeof(Gate));
    });
}

int orc_schedule(uint32_t n, const orc_gate *g, uint64_t ng, int mode, orc_gate *out_gates,
                 uint64_t *offsets, uint8_t *is_meas, uint64_t *nwin) {
    return guard([&] {
        Circuit c = circuit_of(n, g, ng);
        Schedule s = schedule_windows(c, mode ? ScheduleMode::sampling : ScheduleMode::single_shot);
        uint64_t pos = 0;
        offsets[0] = 0;
        for (size_t w = 0; w < s.windows.size(); ++w) {
            for (const Gate &gate : s.windows[w].gates) std::memcpy(out_gates + pos++, &gate, sizeof(Gate));
            offsets[w + 1] = pos;
            is_meas[w] = s.windows[w].is_measurement;
        }
        *nwin = s.windows.size();
    });
}

int orc_basis_state(uint64_t n, const uint8_t *bits, uint64_t *x, uint64_t *z, uint64_t *s) {
    return guard([&] {
        std::vector<bool> init(n, false);
        if (bits) for (uint64_t i = 0; i < n; ++i) init[i] = bits[i] != 0;
        store(T64::basis_state(init), x, z, s);
    });
}

int orc_apply_window(uint64_t n, int layout, uint64_t *x, uint64_t *z, uint64_t *s,
                     const orc_gate *g, uint64_t ng) {
    return guard([&] {
        T64 t = load(n, layout, x, z, s);
        apply_window(t, window_of(g, ng, false));
        store(t, x, z, s);
    });
}

int orc_transpose(uint64_t n, int *layout, uint64_t *x, uint64_t *z) {
    return guard([&] {
        T64 t = load(n, *layout, x, z, nullptr);
        t.transpose_in_place();
        *layout = t.layout() == Layout::RowMajor ? 1 : 0;
        store(t, x, z, nullptr);
    });
}

int orc_find_probabilistic(uint64_t n, int layout, const uint64_t *x, const uint64_t *z,
                           const orc_gate *g, uint64_t ng, int64_t *out) {
    return guard([&] {
        T64 t = load(n, layout, x, z, nullptr);
        auto r = find_probabilistic(t, window_of(g, ng, true));
        std::memcpy(out, r.data(), r.size() * 8);
    });
}

int orc_find_and_compact_pivots(uint64_t n, int layout, const uint64_t *x, const uint64_t *z,
                                uint64_t q, int64_t *entries, uint64_t *count) {
    return guard([&] {
        T64 t = load(n, layout, x, z, nullptr);
        MeasureScratch<uint64_t> scratch;
        PivotList p = find_and_compact_pivots(t, q, scratch);
        std::memcpy(entries, p.entries.data(), p.entries.size() * 8);
        *count = p.count;
    });
}

int orc_parallel_ge(uint64_t n, int layout, uint64_t *x, uint64_t *z, uint64_t *s,
                    const int64_t *entries, uint64_t count, uint64_t block) {
    return guard([&] {
        T64 t = load(n, layout, x, z, s);
        PivotList p;
        p.entries.assign(n, -1);
        for (uint64_t i = 0; i < count && i < n; ++i) p.entries[i] = entries[i];
        p.count = count;
        MeasureScratch<uint64_t> scratch;
        parallel_ge(t, p, scratch, block);
        store(t, x, z, s);
    });
}

int orc_swap_anti_commuting(uint64_t n, int layout, uint64_t *x, uint64_t *z, uint64_t *s,
                            uint64_t p, uint64_t q) {
    return guard([&] {
        T64 t = load(n, layout, x, z, s);
        MeasureScratch<uint64_t> scratch;
        swap_anti_commuting(t, p, q, scratch);
        store(t, x, z, s);
    });
}

int orc_inject_x(uint64_t n, uint64_t *s, uint64_t p) {
    return guard([&] {
        uint64_t k = (n + 63) / 64;
        (void)k;
        uint64_t idx = p;
        s[k + idx / 64] ^= uint64_t(1) << (idx % 64);
    });
}

int orc_deterministic_outcome(uint64_t n, int layout, const uint64_t *x, const uint64_t *z,
                              const uint64_t *s, uint64_t q, uint8_t *out) {
    return guard([&] {
        T64 t = load(n, layout, x, z, s);
        MeasureScratch<uint64_t> scratch;
        *out = deterministic_outcome(t, q, scratch) ? 1 : 0;
    });
}

int orc_measure_window(uint64_t n, int layout, uint64_t *x, uint64_t *z, uint64_t *s,
                       const orc_gate *g, uint64_t ng, uint64_t seed, uint64_t *coin_index,
                       orc_entry *out) {
    return guard([&] {
        T64 t = load(n, layout, x, z, s);
        RandomStream rng(seed, kStreamMeasure);
        for (uint64_t i = 0; i < *coin_index; ++i) rng.next_word();
        // Count coins consumed: a fresh stream at the same index plus the record.
        MeasurementRecord rec;
        MeasureScratch<uint64_t> scratch;
        measure_window(t, window_of(g, ng, true), rng, rec, scratch);
        uint64_t used = 0;
        for (const auto &e : rec.entries) used += e.deterministic ? 0 : 1;
        *coin_index += used;
        std::memcpy(out, rec.entries.data(), rec.entries.size() * sizeof(orc_entry));
        store(t, x, z, s);
    });
}

int orc_run_schedule(uint64_t n, const orc_gate *sg, const uint64_t *off, const uint8_t *is_meas,
                     uint64_t nwin, uint64_t seed, uint64_t *x, uint64_t *z, uint64_t *s,
                     orc_entry *rec, uint64_t *nrec, orc_report *rep) {
    return guard([&] {
        Schedule sched = schedule_of(sg, off, is_meas, nwin);
        Circuit c;
        c.num_qubits = uint32_t(n);
        for (const auto &w : sched.windows)
            c.gates.insert(c.gates.end(), w.gates.begin(), w.gates.end());
        auto r = run_single_shot<uint64_t>(c, sched, seed);
        store(r.tableau, x, z, s);
        *nrec = r.record.entries.size();
        if (rec) std::memcpy(rec, r.record.entries.data(), r.record.entries.size() * sizeof(orc_entry));
        report_of(r.report, rep);
    });
}

int orc_run_single_shot(uint64_t n, const orc_gate *g, uint64_t ng, uint64_t seed, uint64_t *x,
                        uint64_t *z, uint64_t *s, orc_entry *rec, uint64_t *nrec, orc_report *rep) {
    return guard([&] {
        Circuit c = circuit_of(n, g, ng);
        auto r = run_single_shot<uint64_t>(c, seed);
        store(r.tableau, x, z, s);
        *nrec = r.record.entries.size();
        if (rec) std::memcpy(rec, r.record.entries.data(), r.record.entries.size() * sizeof(orc_entry));
        report_of(r.report, rep);
    });
}

int orc_bench_windows(uint32_t n, uint32_t layers, uint64_t seed, double *seconds, uint64_t *gates) {
    return guard([&] {
        Circuit c = generate_random(n, layers, seed, 0.0);
        Schedule s = schedule_windows(c, ScheduleMode::single_shot);
        auto t = T64::zero_state(n);
        for (size_t w = 0; w < s.windows.size() && w < layers; ++w) {
            auto t0 = std::chrono::steady_clock::now();
            apply_window(t, s.windows[w]);
            seconds[w] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            gates[w] = s.windows[w].gates.size();
        }
    });
}

int orc_init_frames(uint64_t n, uint64_t shots, uint64_t seed, uint64_t *xf, uint64_t *zf) {
    return guard([&] {
        auto f = init_frames<uint64_t>(n, shots, seed);
        std::memcpy(xf, f.xf.data(), f.xf.size() * 8);
        std::memcpy(zf, f.zf.data(), f.zf.size() * 8);
    });
}

int orc_apply_window_frames(uint64_t n, uint64_t shots, uint64_t *xf, uint64_t *zf,
                            const orc_gate *g, uint64_t ng) {
    return guard([&] {
        FrameTableau<uint64_t> f;
        f.n = n;
        f.shots = shots;
        f.kf = words_for<uint64_t>(shots);
        f.xf.assign(xf, xf + n * f.kf);
        f.zf.assign(zf, zf + n * f.kf);
        apply_window_frames(f, window_of(g, ng, false));
        std::memcpy(xf, f.xf.data(), f.xf.size() * 8);
        std::memcpy(zf, f.zf.data(), f.zf.size() * 8);
    });
}

int orc_measure_sample(uint64_t n, uint64_t shots, uint64_t *xf, uint64_t *zf, const orc_gate *g,
                       uint64_t ng, uint64_t seed, uint32_t epoch, uint32_t *measured,
                       uint64_t *nrows, uint64_t *words) {
    return guard([&] {
        FrameTableau<uint64_t> f;
        f.n = n;
        f.shots = shots;
        f.kf = words_for<uint64_t>(shots);
        f.xf.assign(xf, xf + n * f.kf);
        f.zf.assign(zf, zf + n * f.kf);
        ShotRecord<uint64_t> rec;
        rec.shots = shots;
        rec.kf = f.kf;
        rec.measured.assign(measured, measured + *nrows);
        rec.words.assign(words, words + *nrows * f.kf);
        measure_sample(f, window_of(g, ng, true), rec, seed, epoch);
        std::memcpy(xf, f.xf.data(), f.xf.size() * 8);
        std::memcpy(zf, f.zf.data(), f.zf.size() * 8);
        *nrows = rec.measured.size();
        std::memcpy(measured, rec.measured.data(), rec.measured.size() * 4);
        std::memcpy(words, rec.words.data(), rec.words.size() * 8);
    });
}

int orc_sample(uint64_t n, const orc_gate *g, uint64_t ng, uint64_t shots, uint64_t seed,
               uint32_t *measured, uint64_t *nrows, uint64_t *words, orc_report *rep) {
    return guard([&] {
        Circuit c = circuit_of(n, g, ng);
        RunReport r;
        auto rec = sample<uint64_t>(c, shots, seed, &r);
        *nrows = rec.measured.size();
        if (measured) std::memcpy(measured, rec.measured.data(), rec.measured.size() * 4);
        if (words) std::memcpy(words, rec.words.data(), rec.words.size() * 8);
        report_of(r, rep);
    });
}

// ---- reference-only entry points (formats either side of the path; no C restatement) ----

static int text_result(const std::string &t, char *buf, uint64_t cap, uint64_t *len) {
    *len = t.size();
    if (buf) std::memcpy(buf, t.data(), std::min<uint64_t>(cap, t.size()));
    return 0;
}

int orc_ref_parse_qasm(const char *text, uint64_t len, uint32_t *n, uint32_t *nclbits, orc_gate *out,
                       uint64_t cap, uint64_t *count, int *line, int *col) {
    *line = *col = 0;
    try {
        Circuit c = parse_qasm(std::string_view(text, len));
        *n = c.num_qubits;
        *nclbits = c.num_clbits;
        *count = c.gates.size();
        if (out) std::memcpy(out, c.gates.data(), std::min<uint64_t>(cap, c.gates.size()) * sizeof(Gate));
        return 0;
    } catch (const QasmError &e) {
        g_err = e.what();
        *line = e.line;
        *col = e.column;
        return 8;
    } catch (const std::exception &e) {
        g_err = e.what();
        return 7;
    }
}

int orc_ref_emit_qasm(uint32_t n, const orc_gate *g, uint64_t ng, char *buf, uint64_t cap, uint64_t *len) {
    return guard([&] { text_result(emit_qasm(circuit_of(n, g, ng)), buf, cap, len); });
}

int orc_ref_schedule_text(uint32_t n, const orc_gate *g, uint64_t ng, int mode, char *buf, uint64_t cap,
                          uint64_t *len) {
    return guard([&] {
        Circuit c = circuit_of(n, g, ng);
        Schedule s = schedule_windows(c, mode ? ScheduleMode::sampling : ScheduleMode::single_shot);
        text_result(schedule_to_text(s), buf, cap, len);
    });
}

int orc_ref_validate_schedule(uint32_t n, const orc_gate *g, uint64_t ng, const orc_gate *sg,
                              const uint64_t *off, const uint8_t *is_meas, uint64_t nwin, char *buf,
                              uint64_t cap, uint64_t *len) {
    return guard([&] {
        text_result(validate_schedule(circuit_of(n, g, ng), schedule_of(sg, off, is_meas, nwin)), buf, cap,
                    len);
    });
}

// sample<W> for W in {8, 16, 32, 64}: rows of kf W-words, written as little-endian bytes.
int orc_ref_sample_w(uint64_t n, const orc_gate *g, uint64_t ng, uint64_t shots, uint64_t seed,
                     unsigned wbits, uint32_t *measured, uint64_t *nrows, uint64_t *kf, uint8_t *bytes) {
    return guard([&] {
        Circuit c = circuit_of(n, g, ng);
        auto run = [&](auto w) {
            using W = decltype(w);
            auto rec = sample<W>(c, shots, seed);
            *nrows = rec.measured.size();
            *kf = rec.kf;
            if (measured) std::memcpy(measured, rec.measured.data(), rec.measured.size() * 4);
            if (bytes)
                for (size_t i = 0; i < rec.words.size(); ++i)
                    for (size_t b = 0; b < sizeof(W); ++b)
                        bytes[i * sizeof(W) + b] = uint8_t((uint64_t(rec.words[i]) >> (8 * b)) & 0xFF);
        };
        switch (wbits) {
        case 8: run(uint8_t{}); break;
        case 16: run(uint16_t{}); break;
        case 32: run(uint32_t{}); break;
        case 64: run(uint64_t{}); break;
        default: throw std::invalid_argument("word size must be one of 8, 16, 32, 64");
        }
    });
}

int orc_ref_check_validity(uint64_t n, int layout, const uint64_t *x, const uint64_t *z, char *buf,
                           uint64_t cap, uint64_t *len) {
    return guard([&] { text_result(load(n, layout, x, z, nullptr).check_group_validity(), buf, cap, len); });
}

} // extern "C"
