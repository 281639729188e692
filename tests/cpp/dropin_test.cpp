// Drop-in check of include/quasar_gpu.hpp: the reference's own API calls, made once through
// the reference (quasar::, CPU) and once through the B200 engine (quasar::gpu::), on the same
// reference types, must agree bit for bit — tableaux under Tableau::operator== (raw storage
// incl. padding, tableau.hpp:250-253), every record entry, every sampled word, the schedule,
// and the caller's RandomStream position. Mirrors test_measure.cpp:315-335,
// test_gates.cpp:176-201, test_frames.cpp:188-204 and test_schedule.cpp:111-129.
// Built by tests/cpp/Makefile against the reference headers; run by tests/test_cpp_dropin.py.
#include <cstdio>
#include <cstdlib>

#include "quasar_gpu.hpp"

using namespace quasar;

static int failures = 0;
#define CHECK(cond)                                                                       \
    do {                                                                                  \
        if (!(cond)) {                                                                    \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);                   \
            ++failures;                                                                   \
        }                                                                                 \
    } while (0)

static bool same_record(const MeasurementRecord &a, const MeasurementRecord &b) {
    if (a.entries.size() != b.entries.size()) return false;
    for (size_t i = 0; i < a.entries.size(); ++i) {
        const auto &x = a.entries[i], &y = b.entries[i];
        if (x.qubit != y.qubit || x.outcome != y.outcome || x.deterministic != y.deterministic)
            return false;
    }
    return true;
}

int main() {
    // run_single_shot over random circuits (both overloads)
    for (uint64_t seed = 0; seed < 24; ++seed) {
        uint32_t n = 2 + uint32_t((seed * 37) % 140);
        Circuit c = generate_random(n, 4 + seed % 40, seed * 31 + 1, (seed % 5) * 0.25);
        auto cpu = run_single_shot<uint64_t>(c, seed);
        auto gpu = gpu::run_single_shot<uint64_t>(c, seed);
        CHECK(cpu.tableau == gpu.tableau);
        CHECK(same_record(cpu.record, gpu.record));
        CHECK(cpu.report.probabilistic_count == gpu.report.probabilistic_count);
        CHECK(gpu.tableau.padding_clean());
        Schedule s = schedule_windows(c, ScheduleMode::single_shot);
        auto gpu2 = gpu::run_single_shot<uint64_t>(c, s, seed + 1);
        auto cpu2 = run_single_shot<uint64_t>(c, s, seed + 1);
        CHECK(cpu2.tableau == gpu2.tableau);
        CHECK(same_record(cpu2.record, gpu2.record));
    }
    // schedule_windows and generate_random
    for (uint64_t seed = 0; seed < 50; ++seed) {
        Circuit c = generate_random(1 + seed % 64, 1 + (seed * 7) % 20, seed, 0.4);
        Circuit g = gpu::generate_random(1 + seed % 64, 1 + (seed * 7) % 20, seed, 0.4);
        CHECK(c == g);
        Schedule a = schedule_windows(c, ScheduleMode::single_shot);
        Schedule b = gpu::schedule_windows(c, ScheduleMode::single_shot);
        CHECK(a.windows.size() == b.windows.size());
        for (size_t w = 0; w < a.windows.size() && w < b.windows.size(); ++w) {
            CHECK(a.windows[w].is_measurement == b.windows[w].is_measurement);
            CHECK(a.windows[w].gates == b.windows[w].gates);
        }
        CHECK(validate_schedule(c, b) == "valid");
    }
    // apply_window + measure_window with a caller stream that is NOT kStreamMeasure
    for (uint64_t seed = 0; seed < 10; ++seed) {
        size_t n = 10 + seed * 13;
        Circuit c = generate_random(uint32_t(n), 14, seed + 100, 0.0);
        Schedule s = schedule_windows(c, ScheduleMode::single_shot);
        auto tc = Tableau<uint64_t>::zero_state(n), tg = tc;
        for (const Window &w : s.windows) {
            apply_window(tc, w);
            gpu::apply_window(tg, w);
        }
        CHECK(tc == tg);
        Window m;
        m.is_measurement = true;
        for (uint32_t q = 0; q < n; q += 2) m.gates.push_back({GateKind::MEASURE, q});
        RandomStream rc(seed * 5 + 3, 9, 4), rg(seed * 5 + 3, 9, 4);
        MeasurementRecord recc, recg;
        MeasureScratch<uint64_t> scratch;
        measure_window(tc, m, rc, recc, scratch);
        gpu::measure_window(tg, m, rg, recg, scratch);
        CHECK(tc == tg);
        CHECK(same_record(recc, recg));
        CHECK(rc.next_word() == rg.next_word()); // both streams advanced by the same count
    }
    // error behaviour: same exception types
    {
        Circuit dup;
        dup.num_qubits = 1;
        dup.gates = {{GateKind::MEASURE, 0}, {GateKind::MEASURE, 0}};
        bool threw = false;
        try { gpu::run_single_shot<uint64_t>(dup, 1); } catch (const std::invalid_argument &) { threw = true; }
        CHECK(threw);
        Circuit bad;
        bad.num_qubits = 2;
        bad.gates = {{GateKind::H, 5}};
        threw = false;
        try { gpu::run_single_shot<uint64_t>(bad, 1); } catch (const std::out_of_range &) { threw = true; }
        CHECK(threw);
        auto t = Tableau<uint64_t>::zero_state(3);
        Window overlap;
        overlap.gates = {{GateKind::H, 0}, {GateKind::CX, 0, 1}};
        threw = false;
        try { gpu::apply_window(t, overlap); } catch (const std::invalid_argument &) { threw = true; }
        CHECK(threw);
    }
    // sample
    for (uint64_t seed = 0; seed < 6; ++seed) {
        Circuit c = generate_random(uint32_t(4 + seed * 5), 10 + uint32_t(seed), 91 + seed, 0.8);
        for (size_t shots : {size_t(1), size_t(64), size_t(130), size_t(1000)}) {
            RunReport rc, rg;
            auto a = sample<uint64_t>(c, shots, 1234 + seed, &rc);
            auto b = gpu::sample<uint64_t>(c, shots, 1234 + seed, &rg);
            CHECK(a.measured == b.measured);
            CHECK(a.words == b.words);
            CHECK(a.kf == b.kf && a.shots == b.shots);
            CHECK(rc.probabilistic_count == rg.probabilistic_count);
        }
    }
    // run_single_shot / apply_window / measure_window / check_group_validity for the other W
    for (uint64_t seed = 0; seed < 6; ++seed) {
        const uint32_t n = 3 + uint32_t(seed * 23);
        Circuit c = generate_random(n, 8 + uint32_t(seed), 700 + seed, 0.5);
        auto a8 = run_single_shot<uint8_t>(c, seed);
        auto b8 = gpu::run_single_shot<uint8_t>(c, seed);
        CHECK(a8.tableau == b8.tableau && same_record(a8.record, b8.record));
        auto a32 = run_single_shot<uint32_t>(c, seed);
        auto b32 = gpu::run_single_shot<uint32_t>(c, seed);
        CHECK(a32.tableau == b32.tableau && same_record(a32.record, b32.record));
        CHECK(gpu::check_group_validity(b32.tableau) == "valid");
        Schedule s = schedule_windows(c, ScheduleMode::single_shot);
        auto ta = Tableau<uint16_t>::zero_state(n), tb = Tableau<uint16_t>::zero_state(n);
        RandomStream ra(seed, kStreamMeasure), rb(seed, kStreamMeasure);
        MeasurementRecord ma, mb;
        MeasureScratch<uint16_t> sa, sb;
        for (const Window &w : s.windows) {
            if (w.is_measurement) {
                measure_window(ta, w, ra, ma, sa);
                gpu::measure_window(tb, w, rb, mb, sb);
            } else {
                apply_window(ta, w);
                gpu::apply_window(tb, w);
            }
        }
        CHECK(ta == tb && same_record(ma, mb) && ra.next_word() == rb.next_word());
    }
    // sample<W> for the reference's other word types
    for (uint64_t seed = 0; seed < 3; ++seed) {
        Circuit c = generate_random(uint32_t(6 + seed * 7), 12, 300 + seed, 0.7);
        for (size_t shots : {size_t(1), size_t(9), size_t(777)}) {
            auto a8 = sample<uint8_t>(c, shots, seed);
            auto b8 = gpu::sample<uint8_t>(c, shots, seed);
            CHECK(a8.measured == b8.measured && a8.words == b8.words && a8.kf == b8.kf);
            auto a16 = sample<uint16_t>(c, shots, seed);
            auto b16 = gpu::sample<uint16_t>(c, shots, seed);
            CHECK(a16.measured == b16.measured && a16.words == b16.words && a16.kf == b16.kf);
            auto a32 = sample<uint32_t>(c, shots, seed);
            auto b32 = gpu::sample<uint32_t>(c, shots, seed);
            CHECK(a32.measured == b32.measured && a32.words == b32.words && a32.kf == b32.kf);
        }
    }
    // parse_qasm / emit_qasm (qasm.hpp), QasmError position and reason
    for (uint64_t seed : {1ull, 2ull, 99ull}) {
        Circuit c = generate_random(100, 60, seed, 0.5);
        std::string text = emit_qasm(c);
        CHECK(gpu::emit_qasm(c) == text);
        Circuit p = gpu::parse_qasm(text);
        CHECK(p == parse_qasm(text) && p.num_clbits == parse_qasm(text).num_clbits);
    }
    for (const char *bad : {"OPENQASM 2.0;\nqreg q[1];\nt q[0];\n", "OPENQASM 2.0;\nqreg q[2];\ncx q[1],q[1];\n",
                            "qreg q[2];\n", "OPENQASM 2.0;\nqreg q[2];\nh q[0]\n"}) {
        std::string ref_what, gpu_what;
        int rl = -1, rc = -1, gl = -2, gc = -2;
        try { parse_qasm(bad); } catch (const QasmError &e) { ref_what = e.what(); rl = e.line; rc = e.column; }
        try { gpu::parse_qasm(bad); } catch (const QasmError &e) { gpu_what = e.what(); gl = e.line; gc = e.column; }
        CHECK(!ref_what.empty() && ref_what == gpu_what && rl == gl && rc == gc);
    }
    // check_group_validity on evolved and on corrupted tableaux
    for (uint64_t seed = 0; seed < 8; ++seed) {
        Circuit c = generate_random(uint32_t(5 + seed * 19), 12, 500 + seed, 0.4);
        auto r = run_single_shot<uint64_t>(c, seed);
        CHECK(gpu::check_group_validity(r.tableau) == "valid");
        auto t = r.tableau;
        t.x_plane()[(seed * 7) % t.num_qubits() * 2 * t.num_words()] ^= uint64_t(1) << (seed % 5);
        CHECK(gpu::check_group_validity(t) == t.check_group_validity());
    }
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "dropin ok", failures);
    return failures ? 1 : 0;
}
