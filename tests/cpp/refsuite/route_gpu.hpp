// Force-included (g++ -include) into the reference's own unit suites
// (/root/reference/proj/tests/test_*.cpp, compiled from where they lie, never copied) so that
// their calls to the hot-path API run on the B200 engine through include/quasar_gpu.hpp.
//
// Each overload below has the reference template's exact signature plus one more constraint:
// C++20 partial ordering by constraints (Word<W> && GpuRoute<W> subsumes Word<W>) makes it the
// better match for every call the suites make — unqualified, `quasar::`-qualified or with
// explicit template arguments — without editing a reference header. What cannot be rerouted
// this way stays the reference's: Tableau members (transpose_in_place, check_group_validity;
// the shim's free quasar::gpu::transpose_in_place is covered by tests/cpp/dropin_test.cpp) and
// non-template inline functions (schedule_windows, generate_random, parse_qasm / emit_qasm;
// their product counterparts are compared with the reference in tests/test_host.py,
// tests/test_qasm.py). Test infrastructure only.
#pragma once

#include "quasar_gpu.hpp"

namespace quasar {

template <typename W>
concept GpuRoute = true;

template <Word W> requires GpuRoute<W>
void apply_window(Tableau<W> &tableau, const Window &window) {
    gpu::apply_window(tableau, window);
}

template <Word W> requires GpuRoute<W>
void measure_window(Tableau<W> &t, const Window &window, RandomStream &rng, MeasurementRecord &record,
                    MeasureScratch<W> &scratch, PhaseTimers *timers = nullptr) {
    gpu::measure_window(t, window, rng, record, scratch, timers);
}

template <Word W> requires GpuRoute<W>
std::vector<int64_t> find_probabilistic(const Tableau<W> &t, const Window &window) {
    return gpu::find_probabilistic(t, window);
}

template <Word W> requires GpuRoute<W>
PivotList find_and_compact_pivots(const Tableau<W> &t, size_t q, MeasureScratch<W> &scratch) {
    return gpu::find_and_compact_pivots(t, q, scratch);
}

template <Word W> requires GpuRoute<W>
void parallel_ge(Tableau<W> &t, const PivotList &pivots, MeasureScratch<W> &scratch,
                 size_t block_targets = kGeBlockTargets) {
    gpu::parallel_ge(t, pivots, scratch, block_targets);
}

template <Word W> requires GpuRoute<W>
void swap_anti_commuting(Tableau<W> &t, size_t p, size_t q, MeasureScratch<W> &scratch) {
    gpu::swap_anti_commuting(t, p, q, scratch);
}

template <Word W> requires GpuRoute<W>
void inject_x(Tableau<W> &t, size_t p) {
    gpu::inject_x(t, p);
}

template <Word W> requires GpuRoute<W>
bool deterministic_outcome(const Tableau<W> &t, size_t q, MeasureScratch<W> &scratch) {
    return gpu::deterministic_outcome(t, q, scratch);
}

template <Word W> requires GpuRoute<W>
SingleShotResult<W> run_single_shot(const Circuit &circuit, const Schedule &schedule, uint64_t seed) {
    return gpu::run_single_shot<W>(circuit, schedule, seed);
}

template <Word W> requires GpuRoute<W>
SingleShotResult<W> run_single_shot(const Circuit &circuit, uint64_t seed) {
    return gpu::run_single_shot<W>(circuit, seed);
}

template <Word W> requires GpuRoute<W>
FrameTableau<W> init_frames(size_t n, size_t shots, uint64_t seed) {
    return gpu::init_frames<W>(n, shots, seed);
}

template <Word W> requires GpuRoute<W>
void apply_window_frames(FrameTableau<W> &f, const Window &window) {
    gpu::apply_window_frames(f, window);
}

template <Word W> requires GpuRoute<W>
void measure_sample(FrameTableau<W> &f, const Window &window, ShotRecord<W> &record, uint64_t seed,
                    uint32_t epoch) {
    gpu::measure_sample(f, window, record, seed, epoch);
}

template <Word W> requires GpuRoute<W>
ShotRecord<W> sample(const Circuit &circuit, size_t shots, uint64_t seed, RunReport *report = nullptr) {
    return gpu::sample<W>(circuit, shots, seed, report);
}

} // namespace quasar
