/*
 * orc.h — CPU oracle interface (TEST INFRASTRUCTURE ONLY).
 *
 * Two implementations export this interface:
 *   oracle/liboracle.so          — qsr_oracle.c, a plain-C restatement of the reference
 *                                  algorithm for the hot path (each function cites the
 *                                  reference file:line it follows);
 *   oracle/_ref/libquasar_ref.so — ref_capi.cpp, the reference's own headers
 *                                  (/root/reference/proj/include/quasar) compiled unmodified
 *                                  behind this interface (built here, travels prebuilt).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load either library. The product (libqsr.so) never links or calls them.
 *
 * Host buffers use the reference's storage layout (tableau.hpp:51-61): x, z = n_pad*2k
 * words, s = 2k words; layout 0 = ColumnMajor, 1 = RowMajor. Status codes match qsr.h.
 */
#ifndef ORC_H_
#define ORC_H_
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_gate { uint8_t kind; uint32_t q0; uint32_t q1; } orc_gate;
typedef struct orc_entry { uint32_t qubit; uint8_t outcome; uint8_t deterministic; } orc_entry;
typedef struct orc_report {
    double to_s, t_s, cmp_s, ge_s;
    uint64_t gate_count, measure_count, probabilistic_count, window_count;
    double total_s;
} orc_report;

const char *orc_last_error(void);
const char *orc_name(void);
void orc_set_threads(unsigned threads);

void orc_philox_block(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
uint64_t orc_philox_word(uint64_t seed, uint32_t stream, uint32_t ctx, uint64_t index);

/* generate_random; writes min(count, cap) gates, *count = total. */
int orc_generate_random(uint32_t n, uint32_t depth, uint64_t seed, double p, orc_gate *out,
                        uint64_t cap, uint64_t *count);
/* schedule_windows: out_gates (cap ng), offsets (cap ng+1), is_meas (cap ng). */
int orc_schedule(uint32_t n, const orc_gate *g, uint64_t ng, int mode, orc_gate *out_gates,
                 uint64_t *offsets, uint8_t *is_meas, uint64_t *nwin);

int orc_basis_state(uint64_t n, const uint8_t *bits, uint64_t *x, uint64_t *z, uint64_t *s);
int orc_apply_window(uint64_t n, int layout, uint64_t *x, uint64_t *z, uint64_t *s,
                     const orc_gate *g, uint64_t ng);
int orc_transpose(uint64_t n, int *layout, uint64_t *x, uint64_t *z);
int orc_find_probabilistic(uint64_t n, int layout, const uint64_t *x, const uint64_t *z,
                           const orc_gate *g, uint64_t ng, int64_t *out);
int orc_find_and_compact_pivots(uint64_t n, int layout, const uint64_t *x, const uint64_t *z,
                                uint64_t q, int64_t *entries, uint64_t *count);
int orc_parallel_ge(uint64_t n, int layout, uint64_t *x, uint64_t *z, uint64_t *s,
                    const int64_t *entries, uint64_t count, uint64_t block);
int orc_swap_anti_commuting(uint64_t n, int layout, uint64_t *x, uint64_t *z, uint64_t *s,
                            uint64_t p, uint64_t q);
int orc_inject_x(uint64_t n, uint64_t *s, uint64_t p);
int orc_deterministic_outcome(uint64_t n, int layout, const uint64_t *x, const uint64_t *z,
                              const uint64_t *s, uint64_t q, uint8_t *out);
int orc_measure_window(uint64_t n, int layout, uint64_t *x, uint64_t *z, uint64_t *s,
                       const orc_gate *g, uint64_t ng, uint64_t seed, uint64_t *coin_index,
                       orc_entry *out);
/* run_single_shot over an explicit schedule (flattened windows). */
int orc_run_schedule(uint64_t n, const orc_gate *sg, const uint64_t *offsets,
                     const uint8_t *is_meas, uint64_t nwin, uint64_t seed, uint64_t *x,
                     uint64_t *z, uint64_t *s, orc_entry *rec, uint64_t *nrec, orc_report *rep);
/* run_single_shot(circuit, seed). */
int orc_run_single_shot(uint64_t n, const orc_gate *g, uint64_t ng, uint64_t seed, uint64_t *x,
                        uint64_t *z, uint64_t *s, orc_entry *rec, uint64_t *nrec, orc_report *rep);

/* CPU-baseline timer: the first `layers` layers of generate_random(n, *, seed, *) are
 * scheduled and applied window by window to a zero state; per-window wall seconds and gate
 * counts are returned (arrays of `layers` entries; unitary layers = unitary windows). */
int orc_bench_windows(uint32_t n, uint32_t layers, uint64_t seed, double *seconds, uint64_t *gates);

/* Frames; xf/zf = n*kf words. */
int orc_init_frames(uint64_t n, uint64_t shots, uint64_t seed, uint64_t *xf, uint64_t *zf);
int orc_apply_window_frames(uint64_t n, uint64_t shots, uint64_t *xf, uint64_t *zf,
                            const orc_gate *g, uint64_t ng);
/* measure_sample with a caller-held record: measured (cap n), *nrows in/out, words (cap n*kf). */
int orc_measure_sample(uint64_t n, uint64_t shots, uint64_t *xf, uint64_t *zf, const orc_gate *g,
                       uint64_t ng, uint64_t seed, uint32_t epoch, uint32_t *measured,
                       uint64_t *nrows, uint64_t *words);
/* sample(circuit, shots, seed): measured (cap n), words (cap n*kf). */
int orc_sample(uint64_t n, const orc_gate *g, uint64_t ng, uint64_t shots, uint64_t seed,
               uint32_t *measured, uint64_t *nrows, uint64_t *words, orc_report *rep);

/* ---- reference-only (oracle/_ref/libquasar_ref.so; the C port has no counterpart) ---- */
/* parse_qasm: 0, or 8 = QasmError (orc_last_error() = what(), *line / *col set). */
int orc_ref_parse_qasm(const char *text, uint64_t len, uint32_t *n, uint32_t *nclbits, orc_gate *out,
                       uint64_t cap, uint64_t *count, int *line, int *col);
/* Text results: *len = full size, min(cap, size) bytes copied to buf (may be NULL). */
int orc_ref_emit_qasm(uint32_t n, const orc_gate *g, uint64_t ng, char *buf, uint64_t cap, uint64_t *len);
int orc_ref_schedule_text(uint32_t n, const orc_gate *g, uint64_t ng, int mode, char *buf, uint64_t cap,
                          uint64_t *len);
int orc_ref_validate_schedule(uint32_t n, const orc_gate *g, uint64_t ng, const orc_gate *sg,
                              const uint64_t *off, const uint8_t *is_meas, uint64_t nwin, char *buf,
                              uint64_t cap, uint64_t *len);
int orc_ref_sample_w(uint64_t n, const orc_gate *g, uint64_t ng, uint64_t shots, uint64_t seed,
                     unsigned wbits, uint32_t *measured, uint64_t *nrows, uint64_t *kf, uint8_t *bytes);
int orc_ref_check_validity(uint64_t n, int layout, const uint64_t *x, const uint64_t *z, char *buf,
                           uint64_t cap, uint64_t *len);

#ifdef __cplusplus
}
#endif
#endif
