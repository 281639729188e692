/*
 * qsr.h — C ABI of the B200-native stabilizer-tableau engine (libqsr.so).
 *
 * This is the drop-in boundary for the hot path named in BASELINE.json's north_star:
 * the reference's single-shot simulate / measure / sample API of proj/include/quasar
 * (arXiv 2603.14641, "QuaSARQ"). Every entry point below replaces one reference
 * function; the citation after each declaration is the reference interface it stands
 * for (paths relative to the reference's proj/include/quasar/).
 *
 * Conventions
 *  - Plain pointers and sizes only; no torch / CUDA types cross the boundary.
 *  - Every function returns a qsr_status. On failure, qsr_last_error() returns a
 *    thread-local message. The reference throws std::invalid_argument /
 *    std::out_of_range / std::logic_error; the status codes map 1:1 onto those types
 *    and the C++ shim (include/quasar_gpu.hpp) rethrows the same exception type.
 *  - Validation happens on the host before any device state is mutated, as the
 *    reference validates before mutating.
 *  - Calls are synchronous (stream-synchronised before return) like the reference.
 *  - Word type is fixed to uint64_t (the reference's default W).
 *  - Host tableau buffers use the reference's storage layout exactly
 *    (tableau.hpp:51-61): ColumnMajor word (q, j) at q*2k + j; RowMajor word
 *    (i, col) at i*2*n_pad + col; signs 2k words. Device storage is private.
 */
#ifndef QSR_H_
#define QSR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QSR_ABI_VERSION 1

typedef int qsr_status;
enum {
    QSR_OK = 0,
    QSR_INVALID_ARGUMENT = 1, /* std::invalid_argument */
    QSR_OUT_OF_RANGE = 2,     /* std::out_of_range */
    QSR_LOGIC_ERROR = 3,      /* std::logic_error (odd phase = corrupted tableau) */
    QSR_CUDA_ERROR = 4,
    QSR_OUT_OF_MEMORY = 5,
    QSR_NCCL_ERROR = 6,
    QSR_INTERNAL = 7,
    QSR_PARSE_ERROR = 8       /* quasar::QasmError (qasm.hpp:33-40) */
};

/* GateKind, same numbering as circuit.hpp:29-42. */
enum {
    QSR_X = 0, QSR_Y, QSR_Z, QSR_H, QSR_S, QSR_SDG,
    QSR_CX, QSR_CY, QSR_CZ, QSR_SWAP, QSR_ISWAP, QSR_MEASURE
};
enum { QSR_COLUMN_MAJOR = 0, QSR_ROW_MAJOR = 1 };   /* tableau.hpp:30 Layout */
enum { QSR_SINGLE_SHOT = 0, QSR_SAMPLING = 1 };     /* schedule.hpp:37 ScheduleMode */

/* Byte-compatible with quasar::Gate (circuit.hpp:85-99): 12 bytes, kind @0, q0 @4, q1 @8,
 * so `circuit.gates.data()` can be passed without repacking. */
typedef struct qsr_gate {
    uint8_t kind;
    uint32_t q0;
    uint32_t q1;
} qsr_gate;

/* Byte-compatible with quasar::MeasurementRecord::Entry (measure.hpp:42-46). */
typedef struct qsr_record_entry {
    uint32_t qubit;
    uint8_t outcome;
    uint8_t deterministic;
} qsr_record_entry;

/* quasar::PhaseTimers (measure.hpp:87-100). Filled from CUDA events (device time). */
typedef struct qsr_phase_timers {
    double to_seconds;
    double t_seconds;
    double cmp_seconds;
    double ge_seconds;
} qsr_phase_timers;

/* quasar::RunReport (simulator.hpp:27-34). */
typedef struct qsr_run_report {
    qsr_phase_timers timers;
    uint64_t gate_count;
    uint64_t measure_count;
    uint64_t probabilistic_count;
    uint64_t window_count;
    double total_seconds;
} qsr_run_report;

/* ---- library ------------------------------------------------------------------- */
const char *qsr_last_error(void);
int qsr_abi_version(void);
qsr_status qsr_device_count(int *count);
/* Tableau planes of destroyed tableaux are cached for reuse by the next tableau of the same
 * shape (QSR_PLANE_CACHE=0 disables); this frees them. */
void qsr_release_cached_memory(void);
/* Kernel launches issued by this library since load (bench `gpu_launches`). */
uint64_t qsr_launch_count(void);
/* Page-locked host buffers for fast tableau / record transfers (cudaHostAlloc). */
qsr_status qsr_host_alloc(uint64_t bytes, void **out);
void qsr_host_free(void *p);

/* ---- Philox-4x32-10 (rng.hpp:28-55) -------------------------------------------- */
void qsr_philox_block(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
uint64_t qsr_philox_word(uint64_t seed, uint32_t stream, uint32_t ctx, uint64_t index);

/* ---- circuits (circuit.hpp:101-173) -------------------------------------------- */
typedef struct qsr_circuit qsr_circuit;
/* Circuit{num_qubits, gates}; check_valid() is applied (circuit.hpp:108-115). */
qsr_status qsr_circuit_create(uint32_t num_qubits, const qsr_gate *gates, uint64_t ngates,
                              qsr_circuit **out);
/* generate_random(n, depth, seed, measure_prob) (circuit.hpp:132-173). */
qsr_status qsr_generate_random(uint32_t n, uint32_t depth, uint64_t seed, double measure_prob,
                               qsr_circuit **out);
qsr_status qsr_circuit_info(const qsr_circuit *c, uint32_t *num_qubits, uint64_t *ngates,
                            uint64_t *nmeasure);
const qsr_gate *qsr_circuit_gates(const qsr_circuit *c);
void qsr_circuit_destroy(qsr_circuit *c);
/* Circuit::num_clbits (circuit.hpp:103-105): classical bits named in the source, labels only.
 * generate_random sets n (circuit.hpp:171), qsr_parse_qasm the last creg size, else 0. */
qsr_status qsr_circuit_clbits(const qsr_circuit *c, uint32_t *num_clbits);
qsr_status qsr_circuit_set_clbits(qsr_circuit *c, uint32_t num_clbits);

/* Host worker threads of the parallel host passes (schedule scatter, QASM parse / emit,
 * fusion); 0 = hardware default. Stands for set_num_threads (parallel.hpp:151). */
void qsr_set_num_threads(unsigned threads);
unsigned qsr_get_num_threads(void);

/* ---- OpenQASM 2.0 subset (qasm.hpp:29-271) -------------------------------------- */
/* parse_qasm (qasm.hpp:159-252): same grammar, same Circuit, same errors. On a syntax error
 * returns QSR_PARSE_ERROR, qsr_last_error() = QasmError::what() ("qasm:L:C: reason") and
 * *err = {line, column}. Large bodies are parsed on all host threads. */
typedef struct qsr_qasm_error { int line; int column; } qsr_qasm_error;
qsr_status qsr_parse_qasm(const char *text, uint64_t len, qsr_circuit **out, qsr_qasm_error *err);
/* emit_qasm (qasm.hpp:254-271). Text outputs: buf == NULL -> *len = size in bytes; else
 * cap >= size is required and exactly *len bytes are written (no NUL terminator). */
qsr_status qsr_emit_qasm(const qsr_circuit *c, char *buf, uint64_t cap, uint64_t *len);

/* ---- schedules (schedule.hpp:32-137) ------------------------------------------- */
typedef struct qsr_schedule qsr_schedule;
/* schedule_windows(circuit, mode) (schedule.hpp:51-137): identical output, O(G). */
qsr_status qsr_schedule_windows(const qsr_circuit *c, int mode, qsr_schedule **out);
/* A caller-built Schedule: windows are [offsets[w], offsets[w+1]) of `gates`. */
qsr_status qsr_schedule_create(const qsr_gate *gates, const uint64_t *offsets,
                               const uint8_t *is_measurement, uint64_t nwindows, int mode,
                               qsr_schedule **out);
qsr_status qsr_schedule_info(const qsr_schedule *s, uint64_t *nwindows, uint64_t *ngates,
                             int *mode);
const qsr_gate *qsr_schedule_gates(const qsr_schedule *s);
const uint64_t *qsr_schedule_offsets(const qsr_schedule *s);      /* nwindows + 1 */
const uint8_t *qsr_schedule_is_measurement(const qsr_schedule *s); /* nwindows */
void qsr_schedule_destroy(qsr_schedule *s);
/* schedule_to_text (schedule.hpp:235-249); text-output convention of qsr_emit_qasm. */
qsr_status qsr_schedule_text(const qsr_schedule *s, char *buf, uint64_t cap, uint64_t *len);
/* validate_schedule (schedule.hpp:143-233): "valid" or the reference's first violation. */
qsr_status qsr_validate_schedule(const qsr_circuit *c, const qsr_schedule *s, char *buf,
                                 uint64_t cap, uint64_t *len);

/* ---- device tableau (tableau.hpp:62-131) --------------------------------------- */
typedef struct qsr_tableau qsr_tableau;
/* Tableau<uint64_t>(n): all-zero planes, ColumnMajor (tableau.hpp:67-72). */
qsr_status qsr_tableau_create(uint64_t n, int device, qsr_tableau **out);
/* Tableau::basis_state(initstate) / zero_state (tableau.hpp:120-131); NULL = |0...0>. */
qsr_status qsr_tableau_basis_state(qsr_tableau *t, const uint8_t *initstate);
qsr_status qsr_tableau_info(const qsr_tableau *t, uint64_t *n, uint64_t *k, uint64_t *n_pad,
                            int *layout);
/* Host buffers in the reference layout: x, z = n_pad*2k words, s = 2k words. */
qsr_status qsr_tableau_upload(qsr_tableau *t, const uint64_t *x, const uint64_t *z,
                              const uint64_t *s, int layout);
qsr_status qsr_tableau_download(const qsr_tableau *t, uint64_t *x, uint64_t *z, uint64_t *s);
qsr_status qsr_tableau_clone(const qsr_tableau *t, qsr_tableau **out);
void qsr_tableau_destroy(qsr_tableau *t);

/* Tableau::transpose_in_place (tableau.hpp:166-176). */
/* Tableau::check_group_validity (tableau.hpp:184-213) on the device: "valid" or the reference's
 * first violation, text-output convention of qsr_emit_qasm. O(n^2 k) word operations as a tiled
 * GF(2) Gram product (seconds at c2, tens of seconds at c5). Whole tableaux only. */
qsr_status qsr_tableau_check_validity(qsr_tableau *t, char *buf, uint64_t cap, uint64_t *len);
qsr_status qsr_transpose_in_place(qsr_tableau *t);

/* apply_window(tableau, window) (gates.hpp:147-197). */
qsr_status qsr_apply_window(qsr_tableau *t, const qsr_gate *gates, uint64_t ngates);

/* Measurement pipeline (measure.hpp:104-442); the tableau must be RowMajor for the
 * first six, as in the reference. */
qsr_status qsr_find_probabilistic(qsr_tableau *t, const qsr_gate *gates, uint64_t ngates,
                                  int64_t *out);                      /* measure.hpp:104 */
qsr_status qsr_find_and_compact_pivots(qsr_tableau *t, uint64_t q, int64_t *entries /* n */,
                                       uint64_t *count);               /* measure.hpp:130 */
qsr_status qsr_parallel_ge(qsr_tableau *t, const int64_t *entries, uint64_t count,
                           uint64_t block_targets);                    /* measure.hpp:161 */
qsr_status qsr_swap_anti_commuting(qsr_tableau *t, uint64_t p, uint64_t q); /* :279 */
qsr_status qsr_inject_x(qsr_tableau *t, uint64_t p);                  /* measure.hpp:335 */
qsr_status qsr_deterministic_outcome(qsr_tableau *t, uint64_t q, uint8_t *outcome); /* :343 */
/* measure_window(t, window, RandomStream(seed, kStreamMeasure) at *coin_index, ...)
 * (measure.hpp:381-442). *coin_index advances by the coins consumed; `out` receives
 * ngates entries in window order. `timers` may be NULL. */
qsr_status qsr_measure_window(qsr_tableau *t, const qsr_gate *gates, uint64_t ngates,
                              uint64_t seed, uint64_t *coin_index, qsr_record_entry *out,
                              qsr_phase_timers *timers);
/* Same, with the coins supplied by the caller: coins[i] & 1 is the i-th coin the window may
 * consume (the caller draws them from its own RandomStream, any stream / context; at most
 * ngates are used, ncoins >= ngates). *used receives how many were consumed, so the caller
 * advances its stream by exactly that many draws (measure.hpp:427). */
qsr_status qsr_measure_window_coins(qsr_tableau *t, const qsr_gate *gates, uint64_t ngates,
                                    const uint8_t *coins, uint64_t ncoins, uint64_t *used,
                                    qsr_record_entry *out, qsr_phase_timers *timers);

/* run_single_shot<uint64_t>(circuit, schedule, seed) (simulator.hpp:46-76).
 * schedule == NULL -> schedule_windows(circuit, single_shot). `record` must hold
 * measure_count entries. If out_tableau != NULL it receives the final tableau (device). */
qsr_status qsr_run_single_shot(const qsr_circuit *c, const qsr_schedule *s, uint64_t seed,
                               int device, qsr_tableau **out_tableau, qsr_record_entry *record,
                               qsr_run_report *report);

/* ---- resident engine (bench / repeated runs; same algorithm as qsr_run_single_shot) */
typedef struct qsr_engine qsr_engine;
qsr_status qsr_engine_create(const qsr_circuit *c, const qsr_schedule *s, int device,
                             qsr_engine **out);
/* One full single-shot pass on device-resident inputs; *device_ms = CUDA-event time. */
qsr_status qsr_engine_run(qsr_engine *e, uint64_t seed, double *device_ms);
/* Per-kernel-class device time of the last run (ms) and launch counts. */
qsr_status qsr_engine_stats(const qsr_engine *e, double *gate_ms, uint64_t *gate_launches,
                            double *transpose_ms, double *measure_ms, uint64_t *launches);
/* Algorithmic bytes of the last run's gate-window launches (kind-exact words of the device
 * gates actually launched — after gate fusion, DESIGN.md §5 — times 8 B x 2kg, + sign words). */
qsr_status qsr_engine_gate_bytes(const qsr_engine *e, double *bytes);
qsr_status qsr_engine_record(const qsr_engine *e, qsr_record_entry *record);
qsr_status qsr_engine_tableau(const qsr_engine *e, uint64_t *x, uint64_t *z, uint64_t *s);
/* Measurement-pass profile (bench.py's per-phase roofline): one more run with CUDA events around
 * every k_batch_absorb launch and a device count of the rows each batch rewrites. Not used by
 * timed runs (the events split the programmatic-launch chain). */
typedef struct qsr_kernel_profile {
    double absorb_ms;          /* summed device time of the absorb launches */
    uint64_t absorb_launches;
    uint64_t absorb_rows;      /* rows that absorbed >= 1 pivot row, summed over the launches */
    uint64_t absorb_slices;    /* 64-word slices per row (one phase byte each) */
    uint64_t row_words;        /* qubit-words per RM row (k) */
    double total_ms;           /* device time of the whole profiled run */
} qsr_kernel_profile;
qsr_status qsr_engine_profile(qsr_engine *e, uint64_t seed, qsr_kernel_profile *out);
/* sample<uint64_t>(circuit, shots, seed) (frames.hpp:163-204) on the resident engine: the
 * engine's run is the reference shot and the Pauli frames ride its (fused) windows on the same
 * stream; *device_ms = CUDA-event time of the call (frames init, run, record fold). The result
 * is the same ShotRecord as qsr_sample (world = 1) or shot-word slice `rank` of `world` as
 * qsr_sample_shard; release it with qsr_frames_destroy. */
typedef struct qsr_frames qsr_frames;
qsr_status qsr_engine_sample(qsr_engine *e, uint64_t shots, uint64_t seed, int world, int rank,
                             qsr_frames **out, double *device_ms);
/* Algorithmic bytes of the last qsr_engine_sample's frames-window launches (frames rule words,
 * no signs: X / Y / Z move nothing, frames.hpp:76-94) = 8 B x shot-words x words, and their
 * summed device time (ms; the frames run on their own stream, beside the reference shot). */
qsr_status qsr_engine_frames_bytes(const qsr_engine *e, double *bytes, double *ms);
void qsr_engine_destroy(qsr_engine *e);

/* ---- Pauli frames (frames.hpp:32-204) ------------------------------------------ */
/* init_frames<uint64_t>(n, shots, seed) (frames.hpp:46-72). */
qsr_status qsr_init_frames(uint64_t n, uint64_t shots, uint64_t seed, int device,
                           qsr_frames **out);
qsr_status qsr_frames_info(const qsr_frames *f, uint64_t *n, uint64_t *shots, uint64_t *kf);
/* Host buffers in the reference layout: word (q, j) at q*kf + j. */
qsr_status qsr_frames_download(const qsr_frames *f, uint64_t *xf, uint64_t *zf);
qsr_status qsr_frames_upload(qsr_frames *f, const uint64_t *xf, const uint64_t *zf);
/* apply_window_frames (frames.hpp:76-94). */
qsr_status qsr_apply_window_frames(qsr_frames *f, const qsr_gate *gates, uint64_t ngates,
                                   int is_measurement);
/* measure_sample(f, window, record, seed, epoch) (frames.hpp:111-158); the ShotRecord
 * lives inside the frames object. */
qsr_status qsr_measure_sample(qsr_frames *f, const qsr_gate *gates, uint64_t ngates,
                              int is_measurement, uint64_t seed, uint32_t epoch);
/* ShotRecord<uint64_t> (frames.hpp:97-107): measured (nrows) and words (nrows*kf).
 * Pass NULL buffers to query *nrows. */
qsr_status qsr_frames_record(const qsr_frames *f, uint64_t *nrows, uint32_t *measured,
                             uint64_t *words);
void qsr_frames_destroy(qsr_frames *f);
/* sample<uint64_t>(circuit, shots, seed, report) (frames.hpp:163-204); the result is the
 * frames object's ShotRecord. */
qsr_status qsr_sample(const qsr_circuit *c, uint64_t shots, uint64_t seed, int device,
                      qsr_frames **out, qsr_run_report *report);
/* sample<uint64_t> sharded by shot: this call computes shot-words
 * [w0, w0+nw) of ceil(shots/64), w0 = kf*rank/world, on `device` (one process per GPU; no
 * communication: the Philox key (q<<24)|j of frames.hpp:63 uses the global word j). The
 * reference shot runs on every rank. The record rows hold nw words each; concatenating the
 * ranks' rows word-wise gives sample()'s ShotRecord exactly. */
qsr_status qsr_sample_shard(const qsr_circuit *c, uint64_t shots, uint64_t seed, int world,
                            int rank, int device, qsr_frames **out, qsr_run_report *report);
/* Global shot-word slice [j0, j0+nw) held by a frames object (j0 = 0, nw = kf unsharded). */
qsr_status qsr_frames_shot_words(const qsr_frames *f, uint64_t *j0, uint64_t *nw);
/* init_frames<W> / sample<W> for the reference's other word types, W = word_bits in
 * {8, 16, 32, 64} (frames.hpp:46-72, 163-204): the Z frames are drawn exactly as the reference
 * draws them for W (one Philox word per W-bit word, low W bits kept), so every shot matches
 * sample<W>. Device and host records keep the 64-bit word layout: shot s is bit s%64 of word
 * s/64 in either case, and the little-endian bytes of a row's first ceil(shots/W)*W/8 bytes are
 * exactly the reference's ShotRecord<W> row. */
qsr_status qsr_init_frames_word(uint64_t n, uint64_t shots, uint64_t seed, unsigned word_bits,
                                int device, qsr_frames **out);
qsr_status qsr_sample_word(const qsr_circuit *c, uint64_t shots, uint64_t seed, unsigned word_bits,
                           int device, qsr_frames **out, qsr_run_report *report);
qsr_status qsr_frames_word_bits(const qsr_frames *f, unsigned *word_bits);

/* ---- generator-row-sharded engine (multi-GPU run_single_shot) ------
 * The tableau is split by generator-words: shard r of `world` holds generator-words
 * [j0, j0+kg) of both halves (destabilizers and stabilizers g = 64*j0 .. 64*(j0+kg)-1) for
 * all qubits. Gate windows run shard-local with no communication; a measurement window
 * exchanges a pivot-leader mask (all-gather of 4 B per shard), the batch's pivot rows
 * (broadcast from the shard holding them), deterministic partial products (all-gather)
 * and the window's flags / record (max-all-reduce). Results are bit-identical to
 * run_single_shot<uint64_t> (simulator.hpp:46-76) for every world size. */
enum { QSR_EXCHANGE_LOCAL = 0, QSR_EXCHANGE_NCCL = 1 };
typedef struct qsr_shard_config {
    int world;              /* number of shards (1 <= world <= ceil(n/64)) */
    int rank;               /* NCCL: the shard this process drives; LOCAL: ignored */
    int device;             /* CUDA device of this process's shard(s) */
    int exchange;           /* QSR_EXCHANGE_LOCAL: all shards in this process on `device`;
                               QSR_EXCHANGE_NCCL: one process per shard (collective create) */
    const uint8_t *nccl_id; /* 128-byte ncclUniqueId shared by all ranks (NCCL only) */
} qsr_shard_config;
typedef struct qsr_sharded qsr_sharded;
/* Shard r's generator-word range for n qubits (host only, no device needed). */
qsr_status qsr_shard_range(uint64_t n, int world, int rank, uint64_t *j0, uint64_t *kg);
/* ncclGetUniqueId (rank 0 creates it, the host rendezvous hands it to every rank). */
qsr_status qsr_nccl_unique_id(uint8_t out[128]);
qsr_status qsr_sharded_create(const qsr_circuit *c, const qsr_schedule *s,
                              const qsr_shard_config *cfg, qsr_sharded **out);
/* One full single-shot pass (collective); *device_ms = CUDA-event time of this process. */
qsr_status qsr_sharded_run(qsr_sharded *e, uint64_t seed, double *device_ms);
/* run_single_shot<uint64_t>(circuit, seed) sharded, end to end from a host circuit (collective):
 * this process's shard is created, the windows are planned, fused and uploaded while the device
 * runs them (the streamed driver of qsr_run_single_shot) and measurement windows use the sharded
 * protocol; `record` (measure_count entries) receives the whole record. One shard per process
 * (QSR_EXCHANGE_NCCL, or QSR_EXCHANGE_LOCAL with world 1). *out keeps the final tableau shard
 * (qsr_sharded_tableau_local / qsr_sharded_tableau / qsr_sharded_destroy). */
qsr_status qsr_sharded_run_circuit(const qsr_circuit *c, const qsr_shard_config *cfg, uint64_t seed,
                                   qsr_record_entry *record, qsr_sharded **out, double *device_ms);
qsr_status qsr_sharded_stats(const qsr_sharded *e, double *gate_ms, uint64_t *gate_launches,
                             double *transpose_ms, double *measure_ms, uint64_t *launches);
/* The full measurement record (identical on every rank). */
qsr_status qsr_sharded_gate_bytes(const qsr_sharded *e, double *bytes); /* this process's shards */
qsr_status qsr_sharded_record(const qsr_sharded *e, qsr_record_entry *record);
/* Writes the generator-word columns of this process's shards into full-size reference-layout
 * CM buffers (x, z: n_pad*2k words; s: 2k words); other columns are left untouched. */
qsr_status qsr_sharded_tableau(const qsr_sharded *e, uint64_t *x, uint64_t *z, uint64_t *s);
/* This process's shards only, compact: per local shard (in rank order) a block of n_pad rows x
 * 2kg words (its destabilizer words, then its stabilizer words) for x and z, and 2kg sign words
 * — 1/world of the tableau per process, no full-size host buffers. */
qsr_status qsr_sharded_tableau_local(const qsr_sharded *e, uint64_t *x, uint64_t *z, uint64_t *s);
void qsr_sharded_destroy(qsr_sharded *e);

#ifdef __cplusplus
}
#endif
#endif /* QSR_H_ */
