// Device object model and kernel launchers of libqsr (sm_100a).
//
// HBM layout:
//   CM plane  : word (q, j) at q*cm_pitch + j, q in [0, n_pad), j in [0, 2k); cm_pitch =
//               round_up(2k, 16) so every qubit row starts on a 128-byte line.
//   RM plane  : generator-major; row r = j*64 + b (r < n_pad destabilizer g = r, else
//               stabilizer g = r - n_pad), word i = qubit-word; at r*rm_pitch + i,
//               rm_pitch = round_up(k, 16). A generator's k words are contiguous, so the
//               measurement row products stream exactly the bytes they need.
//   signs     : 2k words (+ padding to cm_pitch), generator-indexed in both layouts.
// The reference's RowMajor (i-major, tableau.hpp:91-94) is produced only when a caller
// downloads a transposed tableau through the API-parity path.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <utility>
#include <vector>

#include "host.hpp"

namespace qsr {

void cuda_check(cudaError_t e, const char *what);
// The per-device caching allocator behind tableau planes and scratch (capi.cpp): a released
// block is reused by the next acquire of the same size on the same device. `after`: the owner's
// stream when the block may still be read by queued work; the next acquire waits for it.
// Device -> host copy of rows x width bytes (pitched on both sides); pageable destinations are
// staged through pinned buffers (capi.cpp).
void download_2d(void *dst, size_t dpitch, const void *src, size_t spitch, size_t width, size_t rows,
                 cudaStream_t st);
void *cache_acquire(int device, uint64_t bytes);
void cache_release(int device, uint64_t bytes, void *p, cudaStream_t after = nullptr);
#define QSR_CUDA(call) ::qsr::cuda_check((call), #call)

extern uint64_t g_launches; // kernel launches issued by the library
inline void count_launch(uint64_t n = 1) { g_launches += n; }

inline uint64_t round_up(uint64_t v, uint64_t m) { return (v + m - 1) / m * m; }

constexpr int kMaxBatch = 32; // collapses per batched pass (k_batch.cu)
constexpr int kVinfoWords = 8 * kMaxBatch; // per-batch pivot info (k_batch.cu)

// Scratch used by the measurement pipeline; sized for one tableau.
struct MeasureScratch {
    uint64_t *mask = nullptr;       // 2k mask words (column bits of all rows)
    uint32_t *rows = nullptr;       // compacted row list (<= 2*n_pad)
    uint32_t *ctl = nullptr;        // control block (see k_measure.cu)
    uint64_t *partial_x = nullptr;  // deterministic-product partials [kDetChunks][rm_pitch]
    uint64_t *partial_z = nullptr;
    int64_t *partial_e = nullptr;   // [kDetChunks]
    uint8_t *flags = nullptr;       // per-measurement flags of the current window
    qsr_record_entry *out = nullptr;// per-window outcomes
    uint32_t *mqubits = nullptr;    // per-window measured qubits
    uint64_t *coin_index = nullptr; // device coin counter
    int *err = nullptr;             // odd-phase detector
    uint64_t window_cap = 0;
    // batched collapses (k_batch.cu)
    uint32_t *colbits = nullptr;    // [2*ng] column bits at the batch's qubits
    // One contiguous batch block (broadcast as a unit by the sharded engine):
    //   V rows  [kMaxBatch][2][rm_pitch] (x words then z words of pivot row m)
    //   vinfo   [kVinfoWords] u32, bctl [4] u32 (len, stopped, stabilizer OR-mask, -)
    uint64_t *batch_block = nullptr;
    uint64_t batch_block_bytes = 0;
    uint64_t *Vx = nullptr, *Vz = nullptr; // views into batch_block, row stride vstride
    uint64_t vstride = 0;
    uint32_t *vinfo = nullptr;
    uint32_t *bctl = nullptr;
    uint32_t *d_pos = nullptr;      // speculative batch position (k_batch.cu)
    uint32_t *h_bctl = nullptr;     // pinned [2][8] batch control read-back slots (len, stopped,
                                    // OR-mask, skipped, sequence number: k_batch_signs writes them)
    cudaEvent_t bev[2] = {nullptr, nullptr};
    uint8_t *partial = nullptr;     // [slices][2ng] per-(row, slice) phase bytes (k_batch.cu)
    uint64_t partial_bytes = 0;
    uint32_t *nz = nullptr;         // [ng/32] active-stabilizer ballot of the batch
    int *pcount = nullptr;          // [2*kMaxBatch] per-pivot phase / beta counters
    // Second buffer set for chained one-GPU batches (batch_chained): batch k+1's select writes
    // these while batch k still reads the first set.
    uint32_t *vinfo_b = nullptr, *bctl_b = nullptr, *colbits_b = nullptr, *nz_b = nullptr;
    int *pcount_b = nullptr;
    uint32_t *fq = nullptr, *fidx = nullptr; // flagged qubits / window indices [window_cap]
    // Caller-drawn coins for the current measurement window (nullptr = device Philox).
    uint8_t *coin_table = nullptr;
    uint8_t *coin_buf = nullptr;  // [window_cap]
};


// One tableau, or one generator-word shard of it: the shard holds generator
// words [j0, j0+kg) of both halves (destabilizers g and stabilizers g for the same g), for all
// n_pad qubits. Unsharded: j0 = 0, kg = k. CM columns = 2kg local generator-words; RM rows =
// 2ng local generator rows (ng = 64kg; stabilizer row offset ng), each k qubit-words long.
struct DeviceTableau {
    int device = 0;
    cudaStream_t stream = nullptr;
    uint64_t n = 0, k = 0, n_pad = 0; // qubits, qubit-words, CM rows (64k)
    uint64_t kg = 0;                  // generator-words held (per half)
    uint64_t g0 = 0;                  // global index of the first generator held (64*j0)
    uint64_t ng = 0;                  // 64*kg generator rows per half
    uint64_t n_gen = 0;               // valid generators held: clamp(n - g0, 0, ng)
    uint64_t cm_pitch = 0, rm_pitch = 0;
    uint64_t plane_words = 0;        // max(n_pad*cm_pitch, 2*ng*rm_pitch)
    uint64_t *x = nullptr, *z = nullptr;   // current planes
    uint64_t *x2 = nullptr, *z2 = nullptr; // transpose targets
    uint64_t *s = nullptr;                 // signs (cm_pitch words)
    int layout = QSR_COLUMN_MAJOR;
    // Built only from basis states, gates and measurements (a valid tableau). Uploaded
    // tableaux may be corrupt and are measured on the per-collapse path, which checks the
    // phase of every single product (measure.hpp:373-374, tableau.hpp:345-350).
    bool trusted = true;
    // gate-window sign partials
    uint64_t *sign_partials = nullptr;
    uint64_t sign_partial_chunks = 0;
    uint32_t *tile_counters = nullptr;
    uint64_t *gate_buf = nullptr;          // staging for single-window API calls
    uint64_t gate_buf_cap = 0;
    MeasureScratch ms;
    // Optional measurement-pass profile (qsr_engine_profile): events around every absorb launch
    // and a device counter of rows rewritten. Null on every timed path.
    struct AbsorbProfile {
        std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
        unsigned long long *d_rows = nullptr;
    } *prof = nullptr;
    uint8_t *arena = nullptr; // fixed-size scratch (signs, counters, measurement scratch), one block
    uint64_t arena_bytes = 0;
    int num_sms = 148;

    DeviceTableau(uint64_t n, int device, uint64_t j0 = 0, uint64_t kg = 0);
    ~DeviceTableau();
    void ensure_gate_buf(uint64_t ngates);
    void ensure_window_cap(uint64_t m);
    void release_window_cap();
    void sync();
};

// ---- launchers --------------------------------------------------------------------
// Gate window on a CM tableau: `gates` is a device array of packed gate words.
void launch_gate_window(DeviceTableau &t, const uint64_t *gates, uint64_t ngates);
// Gate fusion support (fuse.hpp): the CM rows un-permuted (logical q <- physical perm[q]) into
// the spare planes, which then become the current ones.
void launch_unpermute_rows(DeviceTableau &t, const uint32_t *d_perm);
// Frames rows (n rows of `pitch` words): dst[q] = src[perm[q]].
void launch_unpermute_frame_rows(const uint64_t *src, uint64_t *dst, uint64_t pitch, uint64_t n,
                                 const uint32_t *d_perm, int num_sms, cudaStream_t st);
// Frames: same rules, no signs.
void launch_frame_window(uint64_t *xf, uint64_t *zf, uint64_t pitch, const uint64_t *gates,
                         uint64_t ngates, int num_sms, cudaStream_t st);
// CM <-> internal RM transposes (swap t.x/t.x2 etc).
void transpose_to_rm(DeviceTableau &t);
void transpose_to_cm(DeviceTableau &t);
// Tableau::check_group_validity (tableau.hpp:184-213): "valid" or the reference's first violation.
std::string check_group_validity(DeviceTableau &t);
void launch_zero_state(DeviceTableau &t, const uint8_t *d_init /* nullable */);

// Measurement window on a CM tableau (fused recipe, measure.hpp:381-442 semantics).
// `mq` = device array of measured qubits (m entries) already uploaded to t.ms.mqubits.
struct MeasureTimes { cudaEvent_t t0, t1, t2, t3; };
void measure_window_device(DeviceTableau &t, uint64_t m, uint64_t seed,
                           const std::vector<uint32_t> &qubits, std::vector<uint8_t> &flags_host,
                           bool timed, double *t_ms, double *ge_ms, double *cmp_ms);

void configure_measure_kernels(DeviceTableau &t);
// The three phases of a batch of <= kMaxBatch collapses (the sharded engine exchanges between them):
// column bits + stabilizer OR-mask (bctl[2]); pivots / V rows / coins / record (leader
// shard only); every row absorbs its V's.
void batch_colbits(DeviceTableau &t, const uint32_t *d_fq, uint32_t b, bool zero_block = false);
// Sharded batch plan from the all-gathered masks (k_batch.cu k_shard_plan): plan[4] =
// {this shard leads, lim, deterministic now, skipped}, on the device.
void shard_plan(DeviceTableau &t, const uint32_t *d_masks, int world, int rank, uint32_t b, uint32_t expect,
                uint32_t *d_plan);
// d_pos / expect: speculative batches (the batch is a no-op unless *d_pos == expect; on success
// *d_pos = expect + len). nullptr: unconditional.
// d_plan (sharded): only the plan's leader selects, at most plan[1] collapses.
void batch_pivots(DeviceTableau &t, const uint32_t *d_fq, const uint32_t *d_fidx, uint32_t b,
                  uint64_t seed, uint32_t *d_pos = nullptr, uint32_t expect = 0,
                  const uint32_t *d_plan = nullptr);
void configure_batch_kernels(int device); // per-device kernel attributes (current device)
void set_device_u32(uint32_t *p, uint32_t v, cudaStream_t st);
void batch_apply(DeviceTableau &t);
// One GPU: the whole batch after the column bits in four launches (select; pivot rows +
// memberships; absorb with the signs / coins / record of the V's in CTA 0; sign pass).
// With `host_slot`, the sign pass also writes the batch's control words there (page-locked host
// memory) followed by `seq`, so the host learns the batch length without a copy in the stream.
// One GPU, chained batches: this batch in the tableau's current buffers (ms.vinfo / bctl / colbits
// / nz / pcount), the next one's select inside this batch's absorb (its last CTA) into `nxt`, with
// column bits the membership pass derives (nfq / nb: the next batch's qubits; nfq2 / nb2: the one
// after, whose V bits the sign pass forms). `standalone`: this batch's column bits and select
// are launched first (the window's first batch, or after an early stop).
struct BatchBufs {
    uint32_t *vinfo, *bctl, *colbits, *nz;
    int *pcount;
};
void batch_chained(DeviceTableau &t, const BatchBufs &nxt, const uint32_t *d_fq, const uint32_t *d_fidx,
                   uint32_t b, uint64_t seed, bool standalone, uint32_t *d_pos, uint32_t expect,
                   const uint32_t *nfq, uint32_t nb, const uint32_t *nfq2, uint32_t nb2, uint32_t *host_slot,
                   uint32_t seq);
// With `next_fq` (next_b qubits), the sign pass also computes the next batch's column bits and
// active ballot (what batch_colbits would), so that batch needs no column-bit launch.
void batch_fused(DeviceTableau &t, const uint32_t *d_fq, const uint32_t *d_fidx, uint32_t b, uint64_t seed,
                 uint32_t *d_pos, uint32_t expect, uint32_t *host_slot = nullptr, uint32_t seq = 0,
                 const uint32_t *next_fq = nullptr, uint32_t next_b = 0);
// Deterministic outcome of measuring q (measure.hpp:343-376), sharded form: this shard's
// ordered partial product is written to `slot` ([x: rm_pitch][z: rm_pitch][e: 16 words]);
// det_combine folds `nslots` slots (in shard order, stride det_slot_words) into the outcome,
// written to *out (deterministic entry) and ctl.
uint64_t det_slot_words(const DeviceTableau &t);
void det_local_partial(DeviceTableau &t, uint64_t q, uint64_t *slot);
// slot_stride: words between consecutive shards' slots (0 = det_slot_words).
void det_combine(DeviceTableau &t, uint64_t q, const uint64_t *slots, uint32_t nslots,
                 qsr_record_entry *out, uint64_t slot_stride = 0);
// Probabilistic flags of a measurement window on this tableau/shard (find_probabilistic,
// measure.hpp:104-126) into t.ms.flags (device; m bytes).
void flags_cm(DeviceTableau &t, uint64_t m);
// API-parity kernels on an RM tableau.
void rm_column_mask(DeviceTableau &t, uint64_t q);          // fills t.ms.mask
void rm_find_pivots(DeviceTableau &t, uint64_t q, std::vector<int64_t> &entries, uint64_t &count);
void rm_parallel_ge(DeviceTableau &t, const std::vector<int64_t> &pivots);
void rm_swap_anti_commuting(DeviceTableau &t, uint64_t p, uint64_t q);
bool rm_deterministic_outcome(DeviceTableau &t, uint64_t q);
void rm_find_probabilistic(DeviceTableau &t, const std::vector<uint32_t> &qubits,
                           std::vector<int64_t> &out);
void flip_sign_bit(DeviceTableau &t, uint64_t word, uint64_t bit);
int read_error_flag(DeviceTableau &t); // syncs; returns and clears

// Frames kernels. A frames object may hold a slice of the shot-words: kf words starting at
// global word j0 (sampling sharded by shot); `shots` is the global count.
void launch_frames_init(uint64_t *zf, uint64_t n, uint64_t kf, uint64_t j0, uint64_t pitch,
                        uint64_t shots, uint64_t seed, uint32_t epoch, uint32_t wbits, cudaStream_t st);
// wbits = the reference word type's width (8/16/32/64): Z frames are drawn as sample<W> draws them.
void launch_measure_sample(uint64_t *xf, uint64_t *zf, uint64_t pitch, uint64_t kf, uint64_t j0,
                           uint64_t shots, uint64_t *rec, const uint32_t *qubits,
                           const uint32_t *rows, uint64_t m, uint64_t seed, uint32_t epoch,
                           uint32_t wbits, cudaStream_t st);
void launch_record_fold(uint64_t *rec, uint64_t pitch, uint64_t kf, uint64_t j0, uint64_t shots,
                        const uint32_t *flip_rows, uint64_t nflip, cudaStream_t st);

} // namespace qsr
