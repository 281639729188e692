// Batched projective measurement: up to kMaxBatch consecutive probabilistic collapses of a
// measurement window applied in ONE streaming pass over the RM tableau, bit-identical to
// applying them one by one with the fused recipe of k_measure.cu (itself bit-identical to the
// reference's parallel_ge + swap_anti_commuting + inject_x, measure.hpp:409-431).
//
// Why batching is exact. Collapse m multiplies every row of R_m = {rows other than S_c, D_c
// with X[q_m] set} by V_m = S_{c_m} as it stands at time m, then D_{c_m} <- V_m and
// S_{c_m} <- +/-Z_{q_m}. A row's membership in R_m depends only on its X bit at q_m at time m,
// i.e. its bit at batch start XOR the X bits at q_m of the V's it absorbed before. With
//   colbits_r[m] = X_r[q_m] at batch start            (phase A, a column gather)
//   vb[m'][m]    = X bit of V_{m'} at q_m              (phase B)
// every row's membership vector follows from  member[m] = colbits[m] ^ parity(member[<m] &
// VBcol[m]). Only the pivot rows need sequential treatment (phase B, one CTA): c_m is the
// smallest stabilizer whose current X bit at q_m is set, V_m is S_{c_m} after its own earlier
// memberships, the coin is Philox(seed, 0, 0, coin_index++) & 1.
//
// Why the phase is cheap. For Hermitian Paulis P(a)P(b) = i^g P(a^b) with, summed over qubits,
//   g(a, b) = beta(a) + beta(b) + 2|a_z & b_x| - beta(a^b)   (mod 4),  beta(p) = |p_x & p_z|,
// which is exactly product_phase_counts' (plus - minus) (tableau.hpp:336-342). Absorbing
// V_1..V_k in order (V on the left, as the reference's control*target) therefore telescopes:
//   E = beta(r_start) - beta(r_end) + sum_j beta(V_j) + 2 sum_j |V_jz & cur_{j-1,x}|  (mod 4).
// Every single product of a valid tableau has even phase, so the XOR of the per-product flips
// equals bit 1 of E, and the row's sign becomes s_r ^ XOR_j s(V_j) ^ ((E >> 1) & 1). Per
// absorbed word this costs one AND-XOR into a parity accumulator plus the two row XORs.
// (An odd E flags a corrupted tableau; uploaded, possibly corrupt tableaux are measured on the
// per-collapse path, which checks every product exactly.)
//
// Traffic: one read + write of the touched rows per batch instead of per collapse; the pivot
// rows reach every CTA of the absorb pass as a shared-memory table of their XOR combinations
// per 64-word slice, reused by every row the CTA absorbs into.
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"
#include "device.hpp"

namespace qsr {

namespace {

using u64 = unsigned long long;
constexpr int kB = kMaxBatch; // collapses per batch (<= 32: u32 membership masks)
enum : uint32_t { BL_LEN = 0, BL_DET = 1, BL_STAB_OR = 2, BL_SKIP = 3 };
// vinfo layout (u32 [8*kB]): vb | sign of V_m | c_m (global) | beta(V_m) mod 4 | Mc_m |
// L_m = row m of (I + Mc)^-1 over GF(2) (V_m = XOR_{j in L_m} S_{c_j} at batch start) |
// pair-parity row P_m (bit j' < m: parity(sum_i |V_mz[i] & V_j'x[i]|)) | X bits of V_m at the
// next batch's qubits (one GPU, chained batches)
enum : uint32_t { VI_VB = 0, VI_SIGN = kB, VI_C = 2 * kB, VI_BETA = 3 * kB, VI_MC = 4 * kB, VI_L = 5 * kB,
                  VI_PMAT = 6 * kB, VI_VBN = 7 * kB };
static_assert(8 * kB == kVinfoWords, "vinfo layout");

__device__ __forceinline__ uint32_t parity32(uint32_t v) { return __popc(v) & 1u; }
// Kernels of the batch chain launch with programmatic stream serialization (launch_chain): each
// waits here for its predecessor before touching memory; the launch itself overlaps its tail.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

// Membership vector of a row given its batch-start column bits `cb` (bit m = X at q_m),
// the per-collapse VB columns and the first collapse it can take part in.
__device__ __forceinline__ uint32_t membership(uint32_t cb, const uint32_t *vbcol, uint32_t start,
                                               uint32_t len) {
    uint32_t M = 0;
    for (uint32_t m = start; m < len; ++m) {
        uint32_t bit = ((cb >> m) ^ parity32(M & vbcol[m])) & 1u;
        M |= bit << m;
    }
    return M;
}

// ---- phase A: column bits of all rows at the batch's measured qubits ----------------
// Also ORs the stabilizer rows' bits into *stab_or: bit m set iff some stabilizer held here has
// X at q_m at batch start (the sharded leader protocol, shard.cpp).
__global__ void k_colbits(const uint64_t *__restrict__ x, uint64_t pitch, uint64_t nrows,
                          uint64_t ng, const uint32_t *__restrict__ fq, uint32_t b,
                          uint32_t *__restrict__ colbits, uint32_t *__restrict__ stab_or,
                          uint32_t *__restrict__ nz, uint64_t *__restrict__ zero, uint64_t zero_words) {
    pdl_wait();
    // Sharded engine: the pivot rows + vinfo of this shard's batch block start at zero, so the
    // block exchange can be a root-free max-all-reduce (only the leader writes non-zeros).
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < zero_words;
         i += uint64_t(gridDim.x) * blockDim.x)
        zero[i] = 0;
    __shared__ uint32_t sq[kB];
    if (threadIdx.x < b) sq[threadIdx.x] = fq[threadIdx.x];
    __syncthreads();
    const uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    uint32_t bits = 0;
    if (r < nrows) {
        const uint64_t *row = x + r * pitch;
        uint32_t wi = 0xFFFFFFFFu;
        uint64_t word = 0;
        for (uint32_t m = 0; m < b; ++m) {
            const uint32_t q = sq[m];
            if ((q >> 6) != wi) { wi = q >> 6; word = __ldcg(row + wi); } // measure-all windows: one load per 64
            bits |= uint32_t((word >> (q & 63)) & 1u) << m;
        }
        colbits[r] = bits;
    }
    const uint32_t any = __reduce_or_sync(0xffffffffu, r >= ng && r < nrows ? bits : 0u);
    if ((threadIdx.x & 31) == 0 && any) atomicOr(stab_or, any);
    // Active-stabilizer ballot (bits != 0): rows with no X at any batch qubit can never be a
    // pivot or absorb anything in this batch.
    const uint32_t act = __ballot_sync(0xffffffffu, r >= ng && r < nrows && bits != 0);
    if ((threadIdx.x & 31) == 0 && r >= ng && r < nrows) nz[(r - ng) >> 5] = act;
}

// ---- phase B, split: B1 select (32-bit column logic only), B2 pivot rows (word-parallel),
// B3 signs / coins / record (one warp) ---------------------------------------------------
// B1. The pivot of collapse m, its memberships Mc_m and the X bits of V_m at the batch's
// qubits (vb_m) need only column bits: vb_m = cb(c_m) ^ XOR_{j in Mc_m} vb_j, because V_m is
// S_{c_m}(batch start) times the V_j it absorbed. The candidates are the first kWin active
// stabilizers (ascending, compacted from the nz ballot); each thread keeps their memberships
// incrementally, so a step is O(1) per candidate. If none of them qualifies, the stabilizers
// after the window are scanned with memberships recomputed from the column bits.
constexpr int kSelThreads = 256;
constexpr int kWin = 1024; // candidates (kWin / T per thread)

// X bits of V_j (j < len) at the next batch's qubits nfq[0..nb): lane i reads row S_{c_i} (its
// final state, batch start) at those qubits, and V_j = XOR_{i in L_j} S_{c_i} (one warp).
__device__ __forceinline__ uint32_t vbn_lane(uint32_t lane, bool valid, uint64_t c_local, uint32_t L,
                                             const uint64_t *__restrict__ x, uint64_t pitch, uint64_t ng,
                                             const uint32_t *__restrict__ nfq, uint32_t nb) {
    uint32_t xb = 0;
    if (valid) {
        const uint64_t *row = x + (ng + c_local) * pitch;
        uint32_t wi = 0xFFFFFFFFu;
        uint64_t word = 0;
        for (uint32_t m = 0; m < nb; ++m) {
            const uint32_t q = nfq[m];
            if ((q >> 6) != wi) { wi = q >> 6; word = __ldcg(row + wi); }
            xb |= uint32_t((word >> (q & 63)) & 1u) << m;
        }
    }
    uint32_t v = 0;
    for (uint32_t i = 0; i < 32; ++i) {
        const uint32_t xi = __shfl_sync(0xffffffffu, xb, i);
        if ((L >> i) & 1u) v ^= xi;
    }
    return v;
}

struct SelectArgs {
    const uint32_t *colbits, *nz;
    uint64_t n_gen, ng, g0;
    uint32_t b;
    uint32_t *vinfo, *bctl;
    uint32_t *d_pos; // standalone one-GPU batches: valid iff *d_pos == expect
    uint32_t expect;
    const uint32_t *plan; // sharded: the leader plan (nullptr on one GPU)
    int *pcount;          // one GPU: zeroed here (no reset launch)
    // Chained one-GPU batch (selected inside the previous batch's absorb): valid iff the previous
    // batch collapsed all prev_b of its measurements (its control words, another buffer set).
    const uint32_t *prev_bctl;
    uint32_t prev_b;
    // Standalone one-GPU batch: also the X bits of its V's at the next batch's qubits (VI_VBN).
    const uint64_t *x;
    uint64_t pitch;
    const uint32_t *nfq;
    uint32_t nb;
};

template <int T>
__device__ __forceinline__ void select_body(const SelectArgs &a) {
    constexpr int R = kWin / T;
    const uint32_t *__restrict__ colbits = a.colbits, *__restrict__ nz = a.nz;
    const uint64_t n_gen = a.n_gen, ng = a.ng, g0 = a.g0;
    uint32_t b = a.b;
    uint32_t *__restrict__ vinfo = a.vinfo, *__restrict__ bctl = a.bctl;
    const uint32_t *__restrict__ plan = a.plan;
    if (plan) { // sharded: only the batch's leader selects (the others' blocks stay zero)
        if (!plan[0]) return;
        b = min(b, plan[1]);
    } else { // one GPU, no reset launch: zero the sums k_pivot_rows accumulates into
        if (threadIdx.x < 2 * kB) a.pcount[threadIdx.x] = 0;
        if (threadIdx.x < kB) vinfo[VI_PMAT + threadIdx.x] = 0u;
    }
    __shared__ uint32_t s_rows[kWin];
    __shared__ uint32_t s_vbcol[kB], s_vb[kB], s_c[kB], s_mc[kB];
    __shared__ uint32_t s_scan[T / 32];
    __shared__ uint32_t s_nwin, s_next, s_minb[2], s_len, s_stop;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t nzw = (n_gen + 31) / 32;
    if (tid < kB) s_vbcol[tid] = 0;
    // Speculative batches (measure_window_device): a batch enqueued behind one that stopped
    // early (a chained batch: the previous batch's length; a standalone one: the device position)
    // turns into a no-op.
    const bool stale = !plan && (a.prev_bctl ? (a.prev_bctl[BL_LEN] != a.prev_b || a.prev_bctl[BL_DET] != 0u ||
                                                a.prev_bctl[BL_SKIP] != 0u)
                                             : (a.d_pos && *a.d_pos != a.expect));
    if (stale) {
        if (tid < kB) vinfo[VI_C + tid] = 0xFFFFFFFFu;
        if (tid == 0) { bctl[BL_LEN] = 0; bctl[BL_DET] = 0; bctl[BL_SKIP] = 1; }
        return;
    }
    if (tid == 0) { s_nwin = 0; s_next = uint32_t(n_gen); s_len = b; s_stop = 0; s_minb[0] = s_minb[1] = 0xFFFFFFFFu; }
    __syncthreads();
    // Window: the first kWin active stabilizers in ascending order.
    for (uint64_t base = 0; base < nzw; base += T) {
        const uint64_t w = base + tid;
        const uint32_t word = w < nzw ? nz[w] : 0u;
        const uint32_t cnt = __popc(word);
        uint32_t incl = cnt;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= uint32_t(o)) incl += v;
        }
        if (lane == 31) s_scan[warp] = incl;
        __syncthreads();
        uint32_t off = s_nwin;
        for (uint32_t i = 0; i < warp; ++i) off += s_scan[i];
        uint32_t pos = off + incl - cnt;
        for (uint32_t v = word; v && pos < uint32_t(kWin); v &= v - 1, ++pos) {
            const uint32_t row = uint32_t(w * 32 + __ffs(v) - 1);
            s_rows[pos] = row;
            if (pos == uint32_t(kWin) - 1) s_next = row + 1;
        }
        __syncthreads();
        if (tid == T - 1) s_nwin = min(off + incl, uint32_t(kWin));
        __syncthreads();
        if (s_nwin >= uint32_t(kWin)) break;
    }
    const uint32_t nwin = s_nwin;
    // cur[u]: the candidate's current X bits at the batch's qubits (batch-start bits XOR the vb
    // of every V it absorbed), so its bit at q_m is one shift and absorbing V_m one XOR.
    uint32_t row[R], cur[R], M[R];
#pragma unroll
    for (int u = 0; u < R; ++u) {
        const uint32_t e = tid + u * T;
        row[u] = e < nwin ? s_rows[e] : 0xFFFFFFFFu;
        cur[u] = e < nwin ? colbits[ng + row[u]] : 0u;
        M[u] = 0;
    }
    // Two barriers per collapse; s_minb is double-buffered (step m resets the other slot).
    for (uint32_t m = 0; m < b; ++m) {
        const uint32_t pm = m & 1u;
        uint32_t best = 0xFFFFFFFFu, bits = 0;
#pragma unroll
        for (int u = 0; u < R; ++u) {
            const uint32_t bit = (cur[u] >> m) & 1u;
            bits |= bit << u;
            if (bit) best = min(best, row[u]); // used pivots are inert (cur = 0)
        }
        best = __reduce_min_sync(0xffffffffu, best);
        if (lane == 0 && best != 0xFFFFFFFFu) atomicMin(&s_minb[pm], best);
        __syncthreads();
        if (tid == 0) s_minb[pm ^ 1u] = 0xFFFFFFFFu;
        if (s_minb[pm] == 0xFFFFFFFFu) {
            // Fallback: stabilizers after the window, memberships from the column bits.
            const uint32_t vc = s_vbcol[m];
            for (uint64_t g0r = s_next; g0r < n_gen; g0r += T) {
                const uint64_t g = g0r + tid;
                uint32_t cand = 0xFFFFFFFFu;
                if (g < n_gen) {
                    bool used = false;
                    for (uint32_t j = 0; j < m; ++j) used |= s_c[j] == uint32_t(g);
                    const uint32_t cbg = colbits[ng + g];
                    if (!used && cbg) {
                        const uint32_t Mg = membership(cbg, s_vbcol, 0, m);
                        if (((cbg >> m) ^ parity32(Mg & vc)) & 1u) cand = uint32_t(g);
                    }
                }
                cand = __reduce_min_sync(0xffffffffu, cand);
                if (lane == 0 && cand != 0xFFFFFFFFu) atomicMin(&s_minb[pm], cand);
                __syncthreads();
                if (s_minb[pm] != 0xFFFFFFFFu) break;
                __syncthreads();
            }
        }
        const uint32_t c = s_minb[pm];
        if (c == 0xFFFFFFFFu) { // no stabilizer anticommutes with Z_{q_m}: batch ends here
            if (tid == 0) { s_len = m; s_stop = 1; }
            break;
        }
        // A pivot from the window: its owner holds cur and the memberships in registers.
#pragma unroll
        for (int u = 0; u < R; ++u) {
            if (row[u] == c) {
                s_vb[m] = cur[u];
                s_c[m] = c;
                s_mc[m] = M[u];
            }
        }
        if (tid == 0 && c >= s_next) { // found by the fallback scan after the window
            const uint32_t cbc = colbits[ng + c];
            const uint32_t Mc = membership(cbc, s_vbcol, 0, m);
            uint32_t vb = cbc;
            for (uint32_t U = Mc; U; U &= U - 1) vb ^= s_vb[__ffs(U) - 1];
            s_vb[m] = vb;
            s_c[m] = c;
            s_mc[m] = Mc;
        }
        __syncthreads();
        const uint32_t vb = s_vb[m];
        if (tid < kB) s_vbcol[tid] |= ((vb >> tid) & 1u) << m; // read by the fallback only
#pragma unroll
        for (int u = 0; u < R; ++u) {
            if (row[u] == c) { cur[u] = 0; M[u] = 0; row[u] = 0xFFFFFFFFu; } // now +/-Z_q: inert
            else if ((bits >> u) & 1u) { M[u] |= 1u << m; cur[u] ^= vb; }
        }
    }
    __syncthreads();
    const uint32_t len = s_len;
    if (tid < kB) {
        const bool v = tid < len;
        vinfo[VI_VB + tid] = v ? s_vb[tid] : 0u;
        vinfo[VI_C + tid] = v ? uint32_t(g0 + s_c[tid]) : 0xFFFFFFFFu; // global generator
        const uint32_t mc = v ? s_mc[tid] : 0u;
        vinfo[VI_MC + tid] = mc;
        // L = (I + Mc)^-1: V_m = S_{c_m} * prod_{j in Mc_m} V_j, so L_m = e_m ^ XOR_{j in Mc_m} L_j.
        // Lane m accumulates the L_j of its members as they become final (one shuffle per j).
        uint32_t acc = 0;
        for (uint32_t j = 0; j < kB; ++j) {
            const uint32_t lj = __shfl_sync(0xffffffffu, acc ^ (1u << tid), j); // L_j is final at step j
            if ((mc >> j) & 1u) acc ^= lj;
        }
        vinfo[VI_L + tid] = v ? (acc ^ (1u << tid)) : 0u;
        if (a.nb) vinfo[VI_VBN + tid] = vbn_lane(tid, v, s_c[tid], v ? (acc ^ (1u << tid)) : 0u, a.x, a.pitch, ng,
                                                 a.nfq, a.nb);
    }
    if (tid == 0) {
        bctl[BL_LEN] = len;
        bctl[BL_DET] = s_stop; // (d_pos advances in k_batch_signs, on every shard)
        bctl[BL_SKIP] = 0;
    }
}

__global__ void __launch_bounds__(kSelThreads) k_pivot_select(SelectArgs a) {
    pdl_wait();
    select_body<kSelThreads>(a);
}

__global__ void k_set_u32(uint32_t *p, uint32_t v) { *p = v; }

// Sharded batch plan, computed identically on every shard from the all-gathered stabilizer
// OR-masks (shard.cpp): the leader L = first shard with bit 0 set holds the global pivot of
// collapse 0; a shard d < L has no stabilizer with X at q_m for m < ctz(mask_d), so L can run
// the batch's first lim = min(b, min_{d<L} ctz(mask_d)) collapses alone. No L: the measurement
// is deterministic now (measure.hpp:417-421). A speculative batch whose start is not the device
// position is skipped. plan = {this shard leads, lim, deterministic, skipped}.
__global__ void k_shard_plan(const uint32_t *__restrict__ masks, int world, int rank, uint32_t b,
                             uint32_t expect, const uint32_t *__restrict__ d_pos, uint32_t *__restrict__ plan) {
    pdl_wait();
    if (threadIdx.x != 0) return;
    const bool skip = *d_pos != expect;
    int L = -1;
    for (int r = 0; r < world && L < 0; ++r)
        if (masks[r] & 1u) L = r;
    uint32_t lim = b;
    for (int r = 0; r < L; ++r) lim = min(lim, masks[r] ? uint32_t(__ffs(masks[r]) - 1) : 32u);
    plan[0] = (!skip && L == rank) ? 1u : 0u;
    plan[1] = lim;
    plan[2] = (!skip && L < 0) ? 1u : 0u;
    plan[3] = skip ? 1u : 0u;
}

// Batch start: control words and the pivot kernels' phase sums (one launch instead of two
// memsets, so the whole batch chain is kernel-to-kernel).
__global__ void k_batch_reset(uint32_t *__restrict__ bctl, int *__restrict__ pcount, uint32_t *__restrict__ vinfo) {
    pdl_wait();
    if (threadIdx.x < 4) bctl[threadIdx.x] = 0u;
    if (threadIdx.x < 2 * kB) pcount[threadIdx.x] = 0;
    if (threadIdx.x < kB) vinfo[VI_PMAT + threadIdx.x] = 0u; // accumulated by k_pivot_rows
}

// B2. Pivot rows, parallel over (collapse, word): with L = (I + Mc)^-1 from B1, V_m = XOR over
// j in L_m of the pivot stabilizers S_{c_j} as they stood at batch start, so every V_m word is
// independent. A CTA owns kRowWords words of all V's: it stages the batch-start pivot rows of its
// words in shared memory, thread (m, w) forms V_m, the telescoped phase pieces of V_m (its
// products' cross terms are the pair-parity matrix, file header) and row m of the pair-parity
// matrix over its words; then the pivot pairs are replaced (D_c <- V_m, S_c <- Z_{q_m}).
constexpr int kRowWords = 8;
constexpr int kRowThreads = kB * kRowWords;

struct RowsArgs {
    uint64_t *x, *z;
    uint64_t pitch, ng, g0;
    const uint32_t *fq;
    uint64_t *Vx, *Vz;
    uint64_t vstride;
    uint32_t *vinfo;
    const uint32_t *bctl;
    int *pcount;
};

__device__ __forceinline__ void rows_body(const RowsArgs &a, uint32_t block) {
    uint64_t *__restrict__ x = a.x, *__restrict__ z = a.z, *__restrict__ Vx = a.Vx, *__restrict__ Vz = a.Vz;
    const uint64_t pitch = a.pitch, ng = a.ng, g0 = a.g0, vstride = a.vstride;
    const uint32_t *__restrict__ fq = a.fq;
    uint32_t *__restrict__ vinfo = a.vinfo;
    const uint32_t *__restrict__ bctl = a.bctl;
    int *__restrict__ pcount = a.pcount;
    __shared__ u64 s_sx[kB][kRowWords], s_sz[kB][kRowWords], s_vx[kB][kRowWords];
    __shared__ uint32_t s_c[kB], s_l[kB];
    const uint32_t len = bctl[BL_LEN];
    if (len == 0) return;
    const uint32_t tid = threadIdx.x, m = tid / kRowWords, w = tid % kRowWords;
    if (tid < kB) {
        s_c[tid] = tid < len ? uint32_t(vinfo[VI_C + tid] - g0) : 0u;
        s_l[tid] = tid < len ? vinfo[VI_L + tid] : 0u;
    }
    __syncthreads();
    const uint64_t i = uint64_t(block) * kRowWords + w;
    const bool act = i < pitch;
    {   // stage: thread (m, w) loads S_{c_m} word i (x and z)
        const uint64_t rs = ng + s_c[m];
        const bool ld = act && m < len;
        s_sx[m][w] = ld ? __ldcg(x + rs * pitch + i) : 0ull;
        s_sz[m][w] = ld ? __ldcg(z + rs * pitch + i) : 0ull;
    }
    __syncthreads();
    u64 vx = 0, vz = 0;
    for (uint32_t L = s_l[m]; L; L &= L - 1) {
        const uint32_t j = __ffs(L) - 1;
        vx ^= s_sx[j][w];
        vz ^= s_sz[j][w];
    }
    s_vx[m][w] = vx;
    const u64 x0 = s_sx[m][w], z0 = s_sz[m][w];
    // E_m pieces: beta(S_c) - beta(V_m) + 2 parity(|dz & x0|), dz = V_mz ^ S_cz (the cross terms
    // between members, Q(Mc_m), come from the pair-parity rows in k_pivot_finish).
    int e = __popcll(x0 & z0) - __popcll(vx & vz) + 2 * (__popcll((vz ^ z0) & x0) & 1);
    int bend = __popcll(vx & vz);
    __syncthreads();
    uint32_t prow = 0; // bit j' < m: parity(|V_mz & V_j'x|) over this word
    for (uint32_t jp = 0; jp < m; ++jp) prow |= uint32_t(__popcll(vz & s_vx[jp][w]) & 1) << jp;
    // Reduce over the kRowWords lanes of collapse m (consecutive lanes of one warp).
#pragma unroll
    for (int o = kRowWords / 2; o >= 1; o >>= 1) {
        e += __shfl_xor_sync(0xffffffffu, e, o);
        bend += __shfl_xor_sync(0xffffffffu, bend, o);
        prow ^= __shfl_xor_sync(0xffffffffu, prow, o);
    }
    if (w == 0 && m < len) {
        if (e) atomicAdd(pcount + m, e);
        if (bend) atomicAdd(pcount + kB + m, bend);
        if (prow) atomicXor(vinfo + VI_PMAT + m, prow);
    }
    if (!act || m >= len) return;
    Vx[uint64_t(m) * vstride + i] = vx;
    Vz[uint64_t(m) * vstride + i] = vz;
    // Replace the pivot pairs: D_c <- V_m (bits), S_c <- Z_{q_m}; word i of row S_c was staged
    // above, and only this CTA touches word i.
    const uint64_t c = s_c[m], q = fq[m];
    x[c * pitch + i] = vx;
    z[c * pitch + i] = vz;
    x[(ng + c) * pitch + i] = 0ull;
    z[(ng + c) * pitch + i] = i == (q >> 6) ? (1ull << (q & 63)) : 0ull;
}

__global__ void __launch_bounds__(kRowThreads) k_pivot_rows(RowsArgs a) {
    pdl_wait();
    rows_body(a, blockIdx.x);
}

// B3. Signs of the V_m (telescoped phase, file header), coins, record entries and the signs of
// the replaced pairs. One warp: lane m stages collapse m's inputs and draws its coin (coins depend
// only on their index), lane 0 runs the sign chain over shared memory, lanes write the results.
struct FinishArgs {
    uint64_t *s;
    uint64_t ng, g0;
    const uint32_t *fq, *fidx;
    uint32_t *vinfo;
    const uint32_t *bctl;
    const int *pcount;
    uint64_t seed;
    const uint64_t *coin_index;
    qsr_record_entry *out;
    int *err;
    const uint8_t *coin_table;
};

// One warp (lane = threadIdx.x & 31).
__device__ __forceinline__ void finish_body(const FinishArgs &a) {
    uint64_t *__restrict__ s = a.s;
    const uint64_t ng = a.ng, g0 = a.g0, seed = a.seed;
    const uint32_t *__restrict__ fq = a.fq, *__restrict__ fidx = a.fidx, *__restrict__ bctl = a.bctl;
    uint32_t *__restrict__ vinfo = a.vinfo;
    const int *__restrict__ pcount = a.pcount;
    const uint64_t *__restrict__ coin_index = a.coin_index;
    qsr_record_entry *__restrict__ out = a.out;
    int *__restrict__ err = a.err;
    const uint8_t *__restrict__ coin_table = a.coin_table;
    __shared__ uint32_t s_c[kB], s_mc[kB], s_ss[kB], s_coin[kB], s_vsign[kB], s_beta[kB], s_p[kB];
    __shared__ int s_e[kB];
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t len = bctl[BL_LEN];
    if (len == 0) return;
    const uint64_t idx0 = *coin_index; // advanced by len in k_batch_signs
    if (lane < len) {
        const uint64_t c = vinfo[VI_C + lane] - g0, rs = ng + c;
        s_c[lane] = uint32_t(c);
        s_mc[lane] = vinfo[VI_MC + lane];
        s_e[lane] = pcount[lane];
        s_beta[lane] = uint32_t(pcount[kB + lane]) & 3u;
        s_ss[lane] = uint32_t((s[rs >> 6] >> (rs & 63)) & 1u); // S_c sign at batch start
        s_p[lane] = vinfo[VI_PMAT + lane];
        s_coin[lane] = draw_coin(seed, idx0 + lane, coin_table);
    }
    __syncwarp();
    // Lane m: E_m + sum_{j in Mc_m} beta(V_j) needs no chain (beta(V_j) is known for every j);
    // the signs are a unit-triangular GF(2) system, solved one ballot per collapse.
    uint32_t mc = 0, base = 0;
    bool odd = false;
    if (lane < len) {
        mc = s_mc[lane];
        int E = s_e[lane];
        uint32_t qf = 0; // Q(Mc_m): pairs j' < j of Mc_m with P(j', j) = 1
        for (uint32_t U = mc; U; U &= U - 1) {
            const uint32_t j = __ffs(U) - 1;
            E += int(s_beta[j]);
            qf ^= parity32(mc & s_p[j]);
        }
        E += 2 * int(qf);
        odd = (E & 1) != 0;
        base = s_ss[lane] ^ ((uint32_t(E) >> 1) & 1u);
    }
    uint32_t vs = 0; // bit j = sign of V_j
    for (uint32_t m = 0; m < len; ++m) {
        const uint32_t bit = __shfl_sync(0xffffffffu, base ^ parity32(mc & vs), m);
        vs |= bit << m;
    }
    if (lane < len) {
        s_vsign[lane] = (vs >> lane) & 1u;
        // Replaced pair: D_c <- sign of V_m, S_c <- coin. The c_m are distinct, so every lane owns
        // its two bits; lanes sharing a 64-bit word combine through bitwise atomics.
        const uint64_t c = s_c[lane], rs = ng + c;
        const unsigned long long bc = 1ull << (c & 63), br = 1ull << (rs & 63);
        auto *sw = reinterpret_cast<unsigned long long *>(s);
        if ((vs >> lane) & 1u) atomicOr(sw + (c >> 6), bc); else atomicAnd(sw + (c >> 6), ~bc);
        if (s_coin[lane]) atomicOr(sw + (rs >> 6), br); else atomicAnd(sw + (rs >> 6), ~br);
    }
    if (__any_sync(0xffffffffu, odd) && lane == 0) atomicExch(err, 1);
    __syncwarp();
    if (lane < len) {
        out[fidx[lane]] = qsr_record_entry{fq[lane], uint8_t(s_coin[lane]), 0};
        vinfo[VI_SIGN + lane] = s_vsign[lane];
        vinfo[VI_BETA + lane] = s_beta[lane];
    } else {
        vinfo[VI_SIGN + lane] = 0;
        vinfo[VI_BETA + lane] = 0;
    }
}

__global__ void __launch_bounds__(32) k_pivot_finish(FinishArgs a) {
    pdl_wait();
    finish_body(a);
}

constexpr int kSlice = 64; // words per staged V slice (2 per lane)

// ---- phase C: membership pass, slice-major absorb pass, sign pass -----------------------
// Absorbing V_j1, V_j2, ... (ascending j, the row's membership set M) in order, the telescoped
// phase (file header) needs parity(sum_j |V_jz & cur_x before V_j|). With cur_x = x0 ^
// XOR_{j'<j in M} V_j'x this is  parity(|dz & x0|) ^ Q(M),  dz = XOR_{j in M} V_jz and
// Q(M) = XOR_{j'<j, both in M} P(j', j),  P(j', j) = parity(sum_i |V_jz[i] & V_j'x[i]|).
// So the absorb pass only XORs row deltas; the quadratic form is a per-row 32-bit fold.
// C1 k_batch_member: M[r] (bit m = row r absorbs V_m) for every row, written over colbits (the
//    pair-parity matrix rows P(j', j) arrive with the batch block, from k_pivot_rows).
// C2 k_batch_absorb: persistent, one CTA per SM walks (slice, row) items slice-major; for its
//    64-word slice it stages, per group of 4 consecutive V's, all 16 XOR combinations
//    T[g][S] = XOR_{j in S} V_{4g+j} (x and z; T[g][0] = 0) in shared memory, so a row
//    absorbs its members S = (M >> 4g) & 15 of a group with one branch-free lookup. Per
//    (row, slice) it stores (beta(start) - beta(end) + 2 parity(|dz & x0|)) mod 4 as a byte.
// C3 k_batch_signs: per row, sums its slice bytes, adds sum beta(V_j), 2 Q(M) and the V signs
//    (file header), and flips the sign bit; a warp ballot forms each 32-bit half-word of the
//    sign vector (one writer per half-word, no atomics).
constexpr int kAThreads = 512;
constexpr int kAWarps = kAThreads / 32;
constexpr int kARows = 4;                    // rows in flight per warp
constexpr int kGroups = kB / 4;              // 8 groups of 4 V's
constexpr size_t kTableWords = size_t(kGroups) * 16 * 2 * kSlice; // 128 KB
constexpr size_t kAbsorbSmem = kTableWords * sizeof(u64);

struct MemberArgs {
    uint32_t *colbits;
    uint64_t nrows, ng, g0;
    const uint32_t *vinfo, *bctl;
    unsigned long long *touched;
    // Chained one-GPU batches: the next batch's column bits and active ballot, from each row's
    // current X bits at its qubits (rows other than the pivots are not rewritten before the
    // absorb) and the X bits there of the V's it will absorb (VI_VBN).
    const uint64_t *x;
    uint64_t pitch;
    const uint32_t *nfq;
    uint32_t nb;
    uint32_t *colbits_next, *nz_next;
};

__device__ __forceinline__ void member_body(const MemberArgs &a, uint32_t block) {
    uint32_t *__restrict__ colbits = a.colbits;
    const uint64_t nrows = a.nrows, ng = a.ng, g0 = a.g0;
    const uint32_t *__restrict__ vinfo = a.vinfo, *__restrict__ bctl = a.bctl;
    unsigned long long *__restrict__ touched = a.touched;
    __shared__ uint32_t s_vbcol[kB], s_c[kB], s_vb[kB], s_vbn[kB], s_nq[kB];
    const uint32_t len = bctl[BL_LEN];
    const uint32_t tid = threadIdx.x;
    if (tid < kB) {
        s_vbn[tid] = a.nb ? vinfo[VI_VBN + tid] : 0u;
        if (tid < a.nb) s_nq[tid] = a.nfq[tid];
        s_vb[tid] = vinfo[VI_VB + tid];
        const uint32_t cg = vinfo[VI_C + tid];
        s_c[tid] = (cg != 0xFFFFFFFFu && cg >= g0 && cg < g0 + ng) ? uint32_t(cg - g0) : 0xFFFFFFFFu;
    }
    __syncthreads();
    if (tid < kB) {
        uint32_t col = 0;
        for (uint32_t mp = 0; mp < len && mp < tid; ++mp) col |= ((s_vb[mp] >> tid) & 1u) << mp;
        s_vbcol[tid] = col;
    }
    __syncthreads();
    const uint64_t r = uint64_t(block) * blockDim.x + tid;
    if (len == 0) return;
    uint32_t M = 0, ncb = 0;
    if (r < nrows) {
        // Pivot stabilizers are final already; replaced destabilizers restart from V_m after
        // collapse m; every other row starts from its batch-start column bits.
        uint32_t cb = colbits[r], start = 0;
        bool skip = false;
        for (uint32_t j = 0; j < len; ++j) {
            if (s_c[j] == 0xFFFFFFFFu) continue;
            if (r == ng + s_c[j]) skip = true;
            if (r == s_c[j]) { cb = s_vb[j]; start = j + 1; }
        }
        M = skip ? 0u : membership(cb, s_vbcol, start, len);
        colbits[r] = M;
        if (a.nb) { // (the pivot stabilizers become +/-Z_q: no X bits, ncb = 0)
            if (!skip) {
                if (start) {
                    ncb = s_vbn[start - 1]; // destabilizer D_c <- V_{start-1}
                } else {
                    const uint64_t *row = a.x + r * a.pitch;
                    uint32_t wi = 0xFFFFFFFFu;
                    uint64_t word = 0;
                    for (uint32_t m = 0; m < a.nb; ++m) {
                        const uint32_t q = s_nq[m];
                        if ((q >> 6) != wi) { wi = q >> 6; word = __ldcg(row + wi); }
                        ncb |= uint32_t((word >> (q & 63)) & 1u) << m;
                    }
                }
                for (uint32_t U = M; U; U &= U - 1) ncb ^= s_vbn[__ffs(U) - 1];
            }
            a.colbits_next[r] = ncb;
        }
    }
    if (a.nb) {
        const bool stab = r >= ng && r < nrows;
        const uint32_t act = __ballot_sync(0xffffffffu, stab && ncb != 0u);
        if ((tid & 31) == 0 && stab) a.nz_next[(r - ng) >> 5] = act;
    }
    if (touched) { // profile runs only: rows the absorb pass rewrites
        const uint32_t b = __ballot_sync(0xffffffffu, M != 0u);
        if ((tid & 31) == 0 && b) atomicAdd(touched, (unsigned long long)__popc(b));
    }
}

__global__ void __launch_bounds__(256) k_batch_member(MemberArgs a) {
    pdl_wait();
    member_body(a, blockIdx.x);
}

// One-GPU chain: the pivot rows (blocks < rblocks) and the memberships (the rest) in one launch —
// both need only the select's output.
__global__ void __launch_bounds__(256) k_rows_member(RowsArgs ra, MemberArgs ma, uint32_t rblocks) {
    pdl_wait();
    if (blockIdx.x < rblocks) rows_body(ra, blockIdx.x);
    else member_body(ma, blockIdx.x - rblocks);
}

__global__ void __launch_bounds__(kAThreads, 1)
k_batch_absorb(uint64_t *__restrict__ x, uint64_t *__restrict__ z, uint64_t pitch,
               uint64_t nrows, const uint32_t *__restrict__ member,
               const uint64_t *__restrict__ Vx, const uint64_t *__restrict__ Vz, uint64_t vstride,
               const uint32_t *__restrict__ bctl, uint8_t *__restrict__ partial, uint64_t stride,
               FinishArgs fin, int do_finish, SelectArgs sel, int sel_cta) {
    pdl_wait();
    // Chained one-GPU batches: the last CTA selects the next batch's pivots (from column bits the
    // membership pass already derived) while the others absorb this one; it runs even when this
    // batch is empty, so the next batch's control words are always written.
    if (sel_cta && blockIdx.x == gridDim.x - 1) {
        select_body<kAThreads>(sel);
        return;
    }
    const uint32_t grid = gridDim.x - (sel_cta ? 1u : 0u);
    extern __shared__ __align__(16) u64 tab[]; // [g][S][plane][kSlice]
    const uint32_t len = bctl[BL_LEN];
    if (len == 0) return;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // One-GPU chain: B3 (signs of the V's, coins, record) rides in CTA 0's first warp; only the
    // sign pass after this kernel reads its output.
    if (do_finish && blockIdx.x == 0 && warp == 0) finish_body(fin);
    const uint32_t ngroups = (len + 3) / 4;
    const uint64_t nslices = (pitch + kSlice - 1) / kSlice;
    // Work items are (slice, row group of kARows rows). Within a slice, blocks of kAWarps
    // consecutive groups (one per warp: 64 contiguous rows per CTA step, page-friendly) are
    // visited in the order b -> (b * stride) mod nblk (a bijection, stride coprime with nblk; the
    // tail groups map to themselves): rows that absorb nothing (the growing block of collapsed
    // stabilizers of a measure-all window) spread over all CTAs instead of idling a few.
    const uint64_t ngr = (nrows + kARows - 1) / kARows;
    const uint64_t nblk = nrows / (uint64_t(kARows) * kAWarps), nmapped = nblk * kAWarps;
    const uint64_t total = nslices * ngr;
    const uint64_t item0 = total * blockIdx.x / grid, item1 = total * (blockIdx.x + 1) / grid;
    const uint64_t step = nblk ? stride % nblk : 0;
    uint64_t it = item0;
    while (it < item1) {
        const uint64_t sl = it / ngr;
        const uint64_t g_begin = it - sl * ngr;
        const uint64_t g_end = min(ngr, g_begin + (item1 - it));
        const uint64_t w0 = sl * kSlice;
        // Build the combination table of this slice.
        __syncthreads(); // previous slice's readers are done
        for (uint32_t e = tid; e < ngroups * 2 * (kSlice / 2); e += kAThreads) {
            const uint32_t wp = e % (kSlice / 2), plane = (e / (kSlice / 2)) & 1, g = e / kSlice;
            const uint64_t gw = w0 + 2 * wp;
            ulonglong2 v[4];
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const uint32_t j = 4 * g + b;
                v[b] = make_ulonglong2(0ull, 0ull);
                if (j < len && gw < pitch)
                    v[b] = __ldcg(reinterpret_cast<const ulonglong2 *>((plane ? Vz : Vx) + uint64_t(j) * vstride + gw));
            }
            u64 *dst = tab + (size_t(g) * 16 * 2 + plane) * kSlice + 2 * wp;
#pragma unroll
            for (uint32_t S = 0; S < 16; ++S) {
                u64 a = 0, b2 = 0;
#pragma unroll
                for (int b = 0; b < 4; ++b)
                    if ((S >> b) & 1u) { a ^= v[b].x; b2 ^= v[b].y; }
                *reinterpret_cast<ulonglong2 *>(dst + size_t(S) * 2 * kSlice) = make_ulonglong2(a, b2);
            }
        }
        __syncthreads();
        const uint64_t i = w0 + 2 * lane;
        const bool act = i < pitch;
        // Group u -> first row; pos tracks ((u / kAWarps) * stride) mod nblk incrementally
        // (u advances by kAWarps, so its block by one and its place in the block stays wq).
        uint64_t u = g_begin + warp;
        const uint64_t wq = u % kAWarps;
        uint64_t pos = nblk ? ((u / kAWarps) % nblk) * step % nblk : 0;
        auto first_row = [&](uint64_t uu, uint64_t pp) {
            return (uu < nmapped ? pp * kAWarps + wq : uu) * kARows;
        };
        // Memberships of the next row group are loaded one iteration ahead (their L2 round
        // trip overlaps this group's loads and table lookups).
        uint32_t Mn[kARows];
        {
            const uint64_t b0 = first_row(u, pos);
#pragma unroll
            for (int q = 0; q < kARows; ++q) Mn[q] = u < g_end && b0 + q < nrows ? member[b0 + q] : 0u;
        }
        for (; u < g_end; u += kAWarps) {
            const uint64_t base = first_row(u, pos);
            pos += step;
            if (pos >= nblk) pos -= nblk;
            const uint64_t un = u + kAWarps, nb = first_row(un, pos);
            uint32_t M[kARows];
            uint32_t U = 0;
#pragma unroll
            for (int q = 0; q < kARows; ++q) {
                M[q] = Mn[q];
                U |= M[q];
                Mn[q] = un < g_end && nb + q < nrows ? member[nb + q] : 0u;
            }
            if (U == 0) continue;
            ulonglong2 x0[kARows], z0[kARows], dx[kARows], dz[kARows];
#pragma unroll
            for (int q = 0; q < kARows; ++q) {
                x0[q] = make_ulonglong2(0ull, 0ull);
                z0[q] = x0[q];
                dx[q] = x0[q];
                dz[q] = x0[q];
                if (M[q] && act) {
                    x0[q] = __ldcs(reinterpret_cast<const ulonglong2 *>(x + (base + q) * pitch + i));
                    z0[q] = __ldcs(reinterpret_cast<const ulonglong2 *>(z + (base + q) * pitch + i));
                }
            }
            const u64 *tl = tab + 2 * lane;
            for (uint32_t g = 0; g < ngroups; ++g) {
#pragma unroll
                for (int q = 0; q < kARows; ++q) {
                    const uint32_t S = (M[q] >> (4 * g)) & 15u; // S = 0 reads the zero entry
                    const u64 *te = tl + (size_t(g) * 16 + S) * 2 * kSlice;
                    const ulonglong2 tx = *reinterpret_cast<const ulonglong2 *>(te);
                    const ulonglong2 tz = *reinterpret_cast<const ulonglong2 *>(te + kSlice);
                    dx[q].x ^= tx.x; dx[q].y ^= tx.y;
                    dz[q].x ^= tz.x; dz[q].y ^= tz.y;
                }
            }
            // Per row: (beta(x0,z0) - beta(end) + 2 parity(|dz & x0|)) mod 4 per lane, packed one
            // byte per row (each lane's value < 4, a warp's sum < 256) into a single warp sum.
            uint32_t packed = 0;
#pragma unroll
            for (int q = 0; q < kARows; ++q) {
                const u64 ex = x0[q].x ^ dx[q].x, ey = x0[q].y ^ dx[q].y;
                const u64 fx = z0[q].x ^ dz[q].x, fy = z0[q].y ^ dz[q].y;
                const int v = __popcll(x0[q].x & z0[q].x) + __popcll(x0[q].y & z0[q].y) -
                              __popcll(ex & fx) - __popcll(ey & fy) +
                              2 * (__popcll((dz[q].x & x0[q].x) ^ (dz[q].y & x0[q].y)) & 1);
                packed |= uint32_t(v & 3) << (8 * q);
                if (M[q] && act) {
                    __stcs(reinterpret_cast<ulonglong2 *>(x + (base + q) * pitch + i), make_ulonglong2(ex, ey));
                    __stcs(reinterpret_cast<ulonglong2 *>(z + (base + q) * pitch + i), make_ulonglong2(fx, fy));
                }
            }
            packed = __reduce_add_sync(0xffffffffu, packed);
            if (lane < kARows && M[lane] != 0u) // M[] is warp-uniform; lane q writes row q
                partial[sl * nrows + base + lane] = uint8_t((packed >> (8 * lane)) & 3u);
        }
        it += g_end - g_begin;
    }
}

// The next batch's column-bit pass riding the sign pass (one GPU, speculative successor): b = 0
// means none.
struct NextCols {
    const uint64_t *x;
    uint64_t pitch, ng;
    const uint32_t *fq;
    uint32_t b;
    uint32_t *nz;
};
// Chained batches: the X bits of batch k+1's V's at batch k+2's qubits (VI_VBN of k+1), formed by
// batch k's sign pass, the first point where batch k+1's pivot rows are final. nb = 0: none.
struct VbnNext {
    const uint64_t *x;
    uint64_t pitch, ng;
    uint32_t *vinfo;
    const uint32_t *bctl;
    const uint32_t *nfq;
    uint32_t nb;
};

__global__ void __launch_bounds__(256)
k_batch_signs(uint64_t *__restrict__ s, uint64_t nrows, uint64_t nslices,
              uint32_t *member, const uint8_t *__restrict__ partial,
              const uint32_t *__restrict__ vinfo, const uint32_t *__restrict__ bctl,
              int *__restrict__ err, uint32_t *__restrict__ d_pos, uint64_t *__restrict__ coin_index,
              uint32_t *__restrict__ host_slot, uint32_t seq, NextCols nc, VbnNext vn) {
    pdl_wait();
    __shared__ uint32_t s_vs_mask, s_b0_mask, s_b1_mask, s_p[kB], s_nq[kB];
    if (host_slot && blockIdx.x == 0 && threadIdx.x == 0) { // the batch is decided: tell the host
        volatile uint32_t *h = host_slot;
        for (int i = 0; i < 4; ++i) h[i] = bctl[i];
        __threadfence_system();
        h[4] = seq;
    }
    const uint32_t len = bctl[BL_LEN];
    if (len == 0) return;
    const uint32_t tid = threadIdx.x;
    if (vn.nb && blockIdx.x == 0 && tid < kB) {
        const uint32_t lenn = vn.bctl[BL_SKIP] ? 0u : vn.bctl[BL_LEN];
        if (lenn) {
            const bool v = tid < lenn;
            const uint32_t cg = v ? vn.vinfo[VI_C + tid] : 0u, L = v ? vn.vinfo[VI_L + tid] : 0u;
            vn.vinfo[VI_VBN + tid] = vbn_lane(tid, v, cg, L, vn.x, vn.pitch, vn.ng, vn.nfq, vn.nb);
        }
    }
    // The batch is decided: advance the speculation position and the coin index, on every shard
    // alike (B3 drew coins idx0 .. idx0 + len - 1).
    if (blockIdx.x == 0 && tid == 0) {
        if (d_pos) *d_pos += len;
        *coin_index += len;
    }
    if (tid < kB) { // one warp: lane j loads V_j's words, ballots form the masks (kB == 32)
        const bool v = tid < len;
        const uint32_t sg = v ? vinfo[VI_SIGN + tid] : 0u, beta = v ? vinfo[VI_BETA + tid] : 0u;
        s_p[tid] = v ? vinfo[VI_PMAT + tid] : 0u;
        const uint32_t vs = __ballot_sync(0xffffffffu, sg & 1u), b0 = __ballot_sync(0xffffffffu, beta & 1u),
                       b1 = __ballot_sync(0xffffffffu, (beta >> 1) & 1u);
        if (tid == 0) s_vs_mask = vs, s_b0_mask = b0, s_b1_mask = b1;
        if (tid < nc.b) s_nq[tid] = nc.fq[tid];
    }
    __syncthreads();
    const uint64_t r = uint64_t(blockIdx.x) * blockDim.x + tid;
    uint32_t f = 0;
    bool odd = false;
    uint32_t M = 0;
    if (r < nrows) {
        M = member[r];
        if (M) {
            int E = 0;
            for (uint64_t sl = 0; sl < nslices; ++sl) E += partial[sl * nrows + r];
            uint32_t qf = 0; // Q(M): pairs j' < j of M with P(j', j) = 1
            for (uint32_t U = M; U; U &= U - 1) qf ^= parity32(M & s_p[__ffs(U) - 1]);
            E += 2 * int(qf) + __popc(M & s_b0_mask) + 2 * __popc(M & s_b1_mask);
            odd = (E & 1) != 0;
            f = parity32(M & s_vs_mask) ^ ((uint32_t(E) >> 1) & 1u);
        }
    }
    const uint32_t bits = __ballot_sync(0xffffffffu, f != 0);
    if (__any_sync(0xffffffffu, odd) && (tid & 31) == 0) atomicExch(err, 1);
    if ((tid & 31) == 0 && bits && r < nrows)
        reinterpret_cast<uint32_t *>(s)[r >> 5] ^= bits; // rows r..r+31 own this half-word
    if (nc.b) { // the next batch's column bits and active ballot (k_colbits), from the final rows
        uint32_t cb = 0;
        if (r < nrows) {
            const uint64_t *row = nc.x + r * nc.pitch;
            uint32_t wi = 0xFFFFFFFFu;
            uint64_t word = 0;
            for (uint32_t m = 0; m < nc.b; ++m) {
                const uint32_t q = s_nq[m];
                if ((q >> 6) != wi) { wi = q >> 6; word = __ldcg(row + wi); }
                cb |= uint32_t((word >> (q & 63)) & 1u) << m;
            }
            member[r] = cb; // (this thread read its membership above)
        }
        const uint32_t act = __ballot_sync(0xffffffffu, r >= nc.ng && r < nrows && cb != 0);
        if ((tid & 31) == 0 && r >= nc.ng && r < nrows) nc.nz[(r - nc.ng) >> 5] = act;
    }
}

} // namespace

// QSR_PDL=0 restores plain launches for the batch chain (as for the gate windows).
static bool chain_pdl() {
    static const bool on = [] {
        const char *e = getenv("QSR_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

template <typename... P, typename... A>
static void launch_chain(void (*k)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, A &&...args) {
    if (chain_pdl()) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = block;
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        QSR_CUDA(cudaLaunchKernelEx(&cfg, k, std::forward<A>(args)...));
    } else {
        k<<<grid, block, smem, st>>>(std::forward<A>(args)...);
    }
    QSR_CUDA(cudaGetLastError());
}

void batch_colbits(DeviceTableau &t, const uint32_t *d_fq, uint32_t b, bool zero_block) {
    MeasureScratch &ms = t.ms;
    const uint64_t nrows = 2 * t.ng;
    // Sharded batches: control words and the pivot kernels' phase sums zeroed ahead of the chain
    // on every shard (the one-GPU chain's select does this itself: one launch fewer per batch).
    if (zero_block) {
        launch_chain(k_batch_reset, dim3(1), dim3(2 * kB), 0, t.stream, ms.bctl, ms.pcount, ms.vinfo);
        count_launch();
    }
    // The pivot rows and vinfo of the block (everything before bctl), zeroed for a sharded batch.
    const uint64_t zw = zero_block ? uint64_t(reinterpret_cast<uint64_t *>(ms.vinfo) - ms.batch_block) +
                                         (kVinfoWords * 4 + 7) / 8
                                   : 0;
    launch_chain(k_colbits, dim3(unsigned((nrows + 255) / 256)), dim3(256), 0, t.stream,
                 static_cast<const uint64_t *>(t.x), t.rm_pitch, nrows, t.ng, d_fq, b, ms.colbits,
                 ms.bctl + BL_STAB_OR, ms.nz, ms.batch_block, zw);
    count_launch();
}

void shard_plan(DeviceTableau &t, const uint32_t *d_masks, int world, int rank, uint32_t b, uint32_t expect,
                uint32_t *d_plan) {
    launch_chain(k_shard_plan, dim3(1), dim3(32), 0, t.stream, d_masks, world, rank, b, expect,
                 static_cast<const uint32_t *>(t.ms.d_pos), d_plan);
    count_launch();
}

void set_device_u32(uint32_t *p, uint32_t v, cudaStream_t st) {
    k_set_u32<<<1, 1, 0, st>>>(p, v);
    QSR_CUDA(cudaGetLastError());
    count_launch();
}

namespace {
RowsArgs rows_args(DeviceTableau &t, const uint32_t *d_fq) {
    MeasureScratch &ms = t.ms;
    return RowsArgs{t.x, t.z, t.rm_pitch, t.ng, t.g0, d_fq, ms.Vx, ms.Vz, ms.vstride, ms.vinfo, ms.bctl, ms.pcount};
}
FinishArgs finish_args(DeviceTableau &t, const uint32_t *d_fq, const uint32_t *d_fidx, uint64_t seed) {
    MeasureScratch &ms = t.ms;
    return FinishArgs{t.s, t.ng, t.g0, d_fq, d_fidx, ms.vinfo, ms.bctl, ms.pcount, seed, ms.coin_index, ms.out, ms.err,
                      ms.coin_table};
}
MemberArgs member_args(DeviceTableau &t) {
    MeasureScratch &ms = t.ms;
    return MemberArgs{ms.colbits, 2 * t.ng, t.ng, t.g0, ms.vinfo, ms.bctl, t.prof ? t.prof->d_rows : nullptr,
                      nullptr, 0, nullptr, 0, nullptr, nullptr};
}
SelectArgs select_args(DeviceTableau &t, uint32_t b, uint32_t *d_pos, uint32_t expect, const uint32_t *d_plan) {
    MeasureScratch &ms = t.ms;
    SelectArgs a{};
    a.colbits = ms.colbits;
    a.nz = ms.nz;
    a.n_gen = t.n_gen;
    a.ng = t.ng;
    a.g0 = t.g0;
    a.b = b;
    a.vinfo = ms.vinfo;
    a.bctl = ms.bctl;
    a.d_pos = d_pos;
    a.expect = expect;
    a.plan = d_plan;
    a.pcount = ms.pcount; // (sharded: zeroed by batch_colbits; one GPU: by the select itself)
    return a;
}
void launch_select(const SelectArgs &a, cudaStream_t st) {
    launch_chain(k_pivot_select, dim3(1), dim3(kSelThreads), 0, st, a);
    count_launch();
}
void launch_select(DeviceTableau &t, uint32_t b, uint32_t *d_pos, uint32_t expect, const uint32_t *d_plan) {
    launch_select(select_args(t, b, d_pos, expect, d_plan), t.stream);
}
uint32_t rows_blocks(const DeviceTableau &t) { return uint32_t((t.rm_pitch + kRowWords - 1) / kRowWords); }
} // namespace

void batch_pivots(DeviceTableau &t, const uint32_t *d_fq, const uint32_t *d_fidx, uint32_t b,
                  uint64_t seed, uint32_t *d_pos, uint32_t expect, const uint32_t *d_plan) {
    launch_select(t, b, d_pos, expect, d_plan);
    launch_chain(k_pivot_rows, dim3(rows_blocks(t)), dim3(kRowThreads), 0, t.stream, rows_args(t, d_fq));
    launch_chain(k_pivot_finish, dim3(1), dim3(32), 0, t.stream, finish_args(t, d_fq, d_fidx, seed));
    count_launch(2);
}

// Function attributes are per device context: raise the absorb pass's dynamic shared memory
// limit once on every device it runs on (a process-wide flag left device 1 at 48 KB).
void configure_batch_kernels(int device) {
    static std::mutex mu;
    static std::vector<bool> done;
    std::lock_guard<std::mutex> g(mu);
    if (device < 0) return;
    if (done.size() <= size_t(device)) done.resize(size_t(device) + 1, false);
    if (done[size_t(device)]) return;
    QSR_CUDA(cudaFuncSetAttribute(k_batch_absorb, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(kAbsorbSmem)));
    done[size_t(device)] = true;
}

// A stride coprime with the number of full row blocks, near its golden section (k_batch_absorb).
uint64_t absorb_stride(uint64_t nfull) {
    if (nfull < 2) return 1;
    uint64_t st = std::max<uint64_t>(1, uint64_t(double(nfull) * 0.6180339887));
    auto gcd = [](uint64_t a, uint64_t b) { while (b) { const uint64_t t = a % b; a = b; b = t; } return a; };
    while (gcd(st, nfull) != 1) ++st;
    return st;
}

namespace {
// Member pass (unless `member` is false: the fused chain ran it with the pivot rows), absorb
// (with B3 in CTA 0 when `fin` is set), signs.
void apply_passes(DeviceTableau &t, bool member, const FinishArgs *fin, uint32_t *host_slot = nullptr,
                  uint32_t seq = 0, const uint32_t *next_fq = nullptr, uint32_t next_b = 0,
                  const SelectArgs *chain_sel = nullptr, VbnNext vn = VbnNext{}) {
    MeasureScratch &ms = t.ms;
    const uint64_t nrows = 2 * t.ng;
    configure_batch_kernels(t.device);
    const uint64_t nslices = (t.rm_pitch + kSlice - 1) / kSlice;
    if (!ms.partial || ms.partial_bytes < nslices * nrows) {
        if (ms.partial) cache_release(t.device, ms.partial_bytes, ms.partial, t.stream);
        ms.partial_bytes = nslices * nrows;
        ms.partial = static_cast<uint8_t *>(cache_acquire(t.device, ms.partial_bytes));
    }
    const uint32_t row_blocks = uint32_t((nrows + 255) / 256);
    if (member) {
        launch_chain(k_batch_member, dim3(row_blocks), dim3(256), 0, t.stream, member_args(t));
        count_launch();
    }
    cudaEvent_t ea = nullptr, eb = nullptr;
    if (t.prof) {
        QSR_CUDA(cudaEventCreate(&ea));
        QSR_CUDA(cudaEventCreate(&eb));
        QSR_CUDA(cudaEventRecord(ea, t.stream));
    }
    const FinishArgs none{};
    const SelectArgs no_sel{};
    launch_chain(k_batch_absorb, dim3(unsigned(t.num_sms)), dim3(kAThreads), kAbsorbSmem, t.stream, t.x, t.z,
                 t.rm_pitch, nrows, ms.colbits, ms.Vx, ms.Vz, ms.vstride, ms.bctl, ms.partial,
                 absorb_stride(nrows / (uint64_t(kARows) * kAWarps)), fin ? *fin : none, fin ? 1 : 0,
                 chain_sel ? *chain_sel : no_sel, chain_sel ? 1 : 0);
    if (t.prof) {
        QSR_CUDA(cudaEventRecord(eb, t.stream));
        t.prof->ev.emplace_back(ea, eb);
    }
    launch_chain(k_batch_signs, dim3(row_blocks), dim3(256), 0, t.stream, t.s, nrows, nslices, ms.colbits,
                 ms.partial, ms.vinfo, ms.bctl, ms.err, ms.d_pos, ms.coin_index, host_slot, seq,
                 NextCols{t.x, t.rm_pitch, t.ng, next_fq, next_fq ? next_b : 0u, ms.nz}, vn);
    count_launch(2);
}
} // namespace

void batch_apply(DeviceTableau &t) { apply_passes(t, true, nullptr); }

void batch_fused(DeviceTableau &t, const uint32_t *d_fq, const uint32_t *d_fidx, uint32_t b, uint64_t seed,
                 uint32_t *d_pos, uint32_t expect, uint32_t *host_slot, uint32_t seq, const uint32_t *next_fq,
                 uint32_t next_b) {
    launch_select(t, b, d_pos, expect, nullptr);
    configure_batch_kernels(t.device);
    const uint32_t rb = rows_blocks(t), mb = uint32_t((2 * t.ng + 255) / 256);
    launch_chain(k_rows_member, dim3(rb + mb), dim3(256), 0, t.stream, rows_args(t, d_fq), member_args(t), rb);
    count_launch();
    const FinishArgs fin = finish_args(t, d_fq, d_fidx, seed);
    apply_passes(t, false, &fin, host_slot, seq, next_fq, next_b);
}

void batch_chained(DeviceTableau &t, const BatchBufs &nxt, const uint32_t *d_fq, const uint32_t *d_fidx,
                   uint32_t b, uint64_t seed, bool standalone, uint32_t *d_pos, uint32_t expect,
                   const uint32_t *nfq, uint32_t nb, const uint32_t *nfq2, uint32_t nb2, uint32_t *host_slot,
                   uint32_t seq) {
    MeasureScratch &ms = t.ms;
    configure_batch_kernels(t.device);
    if (standalone) { // column bits + select of this batch, and its V's bits at the next batch's qubits
        batch_colbits(t, d_fq, b);
        SelectArgs a = select_args(t, b, d_pos, expect, nullptr);
        a.x = t.x;
        a.pitch = t.rm_pitch;
        a.nfq = nfq;
        a.nb = nb;
        launch_select(a, t.stream);
    }
    MemberArgs ma = member_args(t);
    if (nb) {
        ma.x = t.x;
        ma.pitch = t.rm_pitch;
        ma.nfq = nfq;
        ma.nb = nb;
        ma.colbits_next = nxt.colbits;
        ma.nz_next = nxt.nz;
    }
    const uint32_t rb = rows_blocks(t), mb = uint32_t((2 * t.ng + 255) / 256);
    launch_chain(k_rows_member, dim3(rb + mb), dim3(256), 0, t.stream, rows_args(t, d_fq), ma, rb);
    count_launch();
    const FinishArgs fin = finish_args(t, d_fq, d_fidx, seed);
    SelectArgs sel{};
    if (nb) { // the next batch's select, in the absorb's last CTA
        sel.colbits = nxt.colbits;
        sel.nz = nxt.nz;
        sel.n_gen = t.n_gen;
        sel.ng = t.ng;
        sel.g0 = t.g0;
        sel.b = nb;
        sel.vinfo = nxt.vinfo;
        sel.bctl = nxt.bctl;
        sel.pcount = nxt.pcount;
        sel.prev_bctl = ms.bctl;
        sel.prev_b = b;
    }
    VbnNext vn{};
    if (nb && nb2) vn = VbnNext{t.x, t.rm_pitch, t.ng, nxt.vinfo, nxt.bctl, nfq2, nb2};
    apply_passes(t, false, &fin, host_slot, seq, nullptr, 0, nb ? &sel : nullptr, vn);
}

} // namespace qsr
