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
// rows are staged through shared memory (cp.async, double-buffered 64-word slices) and each
// staged word is reused by the 4 rows a warp carries.
#include "common.cuh"
#include "device.hpp"

namespace qsr {

namespace {

using u64 = unsigned long long;
constexpr int kB = kMaxBatch; // collapses per batch (<= 32: u32 membership masks)
enum : uint32_t { BL_LEN = 0, BL_DET = 1, BL_STAB_OR = 2 };
// vinfo layout (u32 [4*kB]): vb | sign of V_m | c_m | beta(V_m) mod 4
enum : uint32_t { VI_VB = 0, VI_SIGN = kB, VI_C = 2 * kB, VI_BETA = 3 * kB };

__device__ __forceinline__ uint32_t parity32(uint32_t v) { return __popc(v) & 1u; }

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

__device__ __forceinline__ int block_sum(int v, int *red /* >= 32 ints */) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    int t = 0;
    if (threadIdx.x < 32) {
        t = threadIdx.x < (blockDim.x + 31) / 32 ? red[threadIdx.x] : 0;
        t = warp_sum(t);
    }
    return t; // valid in warp 0
}

// ---- phase A: column bits of all rows at the batch's measured qubits ----------------
// Also ORs the stabilizer rows' bits into *stab_or: bit m set iff some stabilizer held here has
// X at q_m at batch start (the sharded leader protocol, shard.cpp).
__global__ void k_colbits(const uint64_t *__restrict__ x, uint64_t pitch, uint64_t nrows,
                          uint64_t ng, const uint32_t *__restrict__ fq, uint32_t b,
                          uint32_t *__restrict__ colbits, uint32_t *__restrict__ stab_or) {
    __shared__ uint32_t sq[kB];
    if (threadIdx.x < b) sq[threadIdx.x] = fq[threadIdx.x];
    __syncthreads();
    const uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    uint32_t bits = 0;
    if (r < nrows) {
        const uint64_t *row = x + r * pitch;
        for (uint32_t m = 0; m < b; ++m) {
            const uint32_t q = sq[m];
            bits |= uint32_t((__ldcg(row + (q >> 6)) >> (q & 63)) & 1u) << m;
        }
        colbits[r] = bits;
    }
    const uint32_t any = __reduce_or_sync(0xffffffffu, r >= ng && r < nrows ? bits : 0u);
    if ((threadIdx.x & 31) == 0 && any) atomicOr(stab_or, any);
}

// ---- phase B: pivots, pivot rows, coins (one CTA) --------------------------------------
__global__ void __launch_bounds__(1024)
k_batch_pivots(uint64_t *__restrict__ x, uint64_t *__restrict__ z, uint64_t pitch, uint64_t k,
               uint64_t n, uint64_t ng, uint64_t g0, uint64_t *__restrict__ s,
               const uint32_t *__restrict__ colbits, const uint32_t *__restrict__ fq,
               const uint32_t *__restrict__ fidx, uint32_t b, uint64_t *__restrict__ Vx,
               uint64_t *__restrict__ Vz, uint64_t vstride, uint32_t *__restrict__ vinfo,
               uint32_t *__restrict__ bctl,
               uint64_t seed, uint64_t *__restrict__ coin_index, qsr_record_entry *__restrict__ out,
               int *__restrict__ err, const uint8_t *__restrict__ coin_table) {
    __shared__ uint32_t s_vb[kB], s_vsign[kB], s_c[kB], s_q[kB], s_vbcol[kB], s_beta[kB];
    __shared__ uint32_t s_min, s_len;
    __shared__ int s_red[32];
    __shared__ uint32_t s_bits[kB];
    const uint32_t tid = threadIdx.x, nthr = blockDim.x;
    if (tid < b) s_q[tid] = fq[tid];
    if (tid == 0) s_len = b;
    __syncthreads();
    for (uint32_t m = 0; m < b; ++m) {
        // VB columns over the V's found so far (bit m' of vbcol[j] = X of V_{m'} at q_j).
        if (tid < b) {
            uint32_t col = 0;
            for (uint32_t mp = 0; mp < m; ++mp) col |= ((s_vb[mp] >> tid) & 1u) << mp;
            s_vbcol[tid] = col;
        }
        if (tid == 0) s_min = 0xFFFFFFFFu;
        __syncthreads();
        // Smallest stabilizer whose current X bit at q_m is set (pivots already used in this
        // batch are +/-Z now and never qualify). Scanned 1024 rows at a time from g = 0; in a
        // scrambled state the first chunk almost always holds it.
        uint32_t found = 0xFFFFFFFFu;
        for (uint64_t base = 0; base < n; base += nthr) {
            const uint64_t g = base + tid;
            if (g < n) {
                bool used = false;
                for (uint32_t mp = 0; mp < m; ++mp) used |= s_c[mp] == uint32_t(g);
                if (!used) {
                    const uint32_t cb = colbits[ng + g];
                    const uint32_t M = membership(cb, s_vbcol, 0, m);
                    const uint32_t bit = ((cb >> m) ^ parity32(M & s_vbcol[m])) & 1u;
                    if (bit) atomicMin(&s_min, uint32_t(g));
                }
            }
            __syncthreads();
            found = s_min;
            __syncthreads(); // everyone has read s_min before anyone updates it again
            if (found != 0xFFFFFFFFu) break;
        }
        if (found == 0xFFFFFFFFu) { // deterministic at time m: the batch ends before it
            if (tid == 0) { s_len = m; bctl[BL_DET] = 1; }
            __syncthreads();
            break;
        }
        const uint32_t c = found;
        const uint32_t Mc = membership(colbits[ng + c], s_vbcol, 0, m);
        // V_m = S_c after its memberships; phase by the telescoped formula (file header).
        const uint64_t rs = ng + c;
        int e_part = 0, beta_part = 0;
        u64 acc = 0;
        for (uint64_t i = tid; i < k; i += nthr) {
            u64 cx = x[rs * pitch + i], cz = z[rs * pitch + i];
            e_part += __popcll(cx & cz);
            for (uint32_t U = Mc; U; U &= U - 1) {
                const uint32_t j = __ffs(U) - 1;
                const u64 vx = Vx[uint64_t(j) * vstride + i], vz = Vz[uint64_t(j) * vstride + i];
                acc ^= vz & cx;
                cx ^= vx;
                cz ^= vz;
            }
            const int bend = __popcll(cx & cz);
            e_part -= bend;
            beta_part += bend;
            Vx[uint64_t(m) * vstride + i] = cx;
            Vz[uint64_t(m) * vstride + i] = cz;
        }
        e_part += 2 * (__popcll(acc) & 1);
        const int e_tot = block_sum(e_part, s_red);
        const int b_tot = block_sum(beta_part, s_red);
        if (tid == 0) {
            int E = e_tot;
            uint32_t sign = uint32_t((s[rs >> 6] >> (rs & 63)) & 1u);
            for (uint32_t U = Mc; U; U &= U - 1) {
                const uint32_t j = __ffs(U) - 1;
                E += int(s_beta[j]);
                sign ^= s_vsign[j];
            }
            if (E & 1) atomicExch(err, 1);
            sign ^= (uint32_t(E) >> 1) & 1u;
            s_vsign[m] = sign;
            s_beta[m] = uint32_t(b_tot) & 3u;
            s_c[m] = c;
            const uint64_t idx = *coin_index;
            const uint32_t coin = draw_coin(seed, idx, coin_table);
            *coin_index = idx + 1;
            out[fidx[m]] = qsr_record_entry{s_q[m], uint8_t(coin), 0};
            // signs of the replaced pair: D_c <- s(V_m), S_c <- coin
            const uint64_t rd = c;
            s[rd >> 6] = (s[rd >> 6] & ~(1ull << (rd & 63))) | (uint64_t(sign) << (rd & 63));
            s[rs >> 6] = (s[rs >> 6] & ~(1ull << (rs & 63))) | (uint64_t(coin) << (rs & 63));
        }
        __syncthreads(); // V_m (global) and the shared pivot bookkeeping visible to the block
        if (tid < b) {
            const uint32_t qj = s_q[tid];
            s_bits[tid] = uint32_t((Vx[uint64_t(m) * vstride + (qj >> 6)] >> (qj & 63)) & 1u);
        }
        __syncthreads();
        if (tid == 0) {
            uint32_t vb = 0;
            for (uint32_t j = 0; j < b; ++j) vb |= s_bits[j] << j;
            s_vb[m] = vb;
        }
        // Special rows: D_c <- V_m (bits), S_c <- Z_{q_m}.
        const uint32_t qm = s_q[m];
        for (uint64_t i = tid; i < pitch; i += nthr) {
            const bool valid = i < k;
            x[uint64_t(c) * pitch + i] = valid ? Vx[uint64_t(m) * vstride + i] : 0ull;
            z[uint64_t(c) * pitch + i] = valid ? Vz[uint64_t(m) * vstride + i] : 0ull;
            x[rs * pitch + i] = 0ull;
            z[rs * pitch + i] = i == (qm >> 6) ? (1ull << (qm & 63)) : 0ull;
        }
        __syncthreads();
    }
    __syncthreads();
    if (tid < kB) {
        const bool v = tid < s_len;
        vinfo[VI_VB + tid] = v ? s_vb[tid] : 0u;
        vinfo[VI_SIGN + tid] = v ? s_vsign[tid] : 0u;
        vinfo[VI_C + tid] = v ? uint32_t(g0 + s_c[tid]) : 0xFFFFFFFFu; // global generator
        vinfo[VI_BETA + tid] = v ? s_beta[tid] : 0u;
    }
    if (tid == 0) bctl[BL_LEN] = s_len;
}

// ---- phase C: every other row absorbs its V's in one pass --------------------------
constexpr int kCThreads = 256;
constexpr int kCWarps = kCThreads / 32;
constexpr int kRowsPerWarp = 4;
constexpr int kGroupRows = kCWarps * kRowsPerWarp; // 32 consecutive rows per CTA iteration
constexpr int kSlice = 64;                          // words per staged V slice (2 per lane)
constexpr size_t kSliceWords = size_t(kB) * 2 * kSlice;
constexpr size_t kApplySmem = 2 * kSliceWords * sizeof(u64); // double buffer

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned sa = unsigned(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

// Stage words [w0, w0+kSlice) of V_0..V_{len-1} (x and z) into buf[(j*2+plane)*kSlice + w]
// with cp.async (16 bytes per op; pitch % 16 == 0, so past k it reads the zero padding).
__device__ __forceinline__ void stage_slice(u64 *buf, const uint64_t *Vx, const uint64_t *Vz,
                                            uint64_t pitch, uint64_t vstride, uint64_t w0,
                                            uint32_t len) {
    const uint32_t pairs = len * 2 * (kSlice / 2);
    for (uint32_t e = threadIdx.x; e < pairs; e += kCThreads) {
        const uint32_t w = 2 * (e & (kSlice / 2 - 1)), jp = e / (kSlice / 2);
        const uint32_t j = jp >> 1, plane = jp & 1;
        const uint64_t gw = w0 + w;
        u64 *dst = buf + size_t(jp) * kSlice + w;
        if (gw < pitch) cp_async16(dst, (plane ? Vz : Vx) + uint64_t(j) * vstride + gw);
        else { dst[0] = 0; dst[1] = 0; }
    }
    cp_async_commit();
}

__global__ void __launch_bounds__(kCThreads, 2)
k_batch_apply(uint64_t *__restrict__ x, uint64_t *__restrict__ z, uint64_t pitch, uint64_t k,
              uint64_t nrows, uint64_t ng, uint64_t g0, uint64_t *__restrict__ s,
              const uint32_t *__restrict__ colbits, const uint64_t *__restrict__ Vx,
              const uint64_t *__restrict__ Vz, uint64_t vstride, const uint32_t *__restrict__ vinfo,
              const uint32_t *__restrict__ bctl, int *__restrict__ err) {
    __shared__ uint32_t s_vbcol[kB], s_c[kB], s_vb[kB];
    __shared__ uint32_t s_vs_mask, s_b0_mask, s_b1_mask;
    extern __shared__ __align__(16) u64 sv_raw[];
    const uint32_t len = bctl[BL_LEN];
    if (len == 0) return;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < kB) {
        s_vb[tid] = vinfo[VI_VB + tid];
        // Pivot generator (global) -> local generator index, or none if another shard holds it.
        const uint32_t cg = vinfo[VI_C + tid];
        s_c[tid] = (cg != 0xFFFFFFFFu && cg >= g0 && cg < g0 + ng) ? uint32_t(cg - g0)
                                                                       : 0xFFFFFFFFu;
    }
    if (tid == 0) {
        uint32_t vs = 0, b0 = 0, b1 = 0;
        for (uint32_t j = 0; j < len; ++j) {
            vs |= (vinfo[VI_SIGN + j] & 1u) << j;
            b0 |= (vinfo[VI_BETA + j] & 1u) << j;
            b1 |= ((vinfo[VI_BETA + j] >> 1) & 1u) << j;
        }
        s_vs_mask = vs, s_b0_mask = b0, s_b1_mask = b1;
    }
    __syncthreads();
    if (tid < kB) {
        uint32_t col = 0;
        for (uint32_t mp = 0; mp < len && mp < tid; ++mp) col |= ((s_vb[mp] >> tid) & 1u) << mp;
        s_vbcol[tid] = col;
    }
    __syncthreads();
    const uint64_t groups = nrows / kGroupRows;
    const uint32_t nslices = uint32_t((k + kSlice - 1) / kSlice);
    for (uint64_t grp = blockIdx.x; grp < groups; grp += gridDim.x) {
        const uint64_t r0 = grp * kGroupRows + warp * kRowsPerWarp;
        // Membership per row: pivot stabilizers are final already; replaced destabilizers
        // restart from V_m after collapse m; every other row starts from its column bits.
        uint32_t M[kRowsPerWarp];
#pragma unroll
        for (int q = 0; q < kRowsPerWarp; ++q) {
            const uint64_t r = r0 + q;
            uint32_t cb = colbits[r], start = 0;
            bool skip = false;
            for (uint32_t j = 0; j < len; ++j) {
                if (s_c[j] == 0xFFFFFFFFu) continue;
                if (r == ng + s_c[j]) skip = true;
                if (r == s_c[j]) { cb = s_vb[j]; start = j + 1; }
            }
            M[q] = skip ? 0u : membership(cb, s_vbcol, start, len);
        }
        const uint32_t U = M[0] | M[1] | M[2] | M[3];
        u64 acc[kRowsPerWarp];
        int bd[kRowsPerWarp];
#pragma unroll
        for (int q = 0; q < kRowsPerWarp; ++q) acc[q] = 0, bd[q] = 0;
        stage_slice(sv_raw, Vx, Vz, pitch, vstride, 0, len);
        for (uint32_t sl = 0; sl < nslices; ++sl) {
            cp_async_wait_all();
            __syncthreads(); // slice sl staged; everyone is done with the other buffer
            if (sl + 1 < nslices)
                stage_slice(sv_raw + ((sl + 1) & 1) * kSliceWords, Vx, Vz, pitch, vstride,
                            uint64_t(sl + 1) * kSlice, len);
            if (U == 0) continue;
            const u64 *buf = sv_raw + (sl & 1) * kSliceWords;
            const uint64_t i = uint64_t(sl) * kSlice + 2 * lane;
            const bool act = i < pitch;
            ulonglong2 cx[kRowsPerWarp], cz[kRowsPerWarp];
#pragma unroll
            for (int q = 0; q < kRowsPerWarp; ++q) {
                cx[q] = make_ulonglong2(0ull, 0ull);
                cz[q] = cx[q];
                if (M[q] && act) {
                    cx[q] = __ldcs(reinterpret_cast<const ulonglong2 *>(x + (r0 + q) * pitch + i));
                    cz[q] = __ldcs(reinterpret_cast<const ulonglong2 *>(z + (r0 + q) * pitch + i));
                    bd[q] += __popcll(cx[q].x & cz[q].x) + __popcll(cx[q].y & cz[q].y);
                }
            }
            for (uint32_t W = U; W; W &= W - 1) {
                const uint32_t j = __ffs(W) - 1;
                const ulonglong2 vx = *reinterpret_cast<const ulonglong2 *>(buf + (2 * j) * kSlice + 2 * lane);
                const ulonglong2 vz = *reinterpret_cast<const ulonglong2 *>(buf + (2 * j + 1) * kSlice + 2 * lane);
#pragma unroll
                for (int q = 0; q < kRowsPerWarp; ++q) {
                    if ((M[q] >> j) & 1u) {
                        acc[q] ^= (vz.x & cx[q].x) ^ (vz.y & cx[q].y);
                        cx[q].x ^= vx.x; cx[q].y ^= vx.y;
                        cz[q].x ^= vz.x; cz[q].y ^= vz.y;
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < kRowsPerWarp; ++q) {
                if (M[q] && act) {
                    bd[q] -= __popcll(cx[q].x & cz[q].x) + __popcll(cx[q].y & cz[q].y);
                    __stcs(reinterpret_cast<ulonglong2 *>(x + (r0 + q) * pitch + i), cx[q]);
                    __stcs(reinterpret_cast<ulonglong2 *>(z + (r0 + q) * pitch + i), cz[q]);
                }
            }
        }
        cp_async_wait_all();
        __syncthreads(); // buffers free before the next row group stages into them
        if (U == 0) continue;
        uint64_t flips = 0;
        bool odd = false;
#pragma unroll
        for (int q = 0; q < kRowsPerWarp; ++q) {
            const int tot = warp_sum(bd[q] + 2 * (__popcll(acc[q]) & 1));
            if (M[q]) {
                const int E = tot + __popc(M[q] & s_b0_mask) + 2 * __popc(M[q] & s_b1_mask);
                odd |= (E & 1) != 0;
                const uint32_t f = parity32(M[q] & s_vs_mask) ^ ((uint32_t(E) >> 1) & 1u);
                flips |= uint64_t(f) << ((r0 + q) & 63);
            }
        }
        if (lane == 0) {
            if (odd) atomicExch(err, 1);
            if (flips) atomicXor(reinterpret_cast<unsigned long long *>(s + (r0 >> 6)), flips);
        }
    }
}

} // namespace

void batch_colbits(DeviceTableau &t, const uint32_t *d_fq, uint32_t b) {
    MeasureScratch &ms = t.ms;
    const uint64_t nrows = 2 * t.ng;
    QSR_CUDA(cudaMemsetAsync(ms.bctl, 0, 16, t.stream));
    k_colbits<<<unsigned((nrows + 255) / 256), 256, 0, t.stream>>>(t.x, t.rm_pitch, nrows, t.ng, d_fq,
                                                                    b, ms.colbits, ms.bctl + BL_STAB_OR);
    QSR_CUDA(cudaGetLastError());
    count_launch();
}

void batch_pivots(DeviceTableau &t, const uint32_t *d_fq, const uint32_t *d_fidx, uint32_t b,
                  uint64_t seed) {
    MeasureScratch &ms = t.ms;
    k_batch_pivots<<<1, 1024, 0, t.stream>>>(t.x, t.z, t.rm_pitch, t.k, t.n_gen, t.ng, t.g0, t.s,
                                             ms.colbits, d_fq, d_fidx, b, ms.Vx, ms.Vz,
                                             ms.vstride, ms.vinfo, ms.bctl, seed, ms.coin_index,
                                             ms.out, ms.err, ms.coin_table);
    QSR_CUDA(cudaGetLastError());
    count_launch();
}

void batch_apply(DeviceTableau &t) {
    MeasureScratch &ms = t.ms;
    static bool configured = false;
    if (!configured) {
        QSR_CUDA(cudaFuncSetAttribute(k_batch_apply, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(kApplySmem)));
        configured = true;
    }
    k_batch_apply<<<unsigned(t.num_sms * 2), kCThreads, kApplySmem, t.stream>>>(
        t.x, t.z, t.rm_pitch, t.k, 2 * t.ng, t.ng, t.g0, t.s, ms.colbits, ms.Vx, ms.Vz, ms.vstride,
        ms.vinfo, ms.bctl, ms.err);
    QSR_CUDA(cudaGetLastError());
    count_launch();
}

void measure_batch(DeviceTableau &t, const uint32_t *d_fq, const uint32_t *d_fidx, uint32_t b,
                   uint64_t seed, uint32_t &done, bool &det) {
    batch_colbits(t, d_fq, b);
    batch_pivots(t, d_fq, d_fidx, b, seed);
    batch_apply(t);
    uint32_t h[2];
    QSR_CUDA(cudaMemcpyAsync(h, t.ms.bctl, 8, cudaMemcpyDeviceToHost, t.stream));
    QSR_CUDA(cudaStreamSynchronize(t.stream));
    done = h[BL_LEN];
    det = h[BL_DET] != 0;
}

} // namespace qsr
