// Batched projective measurement: B consecutive probabilistic collapses of a measurement
// window applied in ONE streaming pass over the RM tableau (bit-identical to applying them one
// by one with the fused recipe of k_measure.cu, which is itself bit-identical to the
// reference's parallel_ge + swap_anti_commuting + inject_x, measure.hpp:409-431).
//
// Why it is exact. Collapse m multiplies every row of R_m = {rows != S_c, D_c with X[q_m]} by
// V_m = S_{c_m} as it stands at time m, then D_{c_m} <- V_m, S_{c_m} <- +/-Z_{q_m}. A row's
// membership in R_m depends only on its X bit at q_m at time m, which is its bit at batch
// start XORed with the X bits at q_m of the V's it absorbed earlier. So with
//   colbits_r[m] = X_r[q_m] at batch start            (phase A, a column gather)
//   vb[m'][m]    = X bit of V_{m'} at q_m              (phase B)
// the membership vector of every row follows from the recurrence
//   member_r[m] = colbits_r[m] ^ parity(member_r[<m] & VBcol[m]),
// and the row's final value and sign are r ^ sum V_m, s_r ^ sum (s(V_m) ^ flip_m), with the
// mod-4 phase of each product taken against the row as it stands just before it (phase C).
// Only the pivot rows need sequential treatment (phase B, one CTA): c_m is the smallest
// stabilizer whose current X bit at q_m is set, V_m is S_{c_m} after its own earlier
// memberships, and the coin is Philox(seed, 0, 0, coin_index++) & 1.
//
// Traffic: one read + write of the touched rows per batch instead of per collapse
// (B x fewer HBM bytes); the pivot rows V_m are staged through shared memory in 64-word
// slices.
#include "common.cuh"
#include "device.hpp"

namespace qsr {

namespace {

constexpr int kB = kMaxBatch;       // collapses per batch (<= 32: u32 membership masks)
enum : uint32_t { BL_LEN = 0, BL_DET = 1 };

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

// ---- phase A: column bits of all rows at the batch's measured qubits ----------------
__global__ void k_colbits(const uint64_t *__restrict__ x, uint64_t pitch, uint64_t nrows,
                          const uint32_t *__restrict__ fq, uint32_t b, uint32_t *__restrict__ colbits) {
    __shared__ uint32_t sq[kB];
    if (threadIdx.x < b) sq[threadIdx.x] = fq[threadIdx.x];
    __syncthreads();
    const uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= nrows) return;
    const uint64_t *row = x + r * pitch;
    uint32_t bits = 0;
    for (uint32_t m = 0; m < b; ++m) {
        const uint32_t q = sq[m];
        bits |= uint32_t((__ldcg(row + (q >> 6)) >> (q & 63)) & 1u) << m;
    }
    colbits[r] = bits;
}

// ---- phase B: pivots, pivot rows, coins (one CTA) --------------------------------------
// vinfo layout: [0,kB) vb (X bits of V_m at q_0..q_{b-1}), [kB,2kB) sign of V_m,
//               [2kB,3kB) c_m (stabilizer index).
__global__ void __launch_bounds__(1024)
k_batch_pivots(uint64_t *__restrict__ x, uint64_t *__restrict__ z, uint64_t pitch, uint64_t k,
               uint64_t n, uint64_t n_pad, uint64_t *__restrict__ s,
               const uint32_t *__restrict__ colbits, const uint32_t *__restrict__ fq,
               const uint32_t *__restrict__ fidx, uint32_t b, uint64_t *__restrict__ Vx,
               uint64_t *__restrict__ Vz, uint32_t *__restrict__ vinfo, uint32_t *__restrict__ bctl,
               uint64_t seed, uint64_t *__restrict__ coin_index, qsr_record_entry *__restrict__ out,
               int *__restrict__ err) {
    __shared__ uint32_t s_vb[kB], s_vsign[kB], s_c[kB], s_q[kB], s_vbcol[kB];
    __shared__ uint32_t s_min;
    __shared__ int s_red[32][kB];
    __shared__ uint32_t s_len;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nthr = blockDim.x;
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
                    const uint32_t cb = colbits[n_pad + g];
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
        const uint32_t Mc = membership(colbits[n_pad + c], s_vbcol, 0, m);
        // V_m = S_c after its memberships (ordered products with mod-4 phase per product).
        int ph[kB];
#pragma unroll
        for (int j = 0; j < kB; ++j) ph[j] = 0;
        const uint64_t rs = n_pad + c;
        for (uint64_t i = tid; i < k; i += nthr) {
            uint64_t cx = x[rs * pitch + i], cz = z[rs * pitch + i];
#pragma unroll
            for (int j = 0; j < kB; ++j) {
                if ((Mc >> j) & 1u) {
                    const uint64_t vx = Vx[uint64_t(j) * pitch + i], vz = Vz[uint64_t(j) * pitch + i];
                    ph[j] += phase_delta(vx, vz, cx, cz);
                    cx ^= vx;
                    cz ^= vz;
                }
            }
            Vx[uint64_t(m) * pitch + i] = cx;
            Vz[uint64_t(m) * pitch + i] = cz;
        }
#pragma unroll
        for (int j = 0; j < kB; ++j) {
            int v = warp_sum(ph[j]);
            if (lane == 0) s_red[warp][j] = v;
        }
        __syncthreads();
        if (tid == 0) {
            uint32_t sign = uint32_t((s[rs >> 6] >> (rs & 63)) & 1u);
            for (uint32_t j = 0; j < m; ++j) {
                if (!((Mc >> j) & 1u)) continue;
                int tot = 0;
                for (uint32_t w = 0; w < (nthr + 31) / 32; ++w) tot += s_red[w][j];
                if (tot & 1) atomicExch(err, 1);
                sign ^= s_vsign[j] ^ ((uint32_t(tot) >> 1) & 1u);
            }
            s_vsign[m] = sign;
            s_c[m] = c;
            const uint64_t idx = *coin_index;
            const uint32_t coin = uint32_t(d_philox_word(seed, 0, 0, idx) & 1u);
            *coin_index = idx + 1;
            out[fidx[m]] = qsr_record_entry{s_q[m], uint8_t(coin), 0};
            // signs of the replaced pair: D_c <- s(V_m), S_c <- coin
            const uint64_t rd = c;
            s[rd >> 6] = (s[rd >> 6] & ~(1ull << (rd & 63))) | (uint64_t(sign) << (rd & 63));
            s[rs >> 6] = (s[rs >> 6] & ~(1ull << (rs & 63))) | (uint64_t(coin) << (rs & 63));
        }
        __syncthreads(); // V_m visible to the block
        if (tid < b) {
            const uint32_t qj = s_q[tid];
            s_red[0][tid] = uint32_t((Vx[uint64_t(m) * pitch + (qj >> 6)] >> (qj & 63)) & 1u);
        }
        __syncthreads();
        if (tid == 0) {
            uint32_t vb = 0;
            for (uint32_t j = 0; j < b; ++j) vb |= uint32_t(s_red[0][j]) << j;
            s_vb[m] = vb;
        }
        // Special rows: D_c <- V_m (bits), S_c <- Z_{q_m}.
        const uint32_t qm = s_q[m];
        for (uint64_t i = tid; i < pitch; i += nthr) {
            const bool valid = i < k;
            x[uint64_t(c) * pitch + i] = valid ? Vx[uint64_t(m) * pitch + i] : 0ull;
            z[uint64_t(c) * pitch + i] = valid ? Vz[uint64_t(m) * pitch + i] : 0ull;
            x[rs * pitch + i] = 0ull;
            z[rs * pitch + i] = i == (qm >> 6) ? (1ull << (qm & 63)) : 0ull;
        }
        __syncthreads();
    }
    __syncthreads();
    if (tid < kB) {
        vinfo[tid] = tid < s_len ? s_vb[tid] : 0u;
        vinfo[kB + tid] = tid < s_len ? s_vsign[tid] : 0u;
        vinfo[2 * kB + tid] = tid < s_len ? s_c[tid] : 0xFFFFFFFFu;
    }
    if (tid == 0) bctl[BL_LEN] = s_len;
}

// ---- phase C: every other row absorbs its V's in one pass --------------------------
// One warp per row; the CTA's rows share each 128-word slice of the V's staged in shared
// memory. Per absorbed V the mod-4 product phase is kept in a bit-sliced 2-bit counter per bit
// position (c1 = ones, c2 = twos), flushed with two popcounts per slice:
//   x1z2 = vx & cz ; anti = (cx & vz) ^ x1z2 ; (cx, cz) ^= (vx, vz)
//   c2 ^= (c1 ^ cx ^ cz ^ x1z2) & anti ; c1 ^= anti
// which adds +1 (mod 4) for each bit where V*cur picks up +i and -1 where it picks up -i —
// the same count as product_phase_counts (tableau.hpp:336-342), in ~8 logic ops per word.
constexpr int kCThreads = 512;
constexpr int kCWarps = kCThreads / 32;
constexpr int kSlice = 128; // words per staged V slice (4 per lane)

using u64 = unsigned long long;
__device__ __forceinline__ void absorb(u64 vx, u64 vz, u64 &cx, u64 &cz, u64 &c1, u64 &c2) {
    const u64 x1z2 = vx & cz;
    const u64 anti = (cx & vz) ^ x1z2;
    cx ^= vx;
    cz ^= vz;
    c2 ^= (c1 ^ cx ^ cz ^ x1z2) & anti;
    c1 ^= anti;
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned sa = unsigned(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

// Stage words [w0, w0+kSlice) of V_0..V_{len-1} (x and z) into buf[j][plane][word]
// asynchronously (cp.async, 16 bytes per op; pitch % 16 == 0 so slices past k read zeros).
__device__ __forceinline__ void stage_slice(u64 (*buf)[2][kSlice], const uint64_t *Vx,
                                            const uint64_t *Vz, uint64_t pitch, uint64_t w0,
                                            uint32_t len, uint32_t tid) {
    const uint32_t pairs = len * 2 * (kSlice / 2);
    for (uint32_t e = tid; e < pairs; e += kCThreads) {
        const uint32_t w = 2 * (e & (kSlice / 2 - 1)), jp = e / (kSlice / 2);
        const uint32_t j = jp >> 1, plane = jp & 1;
        const uint64_t gw = w0 + w;
        u64 *dst = &buf[j][plane][w];
        if (gw < pitch) cp_async16(dst, (plane ? Vz : Vx) + uint64_t(j) * pitch + gw);
        else { dst[0] = 0; dst[1] = 0; }
    }
    cp_async_commit();
}

__global__ void __launch_bounds__(kCThreads, 2)
k_batch_apply(uint64_t *__restrict__ x, uint64_t *__restrict__ z, uint64_t pitch, uint64_t k,
              uint64_t nrows, uint64_t n_pad, uint64_t *__restrict__ s,
              const uint32_t *__restrict__ colbits, const uint64_t *__restrict__ Vx,
              const uint64_t *__restrict__ Vz, const uint32_t *__restrict__ vinfo,
              const uint32_t *__restrict__ bctl, int *__restrict__ err) {
    __shared__ uint32_t s_vbcol[kB], s_vsign[kB], s_c[kB], s_vb[kB];
    extern __shared__ __align__(16) u64 sv_raw[]; // [2 buffers][kB][2 planes][kSlice]
    u64 (*sv[2])[2][kSlice] = {reinterpret_cast<u64 (*)[2][kSlice]>(sv_raw),
                               reinterpret_cast<u64 (*)[2][kSlice]>(sv_raw + kB * 2 * kSlice)};
    const uint32_t len = bctl[BL_LEN];
    if (len == 0) return;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < kB) {
        s_vb[tid] = vinfo[tid];
        s_vsign[tid] = vinfo[kB + tid];
        s_c[tid] = vinfo[2 * kB + tid];
    }
    __syncthreads();
    if (tid < kB) {
        uint32_t col = 0;
        for (uint32_t mp = 0; mp < len; ++mp)
            if (mp < tid) col |= ((s_vb[mp] >> tid) & 1u) << mp;
        s_vbcol[tid] = col;
    }
    __syncthreads();
    const uint64_t groups = nrows / kCWarps;
    const uint32_t nslices = uint32_t((k + kSlice - 1) / kSlice);
    for (uint64_t grp = blockIdx.x; grp < groups; grp += gridDim.x) {
        const uint64_t r = grp * kCWarps + warp;
        // Membership: pivot stabilizers are final already; replaced destabilizers restart
        // from V_m at collapse m+1; every other row starts from its batch-start column bits.
        uint32_t M;
        {
            uint32_t cb = colbits[r], start = 0;
            bool skip = false;
            for (uint32_t j = 0; j < len; ++j) {
                if (r == n_pad + s_c[j]) skip = true;
                if (r == s_c[j]) { cb = s_vb[j]; start = j + 1; }
            }
            M = skip ? 0u : membership(cb, s_vbcol, start, len);
        }
        int ph[kB];
#pragma unroll
        for (int j = 0; j < kB; ++j) ph[j] = 0;
        uint64_t *xr = x + r * pitch, *zr = z + r * pitch;
        stage_slice(sv[0], Vx, Vz, pitch, 0, len, tid);
        for (uint32_t sl = 0; sl < nslices; ++sl) {
            cp_async_wait_all();
            __syncthreads(); // slice sl staged; everyone is done with slice sl-1's buffer
            if (sl + 1 < nslices)
                stage_slice(sv[(sl + 1) & 1], Vx, Vz, pitch, uint64_t(sl + 1) * kSlice, len, tid);
            if (M == 0) continue;
            u64 (*buf)[2][kSlice] = sv[sl & 1];
            // lane words: [w0 + 2*lane, +1] and [w0 + 64 + 2*lane, +1] (two 512-byte warp runs)
            const uint64_t w0 = uint64_t(sl) * kSlice;
            const uint64_t i0 = w0 + 2 * lane, i1 = i0 + 64;
            const bool a0 = i0 < pitch, a1 = i1 < pitch;
            ulonglong2 xa = make_ulonglong2(0ull, 0ull), za = xa, xb = xa, zb = xa;
            if (a0) {
                xa = __ldcs(reinterpret_cast<const ulonglong2 *>(xr + i0));
                za = __ldcs(reinterpret_cast<const ulonglong2 *>(zr + i0));
            }
            if (a1) {
                xb = __ldcs(reinterpret_cast<const ulonglong2 *>(xr + i1));
                zb = __ldcs(reinterpret_cast<const ulonglong2 *>(zr + i1));
            }
#pragma unroll
            for (int j = 0; j < kB; ++j) {
                if ((M >> j) & 1u) {
                    const ulonglong2 vxa = *reinterpret_cast<const ulonglong2 *>(&buf[j][0][2 * lane]);
                    const ulonglong2 vza = *reinterpret_cast<const ulonglong2 *>(&buf[j][1][2 * lane]);
                    const ulonglong2 vxb = *reinterpret_cast<const ulonglong2 *>(&buf[j][0][64 + 2 * lane]);
                    const ulonglong2 vzb = *reinterpret_cast<const ulonglong2 *>(&buf[j][1][64 + 2 * lane]);
                    u64 c1 = 0, c2 = 0;
                    absorb(vxa.x, vza.x, xa.x, za.x, c1, c2);
                    absorb(vxa.y, vza.y, xa.y, za.y, c1, c2);
                    absorb(vxb.x, vzb.x, xb.x, zb.x, c1, c2);
                    absorb(vxb.y, vzb.y, xb.y, zb.y, c1, c2);
                    ph[j] += __popcll(c1) + 2 * __popcll(c2);
                }
            }
            if (a0) {
                __stcs(reinterpret_cast<ulonglong2 *>(xr + i0), xa);
                __stcs(reinterpret_cast<ulonglong2 *>(zr + i0), za);
            }
            if (a1) {
                __stcs(reinterpret_cast<ulonglong2 *>(xr + i1), xb);
                __stcs(reinterpret_cast<ulonglong2 *>(zr + i1), zb);
            }
        }
        cp_async_wait_all();
        __syncthreads(); // buffers free before the next row group stages into them
        if (M == 0) continue;
        uint32_t dsign = 0;
#pragma unroll
        for (int j = 0; j < kB; ++j) {
            if ((M >> j) & 1u) {
                const int tot = warp_sum(ph[j]);
                if (tot & 1) dsign |= 0x80000000u; // odd phase: corrupted tableau
                dsign ^= s_vsign[j] ^ ((uint32_t(tot) >> 1) & 1u);
            }
        }
        if (lane == 0) {
            if (dsign & 0x80000000u) atomicExch(err, 1);
            if (dsign & 1u)
                atomicXor(reinterpret_cast<unsigned long long *>(s + (r >> 6)), 1ull << (r & 63));
        }
    }
}

constexpr size_t kApplySmem = size_t(2) * kB * 2 * kSlice * sizeof(u64);

} // namespace

void measure_batch(DeviceTableau &t, const uint32_t *d_fq, const uint32_t *d_fidx, uint32_t b,
                   uint64_t seed, uint32_t &done, bool &det) {
    MeasureScratch &ms = t.ms;
    const uint64_t nrows = 2 * t.n_pad;
    QSR_CUDA(cudaMemsetAsync(ms.bctl, 0, 16, t.stream));
    k_colbits<<<unsigned((nrows + 255) / 256), 256, 0, t.stream>>>(t.x, t.rm_pitch, nrows, d_fq, b,
                                                                    ms.colbits);
    QSR_CUDA(cudaGetLastError());
    k_batch_pivots<<<1, 1024, 0, t.stream>>>(t.x, t.z, t.rm_pitch, t.k, t.n, t.n_pad, t.s, ms.colbits,
                                             d_fq, d_fidx, b, ms.Vx, ms.Vz, ms.vinfo, ms.bctl, seed,
                                             ms.coin_index, ms.out, ms.err);
    QSR_CUDA(cudaGetLastError());
    static bool configured = false;
    if (!configured) {
        QSR_CUDA(cudaFuncSetAttribute(k_batch_apply, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(kApplySmem)));
        configured = true;
    }
    k_batch_apply<<<unsigned(t.num_sms * 2), kCThreads, kApplySmem, t.stream>>>(
        t.x, t.z, t.rm_pitch, t.k, nrows, t.n_pad, t.s, ms.colbits, ms.Vx, ms.Vz, ms.vinfo, ms.bctl,
        ms.err);
    QSR_CUDA(cudaGetLastError());
    count_launch(3);
    uint32_t h[2];
    QSR_CUDA(cudaMemcpyAsync(h, ms.bctl, 8, cudaMemcpyDeviceToHost, t.stream));
    QSR_CUDA(cudaStreamSynchronize(t.stream));
    done = h[BL_LEN];
    det = h[BL_DET] != 0;
}

} // namespace qsr
