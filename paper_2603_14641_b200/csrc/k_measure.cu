// K4-K12 — projective Z measurement on the generator-major RM tableau
// (reference measure.hpp:104-442).
//
// Per probabilistic collapse the reference runs find_and_compact_pivots, the three-pass
// parallel_ge, swap_anti_commuting, one coin and inject_x. Inside measure_window the
// control-destabilizer half of parallel_ge is a dead store (swap_anti_commuting overwrites
// D_p with S_p, bits and sign), and the two remaining row sets are disjoint and both
// multiply by the unchanged S_c, so one collapse is exactly:
//   (1) R = {stabilizer t != c : X_t[q]} u {destabilizer g != c : X_g[q]}   (pre-update)
//   (2) every r in R: r ^= S_c, s_r ^= s_c ^ flip(sum phase(S_c, r))
//   (3) D_c <- S_c (bits + sign), S_c <- +Z_q
//   (4) coin = Philox(seed, 0, 0, coin_index++) & 1 ; s(S_c) = coin ; outcome = coin
// Kernels:  k_column_mask  (warp-ballot pivot detection over one qubit column)
//           k_compact      (control c = min pivot, dense ascending row list)
//           k_rowmul       (fused row products with popcount mod-4 phase, step 2)
//           k_det_partial / k_finish (ordered deterministic product, or steps 3-4)
// Every kernel reads its control block from device memory, so a whole measurement window is
// enqueued without a host round trip per collapse.
#include <atomic>

#include "common.cuh"
#include "device.hpp"

namespace qsr {

namespace {

enum : uint32_t { MODE_COLLAPSE = 0, MODE_DET = 1, MODE_SWAP = 2, MODE_NONE = 3 };
// ctl block layout
enum : uint32_t { CTL_COUNT = 0, CTL_C = 1, CTL_MODE = 2, CTL_Q = 3, CTL_OUT = 4, CTL_WORDS = 8 };
constexpr int kDetChunks = 128;

// ---- K4/K5: one qubit column of all 2*ng generator rows -> bit mask (2kg words) ----
__global__ void k_column_mask(const uint64_t *__restrict__ x, uint64_t rm_pitch, uint64_t nrows,
                              uint32_t iq, uint32_t bq, uint32_t *__restrict__ mask32) {
    uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    bool bit = false;
    if (r < nrows)
        bit = (__ldcg(x + r * rm_pitch + iq) >> bq) & 1;
    uint32_t b = __ballot_sync(0xffffffffu, bit);
    if ((threadIdx.x & 31) == 0 && r < nrows)
        mask32[r >> 5] = b;
}

// ---- compaction: single CTA; ctl[CTL_MODE] in: requested mode, out: effective mode ----
// MODE_COLLAPSE request: c = min stabilizer pivot; if none -> MODE_DET.
// MODE_DET: list = destabilizers with X at q (ascending).
// MODE_SWAP: c = ctl[CTL_C] given; list = destabilizers != c with X at q.
__global__ void __launch_bounds__(1024)
k_compact(uint64_t *__restrict__ mask, uint64_t k, uint64_t ng, uint32_t *__restrict__ ctl,
          uint32_t *__restrict__ rows, const uint8_t *__restrict__ active) {
    __shared__ uint32_t s_min;
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_mode;
    const uint32_t tid = threadIdx.x, nthr = blockDim.x;
    if (active && !*active) {
        if (tid == 0) ctl[CTL_MODE] = MODE_NONE, ctl[CTL_COUNT] = 0;
        return;
    }
    uint32_t mode = ctl[CTL_MODE];
    if (tid == 0) s_min = 0xFFFFFFFFu;
    __syncthreads();
    if (mode == MODE_COLLAPSE) {
        for (uint64_t w = tid; w < k; w += nthr) {
            uint64_t v = mask[k + w];
            if (v) atomicMin(&s_min, uint32_t(w * 64 + __ffsll(v) - 1));
        }
        __syncthreads();
        if (s_min == 0xFFFFFFFFu) mode = MODE_DET;
    }
    uint32_t c = mode == MODE_COLLAPSE ? s_min : (mode == MODE_SWAP ? ctl[CTL_C] : 0xFFFFFFFFu);
    // Effective word range of the list and exclusions.
    uint64_t nw = mode == MODE_DET ? k : (mode == MODE_SWAP ? k : 2 * k);
    __syncthreads();
    if (tid == 0) {
        if (mode == MODE_COLLAPSE) {
            mask[c / 64] &= ~(1ull << (c % 64));
            mask[k + c / 64] &= ~(1ull << (c % 64));
        } else if (mode == MODE_SWAP) {
            mask[c / 64] &= ~(1ull << (c % 64));
        }
        s_mode = mode;
    }
    __syncthreads();
    // Contiguous word range per thread, block-wide exclusive scan of popcounts.
    uint64_t per = (nw + nthr - 1) / nthr;
    uint64_t w0 = tid * per, w1 = w0 + per < nw ? w0 + per : nw;
    uint32_t cnt = 0;
    for (uint64_t w = w0; w < w1; ++w) cnt += __popcll(mask[w]);
    // warp scan
    uint32_t lane = tid & 31, warp = tid >> 5;
    uint32_t incl = cnt;
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= uint32_t(o)) incl += v;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint32_t v = lane < (nthr + 31) / 32 ? s_warp[lane] : 0;
        uint32_t inc = v;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= uint32_t(o)) inc += u;
        }
        s_warp[lane] = inc - v; // exclusive warp offsets
        if (lane == 31) ctl[CTL_COUNT] = inc;
    }
    __syncthreads();
    uint32_t pos = s_warp[warp] + incl - cnt;
    for (uint64_t w = w0; w < w1; ++w) {
        uint64_t v = mask[w];
        // Row id: word w < k -> destabilizer rows w*64+b; w >= k -> stabilizer rows
        // ng + (w-k)*64 + b, which equals w*64 + b because ng = 64k (k = generator-words here).
        while (v) {
            uint32_t b = __ffsll(v) - 1;
            v &= v - 1;
            rows[pos++] = uint32_t(w * 64 + b);
        }
    }
    if (tid == 0) {
        ctl[CTL_MODE] = s_mode;
        ctl[CTL_C] = c;
    }
}

// ---- K8+K10 fused: every listed row r ^= control row, with mod-4 phase sign update ----
// ctl_row = control generator row index (RM row); the control row is staged in shared
// memory once per CTA. Only runs when ctl[CTL_MODE] == want_mode (or want_mode == any).
__global__ void __launch_bounds__(512)
k_rowmul(uint64_t *__restrict__ x, uint64_t *__restrict__ z, uint64_t rm_pitch, uint64_t k,
         uint64_t ng, uint64_t *__restrict__ s, const uint32_t *__restrict__ ctl,
         const uint32_t *__restrict__ rows, uint32_t want_mask, int ctl_is_stab,
         int *__restrict__ err) {
    extern __shared__ uint64_t sc[]; // [2][rm_pitch]
    const uint32_t mode = ctl[CTL_MODE];
    if (!((want_mask >> mode) & 1)) return;
    const uint32_t count = ctl[CTL_COUNT];
    if (count == 0) return;
    const uint64_t crow = (ctl_is_stab ? ng : 0) + ctl[CTL_C];
    // Whole pitch (padding words are zero) so the last word pair of an odd k is defined.
    for (uint64_t i = threadIdx.x; i < rm_pitch; i += blockDim.x) {
        sc[i] = x[crow * rm_pitch + i];
        sc[rm_pitch + i] = z[crow * rm_pitch + i];
    }
    __syncthreads();
    const uint64_t sbit = (s[crow >> 6] >> (crow & 63)) & 1;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t e = gw; e < count; e += nwarps) {
        const uint64_t r = rows[e];
        uint64_t *xr = x + r * rm_pitch;
        uint64_t *zr = z + r * rm_pitch;
        int ph = 0;
        for (uint64_t i = lane * 2; i < k; i += 64) {
            // rm_pitch % 16 == 0 and padding words are zero, so a pair never crosses a row.
            ulonglong2 xv = __ldcs(reinterpret_cast<const ulonglong2 *>(xr + i));
            ulonglong2 zv = __ldcs(reinterpret_cast<const ulonglong2 *>(zr + i));
            uint64_t xc0 = sc[i], xc1 = sc[i + 1], zc0 = sc[rm_pitch + i], zc1 = sc[rm_pitch + i + 1];
            ph += phase_delta(xc0, zc0, xv.x, zv.x) + phase_delta(xc1, zc1, xv.y, zv.y);
            __stcs(reinterpret_cast<ulonglong2 *>(xr + i), make_ulonglong2(xv.x ^ xc0, xv.y ^ xc1));
            __stcs(reinterpret_cast<ulonglong2 *>(zr + i), make_ulonglong2(zv.x ^ zc0, zv.y ^ zc1));
        }
        ph = warp_sum(ph);
        if (lane == 0) {
            if (ph & 1) atomicExch(err, 1);
            uint64_t flip = (uint64_t(ph) >> 1) & 1;
            if (sbit ^ flip)
                atomicXor(reinterpret_cast<unsigned long long *>(s + (r >> 6)), 1ull << (r & 63));
        }
    }
}

// ---- K12 partials: ordered product of the listed stabilizers (deterministic outcome) ---
// grid = (word tiles of 64 words, kDetChunks); warp (tile, chunk) walks its chunk of the
// row list in order for its 64 words and leaves the partial product + phase.
__global__ void __launch_bounds__(32)
k_det_partial(const uint64_t *__restrict__ x, const uint64_t *__restrict__ z, uint64_t rm_pitch,
              uint64_t k, uint64_t ng, const uint64_t *__restrict__ s,
              const uint32_t *__restrict__ ctl, const uint32_t *__restrict__ rows,
              uint64_t *__restrict__ px, uint64_t *__restrict__ pz, int64_t *__restrict__ pe) {
    if (ctl[CTL_MODE] != MODE_DET) return;
    const uint32_t count = ctl[CTL_COUNT];
    const uint32_t chunk = blockIdx.y, lane = threadIdx.x;
    const uint64_t e0 = uint64_t(count) * chunk / kDetChunks;
    const uint64_t e1 = uint64_t(count) * (chunk + 1) / kDetChunks;
    const uint64_t i = uint64_t(blockIdx.x) * 64 + lane * 2;
    const bool act = i < k;
    uint64_t ax0 = 0, ax1 = 0, az0 = 0, az1 = 0;
    int ph = 0, sg = 0;
    for (uint64_t e = e0; e < e1; ++e) {
        const uint64_t g = rows[e];          // destabilizer index -> stabilizer row
        const uint64_t r = ng + g;
        if (blockIdx.x == 0 && lane == 0) sg += (s[r >> 6] >> (r & 63)) & 1;
        if (act) {
            ulonglong2 xv = __ldcg(reinterpret_cast<const ulonglong2 *>(x + r * rm_pitch + i));
            ulonglong2 zv = __ldcg(reinterpret_cast<const ulonglong2 *>(z + r * rm_pitch + i));
            ph += phase_delta(ax0, az0, xv.x, zv.x) + phase_delta(ax1, az1, xv.y, zv.y);
            ax0 ^= xv.x; ax1 ^= xv.y; az0 ^= zv.x; az1 ^= zv.y;
        }
    }
    if (act) {
        uint64_t *ox = px + uint64_t(chunk) * rm_pitch + i;
        uint64_t *oz = pz + uint64_t(chunk) * rm_pitch + i;
        ox[0] = ax0; ox[1] = ax1; oz[0] = az0; oz[1] = az1;
    }
    ph = warp_sum(ph);
    if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long *>(pe + chunk),
                             (unsigned long long)(int64_t(ph) + 2 * int64_t(sg)));
}

// ---- finish: deterministic combine, or pivot replacement + coin --------------------
__global__ void __launch_bounds__(1024)
k_finish(uint64_t *__restrict__ x, uint64_t *__restrict__ z, uint64_t rm_pitch, uint64_t k,
         uint64_t ng, uint64_t *__restrict__ s, uint32_t *__restrict__ ctl,
         const uint64_t *__restrict__ px, const uint64_t *__restrict__ pz,
         int64_t *__restrict__ pe, uint64_t seed, uint64_t *__restrict__ coin_index,
         qsr_record_entry *__restrict__ out, int *__restrict__ err,
         const uint8_t *__restrict__ coin_table) {
    const uint32_t mode = ctl[CTL_MODE];
    const uint32_t q = ctl[CTL_Q];
    const uint32_t tid = threadIdx.x;
    if (mode == MODE_NONE) return;
    if (mode == MODE_DET) {
        __shared__ int s_ph;
        if (tid == 0) s_ph = 0;
        __syncthreads();
        int ph = 0;
        for (uint64_t i = tid; i < k; i += blockDim.x) {
            uint64_t ax = 0, az = 0;
            for (int c = 0; c < kDetChunks; ++c) {
                uint64_t bx = px[uint64_t(c) * rm_pitch + i], bz = pz[uint64_t(c) * rm_pitch + i];
                ph += phase_delta(ax, az, bx, bz);
                ax ^= bx;
                az ^= bz;
            }
        }
        ph = warp_sum(ph);
        if ((tid & 31) == 0) atomicAdd(&s_ph, ph);
        __syncthreads();
        if (tid == 0) {
            int64_t e = s_ph;
            for (int c = 0; c < kDetChunks; ++c) {
                e += pe[c];
                pe[c] = 0; // re-arm
            }
            if (e & 1) atomicExch(err, 1);
            uint32_t outcome = uint32_t((e >> 1) & 1);
            ctl[CTL_OUT] = outcome;
            if (out) *out = qsr_record_entry{q, uint8_t(outcome), 1};
        }
        return;
    }
    // MODE_COLLAPSE / MODE_SWAP: D_c <- S_c (bits + sign), S_c <- +Z_q.
    const uint64_t c = ctl[CTL_C];
    const uint64_t rs = ng + c, rd = c;
    const uint64_t iq = q >> 6, bq = q & 63;
    for (uint64_t i = tid; i < k; i += blockDim.x) {
        uint64_t xs = x[rs * rm_pitch + i], zs = z[rs * rm_pitch + i];
        x[rd * rm_pitch + i] = xs;
        z[rd * rm_pitch + i] = zs;
        x[rs * rm_pitch + i] = 0;
        z[rs * rm_pitch + i] = i == iq ? (1ull << bq) : 0ull;
    }
    if (tid == 0) {
        uint64_t sp = (s[rs >> 6] >> (rs & 63)) & 1;
        s[rd >> 6] = (s[rd >> 6] & ~(1ull << (rd & 63))) | (sp << (rd & 63));
        uint64_t coin = 0;
        if (mode == MODE_COLLAPSE) {
            uint64_t idx = *coin_index;
            coin = draw_coin(seed, idx, coin_table);
            *coin_index = idx + 1;
        }
        s[rs >> 6] = (s[rs >> 6] & ~(1ull << (rs & 63))) | (coin << (rs & 63));
        ctl[CTL_OUT] = uint32_t(coin);
        if (out && mode == MODE_COLLAPSE) *out = qsr_record_entry{q, uint8_t(coin), 0};
    }
}

// ---- ordered fold of partial products (deterministic outcome, sharded form) ----------
// Parts c = 0..nparts-1 each hold a product row (x at px + c*stride, z at pz + c*stride) and an
// exponent pe[c*pe_stride] (mod-4 phase incl. 2*signs). Folding them in order keeps the
// product rows and the exponent mod 4 (measure.hpp:343-376 is associative).
// final == 0: write the folded row + exponent to (ox, oz, oe). final == 1: the outcome.
__global__ void __launch_bounds__(1024)
k_det_reduce(const uint64_t *__restrict__ px, const uint64_t *__restrict__ pz,
             int64_t *__restrict__ pe, uint64_t stride, uint64_t pe_stride, uint32_t nparts,
             uint64_t k, int reset_pe, int final, uint64_t *__restrict__ ox,
             uint64_t *__restrict__ oz, int64_t *__restrict__ oe, uint32_t *__restrict__ ctl,
             uint32_t q, qsr_record_entry *__restrict__ out, int *__restrict__ err) {
    __shared__ int s_ph;
    const uint32_t tid = threadIdx.x;
    if (ctl[CTL_MODE] != MODE_DET) return;
    if (tid == 0) s_ph = 0;
    __syncthreads();
    int ph = 0;
    for (uint64_t i = tid; i < k; i += blockDim.x) {
        uint64_t ax = 0, az = 0;
        for (uint32_t c = 0; c < nparts; ++c) {
            const uint64_t bx = px[uint64_t(c) * stride + i], bz = pz[uint64_t(c) * stride + i];
            ph += phase_delta(ax, az, bx, bz);
            ax ^= bx;
            az ^= bz;
        }
        if (!final) { ox[i] = ax; oz[i] = az; }
    }
    ph = warp_sum(ph);
    if ((tid & 31) == 0) atomicAdd(&s_ph, ph);
    __syncthreads();
    if (tid == 0) {
        int64_t e = s_ph;
        for (uint32_t c = 0; c < nparts; ++c) {
            e += pe[uint64_t(c) * pe_stride];
            if (reset_pe) pe[uint64_t(c) * pe_stride] = 0;
        }
        if (!final) {
            *oe = e;
            return;
        }
        if (e & 1) atomicExch(err, 1);
        const uint32_t outcome = uint32_t((e >> 1) & 1);
        ctl[CTL_OUT] = outcome;
        if (out) *out = qsr_record_entry{q, uint8_t(outcome), 1};
    }
}

// ---- window-level helpers ----------------------------------------------------------
// K4 (CM form): probabilistic flag per measured qubit = any stabilizer word of CM row q
// non-zero. Run before the transpose; identical to the reference's RM scan (measure.hpp:
// 104-126) because nothing changes the tableau between the two.
__global__ void k_flags_cm(const uint64_t *__restrict__ x, uint64_t cm_pitch, uint64_t k,
                           const uint32_t *__restrict__ qubits, uint64_t m,
                           uint8_t *__restrict__ flags) {
    const uint64_t wid = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    if (wid >= m) return;
    const uint64_t *row = x + uint64_t(qubits[wid]) * cm_pitch + k;
    uint64_t acc = 0;
    for (uint64_t j = lane; j < k; j += 32) acc |= row[j];
    bool any = __any_sync(0xffffffffu, acc != 0);
    if (lane == 0) flags[wid] = any ? 1 : 0;
}

__global__ void k_set_ctl(uint32_t *ctl, uint32_t mode, uint32_t c, uint32_t q) {
    ctl[CTL_MODE] = mode;
    ctl[CTL_C] = c;
    ctl[CTL_Q] = q;
    ctl[CTL_COUNT] = 0;
}

__global__ void k_flip_sign(uint64_t *s, uint64_t word, uint64_t bit) { s[word] ^= 1ull << bit; }

int rowmul_blocks(const DeviceTableau &t) { return t.num_sms * 2; }
size_t rowmul_smem(const DeviceTableau &t) { return 2 * t.rm_pitch * sizeof(uint64_t); }

void set_ctl(DeviceTableau &t, uint32_t mode, uint32_t c, uint32_t q) {
    k_set_ctl<<<1, 1, 0, t.stream>>>(t.ms.ctl, mode, c, q);
    QSR_CUDA(cudaGetLastError());
    count_launch();
}

void column_mask(DeviceTableau &t, uint64_t q) {
    const uint64_t nrows = 2 * t.ng;
    const unsigned threads = 256;
    k_column_mask<<<unsigned((nrows + threads - 1) / threads), threads, 0, t.stream>>>(
        t.x, t.rm_pitch, nrows, uint32_t(q >> 6), uint32_t(q & 63),
        reinterpret_cast<uint32_t *>(t.ms.mask));
    QSR_CUDA(cudaGetLastError());
    count_launch();
}

void compact(DeviceTableau &t, const uint8_t *active) {
    k_compact<<<1, 1024, 0, t.stream>>>(t.ms.mask, t.kg, t.ng, t.ms.ctl, t.ms.rows, active);
    QSR_CUDA(cudaGetLastError());
    count_launch();
}

void rowmul(DeviceTableau &t, uint32_t want_mask, int ctl_is_stab) {
    size_t smem = rowmul_smem(t);
    k_rowmul<<<rowmul_blocks(t), 512, smem, t.stream>>>(t.x, t.z, t.rm_pitch, t.k, t.ng, t.s,
                                                        t.ms.ctl, t.ms.rows, want_mask,
                                                        ctl_is_stab, t.ms.err);
    QSR_CUDA(cudaGetLastError());
    count_launch();
}

void det_partial(DeviceTableau &t) {
    dim3 grid{unsigned((t.k + 63) / 64), unsigned(kDetChunks)};
    k_det_partial<<<grid, 32, 0, t.stream>>>(t.x, t.z, t.rm_pitch, t.k, t.ng, t.s, t.ms.ctl,
                                              t.ms.rows, t.ms.partial_x, t.ms.partial_z,
                                              t.ms.partial_e);
    QSR_CUDA(cudaGetLastError());
    count_launch();
}

void finish(DeviceTableau &t, uint64_t seed, qsr_record_entry *out) {
    k_finish<<<1, 1024, 0, t.stream>>>(t.x, t.z, t.rm_pitch, t.k, t.ng, t.s, t.ms.ctl,
                                       t.ms.partial_x, t.ms.partial_z, t.ms.partial_e, seed,
                                       t.ms.coin_index, out, t.ms.err, t.ms.coin_table);
    QSR_CUDA(cudaGetLastError());
    count_launch();
}

// QSR_MEASURE_BATCH=0 selects the one-collapse-per-pass path (differential testing / A-B).
bool batch_collapses() {
    static bool on = [] {
        const char *e = getenv("QSR_MEASURE_BATCH");
        return !(e && e[0] == '0');
    }();
    return on;
}

} // namespace

void configure_measure_kernels(DeviceTableau &t) {
    size_t smem = rowmul_smem(t);
    if (smem > 48 * 1024)
        QSR_CUDA(cudaFuncSetAttribute(k_rowmul, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(smem)));
}

namespace {
uint32_t next_batch_seq() {
    static std::atomic<uint32_t> seq{0};
    uint32_t v = ++seq;
    return v ? v : ++seq; // (0 is a fresh slot's value)
}
} // namespace

void measure_window_device(DeviceTableau &t, uint64_t m, uint64_t seed,
                           const std::vector<uint32_t> &qubits, std::vector<uint8_t> &flags_host,
                           bool timed, double *t_ms, double *ge_ms, double *cmp_ms) {
    (void)cmp_ms;
    cudaEvent_t ev[4];
    if (timed)
        for (auto &e : ev) QSR_CUDA(cudaEventCreate(&e));
    // Flags on the CM tableau (find_probabilistic, measure.hpp:405).
    {
        flags_cm(t, m);
        flags_host.resize(m);
        QSR_CUDA(cudaMemcpyAsync(flags_host.data(), t.ms.flags, m, cudaMemcpyDeviceToHost,
                                 t.stream));
    }
    if (timed) QSR_CUDA(cudaEventRecord(ev[0], t.stream));
    transpose_to_rm(t);
    if (timed) QSR_CUDA(cudaEventRecord(ev[1], t.stream));
    QSR_CUDA(cudaStreamSynchronize(t.stream)); // flags_host ready
    // Sequential collapse loop in window order (measure.hpp:409-431); device-resident
    // decisions (pivot, coin, deterministic fallback).
    if (batch_collapses() && t.trusted) {
        // Batched: up to kMaxBatch consecutive flagged collapses per streaming pass.
        std::vector<uint32_t> fq, fidx;
        for (uint64_t i = 0; i < m; ++i)
            if (flags_host[i]) { fq.push_back(qubits[i]); fidx.push_back(uint32_t(i)); }
        if (!fq.empty()) {
            QSR_CUDA(cudaMemcpyAsync(t.ms.fq, fq.data(), fq.size() * 4, cudaMemcpyHostToDevice, t.stream));
            QSR_CUDA(cudaMemcpyAsync(t.ms.fidx, fidx.data(), fidx.size() * 4, cudaMemcpyHostToDevice,
                                     t.stream));
        }
        auto deterministic_at = [&](size_t pos) { // flagged at window start, deterministic now
            set_ctl(t, MODE_DET, 0, fq[pos]);           // (measure.hpp:417-421)
            column_mask(t, fq[pos]);
            compact(t, nullptr);
            det_partial(t);
            finish(t, seed, t.ms.out + fidx[pos]);
        };
        // Speculative double buffering: batch k+1 is enqueued (assuming batch k collapses all
        // of its measurements) before the host reads batch k's length, so the device never
        // waits for the host. A speculative batch behind one that stopped early finds the
        // device position unequal to its start and does nothing (k_pivot_select).
        MeasureScratch &ms = t.ms;
        struct Pending { size_t start; uint32_t b; int slot; };
        Pending queue[2];
        int qhead = 0, qsize = 0, slot = 0;
        size_t pos = 0, spec = 0;
        set_device_u32(ms.d_pos, 0, t.stream);
        // The sign pass of each batch writes its control words + a sequence number into a pinned
        // slot (no copy or event between the batches' kernels, so the launch chain stays
        // programmatic across batches); the host waits for the sequence number. QSR_HOSTPOLL=0:
        // a 16-byte copy + event per batch instead.
        static const bool poll = [] {
            const char *e = getenv("QSR_HOSTPOLL");
            return !(e && e[0] == '0');
        }();
        uint32_t seqs[2] = {0, 0};
        auto wait_slot = [&](int s) {
            if (!poll) {
                QSR_CUDA(cudaEventSynchronize(ms.bev[s]));
                return;
            }
            volatile const uint32_t *h = ms.h_bctl + 8 * s;
            for (uint32_t spin = 1; h[4] != seqs[s]; ++spin) {
                if ((spin & 1023u) == 0) {
                    const cudaError_t q = cudaStreamQuery(t.stream);
                    if (q != cudaSuccess && q != cudaErrorNotReady) QSR_CUDA(q);
                    if (q == cudaSuccess && h[4] != seqs[s])
                        fail(QSR_LOGIC_ERROR, "measure_window: batch control words never arrived");
                }
            }
            std::atomic_thread_fence(std::memory_order_acquire); // the control words, after seq
        };
        // The sign pass of each batch computes its speculative successor's column bits (QSR_FUSE_COLS=0:
        // a separate column-bit launch per batch).
        static const bool fuse_cols = [] {
            const char *e = getenv("QSR_FUSE_COLS");
            return !(e && e[0] == '0');
        }();
        bool cols_ready = false; // the previous batch's sign pass computed this batch's column bits
        // Chained batches (QSR_CHAIN=0: off): batch k+1's select runs in batch k's absorb (its last
        // CTA) on column bits batch k's membership pass derives; the two batches alternate between
        // two buffer sets. A batch after an early stop starts standalone.
        static const bool chain = [] {
            const char *e = getenv("QSR_CHAIN");
            return !(e && e[0] == '0');
        }();
        const BatchBufs sets[2] = {{ms.vinfo, ms.bctl, ms.colbits, ms.nz, ms.pcount},
                                   {ms.vinfo_b, ms.bctl_b, ms.colbits_b, ms.nz_b, ms.pcount_b}};
        auto use_set = [&](int p) {
            ms.vinfo = sets[p].vinfo;
            ms.bctl = sets[p].bctl;
            ms.colbits = sets[p].colbits;
            ms.nz = sets[p].nz;
            ms.pcount = sets[p].pcount;
        };
        int par = 0;
        bool chained = false; // this batch's select already ran in the previous batch's absorb
        auto next_size = [&](size_t at) {
            return at < fq.size() ? uint32_t(std::min<size_t>(kMaxBatch, fq.size() - at)) : 0u;
        };
        while (pos < fq.size()) {
            while (qsize < 2 && spec < fq.size()) {
                const uint32_t b = uint32_t(std::min<size_t>(kMaxBatch, fq.size() - spec));
                const size_t nxt = spec + b;
                seqs[slot] = next_batch_seq(); // process-wide: pinned slots are recycled across tableaux
                uint32_t *hs = poll ? ms.h_bctl + 8 * slot : nullptr;
                if (chain) {
                    const uint32_t nb = next_size(nxt), nb2 = nb ? next_size(nxt + nb) : 0u;
                    use_set(par);
                    batch_chained(t, sets[par ^ 1], ms.fq + spec, ms.fidx + spec, b, seed, !chained, ms.d_pos,
                                  uint32_t(spec), nb ? ms.fq + nxt : nullptr, nb, nb2 ? ms.fq + nxt + nb : nullptr,
                                  nb2, hs, seqs[slot]);
                    chained = nb != 0;
                    par ^= 1;
                } else {
                    if (!cols_ready) batch_colbits(t, ms.fq + spec, b);
                    const uint32_t nb = fuse_cols ? next_size(nxt) : 0u;
                    batch_fused(t, ms.fq + spec, ms.fidx + spec, b, seed, ms.d_pos, uint32_t(spec), hs, seqs[slot],
                                nb ? ms.fq + nxt : nullptr, nb);
                    cols_ready = nb != 0;
                }
                if (!poll) {
                    QSR_CUDA(cudaMemcpyAsync(ms.h_bctl + 8 * slot, ms.bctl, 16, cudaMemcpyDeviceToHost, t.stream));
                    QSR_CUDA(cudaEventRecord(ms.bev[slot], t.stream));
                }
                queue[(qhead + qsize) % 2] = Pending{spec, b, slot};
                ++qsize;
                slot ^= 1;
                spec += b;
            }
            const Pending p = queue[qhead];
            qhead = (qhead + 1) % 2;
            --qsize;
            wait_slot(p.slot);
            volatile const uint32_t *h = ms.h_bctl + 8 * p.slot;
            if (h[3]) continue; // skipped (behind a batch that stopped early)
            pos = p.start + h[0];
            if (h[1]) {         // stopped: the measurement at pos is deterministic now
                while (qsize) { // the speculative batch behind it is a no-op; drain it
                    wait_slot(queue[qhead].slot);
                    qhead = (qhead + 1) % 2;
                    --qsize;
                }
                deterministic_at(pos++);
                set_device_u32(ms.d_pos, uint32_t(pos), t.stream);
                spec = pos;
                cols_ready = false; // the drained batch's successor columns were for another position
                chained = false;
            }
        }
        use_set(0); // (the other paths and the sharded engine use the first set)
    } else {
        for (uint64_t i = 0; i < m; ++i) {
            if (!flags_host[i]) continue;
            set_ctl(t, MODE_COLLAPSE, 0, qubits[i]);
            column_mask(t, qubits[i]);
            compact(t, nullptr);
            rowmul(t, 1u << MODE_COLLAPSE, 1);
            det_partial(t);
            finish(t, seed, t.ms.out + i);
        }
    }
    // Deterministic outcomes of the unflagged measurements (measure.hpp:432-438).
    for (uint64_t i = 0; i < m; ++i) {
        if (flags_host[i]) continue;
        set_ctl(t, MODE_DET, 0, qubits[i]);
        column_mask(t, qubits[i]);
        compact(t, nullptr);
        det_partial(t);
        finish(t, seed, t.ms.out + i);
    }
    if (timed) QSR_CUDA(cudaEventRecord(ev[2], t.stream));
    transpose_to_cm(t);
    if (timed) {
        QSR_CUDA(cudaEventRecord(ev[3], t.stream));
        QSR_CUDA(cudaEventSynchronize(ev[3]));
        float a, b, c;
        QSR_CUDA(cudaEventElapsedTime(&a, ev[0], ev[1]));
        QSR_CUDA(cudaEventElapsedTime(&b, ev[1], ev[2]));
        QSR_CUDA(cudaEventElapsedTime(&c, ev[2], ev[3]));
        if (t_ms) *t_ms += a + c;
        if (ge_ms) *ge_ms += b;
        for (auto &e : ev) QSR_CUDA(cudaEventDestroy(e));
    }
}

uint64_t det_slot_words(const DeviceTableau &t) { return 2 * t.rm_pitch + 16; }

void det_local_partial(DeviceTableau &t, uint64_t q, uint64_t *slot) {
    set_ctl(t, MODE_DET, 0, uint32_t(q));
    column_mask(t, q);
    compact(t, nullptr);
    det_partial(t);
    k_det_reduce<<<1, 1024, 0, t.stream>>>(t.ms.partial_x, t.ms.partial_z, t.ms.partial_e,
                                           t.rm_pitch, 1, kDetChunks, t.k, 1, 0, slot,
                                           slot + t.rm_pitch,
                                           reinterpret_cast<int64_t *>(slot + 2 * t.rm_pitch),
                                           t.ms.ctl, uint32_t(q), nullptr, t.ms.err);
    QSR_CUDA(cudaGetLastError());
    count_launch();
}

void det_combine(DeviceTableau &t, uint64_t q, const uint64_t *slots, uint32_t nslots,
                 qsr_record_entry *out, uint64_t slot_stride) {
    const uint64_t sw = slot_stride ? slot_stride : det_slot_words(t);
    k_det_reduce<<<1, 1024, 0, t.stream>>>(
        slots, slots + t.rm_pitch,
        reinterpret_cast<int64_t *>(const_cast<uint64_t *>(slots) + 2 * t.rm_pitch), sw, sw,
        nslots, t.k, 0, 1, nullptr, nullptr, nullptr, t.ms.ctl, uint32_t(q), out, t.ms.err);
    QSR_CUDA(cudaGetLastError());
    count_launch();
}

void flags_cm(DeviceTableau &t, uint64_t m) {
    if (m == 0) return;
    const unsigned threads = 256;
    const unsigned blocks = unsigned((m * 32 + threads - 1) / threads);
    k_flags_cm<<<blocks, threads, 0, t.stream>>>(t.x, t.cm_pitch, t.kg, t.ms.mqubits, m,
                                                 t.ms.flags);
    QSR_CUDA(cudaGetLastError());
    count_launch();
}

// ---- API-parity operations on a (transposed) RM tableau ------------------------------
void rm_column_mask(DeviceTableau &t, uint64_t q) { column_mask(t, q); }

namespace {
// find_and_compact_pivots' scatter + stable compaction (measure.hpp:130-150,
// bitplane.hpp:126-136) on the device: the stabilizer half of q's column mask (bit g = X bit of
// stabilizer g at q) becomes the ascending pivot list with a -1 tail. One CTA: contiguous word
// chunks per thread, a popcount block scan for the output offsets, then every thread writes its
// pivots in order and the tail.
__global__ void __launch_bounds__(1024)
k_pivot_list(const uint64_t *__restrict__ mask, uint64_t words, uint64_t n, int64_t *__restrict__ entries,
             uint64_t *__restrict__ count) {
    __shared__ uint32_t s_warp[32];
    __shared__ uint32_t s_total;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, T = blockDim.x;
    const uint64_t per = (words + T - 1) / T, w0 = min(words, uint64_t(tid) * per), w1 = min(words, w0 + per);
    uint32_t cnt = 0;
    for (uint64_t w = w0; w < w1; ++w) cnt += uint32_t(__popcll(mask[w]));
    uint32_t incl = cnt; // inclusive scan: warp, then warp totals
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= uint32_t(o)) incl += v;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint32_t v = lane < (T + 31) / 32 ? s_warp[lane] : 0u, x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= uint32_t(o)) x += u;
        }
        s_warp[lane] = x - v; // exclusive warp offsets
        if (lane == 31) s_total = x;
    }
    __syncthreads();
    uint64_t pos = s_warp[warp] + incl - cnt;
    for (uint64_t w = w0; w < w1; ++w)
        for (uint64_t m = mask[w]; m; m &= m - 1) entries[pos++] = int64_t(w * 64 + uint64_t(__ffsll(m) - 1));
    const uint32_t total = s_total;
    for (uint64_t i = uint64_t(total) + tid; i < n; i += T) entries[i] = -1;
    if (tid == 0) *count = total;
}
} // namespace

void rm_find_pivots(DeviceTableau &t, uint64_t q, std::vector<int64_t> &entries, uint64_t &count) {
    column_mask(t, q);
    int64_t *d_entries = nullptr;
    uint64_t *d_count = nullptr;
    QSR_CUDA(cudaMallocAsync(&d_entries, t.n * 8 + 8, t.stream));
    d_count = reinterpret_cast<uint64_t *>(d_entries + t.n);
    k_pivot_list<<<1, 1024, 0, t.stream>>>(t.ms.mask + t.kg, t.kg, t.n, d_entries, d_count);
    QSR_CUDA(cudaGetLastError());
    count_launch();
    entries.resize(t.n);
    QSR_CUDA(cudaMemcpyAsync(entries.data(), d_entries, t.n * 8, cudaMemcpyDeviceToHost, t.stream));
    QSR_CUDA(cudaMemcpyAsync(&count, d_count, 8, cudaMemcpyDeviceToHost, t.stream));
    QSR_CUDA(cudaFreeAsync(d_entries, t.stream));
    QSR_CUDA(cudaStreamSynchronize(t.stream));
}

void rm_find_probabilistic(DeviceTableau &t, const std::vector<uint32_t> &qubits,
                           std::vector<int64_t> &out) {
    out.assign(qubits.size(), -1);
    std::vector<uint64_t> mask(t.kg);
    for (size_t i = 0; i < qubits.size(); ++i) {
        column_mask(t, qubits[i]);
        QSR_CUDA(cudaMemcpyAsync(mask.data(), t.ms.mask + t.kg, t.kg * 8, cudaMemcpyDeviceToHost,
                                 t.stream));
        QSR_CUDA(cudaStreamSynchronize(t.stream));
        for (uint64_t w = 0; w < t.kg; ++w)
            if (mask[w]) { out[i] = qubits[i]; break; }
    }
}

namespace {
// Destabilizer half of parallel_ge (measure.hpp:188-272) for API parity: D_c accumulates the
// targets' destabilizers in order; each target's flip uses the exclusive prefix (control
// snapshot included). One warp per 64-word tile walks the targets sequentially.
__global__ void k_ge_dest(uint64_t *__restrict__ x, uint64_t *__restrict__ z, uint64_t rm_pitch,
                          uint64_t k, const uint32_t *__restrict__ targets, uint64_t ntargets,
                          uint64_t c, int *__restrict__ phase) {
    const uint32_t lane = threadIdx.x;
    const uint64_t i = uint64_t(blockIdx.x) * 64 + lane * 2;
    const bool act = i < k;
    uint64_t px0 = 0, px1 = 0, pz0 = 0, pz1 = 0;
    if (act) {
        px0 = x[c * rm_pitch + i]; px1 = x[c * rm_pitch + i + 1];
        pz0 = z[c * rm_pitch + i]; pz1 = z[c * rm_pitch + i + 1];
    }
    for (uint64_t e = 0; e < ntargets; ++e) {
        const uint64_t r = targets[e];
        int ph = 0;
        if (act) {
            uint64_t tx0 = x[r * rm_pitch + i], tx1 = x[r * rm_pitch + i + 1];
            uint64_t tz0 = z[r * rm_pitch + i], tz1 = z[r * rm_pitch + i + 1];
            ph = phase_delta(px0, pz0, tx0, tz0) + phase_delta(px1, pz1, tx1, tz1);
            px0 ^= tx0; px1 ^= tx1; pz0 ^= tz0; pz1 ^= tz1;
        }
        ph = warp_sum(ph);
        if (lane == 0 && ph) atomicAdd(phase + e, ph);
    }
    if (act) {
        x[c * rm_pitch + i] = px0; x[c * rm_pitch + i + 1] = px1;
        z[c * rm_pitch + i] = pz0; z[c * rm_pitch + i + 1] = pz1;
    }
}
} // namespace

void rm_parallel_ge(DeviceTableau &t, const std::vector<int64_t> &pivots) {
    const uint64_t c = uint64_t(pivots[0]);
    const uint64_t T = pivots.size() - 1;
    if (T == 0) return;
    std::vector<uint32_t> stab_rows(T), dest_rows(T);
    for (uint64_t e = 0; e < T; ++e) {
        stab_rows[e] = uint32_t(t.ng + uint64_t(pivots[e + 1]));
        dest_rows[e] = uint32_t(pivots[e + 1]);
    }
    // Destabilizer half first (reads target destabilizers, which the stabilizer half never
    // touches; the reference computes both histories in one pass before any sign fold).
    uint32_t *d_targets = nullptr;
    int *d_phase = nullptr;
    QSR_CUDA(cudaMallocAsync(&d_targets, T * 4, t.stream));
    QSR_CUDA(cudaMallocAsync(&d_phase, T * 4, t.stream));
    QSR_CUDA(cudaMemcpyAsync(d_targets, dest_rows.data(), T * 4, cudaMemcpyHostToDevice, t.stream));
    QSR_CUDA(cudaMemsetAsync(d_phase, 0, T * 4, t.stream));
    k_ge_dest<<<unsigned((t.k + 63) / 64), 32, 0, t.stream>>>(t.x, t.z, t.rm_pitch, t.k, d_targets,
                                                             T, c, d_phase);
    QSR_CUDA(cudaGetLastError());
    count_launch();
    std::vector<int> phase(T);
    QSR_CUDA(cudaMemcpyAsync(phase.data(), d_phase, T * 4, cudaMemcpyDeviceToHost, t.stream));
    // Stabilizer half: S_t ^= S_c with sign s_t ^= s_c ^ flip (fused row kernel).
    QSR_CUDA(cudaMemcpyAsync(t.ms.rows, stab_rows.data(), T * 4, cudaMemcpyHostToDevice, t.stream));
    set_ctl(t, MODE_COLLAPSE, uint32_t(c), 0);
    uint32_t cnt = uint32_t(T);
    QSR_CUDA(cudaMemcpyAsync(t.ms.ctl + CTL_COUNT, &cnt, 4, cudaMemcpyHostToDevice, t.stream));
    rowmul(t, 1u << MODE_COLLAPSE, 1);
    std::vector<uint64_t> s(2 * t.kg);
    QSR_CUDA(cudaMemcpyAsync(s.data(), t.s, 2 * t.kg * 8, cudaMemcpyDeviceToHost, t.stream));
    QSR_CUDA(cudaStreamSynchronize(t.stream));
    QSR_CUDA(cudaFreeAsync(d_targets, t.stream));
    QSR_CUDA(cudaFreeAsync(d_phase, t.stream));
    if (read_error_flag(t))
        fail(QSR_LOGIC_ERROR, "product of anti-commuting rows (corrupted tableau)");
    // Control destabilizer sign: XOR of s(D_t) ^ flip(prefix phase) (measure.hpp:258-272).
    uint64_t dc = (s[c / 64] >> (c % 64)) & 1;
    for (uint64_t e = 0; e < T; ++e) {
        int ph = phase[e];
        if (ph & 1) fail(QSR_LOGIC_ERROR, "product of anti-commuting rows (corrupted tableau)");
        uint64_t tg = uint64_t(pivots[e + 1]);
        uint64_t st = (s[tg / 64] >> (tg % 64)) & 1;
        dc ^= st ^ ((uint64_t(ph) >> 1) & 1);
    }
    uint64_t cur = (s[c / 64] >> (c % 64)) & 1;
    if (cur != dc) flip_sign_bit(t, c / 64, c % 64);
}

void rm_swap_anti_commuting(DeviceTableau &t, uint64_t p, uint64_t q) {
    set_ctl(t, MODE_SWAP, uint32_t(p), uint32_t(q));
    column_mask(t, q);
    compact(t, nullptr);
    rowmul(t, 1u << MODE_SWAP, 1);
    finish(t, 0, nullptr);
}

bool rm_deterministic_outcome(DeviceTableau &t, uint64_t q) {
    set_ctl(t, MODE_DET, 0, uint32_t(q));
    column_mask(t, q);
    compact(t, nullptr);
    det_partial(t);
    finish(t, 0, nullptr);
    uint32_t out = 0;
    QSR_CUDA(cudaMemcpyAsync(&out, t.ms.ctl + CTL_OUT, 4, cudaMemcpyDeviceToHost, t.stream));
    QSR_CUDA(cudaStreamSynchronize(t.stream));
    if (read_error_flag(t))
        fail(QSR_LOGIC_ERROR, "deterministic_outcome: imaginary phase (corrupted tableau)");
    return out != 0;
}

void flip_sign_bit(DeviceTableau &t, uint64_t word, uint64_t bit) {
    k_flip_sign<<<1, 1, 0, t.stream>>>(t.s, word, bit);
    QSR_CUDA(cudaGetLastError());
    count_launch();
}

int read_error_flag(DeviceTableau &t) {
    int e = 0;
    QSR_CUDA(cudaMemcpyAsync(&e, t.ms.err, 4, cudaMemcpyDeviceToHost, t.stream));
    QSR_CUDA(cudaStreamSynchronize(t.stream));
    if (e) QSR_CUDA(cudaMemsetAsync(t.ms.err, 0, 4, t.stream));
    return e;
}

} // namespace qsr
