// K1 — gate-window kernel (reference gates.hpp:147-197, frames.hpp:76-94).
//
// A window's gates act on disjoint qubits, and every generator-word j is independent, so the
// window is a 2-D domain (gate, j). CTA = 8 warps sharing one j-tile of 64 words (each lane
// owns 2 adjacent words, moved with 128-bit ld/st.global.v2.u64 — a warp touches 512
// contiguous bytes of a qubit row, i.e. four full 128-byte lines). The 8 warps stride over
// one chunk of the window's gates; grid.y splits the window into chunks so that
// tiles x chunks fills every SM. Each lane keeps its two sign words in registers across all
// its gates, the 8 warps combine them with a shared-memory XOR tree, and the per-(chunk,
// tile) partial is folded into S[j] by the last CTA of the tile to arrive (no per-gate or
// per-word global atomics; XOR makes the fold order-free, so the result is bit-identical to
// the reference's partitioned reduce_xor).
//
// Only the operand words a kind actually reads / writes are moved (X/Y/Z never write, S
// writes z0 only, ...), so DRAM traffic equals the kind-exact algorithmic byte model.
// U gates are in flight per warp iteration to raise memory-level parallelism.
#include <algorithm>
#include <string>

#include "common.cuh"
#include "device.hpp"

namespace qsr {

namespace {

struct V2 {
    uint64_t a, b;
    __device__ __forceinline__ V2 operator&(V2 o) const { return {a & o.a, b & o.b}; }
    __device__ __forceinline__ V2 operator^(V2 o) const { return {a ^ o.a, b ^ o.b}; }
    __device__ __forceinline__ V2 operator~() const { return {~a, ~b}; }
    __device__ __forceinline__ V2 &operator^=(V2 o) { a ^= o.a; b ^= o.b; return *this; }
};

__device__ __forceinline__ V2 ld2(const uint64_t *p) {
    ulonglong2 v = __ldcg(reinterpret_cast<const ulonglong2 *>(p));
    return {v.x, v.y};
}
__device__ __forceinline__ void st2(uint64_t *p, V2 v) {
    __stcg(reinterpret_cast<ulonglong2 *>(p), make_ulonglong2(v.a, v.b));
}

// Vectorised word rules (same table as common.cuh apply_rule, both lanes at once).
__device__ __forceinline__ V2 rule2(uint32_t kind, V2 &x0, V2 &z0, V2 &x1, V2 &z1) {
    V2 sign{0, 0};
    switch (kind) {
    case K_H: { sign = x0 & z0; V2 t = x0; x0 = z0; z0 = t; break; }
    case K_S: sign = x0 & z0; z0 ^= x0; break;
    case K_SDG: sign = x0 & ~z0; z0 ^= x0; break;
    case K_X: sign = z0; break;
    case K_Y: sign = x0 ^ z0; break;
    case K_Z: sign = x0; break;
    case K_CX: sign = x0 & z1 & ~(x1 ^ z0); x1 ^= x0; z0 ^= z1; break;
    case K_CZ: sign = x0 & x1 & (z0 ^ z1); z1 ^= x0; z0 ^= x1; break;
    case K_CY: {
        V2 s1 = x1 & ~z1;
        V2 zt = z1 ^ x1;
        V2 s2 = x0 & zt & ~(x1 ^ z0);
        V2 xt = x1 ^ x0;
        V2 zc = z0 ^ zt;
        V2 s3 = xt & zt;
        sign = s1 ^ s2 ^ s3;
        x1 = xt; z0 = zc; z1 = zt ^ xt;
        break;
    }
    case K_SWAP: { V2 t = x0; x0 = x1; x1 = t; t = z0; z0 = z1; z1 = t; break; }
    case K_ISWAP:
    case K_ISWAP_R: { // ISWAP = the swap, then this residual (symmetric in its operands)
        if (kind == K_ISWAP) { V2 t = x0; x0 = x1; x1 = t; t = z0; z0 = z1; z1 = t; }
        V2 s2 = x0 & x1 & (z0 ^ z1);
        V2 zt = z1 ^ x0;
        V2 zc = z0 ^ x1;
        V2 s3 = x1 & zt;
        V2 s4 = x0 & zc;
        sign = s2 ^ s3 ^ s4;
        z1 = zt ^ x1; z0 = zc ^ x0;
        break;
    }
    default: break; // K_C1: only its pre-operation
    }
    return sign;
}

// One of the 24 single-qubit Cliffords (kCliff1 encoding: bits 0-3 matrix m00 m01 m10 m11, bits
// 4-6 sign flips of the images of X, Z, Y) on a word pair; returns the sign-flip words. Each
// element is a compile-time instance (the masks fold away: 2-6 logic ops per word instead of
// table-driven masking), selected by a warp-uniform switch.
template <uint32_t C>
__device__ __forceinline__ V2 cliff1_fixed(V2 &x, V2 &z) {
    V2 f{0, 0}, nx{0, 0}, nz{0, 0};
    if (C & 16u) f ^= x & ~z;
    if (C & 32u) f ^= z & ~x;
    if (C & 64u) f ^= x & z;
    if (C & 1u) nx ^= x;
    if (C & 2u) nx ^= z;
    if (C & 4u) nz ^= x;
    if (C & 8u) nz ^= z;
    x = nx;
    z = nz;
    return f;
}

__device__ __forceinline__ V2 cliff1_apply(uint32_t e, V2 &x, V2 &z) {
    switch (e) { // kCliff1 (common.cuh), element 0 = identity
    case 1: return cliff1_fixed<105>(x, z);
    case 2: return cliff1_fixed<57>(x, z);
    case 3: return cliff1_fixed<89>(x, z);
    case 4: return cliff1_fixed<70>(x, z);
    case 5: return cliff1_fixed<77>(x, z);
    case 6: return cliff1_fixed<29>(x, z);
    case 7: return cliff1_fixed<38>(x, z);
    case 8: return cliff1_fixed<45>(x, z);
    case 9: return cliff1_fixed<125>(x, z);
    case 10: return cliff1_fixed<118>(x, z);
    case 11: return cliff1_fixed<22>(x, z);
    case 12: return cliff1_fixed<14>(x, z);
    case 13: return cliff1_fixed<110>(x, z);
    case 14: return cliff1_fixed<87>(x, z);
    case 15: return cliff1_fixed<7>(x, z);
    case 16: return cliff1_fixed<55>(x, z);
    case 17: return cliff1_fixed<103>(x, z);
    case 18: return cliff1_fixed<62>(x, z);
    case 19: return cliff1_fixed<94>(x, z);
    case 20: return cliff1_fixed<43>(x, z);
    case 21: return cliff1_fixed<75>(x, z);
    case 22: return cliff1_fixed<123>(x, z);
    case 23: return cliff1_fixed<27>(x, z);
    default: return V2{0, 0};
    }
}

// A packed gate on its operand words: the fused single-qubit pre-operations, then the rule.
__device__ __forceinline__ V2 gate2(uint64_t gw, V2 &x0, V2 &z0, V2 &x1, V2 &z1) {
    V2 sign{0, 0};
    const uint32_t p0 = gate_pre0(gw), p1 = gate_pre1(gw);
    if (p0) sign ^= cliff1_apply(p0, x0, z0);
    if (p1) sign ^= cliff1_apply(p1, x1, z1);
    sign ^= rule2(gate_kind(gw), x0, z0, x1, z1);
    return sign;
}

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kTileWords = 64;

// Per-CTA sign fold: shared-memory XOR tree over the 8 warps (the reference's collapse_signs /
// reduce_xor, bitplane.hpp:96-122, done per CTA); with several gate chunks per tile the last
// CTA of the tile to arrive folds the per-chunk partials into S[j].
__device__ __forceinline__ void fold_tile_signs(V2 sacc, uint32_t warp, uint32_t lane, uint64_t j, bool active,
                                                uint64_t pitch, uint64_t *__restrict__ partials,
                                                uint32_t *__restrict__ counters, uint64_t *__restrict__ s) {
    __shared__ uint64_t red[kWarps][kTileWords];
    __shared__ bool last;
    red[warp][lane * 2] = sacc.a;
    red[warp][lane * 2 + 1] = sacc.b;
    __syncthreads();
#pragma unroll
    for (int h = kWarps / 2; h >= 1; h >>= 1) {
        if (warp < uint32_t(h)) {
            red[warp][lane * 2] ^= red[warp + h][lane * 2];
            red[warp][lane * 2 + 1] ^= red[warp + h][lane * 2 + 1];
        }
        __syncthreads();
    }
    if (gridDim.y == 1) {
        if (warp == 0 && active) {
            s[j] ^= red[0][lane * 2];
            s[j + 1] ^= red[0][lane * 2 + 1];
        }
        return;
    }
    if (warp == 0 && active) {
        uint64_t *p = partials + uint64_t(blockIdx.y) * pitch + j;
        __stcg(reinterpret_cast<ulonglong2 *>(p),
               make_ulonglong2(red[0][lane * 2], red[0][lane * 2 + 1]));
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t prev = atomicAdd(counters + blockIdx.x, 1u);
        last = prev == gridDim.y - 1;
    }
    __syncthreads();
    if (last && warp == 0) {
        __threadfence();
        if (active) {
            uint64_t a = 0, b = 0;
            for (uint32_t c = 0; c < gridDim.y; ++c) {
                ulonglong2 v = __ldcg(reinterpret_cast<const ulonglong2 *>(
                    partials + uint64_t(c) * pitch + j));
                a ^= v.x;
                b ^= v.y;
            }
            s[j] ^= a;
            s[j + 1] ^= b;
        }
        if (lane == 0)
            counters[blockIdx.x] = 0; // re-armed for the next window
    }
}

template <bool kSigns, int U, int kMinBlocks>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
k_gate_window(uint64_t *__restrict__ x, uint64_t *__restrict__ z, uint64_t pitch,
              const uint64_t *__restrict__ gates, uint32_t ngates, uint32_t chunk,
              uint64_t *__restrict__ partials, uint32_t *__restrict__ counters,
              uint64_t *__restrict__ s) {
    // Programmatic dependent launch (launch_window_kernel): wait for the previous window to
    // complete, then let the next one's CTAs take the SM slots this grid's tail frees.
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t j = uint64_t(blockIdx.x) * kTileWords + lane * 2;
    const bool active = j < pitch; // pitch % 16 == 0, so j+1 < pitch too
    const uint32_t g_begin = blockIdx.y * chunk;
    const uint32_t g_end = min(g_begin + chunk, ngates);
    V2 sacc{0, 0};

    if (active) {
        uint32_t g = g_begin + warp;
        for (; g + kWarps * (U - 1) < g_end; g += kWarps * U) {
            uint64_t gws[U];
            uint32_t rd[U], wr[U];
            uint64_t o0[U], o1[U];
            V2 X0[U], Z0[U], X1[U], Z1[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint64_t gw = gws[u] = __ldg(gates + g + kWarps * u);
                rd[u] = gate_reads(gw, kSigns);
                wr[u] = gate_writes(gw);
                o0[u] = uint64_t(gate_q0(gw)) * uint32_t(pitch) + j;
                o1[u] = uint64_t(gate_q1(gw)) * uint32_t(pitch) + j;
                X0[u] = Z0[u] = X1[u] = Z1[u] = V2{0, 0};
                if (rd[u] & 1) X0[u] = ld2(x + o0[u]);
                if (rd[u] & 2) Z0[u] = ld2(z + o0[u]);
                if (rd[u] & 4) X1[u] = ld2(x + o1[u]);
                if (rd[u] & 8) Z1[u] = ld2(z + o1[u]);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                V2 sg = gate2(gws[u], X0[u], Z0[u], X1[u], Z1[u]);
                if (kSigns) sacc ^= sg;
                if (wr[u] & 1) st2(x + o0[u], X0[u]);
                if (wr[u] & 2) st2(z + o0[u], Z0[u]);
                if (wr[u] & 4) st2(x + o1[u], X1[u]);
                if (wr[u] & 8) st2(z + o1[u], Z1[u]);
            }
        }
        for (; g < g_end; g += kWarps) {
            uint64_t gw = __ldg(gates + g);
            uint32_t rd = gate_reads(gw, kSigns), wr = gate_writes(gw);
            uint64_t a0 = uint64_t(gate_q0(gw)) * uint32_t(pitch) + j, a1 = uint64_t(gate_q1(gw)) * uint32_t(pitch) + j;
            V2 X0{0, 0}, Z0{0, 0}, X1{0, 0}, Z1{0, 0};
            if (rd & 1) X0 = ld2(x + a0);
            if (rd & 2) Z0 = ld2(z + a0);
            if (rd & 4) X1 = ld2(x + a1);
            if (rd & 8) Z1 = ld2(z + a1);
            V2 sg = gate2(gw, X0, Z0, X1, Z1);
            if (kSigns) sacc ^= sg;
            if (wr & 1) st2(x + a0, X0);
            if (wr & 2) st2(z + a0, Z0);
            if (wr & 4) st2(x + a1, X1);
            if (wr & 8) st2(z + a1, Z1);
        }
    }

    if constexpr (kSigns) fold_tile_signs(sacc, warp, lane, j, active, pitch, partials, counters, s);
}

// Kernel variants (unroll U, min resident CTAs): 0 = <2,3>, 1 = <1,4>, 2 = <2,4>, 3 = <2,2>,
// 4 = <4,2>.
// QSR_GATE_VARIANT selects one for tuning runs; the default is the measured best
// (profiles/r01_gate_tune.log: <2,3> 6.37 TB/s at c5, <1,4> 6.31, <2,4> 6.07 with spills).
// Default: <1,4> (fused c5 windows, ~45k gates: 216.7 vs 226.2 ms per 100 windows at 180k qubits,
// no spills at 64 registers; round 1 kept <2,3> for windows under 16k gates, 20k qubits: 10.5 vs
// 11.1 ms per 300, which no longer holds — see gate_variant).
int gate_variant(uint64_t ngates) {
    static int v = [] {
        const char *e = getenv("QSR_GATE_VARIANT");
        return e ? atoi(e) : -1;
    }();
    if (v >= 0) return v;
    // <1,4> for every window since small windows are chunked at >= 8 gates per warp (pick_chunks):
    // same box, interleaved, c2 32.1 -> 31.1 ms and c4 34.6 -> 32.7 ms against <2,3> below 16 k
    // gates (round 1's choice for them, measured before that chunking and the PDL launches).
    (void)ngates;
    return 1;
}

// Grid of a window launch: tiles x chunks CTAs. Every CTA does the same work, so the grid should
// be a whole number of waves: pick the chunk count (>= ~4 waves when the window is big enough)
// whose tiles x chunks leaves the smallest partial last wave. At least 16 items per warp per
// chunk (8 for windows under 16 k gates) keep the XOR tree and the tile fold negligible: the
// 8 for small windows measured c2 33.3 -> 32.2 ms and c4 35.5 -> 34.8 ms per step, while the
// larger windows (c3 gate phase 188 -> 200 ms) keep 16 and c5 is unaffected (its search range
// stays below the cap). Grows the sign partials as needed.
void pick_chunks(uint64_t pitch, uint64_t nitems, int num_sms, int bps, bool signs, uint64_t **partials,
                 uint64_t *partial_chunks, uint64_t *tiles_out, uint64_t *chunk_out, uint64_t *chunks_out,
                 cudaStream_t st) {
    const uint64_t tiles = (pitch + kTileWords - 1) / kTileWords;
    const uint64_t slots = uint64_t(num_sms) * uint64_t(bps);
    static const uint64_t per_warp_env = [] { // QSR_GATE_MINPW: tuning knob (0 = by window size)
        const char *e = getenv("QSR_GATE_MINPW");
        return e ? std::max<uint64_t>(1, uint64_t(atoll(e))) : uint64_t(0);
    }();
    const uint64_t per_warp = per_warp_env ? per_warp_env : nitems < (uint64_t(1) << 14) ? 8 : 16;
    const uint64_t max_chunks = std::max<uint64_t>(1, nitems / (kWarps * per_warp));
    uint64_t c_min = std::max<uint64_t>(1, (4 * slots + tiles - 1) / tiles);
    // Small windows cannot reach ~4 waves: search the upper half of the allowed range, where a
    // grid just under a whole wave beats one that spills a few CTAs into a second wave.
    if (c_min > max_chunks) c_min = std::max<uint64_t>(1, max_chunks / 2);
    uint64_t chunks = c_min;
    double best = 1e30;
    for (uint64_t c = c_min; c <= std::min<uint64_t>(max_chunks, 4 * c_min); ++c) {
        const uint64_t ctas = tiles * c;
        const uint64_t waves = (ctas + slots - 1) / slots;
        const double eff_time = double(waves) / double(c); // per-CTA work ~ 1/c
        if (eff_time < best * 0.999) { best = eff_time; chunks = c; }
    }
    if (chunks > 65535) chunks = 65535;
    uint64_t chunk = (nitems + chunks - 1) / chunks;
    chunks = (nitems + chunk - 1) / chunk;
    if (signs && chunks > 1 && chunks > *partial_chunks) { // (the owner's device is current)
        int dev = 0;
        QSR_CUDA(cudaGetDevice(&dev));
        if (*partials) cache_release(dev, *partial_chunks * pitch * sizeof(uint64_t), *partials, st);
        *partials = static_cast<uint64_t *>(cache_acquire(dev, chunks * pitch * sizeof(uint64_t)));
        *partial_chunks = chunks;
    }
    *tiles_out = tiles;
    *chunk_out = chunk;
    *chunks_out = chunks;
}

// Gate windows launch with programmatic stream serialization (PDL): back-to-back windows overlap
// the next launch with the previous grid's tail. QSR_PDL=0 restores plain launches.
bool pdl_enabled() {
    static const bool on = [] {
        const char *e = getenv("QSR_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

template <bool kSigns, int U, int B>
void launch_variant(uint64_t *x, uint64_t *z, uint64_t pitch, const uint64_t *gates,
                    uint64_t ngates, int num_sms, cudaStream_t st, uint64_t **partials,
                    uint64_t *partial_chunks, uint32_t *counters, uint64_t *s) {
    static int bps = 0;
    if (bps == 0) {
        QSR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &bps, k_gate_window<kSigns, U, B>, kThreads, 0));
        if (bps < 1)
            bps = 1;
    }
    uint64_t tiles, chunk, chunks;
    pick_chunks(pitch, ngates, num_sms, bps, kSigns, partials, partial_chunks, &tiles, &chunk, &chunks, st);
    dim3 grid{unsigned(tiles), unsigned(chunks)};
    uint64_t *part = kSigns ? *partials : nullptr;
    if (pdl_enabled()) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = 0;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        QSR_CUDA(cudaLaunchKernelEx(&cfg, k_gate_window<kSigns, U, B>, x, z, pitch, gates,
                                    uint32_t(ngates), uint32_t(chunk), part, counters, s));
    } else {
        k_gate_window<kSigns, U, B><<<grid, kThreads, 0, st>>>(x, z, pitch, gates, uint32_t(ngates),
                                                               uint32_t(chunk), part, counters, s);
    }
    QSR_CUDA(cudaGetLastError());
    count_launch();
}

template <bool kSigns>
void launch(uint64_t *x, uint64_t *z, uint64_t pitch, const uint64_t *gates, uint64_t ngates,
            int num_sms, cudaStream_t st, uint64_t **partials, uint64_t *partial_chunks,
            uint32_t *counters, uint64_t *s) {
    if (ngates == 0)
        return;
    switch (gate_variant(ngates)) {
    case 0:
        launch_variant<kSigns, 2, 3>(x, z, pitch, gates, ngates, num_sms, st, partials,
                                     partial_chunks, counters, s);
        break;
    case 3:
        launch_variant<kSigns, 2, 2>(x, z, pitch, gates, ngates, num_sms, st, partials,
                                     partial_chunks, counters, s);
        break;
    case 4:
        launch_variant<kSigns, 4, 2>(x, z, pitch, gates, ngates, num_sms, st, partials,
                                     partial_chunks, counters, s);
        break;
    case 2:
        launch_variant<kSigns, 2, 4>(x, z, pitch, gates, ngates, num_sms, st, partials,
                                     partial_chunks, counters, s);
        break;
    default:
        launch_variant<kSigns, 1, 4>(x, z, pitch, gates, ngates, num_sms, st, partials,
                                     partial_chunks, counters, s);
        break;
    }
}


} // namespace

void launch_gate_window(DeviceTableau &t, const uint64_t *gates, uint64_t ngates) {
    launch<true>(t.x, t.z, t.cm_pitch, gates, ngates, t.num_sms, t.stream, &t.sign_partials,
                 &t.sign_partial_chunks, t.tile_counters, t.s);
}

void launch_frame_window(uint64_t *xf, uint64_t *zf, uint64_t pitch, const uint64_t *gates,
                         uint64_t ngates, int num_sms, cudaStream_t st) {
    launch<false>(xf, zf, pitch, gates, ngates, num_sms, st, nullptr, nullptr, nullptr, nullptr);
}

} // namespace qsr

namespace qsr {

namespace {
// dst row q = src row perm[q] (q < n), rows n .. rows-1 copied as they are (zero padding).
__global__ void k_unpermute_rows(const uint64_t *__restrict__ src, uint64_t *__restrict__ dst, uint64_t pitch,
                                 uint64_t n, uint64_t rows, const uint32_t *__restrict__ perm) {
    const uint64_t chunks = pitch / 2; // 16-byte chunks per row
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < rows * chunks;
         e += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t q = e / chunks, c = e - q * chunks;
        const uint64_t from = q < n ? perm[q] : q;
        __stcs(reinterpret_cast<ulonglong2 *>(dst + q * pitch) + c,
               __ldcs(reinterpret_cast<const ulonglong2 *>(src + from * pitch) + c));
    }
}
} // namespace

void launch_unpermute_frame_rows(const uint64_t *src, uint64_t *dst, uint64_t pitch, uint64_t n,
                                 const uint32_t *d_perm, int num_sms, cudaStream_t st) {
    if (n == 0) return;
    k_unpermute_rows<<<unsigned(num_sms * 8), 512, 0, st>>>(src, dst, pitch, n, n, d_perm);
    QSR_CUDA(cudaGetLastError());
    count_launch();
}

void launch_unpermute_rows(DeviceTableau &t, const uint32_t *d_perm) {
    for (int plane = 0; plane < 2; ++plane) {
        k_unpermute_rows<<<unsigned(t.num_sms * 8), 512, 0, t.stream>>>(plane ? t.z : t.x, plane ? t.z2 : t.x2,
                                                                       t.cm_pitch, t.n, t.n_pad, d_perm);
        QSR_CUDA(cudaGetLastError());
        count_launch();
    }
    std::swap(t.x, t.x2);
    std::swap(t.z, t.z2);
}

} // namespace qsr
