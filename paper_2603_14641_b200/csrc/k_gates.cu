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
    case K_ISWAP: {
        V2 t = x0; x0 = x1; x1 = t; t = z0; z0 = z1; z1 = t;
        V2 s2 = x0 & x1 & (z0 ^ z1);
        V2 zt = z1 ^ x0;
        V2 zc = z0 ^ x1;
        V2 s3 = x1 & zt;
        V2 s4 = x0 & zc;
        sign = s2 ^ s3 ^ s4;
        z1 = zt ^ x1; z0 = zc ^ x0;
        break;
    }
    default: break;
    }
    return sign;
}

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kTileWords = 64;

template <bool kSigns, int U, int kMinBlocks>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
k_gate_window(uint64_t *__restrict__ x, uint64_t *__restrict__ z, uint64_t pitch,
              const uint64_t *__restrict__ gates, uint32_t ngates, uint32_t chunk,
              uint64_t *__restrict__ partials, uint32_t *__restrict__ counters,
              uint64_t *__restrict__ s) {
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t j = uint64_t(blockIdx.x) * kTileWords + lane * 2;
    const bool active = j < pitch; // pitch % 16 == 0, so j+1 < pitch too
    const uint32_t g_begin = blockIdx.y * chunk;
    const uint32_t g_end = min(g_begin + chunk, ngates);
    V2 sacc{0, 0};

    if (active) {
        uint32_t g = g_begin + warp;
        for (; g + kWarps * (U - 1) < g_end; g += kWarps * U) {
            uint32_t kind[U], rd[U], wr[U];
            uint64_t o0[U], o1[U];
            V2 X0[U], Z0[U], X1[U], Z1[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                uint64_t gw = __ldg(gates + g + kWarps * u);
                kind[u] = gate_kind(gw);
                rd[u] = kind_reads(kind[u], kSigns);
                wr[u] = kind_writes(kind[u]);
                o0[u] = uint64_t(gate_q0(gw)) * pitch + j;
                o1[u] = uint64_t(gate_q1(gw)) * pitch + j;
                X0[u] = Z0[u] = X1[u] = Z1[u] = V2{0, 0};
                if (rd[u] & 1) X0[u] = ld2(x + o0[u]);
                if (rd[u] & 2) Z0[u] = ld2(z + o0[u]);
                if (rd[u] & 4) X1[u] = ld2(x + o1[u]);
                if (rd[u] & 8) Z1[u] = ld2(z + o1[u]);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                V2 sg = rule2(kind[u], X0[u], Z0[u], X1[u], Z1[u]);
                if (kSigns) sacc ^= sg;
                if (wr[u] & 1) st2(x + o0[u], X0[u]);
                if (wr[u] & 2) st2(z + o0[u], Z0[u]);
                if (wr[u] & 4) st2(x + o1[u], X1[u]);
                if (wr[u] & 8) st2(z + o1[u], Z1[u]);
            }
        }
        for (; g < g_end; g += kWarps) {
            uint64_t gw = __ldg(gates + g);
            uint32_t kd = gate_kind(gw), rd = kind_reads(kd, kSigns), wr = kind_writes(kd);
            uint64_t a0 = uint64_t(gate_q0(gw)) * pitch + j, a1 = uint64_t(gate_q1(gw)) * pitch + j;
            V2 X0{0, 0}, Z0{0, 0}, X1{0, 0}, Z1{0, 0};
            if (rd & 1) X0 = ld2(x + a0);
            if (rd & 2) Z0 = ld2(z + a0);
            if (rd & 4) X1 = ld2(x + a1);
            if (rd & 8) Z1 = ld2(z + a1);
            V2 sg = rule2(kd, X0, Z0, X1, Z1);
            if (kSigns) sacc ^= sg;
            if (wr & 1) st2(x + a0, X0);
            if (wr & 2) st2(z + a0, Z0);
            if (wr & 4) st2(x + a1, X1);
            if (wr & 8) st2(z + a1, Z1);
        }
    }

    if constexpr (kSigns) {
        // Shared-memory XOR tree over the 8 warps (the reference's collapse_signs /
        // reduce_xor, bitplane.hpp:96-122, done per CTA).
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
}

// Kernel variants (unroll U, min resident CTAs): 0 = <2,3>, 1 = <1,4>, 2 = <2,4>.
// QSR_GATE_VARIANT selects one for tuning runs; the default is the measured best
// (profiles/r01_gate_tune.log: <2,3> 6.37 TB/s at c5, <1,4> 6.31, <2,4> 6.07 with spills).
int gate_variant() {
    static int v = [] {
        const char *e = getenv("QSR_GATE_VARIANT");
        return e ? atoi(e) : 0;
    }();
    return v;
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
    const uint64_t tiles = (pitch + kTileWords - 1) / kTileWords;
    const uint64_t slots = uint64_t(num_sms) * uint64_t(bps);
    // Every CTA does the same work, so the grid should be a whole number of waves: pick the
    // chunk count (>= ~4 waves when the window is big enough) whose tiles x chunks leaves the
    // smallest partial last wave. At least 16 gates per warp per chunk keep the XOR tree and
    // the tile fold negligible.
    const uint64_t max_chunks = std::max<uint64_t>(1, ngates / (kWarps * 16));
    uint64_t c_min = std::max<uint64_t>(1, (4 * slots + tiles - 1) / tiles);
    if (c_min > max_chunks) c_min = max_chunks;
    uint64_t chunks = c_min;
    double best = 1e30;
    for (uint64_t c = c_min; c <= std::min<uint64_t>(max_chunks, 4 * c_min); ++c) {
        const uint64_t ctas = tiles * c;
        const uint64_t waves = (ctas + slots - 1) / slots;
        const double eff_time = double(waves) / double(c); // per-CTA work ~ 1/c
        if (eff_time < best * 0.999) { best = eff_time; chunks = c; }
    }
    if (chunks > 65535) chunks = 65535;
    uint64_t chunk = (ngates + chunks - 1) / chunks;
    chunks = (ngates + chunk - 1) / chunk;
    if (kSigns && chunks > 1 && chunks > *partial_chunks) {
        if (*partials)
            QSR_CUDA(cudaFree(*partials));
        QSR_CUDA(cudaMalloc(partials, chunks * pitch * sizeof(uint64_t)));
        *partial_chunks = chunks;
    }
    dim3 grid{unsigned(tiles), unsigned(chunks)};
    k_gate_window<kSigns, U, B><<<grid, kThreads, 0, st>>>(
        x, z, pitch, gates, uint32_t(ngates), uint32_t(chunk), kSigns ? *partials : nullptr,
        counters, s);
    QSR_CUDA(cudaGetLastError());
    count_launch();
}

template <bool kSigns>
void launch(uint64_t *x, uint64_t *z, uint64_t pitch, const uint64_t *gates, uint64_t ngates,
            int num_sms, cudaStream_t st, uint64_t **partials, uint64_t *partial_chunks,
            uint32_t *counters, uint64_t *s) {
    if (ngates == 0)
        return;
    switch (gate_variant()) {
    case 0:
        launch_variant<kSigns, 2, 3>(x, z, pitch, gates, ngates, num_sms, st, partials,
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
