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
// Default: <1,4> for windows of >= 16k gates (fused c5 windows, ~45k gates: 216.7 vs 226.2 ms per
// 100 windows at 180k qubits,
// no spills at 64 registers), <2,3> for small ones (20k qubits: 10.5 vs 11.1 ms per 300).
int gate_variant(uint64_t ngates) {
    static int v = [] {
        const char *e = getenv("QSR_GATE_VARIANT");
        return e ? atoi(e) : -1;
    }();
    if (v >= 0) return v;
    return ngates >= (uint64_t(1) << 14) ? 1 : 0;
}

// Grid of a window launch: tiles x chunks CTAs. Every CTA does the same work, so the grid should
// be a whole number of waves: pick the chunk count (>= ~4 waves when the window is big enough)
// whose tiles x chunks leaves the smallest partial last wave. At least 16 items per warp per
// chunk keep the XOR tree and the tile fold negligible. Grows the sign partials as needed.
void pick_chunks(uint64_t pitch, uint64_t nitems, int num_sms, int bps, bool signs, uint64_t **partials,
                 uint64_t *partial_chunks, uint64_t *tiles_out, uint64_t *chunk_out, uint64_t *chunks_out) {
    const uint64_t tiles = (pitch + kTileWords - 1) / kTileWords;
    const uint64_t slots = uint64_t(num_sms) * uint64_t(bps);
    static const uint64_t per_warp = [] { // QSR_GATE_MINPW: tuning knob (default 16)
        const char *e = getenv("QSR_GATE_MINPW");
        return e ? std::max<uint64_t>(1, uint64_t(atoll(e))) : uint64_t(16);
    }();
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
        if (*partials) cache_release(dev, *partial_chunks * pitch * sizeof(uint64_t), *partials);
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
    pick_chunks(pitch, ngates, num_sms, bps, kSigns, partials, partial_chunks, &tiles, &chunk, &chunks);
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


// ---- K1p: two consecutive windows as components ------------------------------------------
// Two consecutive unitary windows A, B are each a matching on the qubit rows, so their union
// splits into small paths and cycles. A component of <= kPairRows rows and <= kPairGates gates
// is one record (pair.hpp): its rows are loaded once, A's gates then B's gates are applied, and
// the rows are stored once — a row touched by both windows moves once instead of twice. The
// rows of the component live in the warp's slice of shared memory (lane-private 16-byte slots,
// conflict-free), so the record's local operand indices are plain shared-memory addresses.
// Same tile / chunk / sign-fold structure as k_gate_window.
constexpr int kPairSmemV2 = kWarps * 2 * kPairRows * 2 * 32; // two record buffers per warp
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned sa = unsigned(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
constexpr size_t kPairSmemBytes = size_t(kPairSmemV2) * sizeof(V2);

template <bool kSigns, int kMinBlocks>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
k_gate_pairs(uint64_t *__restrict__ x, uint64_t *__restrict__ z, uint64_t pitch,
             const uint64_t *__restrict__ recs, uint32_t nrec, uint32_t chunk,
             uint64_t *__restrict__ partials, uint32_t *__restrict__ counters,
             uint64_t *__restrict__ s) {
    extern __shared__ V2 pair_smem[];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // Two record buffers per warp: the next record's rows load while this one is computed.
    V2 *const buf0 = pair_smem + warp * (2 * kPairRows * 2 * 32) + lane; // [(row * 2 + plane) * 32]
    V2 *const buf1 = buf0 + kPairRows * 2 * 32;
    const uint64_t j = uint64_t(blockIdx.x) * kTileWords + lane * 2;
    const bool active = j < pitch;
    const uint32_t c_begin = blockIdx.y * chunk;
    const uint32_t c_end = min(c_begin + chunk, nrec);
    V2 sacc{0, 0};
    // Lane l < 16 holds word l of a record (one coalesced 128-byte load); fields are shuffled
    // out on demand.
    auto fetch = [&](uint32_t cc) -> uint64_t {
        return (cc < c_end && lane < uint32_t(kPairRecWords)) ? __ldg(recs + uint64_t(cc) * kPairRecWords + lane) : 0;
    };
    auto offsets = [&](uint64_t rec, uint64_t (&off)[kPairRows]) {
#pragma unroll
        for (int k = 0; k < (kPairRows + 1) / 2; ++k) {
            const uint64_t rw = __shfl_sync(0xFFFFFFFFu, rec, 1 + k);
            off[2 * k] = uint64_t(uint32_t(rw)) * uint32_t(pitch) + j;
            if (2 * k + 1 < kPairRows) off[2 * k + 1] = uint64_t(uint32_t(rw >> 32)) * uint32_t(pitch) + j;
        }
    };
    auto issue = [&](uint64_t rec, V2 *buf) { // the record's read planes -> buf (cp.async)
        const uint32_t rmask = uint32_t(__shfl_sync(0xFFFFFFFFu, rec, 0) >> 8) & 0xFFFFu;
        uint64_t off[kPairRows];
        offsets(rec, off);
        if (active) {
#pragma unroll
            for (int i = 0; i < kPairRows; ++i) {
                if ((rmask >> (2 * i)) & 1u) cp_async16(buf + (2 * i) * 32, x + off[i]);
                if ((rmask >> (2 * i + 1)) & 1u) cp_async16(buf + (2 * i + 1) * 32, z + off[i]);
            }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    uint32_t c = c_begin + warp;
    uint64_t cur = fetch(c), nxt = fetch(c + kWarps);
    if (c < c_end) issue(cur, buf0);
    for (uint32_t it = 0; c < c_end; c += kWarps, ++it) {
        V2 *const b = (it & 1) ? buf1 : buf0;
        const uint64_t nn = fetch(c + 2 * kWarps);
        if (c + kWarps < c_end) issue(nxt, (it & 1) ? buf0 : buf1);
        else asm volatile("cp.async.commit_group;\n" ::: "memory");
        asm volatile("cp.async.wait_group 1;\n" ::: "memory"); // this record's group is complete
        const uint64_t hdr = __shfl_sync(0xFFFFFFFFu, cur, 0);
        const uint32_t ng = uint32_t(hdr >> 4) & 15u, wmask = uint32_t(hdr >> 24) & 0xFFFFu;
        for (uint32_t gi = 0; gi < ng; ++gi) {
            const uint64_t gw = __shfl_sync(0xFFFFFFFFu, cur, 5 + gi);
            const uint32_t a = gate_q0(gw), bq = gate_q1(gw), rd = gate_reads(gw, kSigns), wr = gate_writes(gw);
            V2 X0{0, 0}, Z0{0, 0}, X1{0, 0}, Z1{0, 0};
            if (rd & 1u) X0 = b[(a * 2) * 32];
            if (rd & 2u) Z0 = b[(a * 2 + 1) * 32];
            if (rd & 4u) X1 = b[(bq * 2) * 32];
            if (rd & 8u) Z1 = b[(bq * 2 + 1) * 32];
            const V2 sg = gate2(gw, X0, Z0, X1, Z1);
            if (kSigns) sacc ^= sg;
            if (wr & 1u) b[(a * 2) * 32] = X0;
            if (wr & 2u) b[(a * 2 + 1) * 32] = Z0;
            if (wr & 4u) b[(bq * 2) * 32] = X1;
            if (wr & 8u) b[(bq * 2 + 1) * 32] = Z1;
        }
        uint64_t off[kPairRows];
        offsets(cur, off); // all lanes (the shuffles need the full warp)
        if (active) {
#pragma unroll
            for (int i = 0; i < kPairRows; ++i) {
                if ((wmask >> (2 * i)) & 1u) st2(x + off[i], b[(2 * i) * 32]);
                if ((wmask >> (2 * i + 1)) & 1u) st2(z + off[i], b[(2 * i + 1) * 32]);
            }
        }
        cur = nxt;
        nxt = nn;
    }
    if constexpr (kSigns) fold_tile_signs(sacc, warp, lane, j, active, pitch, partials, counters, s);
}

template <bool kSigns>
void launch_pairs(uint64_t *x, uint64_t *z, uint64_t pitch, const uint64_t *recs, uint64_t nrec, int num_sms,
                  cudaStream_t st, uint64_t **partials, uint64_t *partial_chunks, uint32_t *counters,
                  uint64_t *s) {
    if (nrec == 0) return;
    constexpr int B = 2;
    static int bps = 0;
    if (bps == 0) {
        QSR_CUDA(cudaFuncSetAttribute(k_gate_pairs<kSigns, B>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(kPairSmemBytes)));
        QSR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_gate_pairs<kSigns, B>, kThreads,
                                                               kPairSmemBytes));
        if (bps < 1) bps = 1;
    }
    uint64_t tiles, chunk, chunks;
    pick_chunks(pitch, nrec, num_sms, bps, kSigns, partials, partial_chunks, &tiles, &chunk, &chunks);
    dim3 grid{unsigned(tiles), unsigned(chunks)};
    k_gate_pairs<kSigns, B><<<grid, kThreads, kPairSmemBytes, st>>>(x, z, pitch, recs, uint32_t(nrec), uint32_t(chunk),
                                                       kSigns ? *partials : nullptr, counters, s);
    QSR_CUDA(cudaGetLastError());
    count_launch();
}


// ---- K1b: temporally blocked gate segment ------------------------------------------------
// All windows of a unitary segment in ONE persistent cooperative launch. The CM planes are
// cut into sub-slabs of 16 generator-words (one 128-byte line per qubit row and plane); a step
// processes one window on m consecutive sub-slabs, so the step's working set (m x n_pad x
// 256 B, <= ~40 MB) stays resident in L2 across all windows of the segment while the gate
// list streams through with evict-first loads. Generator-words are independent across windows
// (gates.hpp:173-194), so only window order matters inside a slab group: a grid barrier
// separates consecutive windows. Measured on B200: random 128-byte line read-modify-write runs
// at ~16 TB/s from L2 vs ~4.3 TB/s from HBM (tools/l2_rmw_probe.cu).
// An 8-lane group applies one gate to one sub-slab (lane = 2 words); groups are split into m
// classes, class c always works on sub-slab c of the current group, so each lane's sign words
// stay in registers for the whole segment pass and are folded once (shared-memory XOR, then one
// global atomic per word per CTA).
constexpr int kSegThreads = 512;
constexpr int kSegGroups = kSegThreads / 8;  // 8-lane groups per CTA
constexpr int kSegMaxM = 64;
constexpr int kSegGateBuf = 2048;            // gates per CTA chunk held in shared memory

struct SegArgs {
    uint64_t *x, *z;
    uint64_t pitch;       // row stride in words (16 in the slab-major layout)
    uint64_t sub_stride;  // words between consecutive sub-slabs (n_pad * 16 slab-major)
    const uint64_t *gates;
    const uint64_t *woff; // window offsets into gates, nwin + 1 (device)
    uint32_t nwin;
    uint32_t nsub;        // pitch / 16
    uint32_t m;           // sub-slabs per step (power of two <= 64)
    uint64_t *s;          // signs (kSigns)
    unsigned int *bar;    // grid barrier counter, zero at launch
};

// Sense-reversal grid barrier: arrivals on bar[0]; the last arriver resets it and bumps the
// generation word bar[32] (its own 128-byte line), which the other CTAs poll with back-off, so
// polling never contends with the arrivals' atomics. acq_rel arrivals + release/acquire on the
// generation make every CTA's writes of the step visible to every CTA after the barrier.
__device__ __forceinline__ void grid_barrier(unsigned int *bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int gen, old;
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(gen) : "l"(bar + 32) : "memory");
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
        if (old == gridDim.x - 1) {
            asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(bar) : "memory");
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(bar + 32), "r"(gen + 1) : "memory");
        } else {
            unsigned int v;
            do {
                asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar + 32) : "memory");
            } while (v == gen);
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
    }
    __syncthreads();
}

__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
    const unsigned sa = unsigned(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}

// This CTA's share of window w: gates c0, c0 + NB, c0 + 2NB, ... (cnt of them), NB = gridDim.x.
__device__ __forceinline__ void seg_chunk(const uint64_t *woff, uint32_t w, uint64_t &c0, uint64_t &cnt) {
    const uint64_t g0 = woff[w], n = woff[w + 1] - g0;
    c0 = g0 + blockIdx.x;
    cnt = blockIdx.x < n ? (n - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
}

__device__ __forceinline__ void seg_prefetch(uint64_t *buf, const uint64_t *gates, uint64_t c0,
                                             uint64_t cnt) {
    const uint64_t n = min(cnt, uint64_t(kSegGateBuf));
    for (uint64_t e = threadIdx.x; e < n; e += kSegThreads) cp_async8(buf + e, gates + c0 + e * gridDim.x);
    asm volatile("cp.async.commit_group;\n" ::);
}

template <bool kSigns>
__device__ __forceinline__ void seg_gate(const SegArgs &a, uint64_t gw, uint64_t j, V2 &sacc) {
    const uint32_t rd = gate_reads(gw, kSigns), wr = gate_writes(gw);
    const uint64_t a0 = uint64_t(gate_q0(gw)) * a.pitch + j, a1 = uint64_t(gate_q1(gw)) * a.pitch + j;
    V2 X0{0, 0}, Z0{0, 0}, X1{0, 0}, Z1{0, 0};
    if (rd & 1) X0 = ld2(a.x + a0);
    if (rd & 2) Z0 = ld2(a.z + a0);
    if (rd & 4) X1 = ld2(a.x + a1);
    if (rd & 8) Z1 = ld2(a.z + a1);
    const V2 sg2 = gate2(gw, X0, Z0, X1, Z1);
    if (kSigns) sacc ^= sg2;
    if (wr & 1) st2(a.x + a0, X0);
    if (wr & 2) st2(a.z + a0, Z0);
    if (wr & 4) st2(a.x + a1, X1);
    if (wr & 8) st2(a.z + a1, Z1);
}

template <bool kSigns, int kSegU, int kMinB>
__global__ void __launch_bounds__(kSegThreads, kMinB) k_gate_segment(SegArgs a) {
    __shared__ uint64_t s_sign[kSegMaxM][16];
    __shared__ __align__(16) uint64_t gbuf[2][kSegGateBuf];
    const uint32_t tid = threadIdx.x, l8 = tid & 7, grp = tid >> 3;
    const uint32_t m = a.m, cls = grp % m, gi = grp / m, gstride = kSegGroups / m;
    const uint32_t nsg = (a.nsub + m - 1) / m;
    const uint64_t pitch = a.pitch;
    int cur = 0;
    uint64_t c0, c1;
    seg_chunk(a.woff, 0, c0, c1);
    seg_prefetch(gbuf[0], a.gates, c0, c1);
    for (uint32_t sg = 0; sg < nsg; ++sg) {
        const uint32_t sub = sg * m + cls;
        const bool act = sub < a.nsub;
        const uint64_t j = uint64_t(sub) * a.sub_stride + 2 * l8; // word offset within a row
        V2 sacc{0, 0};
        if (kSigns)
            for (uint32_t e = tid; e < m * 16; e += kSegThreads) s_sign[e / 16][e % 16] = 0;
        for (uint32_t w = 0; w < a.nwin; ++w) {
            // Gates of this step were prefetched during the previous one; start the next.
            asm volatile("cp.async.wait_group 0;\n" ::);
            __syncthreads();
            const uint64_t n0 = c0, ncnt = c1;
            const bool last = (w + 1 == a.nwin) && (sg + 1 == nsg);
            if (!last) {
                seg_chunk(a.woff, w + 1 == a.nwin ? 0 : w + 1, c0, c1);
                seg_prefetch(gbuf[cur ^ 1], a.gates, c0, c1);
            }
            const uint64_t *gb = gbuf[cur];
            const uint64_t nb = min(ncnt, uint64_t(kSegGateBuf));
            if (act) {
                uint64_t t = gi;
                for (; t + uint64_t(gstride) * (kSegU - 1) < nb; t += uint64_t(gstride) * kSegU) {
                    uint64_t gws[kSegU];
                    uint32_t wr[kSegU];
                    uint64_t o0[kSegU], o1[kSegU];
                    V2 X0[kSegU], Z0[kSegU], X1[kSegU], Z1[kSegU];
#pragma unroll
                    for (int u = 0; u < kSegU; ++u) {
                        const uint64_t gw = gws[u] = gb[t + uint64_t(gstride) * u];
                        const uint32_t rd = gate_reads(gw, kSigns);
                        wr[u] = gate_writes(gw);
                        o0[u] = uint64_t(gate_q0(gw)) * pitch + j;
                        o1[u] = uint64_t(gate_q1(gw)) * pitch + j;
                        X0[u] = Z0[u] = X1[u] = Z1[u] = V2{0, 0};
                        if (rd & 1) X0[u] = ld2(a.x + o0[u]);
                        if (rd & 2) Z0[u] = ld2(a.z + o0[u]);
                        if (rd & 4) X1[u] = ld2(a.x + o1[u]);
                        if (rd & 8) Z1[u] = ld2(a.z + o1[u]);
                    }
#pragma unroll
                    for (int u = 0; u < kSegU; ++u) {
                        const V2 sg2 = gate2(gws[u], X0[u], Z0[u], X1[u], Z1[u]);
                        if (kSigns) sacc ^= sg2;
                        if (wr[u] & 1) st2(a.x + o0[u], X0[u]);
                        if (wr[u] & 2) st2(a.z + o0[u], Z0[u]);
                        if (wr[u] & 4) st2(a.x + o1[u], X1[u]);
                        if (wr[u] & 8) st2(a.z + o1[u], Z1[u]);
                    }
                }
                for (; t < nb; t += gstride) seg_gate<kSigns>(a, gb[t], j, sacc);
                // Chunks larger than the buffer (windows > kSegGateBuf * CTAs gates): the rest
                // straight from global memory.
                for (uint64_t t2 = kSegGateBuf + gi; t2 < ncnt; t2 += gstride)
                    seg_gate<kSigns>(a, __ldcs(a.gates + n0 + t2 * gridDim.x), j, sacc);
            }
            cur ^= 1;
            grid_barrier(a.bar);
        }
        if (kSigns) {
            // Fold this pass's sign words: lanes -> shared (per class), CTA -> global.
            if (act) {
                if (sacc.a) atomicXor(reinterpret_cast<unsigned long long *>(&s_sign[cls][2 * l8]), sacc.a);
                if (sacc.b) atomicXor(reinterpret_cast<unsigned long long *>(&s_sign[cls][2 * l8 + 1]), sacc.b);
            }
            __syncthreads();
            for (uint32_t e = tid; e < m * 16; e += kSegThreads) {
                const uint32_t sb = sg * m + e / 16;
                const uint64_t v = s_sign[e / 16][e % 16];
                if (sb < a.nsub && v)
                    atomicXor(reinterpret_cast<unsigned long long *>(a.s + uint64_t(sb) * 16 + e % 16), v);
            }
            __syncthreads();
        }
    }
}

// Opt-in (QSR_GATE_ENGINE=segment). Measured on B200: per-window launches win
// or tie at every width tried (n = 10k..180k); the per-window barrier plus ramp / drain of each
// step costs more than the L2-over-HBM bandwidth advantage of the resident slab.
bool segment_enabled() {
    static bool on = [] {
        const char *e = getenv("QSR_GATE_ENGINE");
        return e && std::string(e) == "segment";
    }();
    return on;
}

// Row-major planes (row q at q * pitch) <-> slab-major (sub-slab s of every row contiguous:
// word (q, 16s + w) at (s * rows + q) * 16 + w). One 16-byte chunk per thread, both sides
// coalesced in 128-byte lines. The segment kernel runs on the slab-major copy: a step's slab is
// then a few contiguous tens of MB (a handful of 2 MB pages) instead of 180k lines spread over
// the whole 8 GB plane, which costs a TLB miss per access (tools/l2_rmw_probe.cu: 16.8 TB/s
// contiguous vs 5.1 TB/s at the c5 row pitch).
template <bool kToSlab>
__global__ void k_slab_permute(const uint64_t *__restrict__ src, uint64_t *__restrict__ dst,
                               uint64_t pitch, uint64_t rows, uint64_t nsub) {
    const uint64_t total = nsub * rows * 8; // 16-byte chunks
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t c = e & 7, line = e >> 3;       // line = s * rows + q (slab-major order)
        const uint64_t sidx = line / rows, q = line - sidx * rows;
        const uint64_t rm = q * pitch + sidx * 16 + 2 * c, sm = line * 16 + 2 * c;
        const uint64_t from = kToSlab ? rm : sm, to = kToSlab ? sm : rm;
        __stcs(reinterpret_cast<ulonglong2 *>(dst + to), __ldcs(reinterpret_cast<const ulonglong2 *>(src + from)));
    }
}

void slab_permute(const uint64_t *src, uint64_t *dst, uint64_t pitch, uint64_t rows, bool to_slab,
                  int num_sms, cudaStream_t st) {
    const unsigned blocks = unsigned(num_sms * 8), threads = 512;
    if (to_slab)
        k_slab_permute<true><<<blocks, threads, 0, st>>>(src, dst, pitch, rows, pitch / 16);
    else
        k_slab_permute<false><<<blocks, threads, 0, st>>>(src, dst, pitch, rows, pitch / 16);
    QSR_CUDA(cudaGetLastError());
    count_launch();
}

template <bool kSigns>
void launch_segment(uint64_t *x, uint64_t *z, uint64_t pitch, uint64_t rows, const uint64_t *gates,
                    const uint64_t *d_woff, uint32_t nwin, int device, int num_sms, cudaStream_t st,
                    unsigned int *bar, uint64_t *s, uint64_t *xs, uint64_t *zs) {
    // Variants (unroll, min CTAs/SM): QSR_SEG_VARIANT 0 = <4,1>, 1 = <2,2>, 2 = <8,1>.
    static const int variant = [] {
        const char *e = getenv("QSR_SEG_VARIANT");
        return e ? atoi(e) : 0;
    }();
    void *fn = variant == 1 ? reinterpret_cast<void *>(k_gate_segment<kSigns, 2, 2>)
             : variant == 2 ? reinterpret_cast<void *>(k_gate_segment<kSigns, 8, 1>)
                            : reinterpret_cast<void *>(k_gate_segment<kSigns, 4, 1>);
    static int bps[2][3] = {{0, 0, 0}, {0, 0, 0}};
    int &b = bps[kSigns ? 1 : 0][variant];
    if (b == 0) {
        QSR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, kSegThreads, 0));
        if (b < 1) fail(QSR_INTERNAL, "k_gate_segment: no resident CTA");
    }
    (void)device;
    SegArgs a;
    a.x = xs; a.z = zs; a.pitch = 16; a.sub_stride = rows * 16;
    a.gates = gates; a.woff = d_woff; a.nwin = nwin;
    a.nsub = uint32_t(pitch / 16);
    // Sub-slabs per step: the step's working set (m x rows x 16 words x 2 planes) <= ~40 MB.
    const uint64_t per_sub = rows * 16 * 16;
    const uint64_t fit = std::max<uint64_t>(1, uint64_t(40e6) / std::max<uint64_t>(per_sub, 1));
    uint64_t m = 1;
    while (m * 2 <= std::min<uint64_t>({fit, uint64_t(a.nsub), uint64_t(kSegMaxM)})) m *= 2;
    a.m = uint32_t(m);
    a.s = s;
    a.bar = bar;
    QSR_CUDA(cudaMemsetAsync(bar, 0, 256, st));
    void *args[] = {&a};
    slab_permute(x, xs, pitch, rows, true, num_sms, st);
    slab_permute(z, zs, pitch, rows, true, num_sms, st);
    QSR_CUDA(cudaLaunchCooperativeKernel(fn, dim3(unsigned(num_sms * b)), dim3(kSegThreads), args, 0, st));
    count_launch();
    slab_permute(xs, x, pitch, rows, false, num_sms, st);
    slab_permute(zs, z, pitch, rows, false, num_sms, st);
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

void launch_gate_pairs(DeviceTableau &t, const uint64_t *recs, uint64_t nrec) {
    launch_pairs<true>(t.x, t.z, t.cm_pitch, recs, nrec, t.num_sms, t.stream, &t.sign_partials,
                       &t.sign_partial_chunks, t.tile_counters, t.s);
}

void launch_frame_pairs(uint64_t *xf, uint64_t *zf, uint64_t pitch, const uint64_t *recs, uint64_t nrec,
                        int num_sms, cudaStream_t st) {
    launch_pairs<false>(xf, zf, pitch, recs, nrec, num_sms, st, nullptr, nullptr, nullptr, nullptr);
}

} // namespace qsr

namespace qsr {

bool gate_segment_enabled() { return segment_enabled(); }

void launch_gate_segment(DeviceTableau &t, const uint64_t *gates, const uint64_t *d_woff,
                         uint32_t nwin) {
    if (!t.seg_bar) t.seg_bar = static_cast<unsigned int *>(cache_acquire(t.device, 256));
    // x2 / z2 (the transpose targets) are free during unitary windows: slab-major copies.
    launch_segment<true>(t.x, t.z, t.cm_pitch, t.n_pad, gates, d_woff, nwin, t.device, t.num_sms,
                         t.stream, t.seg_bar, t.s, t.x2, t.z2);
}

void launch_frame_segment(uint64_t *xf, uint64_t *zf, uint64_t pitch, uint64_t rows,
                          const uint64_t *gates, const uint64_t *d_woff, uint32_t nwin,
                          int num_sms, cudaStream_t st, unsigned int *bar, uint64_t *xs,
                          uint64_t *zs) {
    launch_segment<false>(xf, zf, pitch, rows, gates, d_woff, nwin, 0, num_sms, st, bar, nullptr,
                          xs, zs);
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
