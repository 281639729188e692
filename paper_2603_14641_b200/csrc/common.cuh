// Device helpers shared by the sm_100a kernels: Philox-4x32-10, packed gates, the word-level
// Clifford rules and the Pauli-product phase counter.
#pragma once

#include <cstdint>

namespace qsr {

__device__ __forceinline__ uint64_t d_philox_word(uint64_t seed, uint32_t stream, uint32_t ctx,
                                                  uint64_t index) {
    // Philox-4x32-10, counter {stream, ctx, idx_lo, idx_hi}, key {seed_lo, seed_hi}
    // (reference rng.hpp:34-55).
    uint32_t c0 = stream, c1 = ctx, c2 = uint32_t(index), c3 = uint32_t(index >> 32);
    uint32_t k0 = uint32_t(seed), k1 = uint32_t(seed >> 32);
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
        uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
        c0 = hi1 ^ c1 ^ k0;
        c1 = lo1;
        c2 = hi0 ^ c3 ^ k1;
        c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return (uint64_t(c1) << 32) | c0;
}

// Measurement coin number idx of the run: Philox(seed, kStreamMeasure, 0, idx) & 1
// (measure.hpp:427, simulator.hpp:51), or bit 0 of a caller-supplied table (the C++ shim draws
// the coins from the caller's own RandomStream, whatever its stream / context).
__device__ __forceinline__ uint32_t draw_coin(uint64_t seed, uint64_t idx, const uint8_t *table) {
    return table ? uint32_t(table[idx] & 1u) : uint32_t(d_philox_word(seed, 0, 0, idx) & 1u);
}

enum : uint32_t { K_X = 0, K_Y, K_Z, K_H, K_S, K_SDG, K_CX, K_CY, K_CZ, K_SWAP, K_ISWAP };

enum : uint32_t { K_C1 = 11, K_ISWAP_R = 12 }; // device-only kinds (host.hpp, fuse.cpp)

// Packed gate word (host.hpp): q0 [0,24) kind [24,28) pre0 [28,33) pre1 [33,38) q1 [38,62).
__device__ __forceinline__ uint32_t gate_q0(uint64_t g) { return uint32_t(g) & 0xFFFFFFu; }
__device__ __forceinline__ uint32_t gate_kind(uint64_t g) { return (uint32_t(g) >> 24) & 0xF; }
__device__ __forceinline__ uint32_t gate_pre0(uint64_t g) { return uint32_t(g >> 28) & 31u; }
__device__ __forceinline__ uint32_t gate_pre1(uint64_t g) { return uint32_t(g >> 33) & 31u; }
__device__ __forceinline__ uint32_t gate_q1(uint64_t g) { return uint32_t(g >> 38) & 0xFFFFFFu; }

// The 24 single-qubit Cliffords (fuse.hpp): bits 0-3 = GF(2) matrix m00 m01 m10 m11 acting on
// (x, z) (x' = m00 x ^ m01 z, z' = m10 x ^ m11 z), bits 4-6 = sign flip of the images of X, Z, Y.
// Element 0 is the identity; 0-3 are the Paulis (matrix = identity, code 9).
__device__ __constant__ const uint8_t kCliff1[24] = {9,   105, 57,  89, 70, 77, 29, 38,
                                                     45,  125, 118, 22, 14, 110, 87, 7,
                                                     55,  103, 62,  94, 43, 75, 123, 27};
// Words an element rewrites (x and z) unless its matrix is the identity.
__device__ __forceinline__ bool cliff1_moves(uint32_t e) { return (kCliff1[e] & 0xFu) != 9u; }

// Operand words a packed gate reads / writes, pre-operations included: bit0 x0, bit1 z0,
// bit2 x1, bit3 z1.
// Operand words each kind reads / writes: bit0 x0, bit1 z0, bit2 x1, bit3 z1
// (reference gates.hpp:35-115; X/Y/Z only contribute signs).
__device__ __forceinline__ uint32_t kind_reads(uint32_t kind, bool signs) {
    switch (kind) {
    case K_X: return signs ? 0x2u : 0u;
    case K_Y: return signs ? 0x3u : 0u;
    case K_Z: return signs ? 0x1u : 0u;
    case K_H: return 0x3u;
    case K_S:
    case K_SDG: return 0x3u;
    case K_SWAP: return 0xFu;
    case K_C1: return 0x3u;
    default: return 0xFu; // CX CY CZ ISWAP ISWAP_R
    }
}
__device__ __forceinline__ uint32_t kind_writes(uint32_t kind) {
    switch (kind) {
    case K_H: return 0x3u;
    case K_S:
    case K_SDG: return 0x2u;
    case K_CX: return 0x6u;  // x1, z0
    case K_CZ: return 0xAu;  // z0, z1
    case K_CY: return 0xEu;  // z0, x1, z1
    case K_SWAP:
    case K_ISWAP: return 0xFu;
    case K_ISWAP_R: return 0xAu; // z0, z1
    default: return 0u;          // X Y Z; K_C1 decided by its element (gate_writes)
    }
}

__device__ __forceinline__ uint32_t gate_reads(uint64_t g, bool signs) {
    const uint32_t k = gate_kind(g);
    uint32_t r = kind_reads(k, signs);
    if (gate_pre0(g)) r |= 0x3u;
    if (gate_pre1(g)) r |= 0xCu;
    return r;
}
__device__ __forceinline__ uint32_t gate_writes(uint64_t g) {
    uint32_t w = kind_writes(gate_kind(g));
    if (gate_pre0(g) && cliff1_moves(gate_pre0(g))) w |= 0x3u;
    if (gate_pre1(g) && cliff1_moves(gate_pre1(g))) w |= 0xCu;
    return w;
}

// (plus - minus) contribution of control*target for one word (tableau.hpp:336-342). Only
// the value mod 4 is ever used, so a 32-bit wrap-around sum is exact.
__device__ __forceinline__ int phase_delta(uint64_t xc, uint64_t zc, uint64_t xt, uint64_t zt) {
    uint64_t p = (~xc & zc & xt & ~zt) | (xc & zc & ~xt & zt) | (xc & ~zc & xt & zt);
    uint64_t m = (~xc & zc & xt & zt) | (xc & zc & xt & ~zt) | (xc & ~zc & ~xt & zt);
    return __popcll(p) - __popcll(m);
}

__device__ __forceinline__ int warp_sum(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

} // namespace qsr
