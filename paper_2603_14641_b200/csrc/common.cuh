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

__device__ __forceinline__ uint32_t gate_q0(uint64_t g) { return uint32_t(g) & 0x0FFFFFFFu; }
__device__ __forceinline__ uint32_t gate_kind(uint64_t g) { return (uint32_t(g) >> 28) & 0xF; }
__device__ __forceinline__ uint32_t gate_q1(uint64_t g) { return uint32_t(g >> 32); }

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
    default: return 0xFu; // CX CY CZ ISWAP
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
    default: return 0u;
    }
}

// One word of the column update rules; returns the sign-flip word. Operand 0 = control.
// Restates the frozen conjugation table of gates.hpp:35-115.
__device__ __forceinline__ uint64_t apply_rule(uint32_t kind, uint64_t &x0, uint64_t &z0,
                                               uint64_t &x1, uint64_t &z1) {
    uint64_t sign = 0;
    switch (kind) {
    case K_H: {
        sign = x0 & z0;
        uint64_t t = x0; x0 = z0; z0 = t;
        break;
    }
    case K_S: sign = x0 & z0; z0 ^= x0; break;
    case K_SDG: sign = x0 & ~z0; z0 ^= x0; break;
    case K_X: sign = z0; break;
    case K_Y: sign = x0 ^ z0; break;
    case K_Z: sign = x0; break;
    case K_CX:
        sign = x0 & z1 & ~(x1 ^ z0);
        x1 ^= x0;
        z0 ^= z1;
        break;
    case K_CZ:
        sign = x0 & x1 & (z0 ^ z1);
        z1 ^= x0;
        z0 ^= x1;
        break;
    case K_CY: {
        uint64_t s1 = x1 & ~z1;
        uint64_t zt = z1 ^ x1;
        uint64_t s2 = x0 & zt & ~(x1 ^ z0);
        uint64_t xt = x1 ^ x0;
        uint64_t zc = z0 ^ zt;
        uint64_t s3 = xt & zt;
        sign = s1 ^ s2 ^ s3;
        x1 = xt;
        z0 = zc;
        z1 = zt ^ xt;
        break;
    }
    case K_SWAP: {
        uint64_t t = x0; x0 = x1; x1 = t;
        t = z0; z0 = z1; z1 = t;
        break;
    }
    case K_ISWAP: {
        uint64_t t = x0; x0 = x1; x1 = t;
        t = z0; z0 = z1; z1 = t;
        uint64_t s2 = x0 & x1 & (z0 ^ z1);
        uint64_t zt = z1 ^ x0;
        uint64_t zc = z0 ^ x1;
        uint64_t s3 = x1 & zt;
        uint64_t s4 = x0 & zc;
        sign = s2 ^ s3 ^ s4;
        z1 = zt ^ x1;
        z0 = zc ^ x0;
        break;
    }
    default: break;
    }
    return sign;
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
