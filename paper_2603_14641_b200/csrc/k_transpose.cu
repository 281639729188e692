// K2+K3 — out-of-place layout transpose CM <-> generator-major RM
// (reference Tableau::transpose_in_place = shuffle_tiles + permute_words,
//  tableau.hpp:166-176, 280-322; bit_transpose_tile bitplane.hpp:165-183).
//
// The reference moves 64x64-bit tiles in place in two passes (bit-transpose every tile,
// then permute words per block-row). Here one pass reads each tile once and writes it once:
// a CTA stages an 8x8 block of tiles (512 source rows x 64 contiguous bytes) in shared
// memory, each warp bit-transposes 8 tiles in registers with the same six masked-swap
// rounds (rounds with offset < 32 via __shfl_xor_sync, offset 32 inside the lane), and the
// CTA writes the block to the destination rows, again as 64-byte contiguous runs.
//
//   CM word (q, J)      at q*cm_pitch + J          bits = generators J*64 + b
//   RM word (r = J*64+t, I) at r*rm_pitch + I      bits = qubits I*64 + c
// Tile (I, J): CM rows I*64..I*64+63, word J  <->  RM rows J*64..J*64+63, word I.
#include <algorithm>

#include "common.cuh"
#include "device.hpp"

namespace qsr {

namespace {

constexpr int TB = 8;             // tiles per CTA edge
constexpr int kTileStride = 65;   // padded tile stride in shared memory (bank spread)
constexpr int kThreads = 256;

__device__ __forceinline__ void tile_transpose_warp(uint64_t &a, uint64_t &b, uint32_t lane) {
    // a = tile word `lane`, b = tile word `lane + 32`.
    const uint64_t masks[6] = {0x5555555555555555ull, 0x3333333333333333ull,
                               0x0F0F0F0F0F0F0F0Full, 0x00FF00FF00FF00FFull,
                               0x0000FFFF0000FFFFull, 0x00000000FFFFFFFFull};
#pragma unroll
    for (int l = 0; l < 5; ++l) {
        const uint32_t o = 1u << l;
        const uint64_t m = masks[l];
        uint64_t ya = __shfl_xor_sync(0xffffffffu, a, o);
        uint64_t yb = __shfl_xor_sync(0xffffffffu, b, o);
        if ((lane & o) == 0) {
            a = (a & m) | ((ya & m) << o);
            b = (b & m) | ((yb & m) << o);
        } else {
            a = ((ya & ~m) >> o) | (a & ~m);
            b = ((yb & ~m) >> o) | (b & ~m);
        }
    }
    const uint64_t m = masks[5];
    uint64_t na = (a & m) | ((b & m) << 32);
    uint64_t nb = ((a & ~m) >> 32) | (b & ~m);
    a = na;
    b = nb;
}

// kToRm: src = CM (rows = qubits, words = generator-words), dst = RM.
// !kToRm: src = RM (rows = generators, words = qubit-words), dst = CM.
// Block (bi, bj): source "row tiles" R0 = bi*TB (row-tile index = I for CM, J for RM) and
// source "word" range W0 = bj*TB.
template <bool kToRm>
__global__ void __launch_bounds__(kThreads)
k_transpose(const uint64_t *__restrict__ src, uint64_t *__restrict__ dst, uint64_t src_pitch,
            uint64_t dst_pitch, uint64_t src_row_tiles, uint64_t src_words) {
    extern __shared__ uint64_t sm[]; // TB*TB tiles * kTileStride
    const uint64_t rt0 = uint64_t(blockIdx.x) * TB; // first source row-tile
    const uint64_t w0 = uint64_t(blockIdx.y) * TB;  // first source word
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    // Load: 512 source rows x TB words.
    for (uint32_t e = tid; e < 64 * TB * TB; e += kThreads) {
        uint32_t row = e / TB, w = e % TB;
        uint64_t grow = rt0 * 64 + row, gw = w0 + w;
        uint64_t v = 0;
        if (rt0 + row / 64 < src_row_tiles && gw < src_words)
            v = __ldcs(src + grow * src_pitch + gw);
        // tile (ti = row/64 [source row-tile], tj = w [source word]) element row%64
        sm[((row / 64) * TB + w) * kTileStride + (row % 64)] = v;
    }
    __syncthreads();
    for (uint32_t tile = warp; tile < TB * TB; tile += kThreads / 32) {
        uint64_t *tp = sm + tile * kTileStride;
        uint64_t a = tp[lane], b = tp[lane + 32];
        tile_transpose_warp(a, b, lane);
        tp[lane] = a;
        tp[lane + 32] = b;
    }
    __syncthreads();
    // Store: destination rows = source words * 64 + t, destination words = source row-tiles.
    for (uint32_t e = tid; e < 64 * TB * TB; e += kThreads) {
        uint32_t row = e / TB, w = e % TB; // row: (source word tj = row/64, t = row%64)
        uint64_t dwrow = (w0 + row / 64) * 64 + (row % 64);
        uint64_t dword = rt0 + w;
        if (w0 + row / 64 < src_words && dword < src_row_tiles)
            __stcs(dst + dwrow * dst_pitch + dword,
                   sm[(w * TB + row / 64) * kTileStride + (row % 64)]);
    }
}

// RM row padding (qubit-words k .. rm_pitch-1) must read as zero for the measurement kernels;
// the RM buffer doubles as slab-major scratch of the gate-segment kernel, so it is re-zeroed.
__global__ void k_zero_rm_padding(uint64_t *__restrict__ x, uint64_t *__restrict__ z, uint64_t pitch,
                                  uint64_t k, uint64_t rows) {
    const uint64_t pad = pitch - k;
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < rows * pad;
         e += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t r = e / pad, w = k + e % pad;
        x[r * pitch + w] = 0;
        z[r * pitch + w] = 0;
    }
}

void run(const uint64_t *src, uint64_t *dst, uint64_t src_pitch, uint64_t dst_pitch,
         uint64_t src_row_tiles, uint64_t src_words, bool to_rm, cudaStream_t st) {
    dim3 grid{unsigned((src_row_tiles + TB - 1) / TB), unsigned((src_words + TB - 1) / TB)};
    size_t smem = size_t(TB) * TB * kTileStride * sizeof(uint64_t);
    if (to_rm)
        k_transpose<true><<<grid, kThreads, smem, st>>>(src, dst, src_pitch, dst_pitch,
                                                        src_row_tiles, src_words);
    else
        k_transpose<false><<<grid, kThreads, smem, st>>>(src, dst, src_pitch, dst_pitch,
                                                         src_row_tiles, src_words);
    QSR_CUDA(cudaGetLastError());
    count_launch();
}

} // namespace

void transpose_to_rm(DeviceTableau &t) {
    // CM: row-tiles I in [0,k), words J in [0,2kg).
    run(t.x, t.x2, t.cm_pitch, t.rm_pitch, t.k, 2 * t.kg, true, t.stream);
    run(t.z, t.z2, t.cm_pitch, t.rm_pitch, t.k, 2 * t.kg, true, t.stream);
    if (t.rm_pitch > t.k) {
        const uint64_t rows = 2 * t.ng, work = rows * (t.rm_pitch - t.k);
        const unsigned blocks = unsigned(std::min<uint64_t>((work + 255) / 256, uint64_t(t.num_sms) * 16));
        k_zero_rm_padding<<<blocks, 256, 0, t.stream>>>(t.x2, t.z2, t.rm_pitch, t.k, rows);
        QSR_CUDA(cudaGetLastError());
        count_launch();
    }
    std::swap(t.x, t.x2);
    std::swap(t.z, t.z2);
    t.layout = QSR_ROW_MAJOR;
}

void transpose_to_cm(DeviceTableau &t) {
    // RM: row-tiles J in [0,2kg), words I in [0,k).
    run(t.x, t.x2, t.rm_pitch, t.cm_pitch, 2 * t.kg, t.k, false, t.stream);
    run(t.z, t.z2, t.rm_pitch, t.cm_pitch, 2 * t.kg, t.k, false, t.stream);
    std::swap(t.x, t.x2);
    std::swap(t.z, t.z2);
    t.layout = QSR_COLUMN_MAJOR;
}

} // namespace qsr
