// K2+K3 — out-of-place layout transpose CM <-> generator-major RM
// (reference Tableau::transpose_in_place = shuffle_tiles + permute_words,
//  tableau.hpp:166-176, 280-322; bit_transpose_tile bitplane.hpp:165-183).
//
// The reference moves 64x64-bit tiles in place in two passes (bit-transpose every tile, then
// permute words per block-row). Here one pass reads each tile once and writes it once:
//   * a block = 8 source row-tiles x 16 source words (512 rows x 128 contiguous bytes, 64 KB) is
//     fetched by TMA (two 2-D boxes, cp.async.bulk.tensor) into a ring of three shared-memory
//     buffers: the next two blocks' TMAs are in flight while one is transposed (persistent
//     CTAs, one per SM, mbarrier-tracked);
//   * a thread owns half a tile (32 rows of one word) and transposes it in registers as two
//     32x32 bit transposes of its low and high 32-bit halves (the 64x64 transpose's
//     offset-32 round is pure register renaming): the byte and half-word rounds are `prmt`
//     permutations, the nibble / pair / bit rounds one shift + one lop3 per word;
//   * the transposed halves go through a padded staging area in the buffer the block was just
//     read from (conflict-free 32-bit stores) and leave as 64-byte contiguous runs of 8
//     destination words per destination row; the CTAs running together (one word-block, 148
//     row-blocks) write adjacent runs of the same destination rows.
// Destination words past the source's row-tiles (the RM row padding, qubit-words k .. rm_pitch)
// are read as TMA out-of-bounds zeros and written as zeros, so the padding needs no extra pass.
//
//   CM word (q, J)      at q*cm_pitch + J          bits = generators J*64 + b
//   RM word (r = J*64+t, I) at r*rm_pitch + I      bits = qubits I*64 + c
// Tile (I, J): CM rows I*64..I*64+63, word J  <->  RM rows J*64..J*64+63, word I.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

#include "common.cuh"
#include "device.hpp"

namespace qsr {

namespace {

// Block shape: RT source row-tiles x W source words (RT x 64 rows of W words), two threads per
// tile (row halves); ST blocks in flight per CTA (a TMA ring). The transposed words are staged
// in the buffer the block was just read from, so a CTA needs ST x (block bytes) of shared memory.
template <int RT, int W, int ST>
struct Shape {
    static_assert(W % 16 == 0 && ST >= 2, "block shape");
    static constexpr int kThreads = RT * W * 2;
    static constexpr uint32_t kInWords = RT * 64 * W;
    static constexpr uint32_t kBoxRows = RT * 64 > 256 ? 256 : RT * 64; // TMA box rows
    static constexpr uint32_t kBoxes = RT * 64 / kBoxRows;
    static constexpr uint32_t kStageStride = 32 * RT + 1; // staging words per source word (+1 pad)
    static_assert(W * kStageStride <= kInWords, "staging fits in a block buffer");
    static constexpr size_t kSmemBytes = ST * kInWords * 8 + 64;
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int32_t x, int32_t y, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

// 32x32 bit transpose in registers: out a[c] bit r = in a[r] bit c (delta swaps with offsets
// 16, 8, 4, 2, 1; the first two are byte permutations).
__device__ __forceinline__ void transpose32(uint32_t (&a)[32]) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        const uint32_t x = a[r], y = a[r + 16];
        a[r] = __byte_perm(x, y, 0x5410);
        a[r + 16] = __byte_perm(x, y, 0x7632);
    }
#pragma unroll
    for (int r = 0; r < 32; ++r) {
        if (r & 8) continue;
        const uint32_t x = a[r], y = a[r + 8];
        a[r] = __byte_perm(x, y, 0x6240);
        a[r + 8] = __byte_perm(x, y, 0x7351);
    }
#pragma unroll
    for (int s = 4, sh = 0; s >= 1; s >>= 1, ++sh) {
        const uint32_t m = sh == 0 ? 0x0F0F0F0Fu : sh == 1 ? 0x33333333u : 0x55555555u;
#pragma unroll
        for (int r = 0; r < 32; ++r) {
            if (r & s) continue;
            const uint32_t x = a[r], y = a[r + s];
            a[r] = (x & m) | ((y << s) & ~m);
            a[r + s] = ((x >> s) & m) | (y & ~m);
        }
    }
}

// Persistent CTAs over a virtual block index: groups of gw x gr blocks (gw source word-blocks x
// gr row-tile blocks, word-blocks fastest) so the CTAs running together read ~gw x 128 B of each
// source row and write ~gr x 64 B of each destination row (DRAM page locality on both sides);
// indices past the edges are skipped.
struct BlockMap {
    uint32_t wblocks, rblocks, gw, gr, ngw, per_plane;
    __device__ __forceinline__ bool decode(uint32_t v, uint32_t &plane, uint32_t &wb, uint32_t &rb) const {
        plane = v / per_plane;
        const uint32_t u = v - plane * per_plane, gsz = gw * gr, g = u / gsz, in = u - g * gsz;
        wb = (g % ngw) * gw + in % gw;
        rb = (g / ngw) * gr + in / gw;
        return wb < wblocks && rb < rblocks;
    }
};

template <int kRT, int kW, int kStages>
__global__ void __launch_bounds__(Shape<kRT, kW, kStages>::kThreads)
k_transpose(const __grid_constant__ CUtensorMap src_x, const __grid_constant__ CUtensorMap src_z,
            uint64_t *__restrict__ dst_x, uint64_t *__restrict__ dst_z, uint64_t dst_pitch, uint32_t src_words,
            uint32_t dst_words, BlockMap bm) {
    using S = Shape<kRT, kW, kStages>;
    constexpr uint32_t kStageStride = S::kStageStride, kInWords = S::kInWords;
    constexpr int kThreads = S::kThreads;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t *in0 = reinterpret_cast<uint64_t *>(smem);
    uint64_t *bar = in0 + kStages * kInWords;
    // Thread = (row-tile ti, source word j, row half h); a half-warp reads 16 consecutive words.
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, h = lane >> 4;
    const uint32_t ti = warp / (kW / 16), j = (warp % (kW / 16)) * 16 + (lane & 15);
    const uint32_t nvirt = 2 * bm.per_plane;
    if (tid == 0) {
        for (int i = 0; i < kStages; ++i) mbar_init(&bar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    auto next_valid = [&](uint32_t v) { // v, or the next index of this CTA that is a real block
        uint32_t p, wb, rb;
        while (v < nvirt && !bm.decode(v, p, wb, rb)) v += gridDim.x;
        return v;
    };
    auto issue = [&](uint32_t v, uint32_t buf) {
        uint32_t plane, wb, rb;
        bm.decode(v, plane, wb, rb);
        const CUtensorMap *m = plane ? &src_z : &src_x;
        uint64_t *d = in0 + buf * kInWords;
        mbar_expect_tx(&bar[buf], kInWords * 8);
#pragma unroll
        for (uint32_t bx = 0; bx < S::kBoxes; ++bx)
            tma_load_2d(d + bx * S::kBoxRows * kW, m, int32_t(wb * kW), int32_t(rb * kRT * 64 + bx * S::kBoxRows),
                        &bar[buf]);
    };
    // Ring of kStages buffers: block `it` lives in buffer it % kStages; the block kStages - 1
    // ahead is issued at the top of each iteration, into the buffer read (and synced) in it - 1.
    uint32_t ahead[kStages];
    uint32_t b = next_valid(blockIdx.x);
    ahead[0] = b;
    for (int i = 1; i < kStages; ++i) ahead[i] = ahead[i - 1] < nvirt ? next_valid(ahead[i - 1] + gridDim.x) : nvirt;
    if (tid == 0)
        for (int i = 0; i < kStages - 1; ++i)
            if (ahead[i] < nvirt) issue(ahead[i], uint32_t(i));
    uint32_t it = 0;
    for (; b < nvirt; ++it) {
        const uint32_t buf = it % kStages;
        if (tid == 0 && ahead[kStages - 1] < nvirt) issue(ahead[kStages - 1], (it + kStages - 1) % kStages);
        uint32_t plane, wb, rb;
        bm.decode(b, plane, wb, rb);
        uint64_t *const dst = plane ? dst_z : dst_x;
        mbar_wait(&bar[buf], (it / kStages) & 1u);
        // Rows 64*ti + 32*h .. +31 of source word j: low halves -> bits c < 32 of the
        // destination words, high halves -> c >= 32; this thread's rows are half h of each.
        uint32_t lo[32], hi[32];
        {
            const uint64_t *rows = in0 + buf * kInWords + (ti * 64 + h * 32) * kW + j;
#pragma unroll
            for (int r = 0; r < 32; ++r) {
                const uint64_t v = rows[r * kW];
                lo[r] = uint32_t(v);
                hi[r] = uint32_t(v >> 32);
            }
        }
        __syncthreads(); // every row is in registers: the buffer becomes the staging area
        uint64_t *const stage = in0 + buf * kInWords;
        transpose32(lo);
        transpose32(hi);
        const uint32_t J = wb * kW, I0 = rb * kRT;
#pragma unroll
        for (int pass = 0; pass < 2; ++pass) {
            // Staging: destination word (row (j, c), word ti) at j * kStageStride + c * kRT + ti,
            // half h (the pad spreads 16 consecutive j over all banks).
            uint32_t *st = reinterpret_cast<uint32_t *>(stage) + 2 * (j * kStageStride + ti) + h;
#pragma unroll
            for (int c = 0; c < 32; ++c) st[2 * c * kRT] = pass ? hi[c] : lo[c];
            __syncthreads();
            // kW source words x 32 rows x kRT destination words: thread (c, i) walks every
            // (256 / (32 kRT))-th source word; kRT consecutive lanes write one destination run.
            {
                constexpr uint32_t kJStep = kThreads / (32 * kRT);
                const uint32_t i = tid % kRT, c = (tid / kRT) % 32, j0 = tid / (32 * kRT);
                constexpr uint32_t kPer = kW / kJStep; // 16 destination words per thread and pass
                if (I0 + i < dst_words) {
                    const uint32_t nj = min(uint32_t(kW), src_words - J);
                    uint64_t *d = dst + (uint64_t(J + j0) * 64 + pass * 32 + c) * dst_pitch + I0 + i;
                    const uint64_t *sv = stage + j0 * kStageStride + c * kRT + i;
                    // All staged words first (independent shared loads), then the stores.
                    uint64_t v[kPer];
#pragma unroll
                    for (uint32_t u = 0; u < kPer; ++u) v[u] = sv[u * kJStep * kStageStride];
                    const uint64_t step = uint64_t(kJStep) * 64 * dst_pitch;
#pragma unroll
                    for (uint32_t u = 0; u < kPer; ++u)
                        if (j0 + u * kJStep < nj) __stcs(d + u * step, v[u]);
                }
            }
            __syncthreads();
        }
#pragma unroll
        for (int i = 0; i < kStages - 1; ++i) ahead[i] = ahead[i + 1];
        b = ahead[0];
        ahead[kStages - 1] = ahead[kStages - 2] < nvirt ? next_valid(ahead[kStages - 2] + gridDim.x) : nvirt;
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        QSR_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p) fail(QSR_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

CUtensorMap tensor_map(const uint64_t *base, uint64_t words, uint64_t rows, uint64_t pitch, uint32_t box_words,
                       uint32_t box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {words, rows};
    const cuuint64_t strides[1] = {pitch * 8};
    const cuuint32_t box[2] = {box_words, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<uint64_t *>(base), dims, strides,
                                 box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(QSR_CUDA_ERROR, "cuTensorMapEncodeTiled failed");
    return m;
}

// Dynamic shared memory above 48 KB is a per-device function attribute.
template <int RT, int W, int ST>
void configure(int device) {
    static std::mutex mu;
    static std::vector<bool> done;
    std::lock_guard<std::mutex> g(mu);
    if (done.size() <= size_t(device)) done.resize(size_t(device) + 1, false);
    if (done[size_t(device)]) return;
    QSR_CUDA(cudaFuncSetAttribute(k_transpose<RT, W, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(Shape<RT, W, ST>::kSmemBytes)));
    done[size_t(device)] = true;
}

// src: rows x src_words (pitch src_pitch) -> dst: (64 src_words) rows x dst_words (pitch
// dst_pitch); source row-tiles past src_rows / 64 read as zeros (destination padding words).
template <int RT, int W, int ST>
void run_shape(DeviceTableau &t, const uint64_t *sx, const uint64_t *sz, uint64_t *dx, uint64_t *dz,
               uint64_t src_pitch, uint64_t src_rows, uint64_t src_words, uint64_t dst_pitch, uint64_t dst_words) {
    using S = Shape<RT, W, ST>;
    configure<RT, W, ST>(t.device);
    static int per_sm = 0;
    if (!per_sm) {
        QSR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_transpose<RT, W, ST>, S::kThreads,
                                                               S::kSmemBytes));
        per_sm = std::max(per_sm, 1);
    }
    const CUtensorMap mx = tensor_map(sx, src_words, src_rows, src_pitch, W, S::kBoxRows);
    const CUtensorMap mz = tensor_map(sz, src_words, src_rows, src_pitch, W, S::kBoxRows);
    BlockMap bm;
    bm.wblocks = uint32_t((src_words + W - 1) / W);
    bm.rblocks = uint32_t((dst_words + RT - 1) / RT);
    const uint64_t slots = uint64_t(t.num_sms) * uint64_t(per_sm);
    // Groups of 1 word-block x (resident CTAs) row-blocks: the CTAs running together write
    // adjacent runs of the same destination rows. Measured at c5 (gw x gr): 1 x 148 4.8 TB/s,
    // 2 x 74 4.1, 4 x 37 3.6, 8 x 18 3.6, 148 x 1 3.4 — the write side needs the page locality.
    bm.gw = 1;
    bm.gr = std::max(1u, std::min(bm.rblocks, uint32_t(slots)));
    bm.ngw = (bm.wblocks + bm.gw - 1) / bm.gw;
    const uint32_t ngr = (bm.rblocks + bm.gr - 1) / bm.gr;
    bm.per_plane = bm.ngw * ngr * bm.gw * bm.gr;
    const unsigned grid = unsigned(std::min<uint64_t>(2ull * bm.wblocks * bm.rblocks, slots));
    k_transpose<RT, W, ST><<<grid, S::kThreads, S::kSmemBytes, t.stream>>>(
        mx, mz, dx, dz, dst_pitch, uint32_t(src_words), uint32_t(dst_words), bm);
    QSR_CUDA(cudaGetLastError());
    count_launch();
}

// 8 x 16 blocks (128-byte source runs, 64-byte destination runs), three in flight per CTA, one
// CTA per SM. Measured alternatives (profiles/r02_transpose.md): 4 x 32 ties at c5 and loses
// 15-30 % at 20k-50k qubits; 4 x 16 with two or three CTAs per SM and two-stage rings are
// slower at c5.
void run(DeviceTableau &t, const uint64_t *sx, const uint64_t *sz, uint64_t *dx, uint64_t *dz, uint64_t src_pitch,
         uint64_t src_rows, uint64_t src_words, uint64_t dst_pitch, uint64_t dst_words) {
    run_shape<8, 16, 3>(t, sx, sz, dx, dz, src_pitch, src_rows, src_words, dst_pitch, dst_words);
}

} // namespace

void transpose_to_rm(DeviceTableau &t) {
    // CM: rows n_pad (row-tiles I in [0, k)), words J in [0, 2kg) -> RM rows 2ng, words
    // [0, rm_pitch) (I >= k: zero padding).
    run(t, t.x, t.z, t.x2, t.z2, t.cm_pitch, t.n_pad, 2 * t.kg, t.rm_pitch, t.rm_pitch);
    std::swap(t.x, t.x2);
    std::swap(t.z, t.z2);
    t.layout = QSR_ROW_MAJOR;
}

void transpose_to_cm(DeviceTableau &t) {
    // RM: rows 2ng (row-tiles J in [0, 2kg)), words I in [0, k) -> CM rows n_pad, words
    // [0, cm_pitch) (J >= 2kg: zero padding).
    run(t, t.x, t.z, t.x2, t.z2, t.rm_pitch, 2 * t.ng, t.k, t.cm_pitch, t.cm_pitch);
    std::swap(t.x, t.x2);
    std::swap(t.z, t.z2);
    t.layout = QSR_COLUMN_MAJOR;
}

} // namespace qsr
