// Tableau::check_group_validity (reference tableau.hpp:184-213) on the device.
//
// The reference walks i <= j over n generators and checks three symplectic inner products per
// pair (stabilizers i,j commute; destabilizers i,j commute; destabilizer i vs stabilizer j is 1
// iff i == j), returning the first violation in that order; O(n^2 k) words, days at c5 on a CPU.
// Here the needed half of the 2n x 2n symplectic Gram matrix is computed as a tiled GF(2)
// product over the generator-major (RM) planes, where each generator's qubit words are
// contiguous: a CTA owns a 64 x 128 block of generator pairs, stages 8 qubit-words of both
// blocks' X and Z rows in shared memory, and each thread XOR-accumulates a 4 x 8 pair block
// (rows strided by 16 so a half-warp reads 16 consecutive words: no bank conflicts)
// acc ^= (xa & zb) ^ (za & xb) (four LOP3 per pair-word); parity(popc(acc)) is the inner
// product (the parity of a sum of popcounts is the popcount of the XOR). Violations are
// reduced to the reference's first one with one atomicMin on the key (i*n + j)*3 + check.
#include <algorithm>

#include "common.cuh"
#include "device.hpp"

namespace qsr {

namespace {

constexpr int kRowsA = 64, kRowsB = 128, kWords = 8, kThreads = 256;

__global__ void __launch_bounds__(kThreads, 2) k_sympl_gram(const uint64_t *__restrict__ x,
                                                         const uint64_t *__restrict__ z, uint64_t pitch,
                                                         uint64_t kw, uint64_t ng, uint64_t n,
                                                         unsigned long long *__restrict__ first) {
    const uint64_t b0 = uint64_t(blockIdx.x) * kRowsB;
    const uint64_t na = 2 * ng / kRowsA;
    for (uint64_t ay = blockIdx.y; ay < na; ay += gridDim.y) {
    const uint64_t a0 = ay * kRowsA;
    if (a0 > b0 + kRowsB - 1) return; // only pairs with ga <= gb are needed (a0 grows with ay)
    // +1 word per row of the staging arrays: the 16 words of one source row land in 16
    // different banks (conflict-free stores), and row-consecutive reads stay conflict-free.
    __shared__ uint64_t ax[kWords][kRowsA + 1], az[kWords][kRowsA + 1];
    __shared__ uint64_t bx[kWords][kRowsB + 1], bz[kWords][kRowsB + 1];
    const int t = threadIdx.x, ta = t / 16, tb = t % 16;
    // parity(popc(v)) = parity(popc(lo(v) ^ hi(v))): 32-bit accumulators suffice (and free the
    // registers for two CTAs per SM).
    uint32_t acc[4][8];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0;
    for (uint64_t c = 0; c < kw; c += kWords) {
        // Stage: 8 contiguous words (64 B) per row; RM rows are padded to pitch (multiple of
        // 16) with zeros, so no word-bound checks are needed.
#pragma unroll
        for (int i = 0; i < kRowsA * kWords / kThreads; ++i) {
            const int idx = t + i * kThreads, r = idx / kWords, w = idx % kWords;
            const uint64_t off = (a0 + r) * pitch + c + w;
            ax[w][r] = x[off];
            az[w][r] = z[off];
        }
#pragma unroll
        for (int i = 0; i < kRowsB * kWords / kThreads; ++i) {
            const int idx = t + i * kThreads, r = idx / kWords, w = idx % kWords;
            const uint64_t off = (b0 + r) * pitch + c + w;
            bx[w][r] = x[off];
            bz[w][r] = z[off];
        }
        __syncthreads();
#pragma unroll 4
        for (int w = 0; w < kWords; ++w) {
            uint64_t xa[4], za[4], xb[8], zb[8];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                xa[i] = ax[w][ta + 16 * i];
                za[i] = az[w][ta + 16 * i];
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                xb[j] = bx[w][tb + 16 * j];
                zb[j] = bz[w][tb + 16 * j];
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint64_t v = (xa[i] & zb[j]) ^ (za[i] & xb[j]);
                    acc[i][j] ^= uint32_t(v) ^ uint32_t(v >> 32);
                }
        }
        __syncthreads();
    }
    unsigned long long best = ~0ull;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint64_t ga = a0 + ta + 16 * i, gb = b0 + tb + 16 * j;
            if (ga > gb) continue;
            const bool da = ga < ng, db = gb < ng;
            const uint64_t ia = da ? ga : ga - ng, ib = db ? gb : gb - ng;
            if (ia >= n || ib >= n) continue; // padding generators
            uint64_t ci, cj, check;
            int expect = 0;
            if (da && db) { ci = ia; cj = ib; check = 1; }       // destabilizers i, j
            else if (!da && !db) { ci = ia; cj = ib; check = 0; } // stabilizers i, j
            else if (ib >= ia) { ci = ia; cj = ib; check = 2; expect = ia == ib; } // D_i vs S_j, j >= i
            else continue;                                        // j < i: not checked
            const int bit = __popc(acc[i][j]) & 1;
            if (bit != expect) {
                const unsigned long long key = (ci * n + cj) * 3 + check;
                best = key < best ? key : best;
            }
        }
    if (best != ~0ull) atomicMin(first, best);
    }
}

} // namespace

std::string check_group_validity(DeviceTableau &t) {
    if (t.g0 != 0 || t.kg != t.k) fail(QSR_INVALID_ARGUMENT, "check_group_validity: needs a whole (unsharded) tableau");
    const bool was_cm = t.layout == QSR_COLUMN_MAJOR;
    if (was_cm) transpose_to_rm(t);
    unsigned long long *d_first = nullptr;
    QSR_CUDA(cudaMallocAsync(&d_first, 8, t.stream));
    QSR_CUDA(cudaMemsetAsync(d_first, 0xFF, 8, t.stream));
    const uint64_t rows = 2 * t.ng;
    dim3 grid(unsigned(rows / kRowsB), unsigned(std::min<uint64_t>(rows / kRowsA, 65535)));
    if (t.n) {
        k_sympl_gram<<<grid, kThreads, 0, t.stream>>>(t.x, t.z, t.rm_pitch, t.rm_pitch, t.ng, t.n, d_first);
        QSR_CUDA(cudaGetLastError());
        count_launch();
    }
    unsigned long long first = 0;
    QSR_CUDA(cudaMemcpyAsync(&first, d_first, 8, cudaMemcpyDeviceToHost, t.stream));
    QSR_CUDA(cudaFreeAsync(d_first, t.stream));
    if (was_cm) transpose_to_cm(t);
    t.sync();
    if (first == ~0ull) return "valid";
    const uint64_t check = first % 3, pair = first / 3, i = pair / t.n, j = pair % t.n;
    if (check == 0) return "stabilizers " + std::to_string(i) + "," + std::to_string(j) + " anti-commute";
    if (check == 1) return "destabilizers " + std::to_string(i) + "," + std::to_string(j) + " anti-commute";
    return "destabilizer " + std::to_string(i) + " vs stabilizer " + std::to_string(j) + ": wrong commutation";
}

} // namespace qsr
