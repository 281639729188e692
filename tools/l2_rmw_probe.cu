// Microbenchmark: random 128-byte line read-modify-write throughput (the access pattern of a
// gate window restricted to a 16-word slab: 8 lanes x 16 B per operand row) for buffers that
// fit in L2 and for HBM-sized ones. Decides whether an L2-resident, temporally blocked gate
// pass can beat the HBM-bound one.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2p tools/l2_rmw_probe.cu && /tmp/l2p
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

// Each 8-lane group handles one "gate": two random rows (lines), reads x0,z0,x1,z1 (4 x 128 B),
// writes back x1', z0' (2 x 128 B) like a CX.
template <int L>  // lanes per gate: 8 -> 128-byte segments, 4 -> 64 B, 2 -> 32 B
__global__ void __launch_bounds__(512) k_rmw(ulonglong2 *x, ulonglong2 *z, uint32_t nlines, uint32_t iters,
                                             uint32_t salt, uint32_t stride = 1) {
    const uint32_t lane = threadIdx.x & (L - 1);
    const uint32_t grp = (blockIdx.x * blockDim.x + threadIdx.x) / L;
    ulonglong2 acc = make_ulonglong2(0, 0);
    for (uint32_t it = 0; it < iters; ++it) {
        const uint32_t h = hash32(grp * 0x9E3779B9u + it * 0x85ebca6bu + salt);
        const size_t a = size_t(h % (nlines * (8 / L))) * stride, b = size_t(hash32(h) % (nlines * (8 / L))) * stride;
        ulonglong2 x0 = __ldcg(x + size_t(a) * L + lane), z0 = __ldcg(z + size_t(a) * L + lane);
        ulonglong2 x1 = __ldcg(x + size_t(b) * L + lane), z1 = __ldcg(z + size_t(b) * L + lane);
        x1.x ^= x0.x; x1.y ^= x0.y; z0.x ^= z1.x; z0.y ^= z1.y;
        acc.x ^= x0.x & z1.x; acc.y ^= x0.y & z1.y;
        __stcg(x + size_t(b) * L + lane, x1);
        __stcg(z + size_t(a) * L + lane, z0);
    }
    if (acc.x == 0x1234567ull) x[0] = acc; // keep acc alive
}

template <int L>
void run(int sms) {
    const double mbs[] = {32, 48, 64, 4096};
    for (double mb : mbs) {
        const size_t bytes = size_t(mb * 1e6 / 2); // per plane
        const uint32_t nlines = uint32_t(bytes / 128);
        ulonglong2 *x, *z;
        cudaMalloc(&x, size_t(nlines) * 128);
        cudaMalloc(&z, size_t(nlines) * 128);
        cudaMemset(x, 1, size_t(nlines) * 128);
        cudaMemset(z, 2, size_t(nlines) * 128);
        const uint32_t blocks = sms * 4, threads = 512, iters = 200;
        k_rmw<L><<<blocks, threads>>>(x, z, nlines, iters, 1);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        const int reps = 5;
        for (int r = 0; r < reps; ++r) k_rmw<L><<<blocks, threads>>>(x, z, nlines, iters, 7 + r);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double gates = double(blocks) * threads / L * iters * reps;
        const double moved = gates * 6 * 16 * L;
        printf("%3d-B segments, buffer %6.0f MB: %8.1f GB/s\n", 16 * L, mb, moved / (ms * 1e-3) / 1e9);
        cudaFree(x);
        cudaFree(z);
    }
}

// The gate slab's real layout: 180k qubit rows, one 128-byte line each, row pitch 45,056 B.
void run_strided(int sms, uint32_t rows, uint32_t pitch_lines) {
    ulonglong2 *x, *z;
    const size_t bytes = size_t(rows) * pitch_lines * 128;
    cudaMalloc(&x, bytes);
    cudaMalloc(&z, bytes);
    cudaMemset(x, 1, bytes);
    cudaMemset(z, 2, bytes);
    const uint32_t blocks = sms * 4, threads = 512, iters = 200;
    k_rmw<8><<<blocks, threads>>>(x, z, rows, iters, 1, pitch_lines);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) k_rmw<8><<<blocks, threads>>>(x, z, rows, iters, 7 + r, pitch_lines);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double gates = double(blocks) * threads / 8 * iters * reps;
    printf("strided slab: %u rows x 128 B, pitch %u B (%.1f MB touched): %8.1f GB/s\n", rows,
           pitch_lines * 128, rows * 256.0 / 1e6, gates * 6 * 128 / (ms * 1e-3) / 1e9);
    cudaFree(x);
    cudaFree(z);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<8>(sms);
    run_strided(sms, 180032, 352);   // c5: cm_pitch 5632 words = 352 lines
    run_strided(sms, 180032, 1);     // same lines, contiguous
    run_strided(sms, 180032, 353);   // odd pitch
    run_strided(sms, 90016, 352);
    return 0;
}
