// D2H of a c5-sized CM plane pair: pitched 2-D copy (device pitch 5632 words, host 5626) vs a
// flat 1-D copy of the same bytes, into pinned memory.  nvcc -O2 tools/d2h_probe.cu -o /tmp/d2h
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
int main() {
    const size_t rows = 180032, hw = 5626, dw = 5632;
    uint64_t *d = nullptr, *h = nullptr;
    cudaMalloc(&d, rows * dw * 8);
    cudaMallocHost(&h, rows * dw * 8);
    cudaMemset(d, 1, rows * dw * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 3; ++rep) {
        float ms2 = 0, ms1 = 0;
        cudaEventRecord(a);
        cudaMemcpy2DAsync(h, hw * 8, d, dw * 8, hw * 8, rows, cudaMemcpyDeviceToHost);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms2, a, b);
        cudaEventRecord(a);
        cudaMemcpyAsync(h, d, rows * hw * 8, cudaMemcpyDeviceToHost);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms1, a, b);
        printf("plane %.2f GB: 2-D %.1f ms (%.1f GB/s), 1-D %.1f ms (%.1f GB/s)\n", rows * hw * 8 / 1e9, ms2,
               rows * hw * 8 / ms2 / 1e6, ms1, rows * hw * 8 / ms1 / 1e6);
    }
    return 0;
}
