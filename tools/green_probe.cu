// Probe: can runtime-API kernel launches be confined to an SM subset with a green context
// stream (CUDA 12.4+ driver API), and do they run concurrently with primary-context work on
// the remaining SMs?  nvcc -gencode arch=compute_100a,code=sm_100a tools/green_probe.cu -lcuda -o /tmp/gp
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <set>
#include <vector>

#define CK(x)                                                                                        \
    do {                                                                                             \
        CUresult r = (x);                                                                            \
        if (r != CUDA_SUCCESS) { const char *s; cuGetErrorString(r, &s); printf("%s: %s\n", #x, s); return 1; } \
    } while (0)
#define RK(x)                                                                                        \
    do {                                                                                             \
        cudaError_t r = (x);                                                                         \
        if (r != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(r)); return 1; }         \
    } while (0)

__global__ void k_smid(unsigned *out, long long spin) {
    unsigned id;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(id));
    if (threadIdx.x == 0) out[blockIdx.x] = id;
    const long long t0 = clock64();
    while (clock64() - t0 < spin) {}
}

int main() {
    RK(cudaSetDevice(0));
    RK(cudaFree(0)); // primary context
    CUdevice dev;
    CK(cuDeviceGet(&dev, 0));
    CUdevResource all;
    CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
    printf("device SMs: %u\n", all.sm.smCount);
    CUdevResource part, rest;
    unsigned n = 1;
    CK(cuDevSmResourceSplitByCount(&part, &n, &all, &rest, 0, 96));
    printf("split: %u groups, part %u SMs, rest %u SMs\n", n, part.sm.smCount, rest.sm.smCount);
    CUdevResourceDesc desc;
    CK(cuDevResourceGenerateDesc(&desc, &part, 1));
    CUgreenCtx g;
    CK(cuGreenCtxCreate(&g, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CUstream gs;
    CK(cuGreenCtxStreamCreate(&gs, g, CU_STREAM_NON_BLOCKING, 0));
    const int blocks = 1184;
    unsigned *d = nullptr;
    RK(cudaMalloc(&d, blocks * 4 * 2));
    cudaStream_t ps;
    RK(cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking));
    cudaEvent_t a, b, c, e;
    RK(cudaEventCreate(&a)); RK(cudaEventCreate(&b)); RK(cudaEventCreate(&c)); RK(cudaEventCreate(&e));
    // green stream alone
    RK(cudaEventRecord(a, (cudaStream_t)gs));
    k_smid<<<blocks, 128, 0, (cudaStream_t)gs>>>(d, 200000);
    RK(cudaGetLastError());
    RK(cudaEventRecord(b, (cudaStream_t)gs));
    RK(cudaStreamSynchronize((cudaStream_t)gs));
    std::vector<unsigned> h(blocks);
    RK(cudaMemcpy(h.data(), d, blocks * 4, cudaMemcpyDeviceToHost));
    std::set<unsigned> sms(h.begin(), h.end());
    float ms = 0;
    RK(cudaEventElapsedTime(&ms, a, b));
    printf("green-stream kernel: %zu distinct SMs, %.3f ms\n", sms.size(), ms);
    // both together: green on its part, primary stream on everything
    RK(cudaEventRecord(a, (cudaStream_t)gs));
    k_smid<<<blocks, 128, 0, (cudaStream_t)gs>>>(d, 200000);
    RK(cudaEventRecord(c, ps));
    k_smid<<<52, 128, 0, ps>>>(d + blocks, 200000 * 20);
    RK(cudaEventRecord(e, ps));
    RK(cudaEventRecord(b, (cudaStream_t)gs));
    RK(cudaDeviceSynchronize());
    float mg = 0, mp = 0;
    RK(cudaEventElapsedTime(&mg, a, b));
    RK(cudaEventElapsedTime(&mp, c, e));
    std::vector<unsigned> h2(52);
    RK(cudaMemcpy(h2.data(), d + blocks, 52 * 4, cudaMemcpyDeviceToHost));
    std::set<unsigned> s2(h2.begin(), h2.end()), inter;
    for (unsigned v : s2) if (sms.count(v)) inter.insert(v);
    printf("concurrent: green %.3f ms, primary (52 CTAs, 20x longer each) %.3f ms on %zu SMs, %zu shared with green\n",
           mg, mp, s2.size(), inter.size());
    return 0;
}
