// Profiling probe (not product): do green contexts (SM partitions) give the
// HBM-bound scatter a private share of the SMs beside the latency-bound ack
// path?  Checks the partition (%smid), cross-context events, stream capture
// across the partitions, and a copy kernel's bandwidth on a partition.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <set>
#include <vector>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s_; cuGetErrorString(r_, &s_); printf("%s:%d %s -> %s\n", __FILE__, __LINE__, #x, s_); return 1; } } while (0)
#define CR(x) do { cudaError_t r_ = (x); if (r_ != cudaSuccess) { printf("%s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(r_)); return 1; } } while (0)

__global__ void k_smid(int* out) {
    unsigned s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    if (threadIdx.x == 0) out[blockIdx.x] = s;
}
__global__ void k_copy(int4* __restrict__ d, const int4* __restrict__ s, size_t n) {
    size_t st = (size_t)gridDim.x * blockDim.x;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += 4 * st) {
        int4 a = __ldcs(s + i), b = i + st < n ? __ldcs(s + i + st) : int4{}, c = i + 2 * st < n ? __ldcs(s + i + 2 * st) : int4{},
             e = i + 3 * st < n ? __ldcs(s + i + 3 * st) : int4{};
        __stcs(d + i, a);
        if (i + st < n) __stcs(d + i + st, b);
        if (i + 2 * st < n) __stcs(d + i + 2 * st, c);
        if (i + 3 * st < n) __stcs(d + i + 3 * st, e);
    }
}
__global__ void k_spin(unsigned long long ns) {  // a latency-bound occupant
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > ns) break;
        __nanosleep(200);
    }
}

int main(int argc, char** argv) {
    int chainSms = argc > 1 ? atoi(argv[1]) : 48;
    CK(cuInit(0));
    CUdevice dev;
    CK(cuDeviceGet(&dev, 0));
    CR(cudaSetDevice(0));
    CR(cudaFree(0));  // primary context current
    CUdevResource all;
    CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
    printf("SMs: %u\n", all.sm.smCount);
    CUdevResource part[1], rest;
    unsigned ng = 1;
    CK(cuDevSmResourceSplitByCount(part, &ng, &all, &rest, 0, chainSms));
    printf("chain partition %u SMs, rest %u SMs\n", part[0].sm.smCount, rest.sm.smCount);
    CUdevResourceDesc dA, dB;
    CK(cuDevResourceGenerateDesc(&dA, part, 1));
    CK(cuDevResourceGenerateDesc(&dB, &rest, 1));
    CUgreenCtx gA, gB;
    CK(cuGreenCtxCreate(&gA, dA, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CK(cuGreenCtxCreate(&gB, dB, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CUstream sA, sB;
    CK(cuGreenCtxStreamCreate(&sA, gA, CU_STREAM_NON_BLOCKING, 0));
    CK(cuGreenCtxStreamCreate(&sB, gB, CU_STREAM_NON_BLOCKING, 0));
    int* dsm;
    CR(cudaMalloc(&dsm, 4096 * 4));
    // 1. partition respected by runtime launches on green-context streams?
    for (int which = 0; which < 2; ++which) {
        k_smid<<<2048, 64, 0, which ? (cudaStream_t)sB : (cudaStream_t)sA>>>(dsm);
        CR(cudaGetLastError());
        CR(cudaDeviceSynchronize());
        std::vector<int> h(2048);
        CR(cudaMemcpy(h.data(), dsm, 2048 * 4, cudaMemcpyDeviceToHost));
        std::set<int> s(h.begin(), h.end());
        printf("stream %c: blocks ran on %zu distinct SMs\n", which ? 'B' : 'A', s.size());
    }
    // 2. copy bandwidth: whole GPU, partition B alone, partition B beside spinning chain kernels on A
    size_t bytes = 512ull << 20;
    int4 *src, *dst;
    CR(cudaMalloc(&src, bytes));
    CR(cudaMalloc(&dst, bytes));
    CR(cudaMemset(src, 1, bytes));
    cudaStream_t s0;
    CR(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
    cudaEvent_t e0, e1;
    CR(cudaEventCreate(&e0));
    CR(cudaEventCreate(&e1));
    auto timeit = [&](cudaStream_t st, int blocks, bool spin) -> float {
        for (int w = 0; w < 2; ++w) k_copy<<<blocks, 512, 0, st>>>(dst, src, bytes / 16);
        cudaDeviceSynchronize();
        if (spin) k_spin<<<chainSms * 4, 256, 0, (cudaStream_t)sA>>>(3000000ull);
        cudaEventRecord(e0, st);
        for (int r = 0; r < 5; ++r) k_copy<<<blocks, 512, 0, st>>>(dst, src, bytes / 16);
        cudaEventRecord(e1, st);
        cudaDeviceSynchronize();
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        return 2.0f * bytes * 5 / (ms * 1e-3f) / 1e9f;
    };
    printf("copy, whole GPU (primary stream, 148 x 4 blocks): %.0f GB/s\n", timeit(s0, 148 * 4, false));
    printf("copy, partition B (%u SMs): %.0f GB/s\n", rest.sm.smCount, timeit((cudaStream_t)sB, rest.sm.smCount * 4, false));
    printf("copy, partition B beside %d-SM partition A busy: %.0f GB/s\n", chainSms,
           timeit((cudaStream_t)sB, rest.sm.smCount * 4, true));
    printf("copy, whole GPU beside spinning blocks on A: %.0f GB/s\n", timeit(s0, 148 * 4, true));
    // 3. events across contexts and stream capture across partitions
    cudaEvent_t ev;
    CR(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    cudaGraph_t g;
    cudaStreamBeginCapture(s0, cudaStreamCaptureModeGlobal);
    cudaEventRecord(ev, s0);
    cudaError_t r1 = cudaStreamWaitEvent((cudaStream_t)sA, ev, 0);
    k_smid<<<1, 32, 0, (cudaStream_t)sA>>>(dsm);
    cudaEvent_t ev2;
    cudaEventCreateWithFlags(&ev2, cudaEventDisableTiming);
    cudaError_t r2 = cudaEventRecord(ev2, (cudaStream_t)sA);
    cudaError_t r3 = cudaStreamWaitEvent(s0, ev2, 0);
    cudaError_t r4 = cudaStreamEndCapture(s0, &g);
    printf("capture across partitions: wait %s, record %s, join %s, end %s\n", cudaGetErrorString(r1),
           cudaGetErrorString(r2), cudaGetErrorString(r3), cudaGetErrorString(r4));
    if (r4 == cudaSuccess) {
        cudaGraphExec_t ge;
        cudaError_t r5 = cudaGraphInstantiate(&ge, g, 0);
        cudaError_t r6 = r5 == cudaSuccess ? cudaGraphLaunch(ge, s0) : r5;
        cudaError_t r7 = cudaStreamSynchronize(s0);
        printf("instantiate %s, launch %s, sync %s\n", cudaGetErrorString(r5), cudaGetErrorString(r6),
               cudaGetErrorString(r7));
        std::vector<int> h(1);
        cudaMemcpy(h.data(), dsm, 4, cudaMemcpyDeviceToHost);
        printf("captured kernel ran on SM %d\n", h[0]);
    }
    cudaGetLastError();
    printf("done\n");
    return 0;
}
