// onchip_peaks.cu -- measured L2 and shared-memory read bandwidth of this B200, the on-chip
// roofline denominators SURVEY.md Sec. 8(d) asks for (MEASURED_PEAKS.json has HBM only).
//
//   L2:   every SM streams 16-byte ld.global.cg loads (L1 bypassed) over a 32 MiB buffer that
//         stays L2-resident (126 MB L2), 20 passes after a warm-up pass;
//   SMEM: every SM's threads read 16-byte words of a 32 KiB shared buffer, conflict-free.
// Best of 5 timed launches each (CUDA events); prints one JSON line.
//
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/onchip_peaks tools/onchip_peaks.cu
#include <cstdint>
#include <cstdio>

__global__ void l2_read(const float4* __restrict__ p, size_t n4, int passes, float* sink) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int r = 0; r < passes; ++r) {
        for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
            const float4 v = __ldcg(p + i);
            acc.x += v.x;
            acc.y += v.y;
            acc.z += v.z;
            acc.w += v.w;
        }
    }
    if (acc.x + acc.y + acc.z + acc.w == 12345.f) sink[0] = acc.x;
}

constexpr int kSmemF4 = 2048;   // 32 KiB (static shared memory limit 48 KiB)
__global__ void smem_read(int iters, float* sink) {
    __shared__ float4 buf[kSmemF4];
    for (int i = threadIdx.x; i < kSmemF4; i += blockDim.x) buf[i] = make_float4(i, i + 1, i + 2, i + 3);
    __syncthreads();
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int k = threadIdx.x;
    for (int r = 0; r < iters; ++r) {
#pragma unroll 8
        for (int u = 0; u < 8; ++u) {
            const float4 v = buf[(k + u * blockDim.x) & (kSmemF4 - 1)];
            acc.x += v.x;
            acc.y += v.y;
            acc.z += v.z;
            acc.w += v.w;
        }
        k = (k + 8 * blockDim.x) & (kSmemF4 - 1);
    }
    if (acc.x + acc.y + acc.z + acc.w == 12345.f) sink[0] = acc.x;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const size_t bytes = 32u << 20;
    float4* p;
    float* sink;
    cudaMalloc(&p, bytes);
    cudaMalloc(&sink, 4);
    cudaMemset(p, 0, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int passes = 20;
    double l2_best = 0;
    l2_read<<<sms * 4, 512>>>(p, bytes / 16, 1, sink);   // warm: bring the buffer into L2
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(a);
        l2_read<<<sms * 4, 512>>>(p, bytes / 16, passes, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double gbs = (double)bytes * passes / (ms * 1e-3) / 1e9;
        if (gbs > l2_best) l2_best = gbs;
    }
    const int iters = 4096, threads = 1024;
    double sm_best = 0;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(a);
        smem_read<<<sms, threads>>>(iters, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double gbs = (double)sms * threads * iters * 8 * 16 / (ms * 1e-3) / 1e9;
        if (gbs > sm_best) sm_best = gbs;
    }
    printf("{\"l2_read_gbs\": %.1f, \"smem_read_gbs\": %.1f, \"sms\": %d, \"sm_clock_mhz_attr\": %d, "
           "\"how\": \"tools/onchip_peaks.cu: L2 = %d SMs x 4 blocks x 512 threads of 16-B ld.global.cg over a "
           "32 MiB L2-resident buffer, %d passes; SMEM = one 1024-thread block per SM reading 16-B words of 32 KiB "
           "conflict-free; best of 5, CUDA events\", \"error\": \"%s\"}\n",
           l2_best, sm_best, sms, clk / 1000, sms, passes, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
