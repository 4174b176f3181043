// micro_tput.cu -- per-SM throughput of REDUX / SHFL / LDS / VOTE with many warps.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/micro_tput tools/micro_tput.cu
#include <cstdio>
#include <cstdint>
#define N 4096
template <int OP>
__global__ void k(uint32_t* out, int seed) {
    __shared__ uint32_t s[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = i * 7;
    __syncthreads();
    uint32_t a = threadIdx.x + seed, b = a * 3, c = a * 5, d = a * 7;   // 4 independent chains per warp
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) {
        if (OP == 0) { a = __reduce_min_sync(~0u, a) + threadIdx.x; b = __reduce_min_sync(~0u, b) + threadIdx.x; c = __reduce_min_sync(~0u, c) + threadIdx.x; d = __reduce_min_sync(~0u, d) + threadIdx.x; }
        if (OP == 1) { a = __shfl_sync(~0u, a, (a + 1) & 31); b = __shfl_sync(~0u, b, (b + 1) & 31); c = __shfl_sync(~0u, c, (c + 1) & 31); d = __shfl_sync(~0u, d, (d + 1) & 31); }
        if (OP == 2) { a = s[a & 1023]; b = s[b & 1023]; c = s[c & 1023]; d = s[d & 1023]; }
        if (OP == 3) { a = __ballot_sync(~0u, a & 1) + threadIdx.x; b = __ballot_sync(~0u, b & 1) + threadIdx.x; c = __ballot_sync(~0u, c & 1) + threadIdx.x; d = __ballot_sync(~0u, d & 1) + threadIdx.x; }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) { out[0] = (uint32_t)(t1 - t0); }
    if (a + b + c + d == 0x12345) out[1] = 1;
}
template <int OP>
void run(const char* name, uint32_t* d) {
    for (int warps : {1, 4, 8, 16, 32}) {
        uint32_t h;
        for (int rep = 0; rep < 2; ++rep) { k<OP><<<148, 32 * warps>>>(d, 1); cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost); }
        double cyc = (double)h / N;   // per iteration (4 ops per warp)
        printf("%-6s warps/SM %2d: %6.1f cycles/iter -> %5.2f ops/cycle/SM\n", name, warps, cyc, 4.0 * warps / cyc);
    }
}
int main() { uint32_t* d; cudaMalloc(&d, 64); run<0>("REDUX", d); run<1>("SHFL", d); run<2>("LDS", d); run<3>("VOTE", d); }
