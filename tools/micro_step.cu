// micro_step.cu -- per-step cycles of the construction chain, feature by feature.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/micro_step tools/micro_step.cu
#include <cstdio>
#include <cstdint>
#define STEPS 2000
extern __shared__ uint16_t tab[];
template <int F>
__global__ void k_step(uint32_t* out, int seed) {
    constexpr int rows = 1024;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float* inv = reinterpret_cast<float*>(tab + rows * 32);
    for (int i = threadIdx.x; i < rows * 32; i += blockDim.x) {
        tab[i] = (uint16_t)(((i * 2654435761u) >> 12) & 1023);
        inv[i] = 1.0f + (i & 255);
    }
    __syncthreads();
    uint32_t word = lane * 0x01000001u;
    uint32_t cur = (seed + warp * 7) & 1023;
    uint32_t stage = 0;
    float L = -1.5f - lane;
    long long t0 = clock64();
    for (int s = 0; s < STEPS; ++s) {
        uint32_t c = tab[cur * 32 + lane];
        uint32_t key;
        if (F & 4) {
            float iv = inv[cur * 32 + lane];
            key = __float_as_uint(L * iv) & 0x7fffffffu;
        } else {
            key = (c * 2654435761u + s) & 0x7fffffffu;
        }
        uint32_t w = __shfl_sync(0xffffffffu, word, c >> 5);
        uint32_t mag = ((w << (~c & 31)) & 0x80000000u) | key;
        uint32_t b = __reduce_min_sync(0xffffffffu, mag);
        uint32_t nxt = __reduce_min_sync(0xffffffffu, mag == b ? c : 0xffffffffu);
        if (F & 1) {   // tabu mark
            if (lane == (int)(nxt >> 5)) word ^= 1u << (nxt & 31);
        }
        if (F & 2) {   // route staging + rare fallback branch
            if (b >= 0xF0000000u) nxt = (nxt + 1) & 1023;
            if (lane == (s & 31)) stage = nxt;
            if ((s & 31) == 31) out[64 + blockIdx.x * 32 + lane] = stage;
        }
        cur = nxt & 1023;
    }
    long long t1 = clock64();
    if (lane == 0 && warp == 0 && blockIdx.x == 0) { out[0] = (uint32_t)(t1 - t0); out[1] = cur; }
}
template <int F>
void run(uint32_t* d) {
    cudaFuncSetAttribute(k_step<F>, cudaFuncAttributeMaxDynamicSharedMemorySize, 1024 * 32 * 6);
    for (int warps : {1, 7, 14}) {
        uint32_t h[2];
        for (int rep = 0; rep < 2; ++rep) {
            k_step<F><<<148, warps * 32, 1024 * 32 * 6>>>(d, 1);
            cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
        }
        printf("features mark=%d stage+fb=%d ivload=%d  warps/SM %2d: %6.1f cycles/step\n", F & 1, (F >> 1) & 1,
               (F >> 2) & 1, warps, (double)h[0] / STEPS);
    }
}
int main() {
    uint32_t* d; cudaMalloc(&d, 1 << 20);
    run<0>(d); run<1>(d); run<2>(d); run<3>(d); run<4>(d); run<7>(d);
    return 0;
}
