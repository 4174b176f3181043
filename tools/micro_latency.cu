// micro_latency.cu -- dependent-chain latencies of the ops on the construction step's critical path.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/micro_latency tools/micro_latency.cu
// One warp, 4096 dependent iterations, clock64() around the loop; prints cycles per iteration.
#include <cstdio>
#include <cstdint>

#define ITERS 4096

__global__ void k_lds(uint32_t* out, int seed) {
    __shared__ uint32_t s[1024];
    for (int i = threadIdx.x; i < 1024; i += 32) s[i] = (i * 7 + 3) & 1023;
    __syncwarp();
    uint32_t x = threadIdx.x + seed;
    long long t0 = clock64();
    for (int i = 0; i < ITERS; ++i) x = s[x & 1023];
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = (uint32_t)(t1 - t0); out[1] = x; }
}

__global__ void k_shfl(uint32_t* out, int seed) {
    uint32_t x = threadIdx.x + seed;
    long long t0 = clock64();
    for (int i = 0; i < ITERS; ++i) x = __shfl_sync(0xffffffffu, x, (x + threadIdx.x) & 31);
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = (uint32_t)(t1 - t0); out[1] = x; }
}

__global__ void k_redux(uint32_t* out, int seed) {
    uint32_t x = threadIdx.x * 2654435761u + seed;
    long long t0 = clock64();
    for (int i = 0; i < ITERS; ++i) x = __reduce_min_sync(0xffffffffu, x ^ threadIdx.x) + threadIdx.x;
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = (uint32_t)(t1 - t0); out[1] = x; }
}

__global__ void k_redux2(uint32_t* out, int seed) {
    // the warp_select pattern: min of mag, then min of city among equal mags
    uint32_t mag = threadIdx.x * 2654435761u + seed, c = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < ITERS; ++i) {
        uint32_t b = __reduce_min_sync(0xffffffffu, mag);
        uint32_t w = __reduce_min_sync(0xffffffffu, mag == b ? c : 0xffffffffu);
        mag = (mag ^ w) * 2654435761u;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = (uint32_t)(t1 - t0); out[1] = mag; }
}

__global__ void k_ballot(uint32_t* out, int seed) {
    // min via redux, winner via ballot + ffs + shfl
    uint32_t mag = threadIdx.x * 2654435761u + seed, c = threadIdx.x * 3;
    long long t0 = clock64();
    for (int i = 0; i < ITERS; ++i) {
        uint32_t b = __reduce_min_sync(0xffffffffu, mag);
        uint32_t bal = __ballot_sync(0xffffffffu, mag == b);
        uint32_t w = __shfl_sync(0xffffffffu, c, __ffs(bal) - 1);
        mag = (mag ^ w) * 2654435761u;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = (uint32_t)(t1 - t0); out[1] = mag; }
}

__global__ void k_imadhi(uint32_t* out, int seed) {
    uint32_t x = threadIdx.x + seed;
    long long t0 = clock64();
    for (int i = 0; i < ITERS; ++i) x = __umulhi(x, 0xD2511F53u) ^ x;
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = (uint32_t)(t1 - t0); out[1] = x; }
}

__global__ void k_fma(uint32_t* out, int seed) {
    float x = threadIdx.x + seed;
    long long t0 = clock64();
    for (int i = 0; i < ITERS; ++i) x = __fmaf_rn(x, 0.999f, 0.5f);
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = (uint32_t)(t1 - t0); out[1] = __float_as_uint(x); }
}

__global__ void k_lds_shfl(uint32_t* out, int seed) {
    // step-like: LDS(id) -> SHFL(tabu word) -> bit test -> REDUX -> REDUX
    __shared__ uint16_t tab[512 * 32];
    for (int i = threadIdx.x; i < 512 * 32; i += 32) tab[i] = (uint16_t)((i * 2654435761u) >> 22);
    __syncwarp();
    uint32_t word = threadIdx.x * 0x01010101u;
    uint32_t cur = seed & 511;
    long long t0 = clock64();
    for (int i = 0; i < ITERS; ++i) {
        uint32_t c = tab[cur * 32 + threadIdx.x];
        uint32_t w = __shfl_sync(0xffffffffu, word, c >> 5);
        uint32_t mag = ((w >> (c & 31)) & 1u) ? 0xffffffffu : (c * 2654435761u) >> 1;
        uint32_t b = __reduce_min_sync(0xffffffffu, mag);
        cur = __reduce_min_sync(0xffffffffu, mag == b ? c : 0xffffffffu) & 511;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = (uint32_t)(t1 - t0); out[1] = cur; }
}

int main() {
    uint32_t* d;
    cudaMalloc(&d, 64);
    uint32_t h[2];
    struct { const char* name; void (*k)(uint32_t*, int); } ks[] = {
        {"LDS chain", k_lds}, {"SHFL.IDX chain", k_shfl}, {"REDUX.MIN chain (+IADD)", k_redux},
        {"warp_select (2x REDUX)", k_redux2}, {"REDUX+BALLOT+FFS+SHFL", k_ballot},
        {"IMAD.HI+LOP chain", k_imadhi}, {"FFMA chain", k_fma}, {"step model LDS->SHFL->2xREDUX", k_lds_shfl}};
    for (auto& k : ks) {
        for (int rep = 0; rep < 2; ++rep) {
            k.k<<<1, 32>>>(d, 1);
            cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
        }
        printf("%-34s %7.1f cycles/iter\n", k.name, (double)h[0] / ITERS);
    }
    return 0;
}
