// micro_halfwarp.cu -- feasibility of two ants per warp (one half-warp each) for the cl = 32
// construction step, against one ant per warp (construct_cl_kernel's layout).
//
// Both variants run the step chain  cur -> LDS row -> tabu SHFL -> key merge -> 2x REDUX.MIN
// -> cur  plus RNGW independent ALU instructions per candidate slot per step (a stand-in for
// the Philox + det_log2 work, which does not depend on cur).  One ant per warp: one slot per
// lane.  Two ants per warp: lanes 0-15 / 16-31 each own 2 slots of their ant; the argmax is a
// local (mag, id) min of the two slots then REDUX.MIN with a half-warp membermask (each half
// passes its own mask -- also checked for correctness against a shuffle reduction).
// Reports cycles per step of one warp (1 or 2 ants) at several warps per SM.
//
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/micro_halfwarp tools/micro_halfwarp.cu
#include <cstdint>
#include <cstdio>

#define STEPS 2000
constexpr int kRows = 1024;
extern __shared__ uint16_t tab[];

template <int RNGW>
__device__ __forceinline__ uint32_t rng_work(uint32_t x) {
#pragma unroll
    for (int r = 0; r < RNGW / 2; ++r) x = (x * 0xD2511F53u) ^ (x >> 7);
    return x;
}

__device__ void fill(float*& inv) {
    inv = reinterpret_cast<float*>(tab + kRows * 32);
    for (int i = threadIdx.x; i < kRows * 32; i += blockDim.x) {
        tab[i] = (uint16_t)(((i * 2654435761u) >> 12) & 1023);
        inv[i] = 1.0f + (i & 255);
    }
    __syncthreads();
}

// one ant per warp (lane = slot)
template <int RNGW>
__global__ void k_full(uint32_t* out, int seed) {
    float* inv;
    fill(inv);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t word = lane * 0x01000001u;
    uint32_t cur = (seed + warp * 7) & 1023;
    uint32_t rs = lane * 77u + warp;
    long long t0 = clock64();
    for (int s = 0; s < STEPS; ++s) {
        const uint32_t c = tab[cur * 32 + lane];
        const float iv = inv[cur * 32 + lane];
        rs = rng_work<RNGW>(rs + s);
        const float L = -1.0f - (float)(rs & 255) * 0.001f;
        const uint32_t key = __float_as_uint(L * iv) & 0x7fffffffu;
        const uint32_t w = __shfl_sync(0xffffffffu, word, c);
        const uint32_t mag = ((w << (~(c >> 5) & 31)) & 0x80000000u) | key;
        const uint32_t b = __reduce_min_sync(0xffffffffu, mag);
        const uint32_t nxt = __reduce_min_sync(0xffffffffu, mag == b ? c : 0xffffffffu);
        if (lane == (int)(nxt & 31)) word ^= 1u << ((nxt >> 5) & 31);
        cur = nxt & 1023;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (uint32_t)(t1 - t0);
    out[64 + blockIdx.x * 32 + warp] = cur;
}

// two ants per warp: half h = lane >> 4 owns ant h; lane l of the half owns slots l, l + 16
template <int RNGW>
__global__ void k_half(uint32_t* out, int seed) {
    float* inv;
    fill(inv);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int h = lane >> 4, hl = lane & 15;
    const uint32_t hmask = h ? 0xFFFF0000u : 0x0000FFFFu;
    // tabu: half h, lane hl holds cities c with (c & 15) == hl: bit (c >> 4) of a 64-bit word
    uint64_t word = (uint64_t)hl * 0x0001000100010001ull;
    uint32_t cur = (seed + warp * 7 + h * 3) & 1023;
    uint32_t rs0 = lane * 77u + warp, rs1 = lane * 91u + warp;
    uint32_t bad = 0;
    long long t0 = clock64();
    for (int s = 0; s < STEPS; ++s) {
        const uint32_t c0 = tab[cur * 32 + hl], c1 = tab[cur * 32 + hl + 16];
        const float iv0 = inv[cur * 32 + hl], iv1 = inv[cur * 32 + hl + 16];
        rs0 = rng_work<RNGW>(rs0 + s);
        rs1 = rng_work<RNGW>(rs1 + s);
        const float L0 = -1.0f - (float)(rs0 & 255) * 0.001f, L1 = -1.0f - (float)(rs1 & 255) * 0.001f;
        const uint32_t k0 = __float_as_uint(L0 * iv0) & 0x7fffffffu, k1 = __float_as_uint(L1 * iv1) & 0x7fffffffu;
        // tabu words of the two candidates: source lane (c & 15) of this half
        const uint32_t wlo = (uint32_t)word, whi = (uint32_t)(word >> 32);
        const int src0 = (h << 4) | (c0 & 15), src1 = (h << 4) | (c1 & 15);
        const uint32_t a0 = __shfl_sync(0xffffffffu, (c0 >> 4) & 32 ? whi : wlo, src0);
        const uint32_t a1 = __shfl_sync(0xffffffffu, (c1 >> 4) & 32 ? whi : wlo, src1);
        const uint32_t m0 = ((a0 >> ((c0 >> 4) & 31)) & 1u) << 31 | k0;
        const uint32_t m1 = ((a1 >> ((c1 >> 4) & 31)) & 1u) << 31 | k1;
        // local (mag, id) min of the two slots
        const bool t1 = (m1 < m0) | ((m1 == m0) & (c1 < c0));
        const uint32_t m = t1 ? m1 : m0, c = t1 ? c1 : c0;
        const uint32_t b = __reduce_min_sync(hmask, m);
        const uint32_t nxt = __reduce_min_sync(hmask, m == b ? c : 0xffffffffu);
        if (s < 64) {   // check the split-mask reductions against shuffles within the half
            uint32_t rb = m, rc = c;
            for (int o = 8; o > 0; o >>= 1) {
                const uint32_t ob = __shfl_xor_sync(0xffffffffu, rb, o), oc = __shfl_xor_sync(0xffffffffu, rc, o);
                if (ob < rb || (ob == rb && oc < rc)) { rb = ob; rc = oc; }
            }
            bad += (rb != b) | (rc != nxt);
        }
        if (hl == (int)(nxt & 15)) word ^= 1ull << ((nxt >> 4) & 63);
        cur = nxt & 1023;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (uint32_t)(t1 - t0);
    if (bad) atomicAdd(out + 1, bad);
    out[64 + blockIdx.x * 32 + warp] = cur;
}

template <class K>
double run(K kern, uint32_t* d, int warps) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kRows * 32 * 6);
    uint32_t h[2];
    for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(d, 0, 8);
        kern<<<148, warps * 32, kRows * 32 * 6>>>(d, 1);
        cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    }
    if (h[1]) printf("  !! %u split-mask reduction mismatches\n", h[1]);
    return (double)h[0] / STEPS;
}

template <int RNGW>
void sweep() {
    uint32_t* d;
    cudaMalloc(&d, 1 << 20);
    printf("RNG stand-in: %d instructions per slot per step\n", RNGW);
    for (int w : {1, 2, 4, 7, 8}) {
        const double f = run(k_full<RNGW>, d, w);
        printf("  one ant / warp : %2d warps/SM (%2d ants/SM): %6.1f cycles/step  -> %6.1f cycles per ant-step per SM\n",
               w, w, f, f / w);
    }
    for (int w : {1, 2, 4}) {
        const double f = run(k_half<RNGW>, d, w);
        printf("  two ants / warp: %2d warps/SM (%2d ants/SM): %6.1f cycles/step  -> %6.1f cycles per ant-step per SM\n",
               w, 2 * w, f, f / (2 * w));
    }
    cudaFree(d);
}

int main() {
    sweep<2>();
    sweep<16>();
    sweep<30>();
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
