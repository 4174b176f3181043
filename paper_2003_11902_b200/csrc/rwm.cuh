// rwm.cuh -- construction with the parallel roulette wheel (PRWM), the node
// selection the paper compares WRS against (Sec. 4.2.1; SURVEY NEXT-1;
// DESIGN.md R28).  Written from the contract in DESIGN.md, independently of the
// oracle.  Included by kernels.cuh after construct.cuh.
#pragma once

namespace mmas {

// choice_info of edge (cur, v): tau^alpha * eta^beta as one fp32 product
__device__ __forceinline__ float rwm_weight(const ConstructArgs& A, size_t rowoff, uint32_t v) {
    return __fmul_rn(pow_alpha(__ldg(A.tau + rowoff + v), A.alpha), __ldg(A.heur + rowoff + v));
}

// PRWM over items 0..len-1 with p = 32 lanes (R28).  wf(i) = weight of item i (0 =
// visited).  Stage: chunk c = ceil(len'/32); lane t sums its chunk sequentially, a
// Hillis-Steele inclusive scan of the 32 sums, r = u * total in the first stage, the
// winner is the first lane with prefix > r and a positive sum (else the last lane with
// a positive sum), r -= the preceding prefix, repeat on the winner's chunk until one
// item is left.  Returns the item (warp-uniform) or -1 when every weight is 0.
template <class WF>
__device__ __forceinline__ int rwm_select(WF&& wf, int len, float u, int lane) {
    int lo = 0, hi = len;
    float r = 0.f;
    bool first = true;
    do {
        const int c = (hi - lo + 31) >> 5;
        const int b = lo + lane * c;
        const int e = min(b + c, hi);
        float acc = 0.f;
        for (int i = b; i < e; ++i) acc = __fadd_rn(acc, wf(i));
        float pre = acc;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const float o = __shfl_up_sync(kFull, pre, d);
            if (lane >= d) pre = __fadd_rn(pre, o);
        }
        if (first) {
            const float total = __shfl_sync(kFull, pre, 31);
            if (total == 0.f) return -1;
            r = __fmul_rn(u, total);
            first = false;
        }
        const uint32_t hit = __ballot_sync(kFull, pre > r && acc > 0.f);
        const int win = hit ? __ffs(hit) - 1 : 31 - __clz(__ballot_sync(kFull, acc > 0.f));
        const float below = __shfl_sync(kFull, pre, (win + 31) & 31);
        if (win > 0) r = __fsub_rn(r, below);
        lo += win * c;
        hi = min(lo + c, hi);
    } while (hi - lo > 1);
    return lo;
}

// One warp per ant.  Bitmask tabu (cand lists / all nodes) or compact tabu (cl = 0,
// R27) in shared memory.  One uniform per step: counter (0x20000000, s, a, it), word 0.
template <bool kCT>
__global__ void __launch_bounds__(128) construct_rwm_kernel(ConstructArgs A) {
    if (blockIdx.y) colony_offset(A, (int)blockIdx.y);
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int n = A.n;
    const int words = kCT ? ((n + 1) >> 1) : ((n + 31) >> 5);     // u32 words per warp
    const int stride = (words + 3) & ~3;
    uint32_t* tabu = reinterpret_cast<uint32_t*>(g_smem + 128) + (size_t)warp * stride;
    uint16_t* ent = reinterpret_cast<uint16_t*>(tabu);
    const uint32_t iter = *A.iter_dev;
    unsigned long long wbest = ~0ull;
    unsigned long long wfb = 0;

    for (int al = blockIdx.x * A.warps_per_block + warp; al < A.m_local; al += gridDim.x * A.warps_per_block) {
        const uint32_t ant = (uint32_t)(A.ant_lo + al);
        if (kCT) {
            for (int i = lane; i < n; i += 32) ent[i] = (uint16_t)i;
        } else {
            for (int i = lane; i < words; i += 32) tabu[i] = 0u;
        }
        __syncwarp();
        const uint32_t start = __umulhi(philox4x32_10(ctr_start(ant, iter), A.key).x, (uint32_t)n);
        if (lane == 0) {
            if (kCT) ct_mark(ent, n, n, start);
            else tabu[start >> 5] |= 1u << (start & 31);
        }
        __syncwarp();
        uint16_t* route = A.routes + (size_t)al * A.ldr;
        uint32_t stage = (lane == 0) ? start : 0u;
        uint32_t cur = start;
        for (int s = 1; s < n; ++s) {
            const float u = uniform_open(philox4x32_10(make_uint4(0x20000000u, (uint32_t)s, ant, iter), A.key).x);
            const size_t rowoff = (size_t)cur * A.ld;
            int nxt = -1;
            if (kCT) {
                const int L = n - s;
                nxt = ent[rwm_select([&](int i) { return rwm_weight(A, rowoff, ent[i]); }, L, u, lane)];
                __syncwarp();
                if (lane == 0) ct_mark(ent, L, n, (uint32_t)nxt);
            } else {
                auto visited = [&](uint32_t v) { return (tabu[v >> 5] >> (v & 31)) & 1u; };
                if (A.cl > 0) {
                    const uint16_t* crow = A.cand_id + (size_t)cur * A.cl;
                    const int k = rwm_select(
                        [&](int k) {
                            const uint32_t c = crow[k];
                            return visited(c) ? 0.f : rwm_weight(A, rowoff, c);
                        },
                        A.cl, u, lane);
                    if (k >= 0) nxt = crow[k];
                    else wfb += (lane == 0);
                }
                if (nxt < 0)
                    nxt = rwm_select([&](int i) { return visited((uint32_t)i) ? 0.f : rwm_weight(A, rowoff, (uint32_t)i); },
                                     n, u, lane);
                __syncwarp();
                if (lane == 0) tabu[nxt >> 5] |= 1u << (nxt & 31);
            }
            stage_route(route, s, (uint32_t)nxt, lane, stage);
            __syncwarp();
            cur = (uint32_t)nxt;
        }
        flush_route(route, n, lane, stage);
        __syncwarp();
        if (!A.skip_finish) wbest = min(wbest, finish_ant(A, route, al, ant, lane));
    }
    pdl_trigger();   // this block is done with its ants: let the next kernel's blocks in
    block_finish(A, wbest, wfb, lane, warp);
}

}  // namespace mmas
