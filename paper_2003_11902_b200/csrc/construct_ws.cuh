// construct_ws.cuh -- warp-specialised candidate-list construction (rows a1-a3, a5-local).
//
// Why: a construction step is a chain of dependent latencies (table LDS -> tabu
// SHFL -> 2 x CREDUX, ~150 cycles), and only ~7 ants share an SM (C2), so each
// SM sub-partition runs < 2 warps.  Each ant's warp also has to produce its
// random keys (one Philox per lane per 4 steps + one det_log2 per lane per step,
// ~35 of its ~70 instructions per step); with in-order issue those instructions
// lengthen the step instead of filling the chain's bubbles.
//
// So every ant gets TWO warps: a consumer warp that runs the selection chain and
// a partner producer warp that computes the log2(u) key factors of the ant's
// candidate slots (R13/R14) into a shared-memory ring ahead of it.
// The two synchronise through two monotonic step counters in shared memory
// (checked once per 8-step chunk).  Results are identical to construct_cl_kernel:
// the same counters, the same det_log2, the same argmax.
#pragma once
#include <cstdint>
#include <type_traits>

namespace mmas {

__device__ __forceinline__ int ld_volatile_s32(const int* p) {
    int v;
    asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_volatile_s32(int* p, int v) {
    asm volatile("st.volatile.shared.s32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_s32(const int* p) {
    int v;
    asm volatile("ld.acquire.cta.shared.s32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}
// acquire-load polling: the ring values read after it are the ones produced before
// the producer's release (fence + counter store)
template <int kSleepNs = 20>
__device__ __forceinline__ void wait_at_least(const int* cnt, int target) {
    while (ld_acquire_s32(cnt) < target) __nanosleep(kSleepNs);
}

constexpr int kRing = 32;    // steps buffered per ant (power of two)
constexpr int kChunk = 8;    // steps per producer hand-off (two Philox groups)

// smem layout:
//   [0, 128)                          mbarrier (+ pad)
//   [128, 128 + Tinv + Tid)           candidate table (kSmemTable)
//   counters: W x {produced, consumed} int32, padded to 16 B
//   ring: W x kRing x (kSlots*32) float
//   tabu: W x nwords u32 (SmemTabu only)
template <int kSlots, bool kSmemTable, bool kRegTabu, bool kFull32>
__global__ void __launch_bounds__(512, 1) construct_ws_kernel(ConstructArgs A) {
    static_assert(!kFull32 || kSlots == 1, "kFull32: cl == 32, one slot per lane");
    using Tabu = typename std::conditional<kRegTabu, RegTabu, SmemTabu>::type;
    constexpr int kRow = kSlots * 32;                 // floats per ring step
    const int lane = threadIdx.x & 31;
    const int W = A.warps_per_block;                  // consumer warps (ants in flight)
    const int wid = threadIdx.x >> 5;
    // producers take the LOW warp ids: the issue arbiter favours higher warp ids, so a
    // consumer (the latency-critical chain) wins every slot it is ready for
    const bool producer = wid < W;
    const int pair = producer ? wid : wid - W;        // the ant slot this warp serves
    const int n = A.n, cl = A.cl;
    const int nwords = (((n + 31) >> 5) + 3) & ~3;
    const int NS = (n + kChunk - 1) / kChunk * kChunk;   // virtual steps per ant
    uint64_t* bar = reinterpret_cast<uint64_t*>(g_smem);
    const uint32_t tab_bytes = kSmemTable ? A.table_bytes_inv + A.table_bytes_id : 0u;
    int* counters = reinterpret_cast<int*>(g_smem + 128 + tab_bytes);
    float* ring_all = reinterpret_cast<float*>(g_smem + 128 + tab_bytes + ((8 * W + 15) & ~15));
    uint32_t* tabu_all = reinterpret_cast<uint32_t*>(ring_all + (size_t)W * kRing * kRow);
    int* produced = counters + 2 * pair;
    int* consumed = counters + 2 * pair + 1;
    float* ring = ring_all + (size_t)pair * kRing * kRow;

    if (threadIdx.x == 0 && kSmemTable) {
        mbar_init(bar, 1);
        mbar_expect_tx(bar, A.table_bytes_inv + A.table_bytes_id);
        constexpr uint32_t kCopy = 32768;
        const uint32_t s_base = smem_u32(g_smem);
        for (uint32_t off = 0; off < A.table_bytes_inv; off += kCopy)
            bulk_g2s(s_base + 128u + off, reinterpret_cast<const unsigned char*>(A.cand_inv) + off,
                     min(kCopy, A.table_bytes_inv - off), bar);
        for (uint32_t off = 0; off < A.table_bytes_id; off += kCopy)
            bulk_g2s(s_base + 128u + A.table_bytes_inv + off, reinterpret_cast<const unsigned char*>(A.cand_id) + off,
                     min(kCopy, A.table_bytes_id - off), bar);
    }
    if (threadIdx.x < 2 * W) counters[threadIdx.x] = 0;
    const uint32_t iter = *A.iter_dev;
    __syncthreads();   // counters zeroed, mbarrier initialised

    unsigned long long wbest = ~0ull;
    long long wfb = 0;
    const int stride = gridDim.x * W;

    if (producer) {
        // ---------------- producer: log2(u) of every candidate slot, kChunk steps at a time
        int k = 0;
        for (int al = blockIdx.x * W + pair; al < A.m_local; al += stride, ++k) {
            const uint32_t ant = (uint32_t)(A.ant_lo + al);
            for (int cs = 0; cs < NS; cs += kChunk) {
                const int v0 = k * NS + cs;
                wait_at_least<200>(consumed, v0 + kChunk - kRing);   // the ring slots are free
#pragma unroll
                for (int gg = 0; gg < kChunk / 4; ++gg) {
                    const uint32_t g = (uint32_t)(cs / 4 + gg);
#pragma unroll
                    for (int q = 0; q < kSlots; ++q) {
                        // R13: slot counter (k, s>>2, a, iter), word s&3 -> steps 4g .. 4g+3
                        const uint4 x = philox4x32_10(ctr_slot((uint32_t)(lane + 32 * q), g, ant, iter), A.key);
                        const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const int v = v0 + 4 * gg + j;
                            ring[(v & (kRing - 1)) * kRow + q * 32 + lane] = det_log2(uniform_open(xs[j]));
                        }
                    }
                }
                __threadfence_block();
                __syncwarp();
                if (lane == 0) st_volatile_s32(produced, v0 + kChunk);
            }
        }
    } else {
        // ---------------- consumer: the ant's selection chain
        uint32_t s_inv = smem_u32(g_smem) + 128u;
        uint32_t s_id = s_inv + A.table_bytes_inv;
        asm volatile("" : "+r"(s_inv), "+r"(s_id));
        const uint32_t id_lane = s_id + 2u * (uint32_t)lane;
        const uint32_t inv_lane = s_inv + 4u * (uint32_t)lane;
        const uint32_t ring_lane = smem_u32(ring) + 4u * (uint32_t)lane;
        uint32_t* tabu_base = tabu_all + (size_t)pair * nwords;
        if (kSmemTable) mbar_wait(bar, 0);
        int k = 0;
        for (int al = blockIdx.x * W + pair; al < A.m_local; al += stride, ++k) {
            const uint32_t ant = (uint32_t)(A.ant_lo + al);
            Tabu tabu;
            tabu.init(tabu_base, nwords, lane);
            const uint32_t start = __umulhi(philox4x32_10(ctr_start(ant, iter), A.key).x, (uint32_t)n);
            tabu.mark(start, lane);
            tabu.sync();
            uint16_t* route = A.routes + (size_t)al * A.ldr;
            uint32_t stage = (lane == 0) ? start : 0u;
            uint32_t cur = start;
            long long fb = 0;
            const int vbase = k * NS;
            auto cstep = [&](int s) {
                const int v = vbase + s;
                const uint32_t rbase = ring_lane + 4u * (uint32_t)((v & (kRing - 1)) * kRow);
                uint32_t bm = kNone, bc = kNone;
                if constexpr (kFull32) {
                    uint32_t c;
                    float iv;
                    if (kSmemTable) {
                        c = lds_u16(id_lane + cur * 64u);
                        iv = lds_f32(inv_lane + cur * 128u);
                    } else {
                        c = __ldg(A.cand_id + cur * 32u + lane);
                        iv = __ldg(A.cand_inv + cur * 32u + lane);
                    }
                    const float L = lds_f32(rbase);
                    const uint32_t t = tabu.top_bit(c);
                    bm = (__float_as_uint(__fmul_rn(L, iv)) & 0x7FFFFFFFu) | (t & 0x80000000u);
                    bc = c;
                } else {
#pragma unroll
                    for (int q = 0; q < kSlots; ++q) {
                        const int slot = lane + 32 * q;
                        const bool has = slot < cl;
                        const int idx = (int)cur * cl + (has ? slot : 0);
                        uint32_t c;
                        float iv;
                        if (kSmemTable) {
                            c = lds_u16(s_id + 2u * (uint32_t)idx);
                            iv = lds_f32(s_inv + 4u * (uint32_t)idx);
                        } else {
                            c = __ldg(A.cand_id + idx);
                            iv = __ldg(A.cand_inv + idx);
                        }
                        const float L = lds_f32(rbase + 128u * q);
                        const bool vis = tabu.visited(has ? c : cur);
                        const uint32_t mag = vis ? kNone : key_magnitude(__fmul_rn(L, iv));
                        if (mag < bm || (mag == bm && c < bc)) {
                            bm = mag;
                            bc = c;
                        }
                    }
                }
                const uint32_t best = __reduce_min_sync(kFull, bm);
                uint32_t nxt = __reduce_min_sync(kFull, bm == best ? bc : kNone);
                if (__builtin_expect(best >= 0x80000000u, 0)) {   // R9 fallback (row a3)
                    ++fb;
                    const float* row = A.inv_w + (size_t)cur * A.ld;
                    nxt = A.fallback_argmax
                              ? fallback_select<true>(row, tabu, n, (uint32_t)s, ant, iter, A.key, lane)
                              : fallback_select<false>(row, tabu, n, (uint32_t)s, ant, iter, A.key, lane);
                }
                tabu.mark(nxt, lane);
                stage_route(route, s, nxt, lane, stage);
                tabu.sync();
                cur = nxt;
            };
            // chunk hand-off: give back the previous chunk, wait until this one is produced
            auto handoff = [&](int c0) {
                if (lane == 0 && c0 > 0) st_volatile_s32(consumed, vbase + c0);
                wait_at_least(produced, vbase + c0 + kChunk);
            };
            // chunk 0 (holds s = 0) and the ragged last chunk are guarded; the others are
            // straight-line code (8 unrolled steps, no branch but the rare fallback)
            const int last_c0 = (n - 1) / kChunk * kChunk;
            handoff(0);
#pragma unroll
            for (int j = 1; j < kChunk; ++j)
                if (j < n) cstep(j);
            int c0 = kChunk;
            for (; c0 < last_c0; c0 += kChunk) {
                handoff(c0);
#pragma unroll
                for (int j = 0; j < kChunk; ++j) cstep(c0 + j);
            }
            if (c0 == last_c0 && last_c0 > 0) {
                handoff(c0);
#pragma unroll
                for (int j = 0; j < kChunk; ++j)
                    if (c0 + j < n) cstep(c0 + j);
            }
            if (lane == 0) st_volatile_s32(consumed, vbase + NS);   // the whole ant is consumed
            flush_route(route, n, lane, stage);
            __syncwarp();
            if (!A.skip_finish) wbest = min(wbest, finish_ant(A, route, al, ant, lane));
            wfb += fb;
        }
    }
    block_finish(A, wbest, wfb, lane, wid - W);   // select runs on consumer warp 0 (wid - W == 0)
}

}  // namespace mmas
