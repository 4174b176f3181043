// two_opt.cuh -- row a8: 2-opt local search on every ant's route (Sec. 5.7,
// PAPER.md P:1727-1744; Bentley 1992), written from DESIGN.md R25.
//
// One warp per ant.  The paper lets several warps search for an improving pair
// of edges and "any" that succeeds applies its move; which one wins depends on
// the schedule, so here the search order is fixed instead (R25): the active
// nodes form a FIFO queue, and for the popped node a the warp evaluates all of
// a's neighbour-list moves in both tour directions AT ONCE (lane k = the k-th
// nearest neighbour c of a), then takes the first improving one in the
// sequential (direction, k) order with a ballot + find-first-set.  The move is
// applied by all 32 lanes reversing disjoint position pairs of the shorter side.
#pragma once
#include <cstdint>

namespace mmas {

struct TwoOptArgs {
    const double2* __restrict__ xy;
    const short2* __restrict__ xys;    // integral coordinates, |x|, |y| <= 16383 (kIntXY kernels), else null
    const int32_t* __restrict__ nnd;   // n x K: d(a, nn[a][k]) (setup, exact R12 distances)
    const uint32_t* __restrict__ nnp;  // kIntXY: n x K packed nn[a][k] | d(a, nn[a][k]) << 16 (d < 46339)
    const uint16_t* __restrict__ nn;   // n x K neighbour lists (R10 order)
    int n, K, ldr, m_local, warps_per_block, nwords;
    uint16_t* routes;                  // m_local x ldr (in: constructed routes; out: improved)
    uint16_t* pos;                     // m_local x ldr scratch
    uint16_t* queue;                   // m_local x ldr scratch
    uint32_t* inq;                     // m_local x nwords scratch ("don't-look bit" clear <=> queued)
    unsigned long long* moves;         // total applied moves (stats)
};
__device__ __forceinline__ void colony_offset(TwoOptArgs& T, ConstructArgs& A, int c) {
    T.routes += c * A.cs.routes;
    T.pos += c * A.cs.routes;
    T.queue += c * A.cs.routes;
    T.inq += (long long)c * A.cs.inq;
    colony_offset(A, c);
}

// ---- coordinates and EUC_2D distances of the local search (euc2d_int: kernels.cuh) ----
template <bool kInt>
struct Pts;
template <>
struct Pts<false> {
    using P = double2;
    const double2* __restrict__ p;
    __device__ __forceinline__ explicit Pts(const TwoOptArgs& T) : p(T.xy) {}
    __device__ __forceinline__ P at(int i) const { return __ldg(p + i); }
    __device__ __forceinline__ static int64_t dist(P a, P b) { return euc2d(a, b); }
};
template <>
struct Pts<true> {
    using P = short2;
    const short2* __restrict__ p;
    __device__ __forceinline__ explicit Pts(const TwoOptArgs& T) : p(T.xys) {}
    __device__ __forceinline__ P at(int i) const { return __ldg(p + i); }
    __device__ __forceinline__ static int64_t dist(P a, P b) { return euc2d_int(a, b); }
};

// integral coordinates staged in shared memory (two_opt_group_kernel): one LDS per point
struct PtsSmem {
    using P = short2;
    uint32_t base;   // shared-window address of the n short2
    __device__ __forceinline__ P at(int i) const {
        uint32_t v;
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(base + 4u * (uint32_t)i));
        return make_short2((short)(v & 0xFFFFu), (short)(v >> 16));
    }
    __device__ __forceinline__ static int64_t dist(P a, P b) { return euc2d_int(a, b); }
};

// neighbour k of a and d(a, it): one 4-byte load of the packed table (integer path), else two
template <bool kInt>
__device__ __forceinline__ void load_nbr(const TwoOptArgs& T, int a, int k, int& c, int64_t& d) {
    if (kInt) {
        const uint32_t v = __ldg(T.nnp + (size_t)a * T.K + k);
        c = (int)(v & 0xFFFFu);
        d = (int64_t)(v >> 16);
    } else {
        c = T.nn[(size_t)a * T.K + k];
        d = __ldg(T.nnd + (size_t)a * T.K + k);
    }
}

__device__ __forceinline__ int wrap_inc(int i, int n) { return i + 1 == n ? 0 : i + 1; }
__device__ __forceinline__ int wrap_dec(int i, int n) { return i == 0 ? n - 1 : i - 1; }

// Reverse the forward cyclic segment i..j of the route, or its complement when that is
// strictly shorter (R25).  Lanes swap disjoint position pairs.
__device__ __forceinline__ void warp_reverse(uint16_t* route, uint16_t* pos, int n, int i, int j, int lane) {
    int len = j - i;
    if (len < 0) len += n;
    len += 1;
    if (2 * len > n) {
        const int ni = wrap_inc(j, n), nj = wrap_dec(i, n);
        i = ni;
        j = nj;
        len = n - len;
    }
    for (int k = lane; k < len / 2; k += 32) {
        int p = i + k;
        if (p >= n) p -= n;
        int q = j - k;
        if (q < 0) q += n;
        const uint16_t vp = route[p], vq = route[q];
        route[p] = vq;
        route[q] = vp;
        pos[vq] = (uint16_t)p;
        pos[vp] = (uint16_t)q;
    }
    __syncwarp();
}

// Local search of one route (the whole warp).  Returns the number of applied moves.
template <bool kInt>
__device__ __forceinline__ long long two_opt_route(const TwoOptArgs& T, uint16_t* route, uint16_t* pos,
                                                   uint16_t* queue, uint32_t* inq, int lane) {
    const int n = T.n, K = T.K;
    const Pts<kInt> X(T);
    using P = typename Pts<kInt>::P;
    for (int i = lane; i < n; i += 32) pos[route[i]] = (uint16_t)i;
    long long moves = 0, sweep_moves;
    do {
        // (re-)seed the queue with every node in route order
        for (int i = lane; i < n; i += 32) queue[i] = route[i];
        for (int w = lane; w < T.nwords; w += 32) inq[w] = 0xFFFFFFFFu;
        __syncwarp();
        int head = 0, count = n;
        sweep_moves = 0;
        // the static data of a popped node (its neighbour list entry per lane and the
        // coordinates) is loaded one pop AHEAD, behind the current pop's work
        int a = queue[0];
        int c = a;
        int64_t dac = 0;
        if (lane < K) load_nbr<kInt>(T, a, lane, c, dac);
        P xa = X.at(a), xc = X.at(c);
        while (count > 0) {
            head = wrap_inc(head, n);
            --count;
            if (lane == 0) atomicAnd(inq + (a >> 5), ~(1u << (a & 31)));   // fire-and-forget (RED), no load on the pop path
            const bool ahead = count > 0;                  // the next pop is already queued
            const int a2 = ahead ? (int)queue[head] : a;
            const int pa = pos[a];
            const int sa = route[wrap_inc(pa, n)];      // successor of a
            const int pr = route[wrap_dec(pa, n)];      // predecessor of a
            int c2 = a2;
            int64_t dac2 = 0;
            if (lane < K) load_nbr<kInt>(T, a2, lane, c2, dac2);
            const P xa2 = X.at(a2);
            const P xs = X.at(sa), xp = X.at(pr);
            const int64_t d_as = X.dist(xa, xs);
            const int64_t d_ap = X.dist(xa, xp);
            // lane k: the k-th nearest neighbour c of a, in both directions
            bool imp_s = false, imp_p = false;
            int sc = 0, pc = 0;
            const P xc2 = X.at(c2);
            if (lane < K) {
                const int64_t d_ac = dac;
                const int qc = pos[c];
                sc = route[wrap_inc(qc, n)];
                pc = route[wrap_dec(qc, n)];
                if (d_ac < d_as && c != sa && sc != a) {   // Bentley pruning + degenerate moves
                    const P xsc = X.at(sc);
                    imp_s = d_ac + X.dist(xs, xsc) - d_as - X.dist(xc, xsc) < 0;
                }
                if (d_ac < d_ap && c != pr && pc != a) {
                    const P xpc = X.at(pc);
                    imp_p = d_ac + X.dist(xp, xpc) - d_ap - X.dist(xc, xpc) < 0;
                }
            }
            // the pruning is a prefix of k (lists are sorted by d(a, .)), so "first improving
            // in (direction, k) order" is the lowest improving lane of the successor direction,
            // else of the predecessor direction
            const uint32_t ms = __ballot_sync(kFull, imp_s);
            const uint32_t mp = __ballot_sync(kFull, imp_p);
            if (ms | mp) {
                const int dir = ms ? 0 : 1;
                const int kk = __ffs(ms ? ms : mp) - 1;
                const int cc = __shfl_sync(kFull, c, kk);
                const int dd = __shfl_sync(kFull, dir == 0 ? sc : pc, kk);
                const int b = dir == 0 ? sa : pr;
                if (dir == 0)   // edges (a,b),(c,d) -> (a,c),(b,d): reverse b .. c
                    warp_reverse(route, pos, n, pos[b], pos[cc], lane);
                else            // edges (b,a),(d,c) -> (b,d),(a,c): reverse a .. d
                    warp_reverse(route, pos, n, pos[a], pos[dd], lane);
                // enqueue a, b, c, d in that order (four distinct nodes: c != a, c != b,
                // d != a and b != d for a valid move), all queued-bits read up front
                const int ends[4] = {a, b, cc, dd};
                uint32_t w4[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) w4[e] = inq[ends[e] >> 5];
                __syncwarp();
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int v = ends[e];
                    const uint32_t bit = 1u << (v & 31);
                    if (!(w4[e] & bit)) {
                        int t = head + count;
                        if (t >= n) t -= n;
                        if (lane == 0) {
                            queue[t] = (uint16_t)v;
                            atomicOr(inq + (v >> 5), bit);   // two endpoints may share a word
                        }
                        ++count;
                    }
                }
                __syncwarp();
                ++sweep_moves;
            }
            __syncwarp();
            if (ahead) {
                a = a2;
                c = c2;
                dac = dac2;
                xa = xa2;
                xc = xc2;
            } else if (count > 0) {   // the queue had run empty: the next pop was just enqueued
                a = queue[head];
                c = a;
                dac = 0;
                if (lane < K) load_nbr<kInt>(T, a, lane, c, dac);
                xa = X.at(a);
                xc = X.at(c);
            }
        }
        moves += sweep_moves;
    } while (sweep_moves > 0);
    return moves;
}

}  // namespace mmas

namespace mmas {

// Row a8 over every ant of the shard, then the per-ant length and the block-level
// iteration-best bookkeeping (row a5) on the IMPROVED routes (R26: the local-search
// output replaces the ant's tour).
template <bool kInt>
__global__ void __launch_bounds__(128) two_opt_kernel(TwoOptArgs T, ConstructArgs A) {
    if (blockIdx.y) colony_offset(T, A, (int)blockIdx.y);
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    unsigned long long wbest = ~0ull;
    long long moves = 0;
    for (int al = blockIdx.x * T.warps_per_block + warp; al < T.m_local; al += gridDim.x * T.warps_per_block) {
        uint16_t* route = T.routes + (size_t)al * T.ldr;
        moves += two_opt_route<kInt>(T, route, T.pos + (size_t)al * T.ldr, T.queue + (size_t)al * T.ldr,
                               T.inq + (size_t)al * T.nwords, lane);
        __syncwarp();
        wbest = min(wbest, finish_ant(A, route, al, (uint32_t)(A.ant_lo + al), lane));
    }
    if (lane == 0 && moves) atomicAdd(T.moves, (unsigned long long)moves);
    pdl_trigger();   // this block is done with its ants: let the next kernel's blocks in
    block_finish(A, wbest, 0, lane, warp);
}

}  // namespace mmas

namespace mmas {

}  // namespace mmas

namespace mmas {

// ---------------------------------------------------------------------------
// Cooperative 2-opt: one BLOCK of kLsWarps warps per ant, route + pos in shared
// memory.  Speculative parallel FIFO: in each round warp w evaluates the w-th
// queued node on the SAME route; the results are then taken in queue order up
// to and including the first improving one (exactly what the sequential FIFO of
// R24 would do, since nothing changes the route until that move), the rest are
// discarded and re-evaluated in the next round.  ~3/4 of the pops find no move,
// so a round retires several pops for the latency of one evaluation; the
// reversal of an applied move is spread over all kLsWarps * 32 lanes.
// ---------------------------------------------------------------------------
#ifndef MMAS_LS_WARPS
#define MMAS_LS_WARPS 5   // warps per ant (sweep on C5: 2: 192, 3: 158, 4: 147, 5: 143, 6: 145, 8: 150, 12: 187, 16: 221 ms)
#endif
constexpr int kLsWarps = MMAS_LS_WARPS;   // (MMAS_LS_WARPS: A/B builds)

struct MoveEval {
    int found, dir, b, c, d;
    int i, j;   // the forward segment to reverse (before the shorter-side choice), read during
                // the evaluation so the apply step needs no position reads (and no barrier)
};
// Shared-memory form (16 B: found, b | c << 16, d, i | j << 16).  The size matters: three
// 76.4 KB blocks per SM (C5) leave only ~350 B of static shared memory per block.
__device__ __forceinline__ uint4 pack_eval(const MoveEval& m) {
    return make_uint4((uint32_t)m.found, (uint32_t)m.b | ((uint32_t)m.c << 16), (uint32_t)m.d,
                      (uint32_t)m.i | ((uint32_t)m.j << 16));
}

// Evaluate node a on the current route (one warp).  Lane k: the k-th neighbour.
// d(a, c) comes from the setup's neighbour-distance table (loaded with the neighbour id).
template <bool kInt, class Xs>
__device__ __forceinline__ MoveEval eval_node(const TwoOptArgs& T, const Xs& X, const uint16_t* route,
                                              const uint16_t* pos, int a, int lane) {
    const int n = T.n, K = T.K;
    using P = typename Xs::P;
    int c = a, sc = 0, pc = 0;
    int64_t d_ac = 0;
    if (lane < K) load_nbr<kInt>(T, a, lane, c, d_ac);
    const int pa = pos[a];
    const int sa = route[wrap_inc(pa, n)];
    const int pr = route[wrap_dec(pa, n)];
    const P xs = X.at(sa), xp = X.at(pr), xa = X.at(a);
    const P xc = X.at(c);
    const int64_t d_as = X.dist(xa, xs);
    const int64_t d_ap = X.dist(xa, xp);
    bool imp_s = false, imp_p = false;
    if (lane < K) {
        const int qc = pos[c];
        sc = route[wrap_inc(qc, n)];
        pc = route[wrap_dec(qc, n)];
        if (d_ac < d_as && c != sa && sc != a) {   // Bentley pruning + degenerate moves
            const P xsc = X.at(sc);
            imp_s = d_ac + X.dist(xs, xsc) - d_as - X.dist(xc, xsc) < 0;
        }
        if (d_ac < d_ap && c != pr && pc != a) {
            const P xpc = X.at(pc);
            imp_p = d_ac + X.dist(xp, xpc) - d_ap - X.dist(xc, xpc) < 0;
        }
    }
    const uint32_t ms = __ballot_sync(kFull, imp_s);
    const uint32_t mp = __ballot_sync(kFull, imp_p);
    MoveEval m{0, 0, 0, 0, 0, 0, 0};
    if (ms | mp) {
        m.found = 1;
        m.dir = ms ? 0 : 1;
        const int kk = __ffs(ms ? ms : mp) - 1;
        m.c = __shfl_sync(kFull, c, kk);
        m.d = __shfl_sync(kFull, m.dir == 0 ? sc : pc, kk);
        m.b = m.dir == 0 ? sa : pr;
        const int qk = __shfl_sync(kFull, lane < K ? (int)pos[c] : 0, kk);
        // dir 0: reverse b .. c = pos[a]+1 .. pos[c];  dir 1: reverse a .. d = pos[a] .. pos[c]-1
        m.i = m.dir == 0 ? wrap_inc(pa, n) : pa;
        m.j = m.dir == 0 ? qk : wrap_dec(qk, n);
    }
    return m;
}

// One ant's cooperative 2-opt by a group of kLsWarps warps (tid, warp: within the group),
// synchronised by `sync` (the block barrier, or the group's named barrier).
template <bool kInt, class Xs, class Sync>
__device__ __forceinline__ long long coop_route(const TwoOptArgs& T, const Xs& X, uint16_t* route, uint16_t* queue,
                                                uint16_t* s_route, uint16_t* s_pos, uint32_t* inq, uint4* s_eval,
                                                int* s_ctl, int tid, int nthr, int lane, int warp, Sync sync) {
    const int n = T.n;
    long long moves = 0;
    for (int i = 2 * tid; i < T.ldr; i += 2 * nthr)
        *reinterpret_cast<uint32_t*>(s_route + i) = *reinterpret_cast<const uint32_t*>(route + i);
    sync();
    for (int i = tid; i < n; i += nthr) s_pos[s_route[i]] = (uint16_t)i;
    int sweep_moves;
    do {
        // (re-)seed the queue with every node in route order
        for (int i = tid; i < n; i += nthr) queue[i] = s_route[i];
        for (int w = tid; w < T.nwords; w += nthr) inq[w] = 0xFFFFFFFFu;
        if (tid == 0) {
            s_ctl[0] = 0;
            s_ctl[1] = n;
            s_ctl[2] = 0;
        }
        sync();
        while (true) {
            const int head = s_ctl[0], count = s_ctl[1];
            if (count == 0) break;
            // warp w evaluates the w-th queued node (all on the same route)
            if (warp < count) {
                int q = head + warp;
                if (q >= n) q -= n;
                const MoveEval m = eval_node<kInt>(T, X, s_route, s_pos, (int)queue[q], lane);
                if (lane == 0) s_eval[warp] = pack_eval(m);
            }
            sync();
            // take the results in queue order up to the first improving one
            const int avail = min(count, kLsWarps);
            uint32_t fmask = 0;
#pragma unroll
            for (int w = 0; w < kLsWarps; ++w) fmask |= (w < avail && s_eval[w].x) ? 1u << w : 0u;
            const int win = fmask ? __ffs(fmask) - 1 : -1;
            const int retired = win >= 0 ? win + 1 : avail;
            if (warp == 0 && lane < retired) {
                int q = head + lane;
                if (q >= n) q -= n;
                const int a = queue[q];
                atomicAnd(inq + (a >> 5), ~(1u << (a & 31)));
            }
            int nhead = head + retired;
            if (nhead >= n) nhead -= n;
            int ncount = count - retired;
            if (tid == 0) trace_ls_round(retired, avail - retired);
            if (win >= 0) {
                const uint4 pe = s_eval[win];
                const int mb = (int)(pe.y & 0xFFFFu), mc = (int)(pe.y >> 16), md = (int)pe.z;
                int q = head + win;
                if (q >= n) q -= n;
                const int a = queue[q];
                // reverse (all lanes of all warps; disjoint pairs); the segment's positions
                // come with the evaluation, so no thread reads pos before it changes
                int i = (int)(pe.w & 0xFFFFu);
                int j = (int)(pe.w >> 16);
                int len = j - i;
                if (len < 0) len += n;
                len += 1;
                if (2 * len > n) {
                    const int ni = wrap_inc(j, n), nj = wrap_dec(i, n);
                    i = ni;
                    j = nj;
                    len = n - len;
                }
                if (tid == 0) trace_ls_len(len);
                for (int k = tid; k < len / 2; k += nthr) {
                    int p = i + k;
                    if (p >= n) p -= n;
                    int qq = j - k;
                    if (qq < 0) qq += n;
                    const uint16_t vp = s_route[p], vq = s_route[qq];
                    s_route[p] = vq;
                    s_route[qq] = vp;
                    s_pos[vq] = (uint16_t)p;
                    s_pos[vp] = (uint16_t)qq;
                }
                // enqueue a, b, c, d in that order (thread 0; the bits of a .. d)
                if (tid == 0) {
                    const int ends[4] = {a, mb, mc, md};
                    __threadfence_block();
                    for (int e = 0; e < 4; ++e) {
                        const int v = ends[e];
                        const uint32_t bit = 1u << (v & 31);
                        if (!(atomicOr(inq + (v >> 5), bit) & bit)) {
                            int t = nhead + ncount;
                            if (t >= n) t -= n;
                            queue[t] = (uint16_t)v;
                            ++ncount;
                        }
                    }
                    s_ctl[2] += 1;
                }
            }
            // every thread read head / count before the first barrier of this round, so
            // thread 0 may publish the next round's values now; one barrier covers both
            // the reversal and the queue state
            if (tid == 0) {
                s_ctl[0] = nhead;
                s_ctl[1] = ncount;
            }
            sync();
        }
        sweep_moves = s_ctl[2];
        moves += sweep_moves;
        sync();
    } while (sweep_moves > 0);
    for (int i = 2 * tid; i < T.ldr; i += 2 * nthr)
        *reinterpret_cast<uint32_t*>(route + i) = *reinterpret_cast<const uint32_t*>(s_route + i);
    sync();
    return moves;
}

template <bool kInt>
__global__ void __launch_bounds__(kLsWarps * 32) two_opt_coop_kernel(TwoOptArgs T, ConstructArgs A) {
    if (blockIdx.y) colony_offset(T, A, (int)blockIdx.y);
    pdl_wait();
    extern __shared__ __align__(16) uint16_t ls_smem[];
    __shared__ uint4 s_eval[kLsWarps];
    __shared__ int s_ctl[4];   // head, count, sweep_moves, winner
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    uint16_t* s_route = ls_smem;
    uint16_t* s_pos = ls_smem + T.ldr;
    uint32_t* inq = reinterpret_cast<uint32_t*>(ls_smem + 2 * T.ldr);   // queued bits (smem atomics)
    const Pts<kInt> X(T);
    unsigned long long wbest = ~0ull;
    long long moves = 0;
    for (int al = blockIdx.x; al < T.m_local; al += gridDim.x) {
        uint16_t* route = T.routes + (size_t)al * T.ldr;
        moves += coop_route<kInt>(T, X, route, T.queue + (size_t)al * T.ldr, s_route, s_pos, inq, s_eval, s_ctl, tid,
                                  (int)blockDim.x, lane, warp, [] { __syncthreads(); });
        if (warp == 0) wbest = min(wbest, finish_ant(A, route, al, (uint32_t)(A.ant_lo + al), lane));
        __syncthreads();
    }
    if (tid == 0 && moves) atomicAdd(T.moves, (unsigned long long)moves);
    pdl_trigger();   // this block is done with its ants: let the next kernel's blocks in
    block_finish(A, wbest, 0, lane, warp);
}

// ---------------------------------------------------------------------------
// Grouped cooperative 2-opt (integral coordinates, large n: C5).  The coordinate loads of an
// evaluation (the popped node's two tour neighbours, each neighbour's successor or
// predecessor) were L2 round trips on its chain: three 76 KB one-ant blocks per SM leave no
// L1 for 74 KB of coordinates.  Here one block holds the coordinates once in shared memory
// and runs kGroups ants side by side (kLsWarps warps each, the group's own named barrier
// 1 + g), each with its own route / pos / queued bits.  Same rounds, same moves.  Measured on
// C5: rounds ~20 % shorter, but two ants per SM instead of three: 125 -> 151 ms; opt-in only.
// Shared memory: coordinates (n short2, 16 B aligned), then per group route, pos, inq.
// ---------------------------------------------------------------------------
constexpr int kLsGroupsMax = 2;
template <int kGroups>
__global__ void __launch_bounds__(kGroups * kLsWarps * 32) two_opt_group_kernel(TwoOptArgs T, ConstructArgs A) {
    if (blockIdx.y) colony_offset(T, A, (int)blockIdx.y);
    pdl_wait();
    extern __shared__ __align__(16) uint16_t ls_smem[];
    __shared__ uint4 s_eval[kGroups][kLsWarps];
    __shared__ int s_ctl[kGroups][4];
    const int n = T.n;
    const int lane = threadIdx.x & 31;
    const int g = (int)(threadIdx.x >> 5) / kLsWarps;
    const int tid = (int)threadIdx.x - g * kLsWarps * 32;
    const int warp = tid >> 5;
    const uint32_t xy_bytes = ((uint32_t)n * 4u + 15u) & ~15u;
    {   // the coordinates, once per block
        const uint32_t* src = reinterpret_cast<const uint32_t*>(T.xys);
        uint32_t* dst = reinterpret_cast<uint32_t*>(ls_smem);
        for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = __ldg(src + i);
    }
    __syncthreads();
    const uint32_t per_ant = (uint32_t)(4 * T.ldr + 4 * T.nwords);
    uint16_t* s_route = reinterpret_cast<uint16_t*>(reinterpret_cast<unsigned char*>(ls_smem) + xy_bytes + g * per_ant);
    uint16_t* s_pos = s_route + T.ldr;
    uint32_t* inq = reinterpret_cast<uint32_t*>(s_pos + T.ldr);
    PtsSmem X;
    X.base = (uint32_t)__cvta_generic_to_shared(ls_smem);
    const int bar = 1 + g;
    auto sync = [bar] { asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(kLsWarps * 32) : "memory"); };
    unsigned long long wbest = ~0ull;
    long long moves = 0;
    for (int al = blockIdx.x * kGroups + g; al < T.m_local; al += gridDim.x * kGroups) {
        uint16_t* route = T.routes + (size_t)al * T.ldr;
        moves += coop_route<true>(T, X, route, T.queue + (size_t)al * T.ldr, s_route, s_pos, inq, s_eval[g], s_ctl[g],
                                  tid, kLsWarps * 32, lane, warp, sync);
        if (warp == 0) wbest = min(wbest, finish_ant(A, route, al, (uint32_t)(A.ant_lo + al), lane));
        sync();
    }
    if (tid == 0 && moves) atomicAdd(T.moves, (unsigned long long)moves);
    pdl_trigger();   // this block is done with its ants: let the next kernel's blocks in
    block_finish(A, wbest, 0, lane, (int)(threadIdx.x >> 5));
}

}  // namespace mmas
