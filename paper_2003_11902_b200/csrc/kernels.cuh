// kernels.cuh -- sm_100a kernels of the MMAS hot path.
//
// Rows of SURVEY.md Sec. 8(a):
//   a1-a3, a5(local)  construct_cl_kernel   one warp per ant, candidate-list WRS
//   a1, a4, a5(local) construct_full_kernel one warp per ant, full-row WRS (cl = 0)
//   a5                select_best_kernel    iteration best / global best / limits
//   a6                pheromone_update_kernel evaporate + deposit + clamp + choice_info
//   a0                setup kernels (heuristic matrix, trail init, candidate gather)
//
// Floating point: every op that feeds a result compared with the oracle is an
// explicit round-to-nearest intrinsic and the TU is compiled with -fmad=false,
// so nothing is contracted or flushed.
#pragma once
#include <cstdint>

#include "rng.cuh"

namespace mmas {

constexpr unsigned kFull = 0xFFFFFFFFu;

// Device-side bounds checks (-DMMAS_CHECKED builds: tools/checked_runs.py; compute-sanitizer is
// not available on the GPU pool).  A failed check records its line in g_check_line and traps,
// so the launch fails with an error instead of reading or writing out of bounds.
#ifdef MMAS_CHECKED
__device__ int g_check_line;
#define MMAS_CHECK(cond)                                   \
    do {                                                   \
        if (!(cond)) {                                     \
            atomicExch(&::mmas::g_check_line, __LINE__);   \
            __threadfence_system();                        \
            __trap();                                      \
        }                                                  \
    } while (0)
#else
#define MMAS_CHECK(cond) \
    do {                 \
    } while (0)
#endif

// Programmatic dependent launch: the iteration's kernels are launched with
// programmatic stream serialisation, so a kernel's blocks are resident before its
// predecessor finishes; each waits here before touching the predecessor's output
// (a no-op when launched without the attribute).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Lets the next kernel on the stream launch its blocks now (they run their prologue up to
// their own pdl_wait).  Construction and 2-opt kernels trigger right after their wait, so the
// update's blocks are resident during the construction tail and prefetch the trails.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
constexpr uint32_t kNone = 0xFFFFFFFFu;

// Device error word of a context (mmas_status): a device-side wait that gave up sets a bit
// and the iteration's selection + update are skipped from then on (the replicas stay at the
// last completed iteration instead of silently diverging).
constexpr uint32_t kErrPeerTimeout = 1u;   // a peer's exchange flag did not arrive (row a7)
constexpr uint32_t kErrGridBarrier = 2u;   // the fused launch's grid barrier did not release
// Default bound of every device-side spin: ~2^34 cycles (~9 s at 1.9 GHz); MMAS_SPIN_BOUND
// (cycles, read at create) overrides it -- the failure-path tests use a short one
constexpr long long kSpinBound = 1ll << 34;
// Epoch word of the fused launch's grid barrier: bit 31 marks an aborted iteration (sticky)
constexpr uint32_t kEpochAbort = 0x80000000u;

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t* p) { return *(const volatile uint32_t*)p; }

// Phase timestamps of construct_cl_kernel (tools/trace_phases.py; only with -DMMAS_TRACE):
// per block [entry, table staged, warp 0's ants done, block_finish done (the last block:
// + selection), barrier released, end], %globaltimer ns, thread 0.  No code otherwise.
#ifdef MMAS_TRACE
__device__ unsigned long long g_trace[1024 * 8];
// per (block, warp): %globaltimer when the warp finished its last ant (tools/trace_warps.py)
__device__ unsigned long long g_trace_w[1024 * 16];
__device__ __forceinline__ void trace_warp_done(int warp, int lane) {
    if (lane == 0 && blockIdx.x < 1024 && warp < 16) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
        g_trace_w[blockIdx.x * 16 + warp] = t;
    }
}
__device__ __forceinline__ void trace_mark(int k) {
    if (threadIdx.x == 0 && blockIdx.x < 1024) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
        g_trace[blockIdx.x * 8 + k] = t;
    }
}
// fallback scans: [0] cycles summed over every fallback (lane 0's clock), [1] their count;
// cooperative 2-opt: [2] rounds, [3] evaluations retired, [4] evaluations discarded behind a winner,
// [5..14] applied reversals by length (log2 buckets: < 2, < 4, ... , >= 512), [15] total length
// [16] compacted fallbacks, [17..19] their phase cycles (count | keys | select); from the
// fallback's start to the compacted scan's entry: ([21] - [22]) / [16] (summed clocks);
// [32 + b] cycles and [40 + b] count of the fallbacks with U unvisited cities, b = the bucket
// U < 16, < 32, ..., < 1024, >= 1024 (U known to the caller: n - step)
__device__ unsigned long long g_fbcyc[64];
__device__ __forceinline__ long long trace_clock() { return clock64(); }
__device__ __forceinline__ void trace_fallback(long long t0, int lane, int unvisited = -1) {
    if (lane == 0) {
        const unsigned long long dt = (unsigned long long)(clock64() - t0);
        atomicAdd(&g_fbcyc[0], dt);
        atomicAdd(&g_fbcyc[1], 1ull);
        if (unvisited > 0) {
            const int b = min(7, max(0, 31 - __clz(unvisited) - 3));
            atomicAdd(&g_fbcyc[32 + b], dt);
            atomicAdd(&g_fbcyc[40 + b], 1ull);
        }
    }
}
__device__ __forceinline__ void trace_compact(int lane, long long t0, long long t1, long long t2, long long t3) {
    if (lane == 0) {
        atomicAdd(&g_fbcyc[16], 1ull);
        atomicAdd(&g_fbcyc[17], (unsigned long long)(t1 - t0));
        atomicAdd(&g_fbcyc[18], (unsigned long long)(t2 - t1));
        atomicAdd(&g_fbcyc[19], (unsigned long long)(t3 - t2));
        atomicAdd(&g_fbcyc[21], (unsigned long long)t0);   // summed entry clocks
    }
}
// [48], [49]: cycles and count of the speculative groups that hit a fallback (the whole group:
// speculation, rollback, fallback scan, generic redo); [50], [51]: the same for clean groups
__device__ __forceinline__ void trace_group(long long t0, int lane, bool hit) {
#ifndef MMAS_TRACE_GROUPS   // (two atomics per group: only in builds that ask for them)
    return;
#endif
    if (lane == 0) {
        atomicAdd(&g_fbcyc[hit ? 48 : 50], (unsigned long long)(clock64() - t0));
        atomicAdd(&g_fbcyc[hit ? 49 : 51], 1ull);
    }
}
__device__ __forceinline__ void trace_compact_entry(int lane, long long t_fb) {
    if (lane == 0) atomicAdd(&g_fbcyc[22], (unsigned long long)t_fb);   // summed fallback start clocks
}
__device__ __forceinline__ void trace_ls_len(int len) {
    const int b = min(9, max(0, 31 - __clz(max(len, 1)) ));
    atomicAdd(&g_fbcyc[5 + b], 1ull);
    atomicAdd(&g_fbcyc[15], (unsigned long long)len);
}
__device__ __forceinline__ void trace_ls_round(int retired, int discarded) {
    atomicAdd(&g_fbcyc[2], 1ull);
    atomicAdd(&g_fbcyc[3], (unsigned long long)retired);
    atomicAdd(&g_fbcyc[4], (unsigned long long)discarded);
}
#else
__device__ __forceinline__ void trace_ls_len(int) {}
__device__ __forceinline__ void trace_ls_round(int, int) {}
__device__ __forceinline__ void trace_mark(int) {}
__device__ __forceinline__ void trace_warp_done(int, int) {}
__device__ __forceinline__ long long trace_clock() { return 0; }
__device__ __forceinline__ void trace_fallback(long long, int, int = -1) {}
__device__ __forceinline__ void trace_compact(int, long long, long long, long long, long long) {}
__device__ __forceinline__ void trace_compact_entry(int, long long) {}
__device__ __forceinline__ void trace_group(long long, int, bool) {}
#endif

// TSPLIB EUC_2D (R12): (int)(sqrt(dx*dx + dy*dy) + 0.5) in double.
__device__ __forceinline__ int32_t euc2d(double2 p, double2 q) {
    const double dx = __dsub_rn(p.x, q.x);
    const double dy = __dsub_rn(p.y, q.y);
    const double r = __dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
    return (int32_t)__dadd_rn(r, 0.5);
}

// Integer EUC_2D (the local search and the lean pheromone's fallback scans):
// kIntXY: every coordinate is an integer with |x|, |y| <= 16383 (checked at setup), so
// S = dx^2 + dy^2 < 2^31 is exact in 32 bits and nint(sqrt(S)) -- the R12 distance, which
// the double formula computes exactly for such S (sqrt(S) is never within 2^-30 of a
// half-integer) -- comes from an approximate sqrt rounded to the nearest integer k0
// (|error| << 1/2 except next to a half-integer) and one integer correction:
// (2k-1)^2 <= 4S < (2k+1)^2  <=>  k^2 - k < S <= k^2 + k   (4S is even, (2k+-1)^2 odd).
// No fp64 (DSQRT is a ~20-instruction subroutine with a long DFMA chain).  Pinned against
// the double formula in tests/test_int_distance.py (exhaustive S <= 2^22, random S < 2^31, and the
// near-half-integer cases k^2 + k, k^2 + k + 1).
__device__ __forceinline__ int32_t euc2d_int(short2 p, short2 q) {
    const int dx = (int)p.x - (int)q.x, dy = (int)p.y - (int)q.y;
    const uint32_t S = (uint32_t)(dx * dx) + (uint32_t)(dy * dy);
    float r;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(__uint2float_rn(S)));
    uint32_t k = (uint32_t)__float2int_rn(r);
    const uint32_t kk = k * k;
    if (kk + k < S) ++k;
    else if (k > 0u && kk - k >= S) --k;
    return (int32_t)k;
}

// tau^alpha for integer alpha (R17) by repeated fp32 multiplication.
__device__ __forceinline__ float pow_alpha(float t, int alpha) {
    if (alpha == 1) return t;
    if (alpha == 0) return 1.0f;
    float p = t;
    for (int k = 1; k < alpha; ++k) p = __fmul_rn(p, t);
    return p;
}

// 1 / choice_info (R19)
__device__ __forceinline__ float inv_weight(float tau, float heur, int alpha) {
    return __fdiv_rn(1.0f, __fmul_rn(pow_alpha(tau, alpha), heur));
}

// eta^beta of edge (p, q) (R11, R12, R18 integer beta): (float)(1.0 / max(d,1)^beta) in double
__device__ __forceinline__ float heur_edge(double2 p, double2 q, int beta) {
    const int32_t d = euc2d(p, q);
    const double D = (double)(d > 1 ? d : 1);
    double Db = 1.0;
    for (int k = 0; k < beta; ++k) Db = __dmul_rn(Db, D);
    return __double2float_rn(__ddiv_rn(1.0, Db));
}

// Keys are strictly negative (log2 u < 0, inv_w > 0), so "largest key" is
// "smallest magnitude": the magnitude bits order like unsigned integers.
// kNone marks "no candidate" (R15: initial key -inf).
__device__ __forceinline__ uint32_t key_magnitude(float key) { return __float_as_uint(key) & 0x7FFFFFFFu; }

// warp-wide argmax over (key, city): returns the winning city (uniform over the
// warp) or kNone when no lane holds a candidate.  Ties -> lowest city id (R16).
__device__ __forceinline__ uint32_t warp_select(uint32_t mag, uint32_t city) {
    const uint32_t best = __reduce_min_sync(kFull, mag);
    if (best == kNone) return kNone;
    return __reduce_min_sync(kFull, mag == best ? city : kNone);
}

// ---------------------------------------------------------------------------
// Concurrent independent colonies (the paper's repeated runs, P:1143-1145,
// and its colony-size study, Sec. 5.4).  A context may hold k colonies: colony c
// is an independent MMAS run with Philox key seed + c (R29), its own trails,
// inv_w, candidate 1/w table, routes, best-so-far and limits; the heuristic matrix, candidate
// ids and coordinates are shared.  Every kernel runs all colonies in one launch with
// blockIdx.y = colony and shifts its per-colony pointers by these strides at entry.
// ---------------------------------------------------------------------------
struct ColonyStride {
    long long nn;      // floats between two colonies' tau (and inv_w) matrices: n * ld
    long long cand;    // floats between two colonies' cand_inv tables
    long long routes;  // u16 between two colonies' route blocks (also 2-opt pos / queue): m_local * ldr
    int ants;          // lengths per colony: m_local
    int vec;           // u16 between two colonies' n-vectors (ib / gb route, succ, pred): ldr
    int inq;           // u32 words of 2-opt queued bits per colony
};
__device__ __forceinline__ PhiloxKey colony_key(PhiloxKey k, uint32_t c) {
    const unsigned long long s = ((unsigned long long)k.k1 << 32 | k.k0) + c;   // R29: seed + c
    return PhiloxKey{(uint32_t)s, (uint32_t)(s >> 32)};
}

// ---------------------------------------------------------------------------
// Iteration best + global best + limits (row a5; Alg. 1), then the
// deposit route's successor / predecessor tables for the update.  Either from
// this context's local best key (world == 1) or from `count` gathered per-rank
// records [u64 key][u16 route[n]] (world > 1).  Run by ONE warp: either the
// last construction warp to finish (world == 1, fused) or select_best_kernel.
// ---------------------------------------------------------------------------
struct SelectArgs {
    const unsigned char* records;  // nullptr = local mode
    int count, rec_bytes;
    unsigned long long* local_key;
    const uint16_t* routes;
    int ldr, ant_lo, n;
    double rho, factor;
    int deposit_global;
    uint16_t* ib_route;
    uint16_t* gb_route;
    long long* gb_len;   // -1 = empty (Alg. 1)
    long long* ib_len;
    int* ib_ant;
    float* scal;         // [tau_min, tau_max, delta]
    uint16_t* succ;
    uint16_t* pred;
    const uint32_t* err;  // split path: skip the selection once the context's error word is set
    ColonyStride cs;      // select_best_kernel: grid.y = colonies
};
__device__ __forceinline__ void colony_offset(SelectArgs& S, int c) {
    const ColonyStride& cs = S.cs;
    S.local_key += c;
    S.routes += c * cs.routes;
    S.ib_route += (long long)c * cs.vec;
    S.gb_route += (long long)c * cs.vec;
    S.gb_len += c;
    S.ib_len += c;
    S.ib_ant += c;
    S.scal += 4 * c;
    S.succ += (long long)c * cs.vec;
    S.pred += (long long)c * cs.vec;
}

__device__ __noinline__ void select_best_warp(const SelectArgs S, int lane) {
    const int n = S.n;
    unsigned long long key = 0;
    const uint16_t* src = nullptr;
    int improved = 0;
    long long gbl = 0;
    if (lane == 0) {
        if (S.records) {
            int bi = 0;
            key = __ldcg(reinterpret_cast<const unsigned long long*>(S.records));
            for (int r = 1; r < S.count; ++r) {
                const unsigned long long k =
                    __ldcg(reinterpret_cast<const unsigned long long*>(S.records + (size_t)r * S.rec_bytes));
                if (k < key) { key = k; bi = r; }
            }
            src = reinterpret_cast<const uint16_t*>(S.records + (size_t)bi * S.rec_bytes + 8);
        } else {
            key = __ldcg(S.local_key);
            src = S.routes + (size_t)((int)(key & 0xFFFFFFu) - S.ant_lo) * S.ldr;
        }
        const long long len = (long long)(key >> 24);
        gbl = __ldcg(S.gb_len);
        improved = (gbl < 0 || len < gbl);   // strictly shorter (R8)
        if (improved) {
            *S.gb_len = len;
            // R2: tau_max = 1/((1-rho) C_gb), tau_min = tau_max * F, clamped <= tau_max
            const double tx = __ddiv_rn(1.0, __dmul_rn(__dsub_rn(1.0, S.rho), (double)len));
            double tn = __dmul_rn(tx, S.factor);
            if (tn > tx) tn = tx;
            S.scal[0] = __double2float_rn(tn);
            S.scal[1] = __double2float_rn(tx);
        }
        const long long dep = S.deposit_global ? (improved ? len : gbl) : len;
        S.scal[2] = __double2float_rn(__ddiv_rn(1.0, (double)dep));   // R6
        *S.ib_len = len;
        *S.ib_ant = (int)(key & 0xFFFFFFu);
        if (!S.records) *S.local_key = ~0ull;
    }
    improved = __shfl_sync(kFull, improved, 0);
    src = reinterpret_cast<const uint16_t*>(__shfl_sync(kFull, reinterpret_cast<unsigned long long>(src), 0));
    // deposit route: the iteration best, or the (possibly just replaced) global best (R7)
    const uint16_t* dep = (!S.deposit_global || improved) ? src : S.gb_route;
    // 4 cities per 8-byte vector (routes and records are 8-byte aligned); every load of
    // the warp is issued before any store, so the copy costs ~one L2 round trip
    constexpr int kVecPerLane = 8;    // n <= 1024 in one pass; larger n loops
    const int nvec = (n + 3) >> 2;
    for (int v0 = 0; v0 < nvec; v0 += 32 * kVecPerLane) {
        uint2 r[kVecPerLane], d[kVecPerLane];
        uint16_t nx[kVecPerLane];
#pragma unroll
        for (int u = 0; u < kVecPerLane; ++u) {
            const int v = v0 + u * 32 + lane;
            if (v < nvec) {
                r[u] = __ldcg(reinterpret_cast<const uint2*>(src) + v);
                d[u] = (dep == src) ? r[u] : __ldcg(reinterpret_cast<const uint2*>(dep) + v);
                const int k = 4 * v + 4;
                nx[u] = __ldcg(dep + (k < n ? k : 0));
            }
        }
#pragma unroll
        for (int u = 0; u < kVecPerLane; ++u) {
            const int v = v0 + u * 32 + lane;
            if (v >= nvec) break;
            if (improved) reinterpret_cast<uint2*>(S.gb_route)[v] = r[u];   // gb <- ib (padding ok: ld >= 4*nvec)
            const uint16_t c[5] = {(uint16_t)(d[u].x & 0xFFFFu), (uint16_t)(d[u].x >> 16),
                                   (uint16_t)(d[u].y & 0xFFFFu), (uint16_t)(d[u].y >> 16), nx[u]};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int k = 4 * v + e;
                if (k >= n) break;
                const uint16_t i = c[e];
                const uint16_t j = (k + 1 < n) ? ((e < 3) ? c[e + 1] : c[4]) : nx[u];
                S.succ[i] = j;
                S.pred[j] = i;
            }
        }
    }
}

// Row a5 by a whole block (the fused launch's last block): thread 0 reads the key and sets
// gb / limits / Delta exactly as select_best_warp does; every thread then copies and links
// a share of the deposit route (succ / pred), so one warp does not issue ~2n scattered
// stores in sequence.  Called by every thread of the block.
__device__ __noinline__ void select_best_block(const SelectArgs S) {
    __shared__ const uint16_t* s_src;
    __shared__ int s_improved;
    const int n = S.n;
    if (threadIdx.x == 0) {
        const unsigned long long key = __ldcg(S.local_key);
        const long long gbl = __ldcg(S.gb_len);
        const uint16_t* src = S.routes + (size_t)((int)(key & 0xFFFFFFu) - S.ant_lo) * S.ldr;
        const long long len = (long long)(key >> 24);
        const int improved = (gbl < 0 || len < gbl);   // strictly shorter (R8)
        if (improved) {
            *S.gb_len = len;
            // R2: tau_max = 1/((1-rho) C_gb), tau_min = tau_max * F, clamped <= tau_max
            const double tx = __ddiv_rn(1.0, __dmul_rn(__dsub_rn(1.0, S.rho), (double)len));
            double tn = __dmul_rn(tx, S.factor);
            if (tn > tx) tn = tx;
            S.scal[0] = __double2float_rn(tn);
            S.scal[1] = __double2float_rn(tx);
        }
        const long long dep = S.deposit_global ? (improved ? len : gbl) : len;
        S.scal[2] = __double2float_rn(__ddiv_rn(1.0, (double)dep));   // R6
        *S.ib_len = len;
        *S.ib_ant = (int)(key & 0xFFFFFFu);
        *S.local_key = ~0ull;
        s_src = src;
        s_improved = improved;
    }
    __syncthreads();
    const uint16_t* src = s_src;
    const int improved = s_improved;
    const uint16_t* dep = (!S.deposit_global || improved) ? src : S.gb_route;
    // gb <- ib first when the deposit route is the old gb (deposit_global && !improved never
    // copies, so dep is never overwritten while it is read)
    for (int k = (int)threadIdx.x; k < n; k += (int)blockDim.x) {
        const uint16_t i = __ldcg(dep + k);
        const uint16_t j = __ldcg(dep + (k + 1 < n ? k + 1 : 0));
        if (improved) S.gb_route[k] = __ldcg(src + k);
        S.succ[i] = j;
        S.pred[j] = i;
    }
}

__global__ void select_best_kernel(SelectArgs S) {
    pdl_wait();
    if (S.err && ld_volatile_u32(S.err)) return;   // a lost peer: no selection (mmas_status)
    if (blockIdx.y) colony_offset(S, (int)blockIdx.y);
    if (threadIdx.x < 32) select_best_warp(S, threadIdx.x);
}

// peer-memory exchange (row a7; see publish_peers_kernel below)
struct ExchangeArgs {
    unsigned char* const* peers;   // device array: every rank's exchange buffer (peer-mapped)
    int world, rank, rec_bytes;
    uint32_t parity, seq;
    long long spin_bound;          // cycles before a wait for a peer's flag gives up (kSpinBound)
};

__device__ __forceinline__ unsigned char* xrecord(unsigned char* buf, const ExchangeArgs& X, int p, int r) {
    return buf + ((size_t)p * X.world + r) * X.rec_bytes;
}
__device__ __forceinline__ uint32_t* xflag(unsigned char* buf, const ExchangeArgs& X, int p, int r) {
    return reinterpret_cast<uint32_t*>(buf + (size_t)2 * X.world * X.rec_bytes) + p * X.world + r;
}

// ---------------------------------------------------------------------------
// Memory-lean pheromone (the O(n^2) pheromone memory is the limit the paper
// names).  EXACT, not an approximation (R30): every trail
// that was never deposited on undergoes the same fp32 operations, so it equals one scalar, the
// background b (b_0 = tau_max; b <- min(max(rho b, tau_min), tau_max) each iteration); and a
// deposited trail equals b again at most L + 1 iterations after its last deposit
// (L = ceil(ln F / ln rho), F = tau_min / tau_max).  So a row keeps its cl candidate trails
// densely and at most 2 (L + 1) other trails (each iteration deposits on <= 2 edges of a row)
// in a small sparse list; every other trail is b, its choice_info recomputed from the
// coordinates (eta^beta by heur_edge).  Memory O(n (cl + cap)) instead of 3 n^2 floats.
// ---------------------------------------------------------------------------
constexpr uint16_t kLeanEmpty = 0xFFFFu;
constexpr uint32_t kErrLeanFull = 4u;    // a sparse row overflowed (the bound makes this impossible)
struct LeanArgs {
    float* cand_tau;         // n x cl_ld: trails of the candidate edges
    const float* cand_heur;  // n x cl_ld: eta^beta of the candidate edges
    uint16_t* sp_id;         // n x cap: off-candidate trails different from b (kLeanEmpty = free)
    float* sp_tau;           // n x cap
    float* sp_inv;           // n x cap: 1 / choice_info of those trails
    float* bg;               // [2]: background trail before (bg[p]) / after (bg[p ^ 1]) this update
    int cap;                 // slots per row (multiple of 32)
    int parity;              // p = iteration & 1
    int beta;
    // integral coordinates with |x|, |y| <= 16383 (else null): the fallback scans take the
    // distance in 32-bit integer arithmetic (euc2d_int, exactly R12) and the background's
    // 1 / choice_info from a table by distance, rewritten by every update for the new b
    const short2* xys;
    const float* heur_tab;   // [dtab]: eta^beta of distance d (R11, R18), setup
    float* inv_tab;          // [dtab]: 1 / (b^alpha eta^beta(d)) for the current background b
    int dtab;
};

// pheromone update arguments (row a6; pheromone_update_kernel below)
struct UpdateArgs {
    float* tau;
    float* inv_w;
    const float* heur;
    int n, ld, alpha;
    float rho_f;
    const float* scal;
    const uint16_t* succ;
    const uint16_t* pred;
    const uint16_t* cand_id;
    float* cand_inv;
    int cl;
    int smem_row;      // 1: the new inv_w row is staged in smem for the cand gather (ld floats fit)
    uint32_t* iter_dev;
    uint32_t* err;     // context error word: set -> the update is skipped (kernel) / set on a
                       // grid-barrier timeout (fused)
    long long spin_bound;  // cycles before the fused launch's grid barrier gives up (kSpinBound)
    ColonyStride cs;       // pheromone_update_kernel: grid.y = colonies
    LeanArgs lean;         // lean_update_kernel (cand_tau != null)
    const double2* xy;     // coordinates (lean: eta^beta of the sparse trails)
};
__device__ __forceinline__ void colony_offset(UpdateArgs& U, int c) {
    const ColonyStride& cs = U.cs;
    U.tau += c * cs.nn;
    U.inv_w += c * cs.nn;
    U.scal += 4 * c;
    U.succ += (long long)c * cs.vec;
    U.pred += (long long)c * cs.vec;
    U.cand_inv += c * cs.cand;
    U.iter_dev += c;
}

// Row a6 on one float4 of row i (columns c0 .. c0+3): evaporation, deposit along the
// succ/pred edges of T_dep, clamp (R1, R4-R6), then 1/choice_info (R19).  Shared by the
// update kernel and the update fused into the construction launch (bit-identical).
__device__ __forceinline__ float4 update_quad(float4& t, float4 h, int c0, int si, int pi, float rho_f, float tmin,
                                              float tmax, float delta, int alpha) {
    float tv[4] = {t.x, t.y, t.z, t.w};
    const float hv[4] = {h.x, h.y, h.z, h.w};
    float wv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int c = c0 + j;
        float v = fmaxf(__fmul_rn(rho_f, tv[j]), tmin);
        if (c == si || c == pi) v = __fadd_rn(v, delta);
        v = fminf(v, tmax);
        tv[j] = v;
        wv[j] = inv_weight(v, hv[j], alpha);
    }
    t = make_float4(tv[0], tv[1], tv[2], tv[3]);
    return make_float4(wv[0], wv[1], wv[2], wv[3]);
}

struct ConstructArgs {
    const double2* __restrict__ xy;
    const float* __restrict__ inv_w;        // n x ld
    const uint16_t* __restrict__ cand_id;   // n x cl
    const float* __restrict__ cand_inv;     // n x cl, = inv_w[i][cand_id[i][k]]
    const uint32_t* __restrict__ iter_dev;  // global iteration counter (R20)
    PhiloxKey key;
    int n, ld, cl, ldr;
    int ant_lo, m_local;
    int fallback_argmax;
    int prune_fallback;          // L2-table kernel: pruned (lagged-threshold) fallback scans
    uint32_t fb_row_off;         // L2-table kernel: shared-memory offset of the fallback row buffer (0 = none)
    int fb_lane_cap;             // lane-compacted fallback (construct.cuh fallback_compact): taken at steps with at
                                 // most this many unvisited cities (0 = the trip scans only)
    int warps_per_block;
    uint32_t table_bytes_inv, table_bytes_id;  // smem-table variant: padded table sizes
    // > 0: every block asks L2 for its share of the inv_w matrix (n x ld f32, this many bytes)
    // at launch start, so the fallback rows (row a3) are L2 hits, not HBM round trips
    unsigned long long l2_prefetch_bytes;
    int coop_fb;                 // L2-table kernel, few ant warps per SM (C5): warps paired, helper scans
    uint16_t* __restrict__ routes;          // m_local x ldr
    long long* __restrict__ lengths;        // m_local
    unsigned long long* __restrict__ best_key;       // local min (len << 24 | ant)
    unsigned long long* __restrict__ fallback_count;
    // world == 1: the last warp to finish runs the iteration-best selection (row a5)
    int fuse_select;
    int skip_finish;             // local search follows: lengths / best keys come from two_opt_kernel
    unsigned int* done;          // ants finished this launch (reset by the last warp)
    SelectArgs sel;
    // roulette-wheel selection (R28) reads choice_info = tau^alpha * heur
    const float* __restrict__ tau;   // n x ld
    const float* __restrict__ heur;  // n x ld
    int alpha;
    // world == 1, persistent shared-memory-table grid: the pheromone update (row a6) runs in
    // the same launch after a grid barrier (construct.cuh fused_update)
    int fuse_update;
    unsigned int* epoch;   // grid-barrier generation word (bumped once per fused launch)
    UpdateArgs upd;
    // world > 1, fused launch (mmas_iterate_exchange): the last block publishes this shard's
    // record to every peer, waits for theirs and selects over them (block_finish)
    int xchg;
    ExchangeArgs X;
    unsigned char* xown;   // this rank's exchange buffer
    uint32_t* xerr;        // set when a peer's flag does not arrive (bounded wait)
    ColonyStride cs;       // colonies (grid.y): per-colony pointer strides
    LeanArgs lean;         // memory-lean pheromone (R30; lean.cand_tau != null): the fallback scans
                           // recompute inv_w rows from the coordinates and the background trail
};
// The arguments of colony c (blockIdx.y) -- every per-colony pointer shifted (R29 key)
__device__ __forceinline__ void colony_offset(ConstructArgs& A, int c) {
    const ColonyStride& cs = A.cs;
    A.inv_w += c * cs.nn;
    A.tau += c * cs.nn;
    A.cand_inv += c * cs.cand;
    A.iter_dev += c;
    A.key = colony_key(A.key, (uint32_t)c);
    A.routes += c * cs.routes;
    A.lengths += (long long)c * cs.ants;
    A.best_key += c;
    A.done += 2 * c;
    A.epoch += 2 * c;
    colony_offset(A.sel, c);
    colony_offset(A.upd, c);
}

}  // namespace mmas

#include "construct.cuh"
#include "rwm.cuh"
#include "two_opt.cuh"

namespace mmas {

// world > 1: copy this shard's best route into its exchange record.
__global__ void publish_kernel(unsigned long long* local_key, const uint16_t* routes, int ldr, int ant_lo, int n,
                               unsigned char* record) {
    __shared__ unsigned long long key;
    if (threadIdx.x == 0) key = *local_key;
    __syncthreads();
    const int al = (int)(key & 0xFFFFFFu) - ant_lo;
    uint16_t* dst = reinterpret_cast<uint16_t*>(record + 8);
    for (int k = threadIdx.x; k < n; k += blockDim.x) dst[k] = routes[(size_t)al * ldr + k];
    __syncthreads();
    if (threadIdx.x == 0) {
        *reinterpret_cast<unsigned long long*>(record) = key;
        *local_key = ~0ull;
    }
}

// ---------------------------------------------------------------------------
// Peer-memory exchange (row a7 without a collective library): every rank's exchange
// buffer holds [2 parities][world] records then [2][world] u32 flags.  Iteration t uses
// parity t & 1 and sequence number t + 1.  A rank writes its record straight into slot
// `rank` of every peer's buffer (NVLink P2P stores; its own buffer included), fences
// system-wide, then raises its flag in every peer.  Double buffering by parity is enough:
// a rank publishes iteration t + 2 only after its update t + 1, which waited for every
// rank's record of t + 1, published after that rank had finished reading iteration t.
// ---------------------------------------------------------------------------
// One block: this shard's best record (key = len << 24 | global ant, route) to every peer.
__global__ void publish_peers_kernel(unsigned long long* local_key, const uint16_t* routes, int ldr, int ant_lo,
                                     int n, int m_local, ExchangeArgs X) {
    pdl_wait();
    __shared__ unsigned long long key;
    if (threadIdx.x == 0) key = m_local > 0 ? *local_key : ~0ull;   // an empty shard never wins
    __syncthreads();
    const int al = (int)(key & 0xFFFFFFu) - ant_lo;
    for (int p = 0; p < X.world; ++p) {
        unsigned char* rec = xrecord(X.peers[p], X, (int)X.parity, X.rank);
        if (m_local > 0) {
            uint16_t* dst = reinterpret_cast<uint16_t*>(rec + 8);
            for (int k = threadIdx.x; k < n; k += blockDim.x) dst[k] = routes[(size_t)al * ldr + k];
        }
        if (threadIdx.x == 0) *reinterpret_cast<volatile unsigned long long*>(rec) = key;
    }
    __syncthreads();
    // one system-scope fence (cumulative over the block barrier) by the thread that then
    // raises the flags: records visible to every peer before any flag
    if (threadIdx.x == 0) {
        __threadfence_system();
        for (int p = 0; p < X.world; ++p) *(volatile uint32_t*)xflag(X.peers[p], X, (int)X.parity, X.rank) = X.seq;
    }
    if (threadIdx.x == 0 && m_local > 0) *local_key = ~0ull;
}

// One warp: wait until every rank's flag of this parity carries this iteration's sequence
// number (bounded: after ~2^34 cycles the error word is set and the wait gives up, so a
// lost peer fails the context instead of hanging the GPU), then acquire.
__global__ void wait_peers_kernel(unsigned char* own, ExchangeArgs X, uint32_t* err) {
    pdl_wait();
    const int r = threadIdx.x;
    if (r < X.world) {
        // the flag is written by another device: acquire at system scope (pairs with the
        // writer's __threadfence_system before its flag store)
        const uint32_t* f = xflag(own, X, (int)X.parity, r);
        const long long t0 = clock64();
        while (ld_acquire_sys(f) != X.seq) {
            if (clock64() - t0 > X.spin_bound) {
                atomicOr(err, kErrPeerTimeout);
                break;
            }
            __nanosleep(200);
        }
    }
    __syncwarp();
    __threadfence_system();
}

// ---------------------------------------------------------------------------
// Pheromone update (row a6; Alg. 1, R1/R4-R6, R22):
//   tau <- min(max(rho tau, tau_min) + Delta [(i,j) in T_dep], tau_max)
//   inv_w <- 1 / (tau^alpha heur);  cand_inv[i][k] <- inv_w[i][cand_id[i][k]]
// One block per row (the paper's evaporation geometry), float4
// streaming; the deposit is the row's succ/pred test, so evaporation and
// deposit fuse into one non-conflicting pass.
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(256) pheromone_update_kernel(UpdateArgs U) {
    extern __shared__ __align__(16) float s_row[];   // new inv_w row (cl > 0: for the gather)
    if (blockIdx.y) colony_offset(U, (int)blockIdx.y);
    const int n4 = (U.n + 3) >> 2;
    // Prologue before the dependency wait: tau, heur and the candidate ids are not written
    // by the construction / 2-opt / selection kernels this one depends on (tau's last writer
    // is the previous update, complete before the construction passed its own wait and
    // triggered this launch), so the first row chunk is fetched while they drain.
    float4 t[4], h[4];
    int cid = 0;
    if ((int)blockIdx.x < U.n) {
        const size_t r0 = (size_t)blockIdx.x * U.ld;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int q = (int)threadIdx.x + u * (int)blockDim.x;
            if (q < n4) {
                t[u] = reinterpret_cast<const float4*>(U.tau + r0)[q];
                h[u] = __ldg(reinterpret_cast<const float4*>(U.heur + r0) + q);
            }
        }
        if (U.cl > 0 && (int)threadIdx.x < U.cl) cid = U.cand_id[(size_t)blockIdx.x * U.cl + threadIdx.x];
    }
    pdl_wait();
    if (U.err && ld_volatile_u32(U.err)) {   // a lost peer: the replica keeps its trails (mmas_status)
        if (blockIdx.x == 0 && threadIdx.x == 0) *U.iter_dev += 1u;
        return;
    }
    const float tmin = U.scal[0], tmax = U.scal[1], delta = U.scal[2];
    bool first = true;
    for (int i = blockIdx.x; i < U.n; i += gridDim.x) {
        const int si = U.succ[i], pi = U.pred[i];
        // candidate ids of the row, loaded before the barrier so the gather does not wait
        if (!first && U.cl > 0 && (int)threadIdx.x < U.cl) cid = U.cand_id[(size_t)i * U.cl + threadIdx.x];
        float4* trow = reinterpret_cast<float4*>(U.tau + (size_t)i * U.ld);
        float4* wrow = reinterpret_cast<float4*>(U.inv_w + (size_t)i * U.ld);
        const float4* hrow = reinterpret_cast<const float4*>(U.heur + (size_t)i * U.ld);
        // up to 4 float4 per thread in flight: all loads first, then compute + store
        for (int q0 = threadIdx.x; q0 < n4; q0 += 4 * blockDim.x) {
            if (!first) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int q = q0 + u * blockDim.x;
                    if (q < n4) {
                        t[u] = trow[q];
                        h[u] = __ldg(hrow + q);
                    }
                }
            }
            first = false;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int q = q0 + u * blockDim.x;
                if (q >= n4) break;
                const float4 w4 = update_quad(t[u], h[u], 4 * q, si, pi, U.rho_f, tmin, tmax, delta, U.alpha);
                trow[q] = t[u];
                wrow[q] = w4;
                if (U.cl > 0 && U.smem_row) reinterpret_cast<float4*>(s_row)[q] = w4;
            }
        }
        first = false;   // the prologue's prefetch belongs to the first row only
        if (U.cl > 0) {
            __syncthreads();
            // cl <= 128; rows too long for smem are gathered from the block's own global writes
            if ((int)threadIdx.x < U.cl)
                U.cand_inv[(size_t)i * U.cl + threadIdx.x] =
                    U.smem_row ? s_row[cid] : U.inv_w[(size_t)i * U.ld + cid];
            __syncthreads();
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *U.iter_dev += 1u;
}

// ---------------------------------------------------------------------------
// Setup kernels (row a0).
// ---------------------------------------------------------------------------
// eta^beta for integer beta (R11, R18): (float)(1 / D^beta), D = max(d, 1).
// Pad columns (n <= c < ld) get 1.0 so every float4 of a row is finite.
// Row a6 in the lean representation (R30): one warp per row i -- the candidate trails, the
// sparse trails (dropped when equal to the new background), then the deposits on edges
// (i, succ i), (i, pred i) that are in neither (inserted at the value the dense update gives
// a trail that was at the background).  Same fp32 operations as update_quad, element by element.
__device__ __forceinline__ float evap_deposit_clamp(float tau, bool dep, float rho_f, float tmin, float tmax,
                                                    float delta) {
    float t = fmaxf(__fmul_rn(rho_f, tau), tmin);
    if (dep) t = __fadd_rn(t, delta);
    return fminf(t, tmax);
}
__global__ void __launch_bounds__(256) lean_update_kernel(UpdateArgs U) {
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int i = (int)(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5));
    const LeanArgs& Ln = U.lean;
    if (U.err && ld_volatile_u32(U.err)) {   // a lost peer: keep the trails (mmas_status)
        if (blockIdx.x == 0 && threadIdx.x == 0) *U.iter_dev += 1u;
        return;
    }
    const float tmin = U.scal[0], tmax = U.scal[1], delta = U.scal[2];
    const float b0 = Ln.bg[Ln.parity];
    const float b1 = evap_deposit_clamp(b0, false, U.rho_f, tmin, tmax, delta);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        Ln.bg[Ln.parity ^ 1] = b1;
        *U.iter_dev += 1u;
    }
    if (Ln.inv_tab)   // the next construction's background 1 / choice_info by distance
        for (int d = blockIdx.x * blockDim.x + threadIdx.x; d < Ln.dtab; d += gridDim.x * blockDim.x)
            Ln.inv_tab[d] = inv_weight(b1, Ln.heur_tab[d], U.alpha);
    if (i >= U.n) return;
    const int si = U.succ[i], pi = U.pred[i];
    bool has_s = false, has_p = false;
    // candidate trails (dense)
    for (int k = lane; k < U.cl; k += 32) {
        const size_t e = (size_t)i * U.cl + k;
        const int c = U.cand_id[e];
        const float t = evap_deposit_clamp(Ln.cand_tau[e], c == si || c == pi, U.rho_f, tmin, tmax, delta);
        Ln.cand_tau[e] = t;
        U.cand_inv[e] = inv_weight(t, Ln.cand_heur[e], U.alpha);
        has_s |= c == si;
        has_p |= c == pi;
    }
    // sparse trails: update, drop the ones equal to the background
    const double2 xi = U.xy[i];
    uint32_t free_mask_lo = 0;   // free slots among the lane's first 32 (bit = slot / 32)
    for (int k = lane; k < Ln.cap; k += 32) {
        const size_t e = (size_t)i * Ln.cap + k;
        const int j = Ln.sp_id[e];
        if (j == kLeanEmpty) {
            free_mask_lo |= 1u << (k >> 5);
            continue;
        }
        const bool dep = j == si || j == pi;
        has_s |= j == si;
        has_p |= j == pi;
        const float t = evap_deposit_clamp(Ln.sp_tau[e], dep, U.rho_f, tmin, tmax, delta);
        if (t == b1) {
            Ln.sp_id[e] = kLeanEmpty;
            free_mask_lo |= 1u << (k >> 5);
        } else {
            Ln.sp_tau[e] = t;
            Ln.sp_inv[e] = inv_weight(t, heur_edge(xi, U.xy[j], Ln.beta), U.alpha);
        }
    }
    has_s = __any_sync(kFull, has_s);
    has_p = __any_sync(kFull, has_p);
    // deposits on trails that were at the background: insert where the result differs from it
    const float tdep = evap_deposit_clamp(b0, true, U.rho_f, tmin, tmax, delta);
    int want[2] = {has_s || si == i ? -1 : si, has_p || pi == i || pi == si ? -1 : pi};
    for (int w = 0; w < 2; ++w) {
        if (want[w] < 0 || tdep == b1) continue;
        // the lowest free slot: (lane, round) with round-major order
        int slot = -1;
        for (int r = 0; r * 32 < Ln.cap && slot < 0; ++r) {
            const unsigned m = __ballot_sync(kFull, (free_mask_lo >> r) & 1u);
            if (m) slot = r * 32 + __ffs(m) - 1;
        }
        if (slot < 0) {
            if (lane == 0) atomicOr(U.err, kErrLeanFull);
            break;
        }
        if (lane == (slot & 31)) {
            free_mask_lo &= ~(1u << (slot >> 5));
            const size_t e = (size_t)i * Ln.cap + slot;
            Ln.sp_id[e] = (uint16_t)want[w];
            Ln.sp_tau[e] = tdep;
            Ln.sp_inv[e] = inv_weight(tdep, heur_edge(xi, U.xy[want[w]], Ln.beta), U.alpha);
        }
        __syncwarp();
    }
}

// Lean setup: the candidate edges' eta^beta, trails tau_max and 1 / choice_info; every
// sparse slot free; background tau_max
__global__ void lean_init_kernel(const double2* __restrict__ xy, int n, int cl, const uint16_t* cand_id, int beta,
                                 int alpha, const float* scal, LeanArgs Ln, float* cand_inv) {
    const float tmax = scal[1];
    const size_t total = (size_t)n * cl;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
        const int i = (int)(e / cl);
        const float h = heur_edge(xy[i], xy[cand_id[e]], beta);
        const_cast<float*>(Ln.cand_heur)[e] = h;
        Ln.cand_tau[e] = tmax;
        cand_inv[e] = inv_weight(tmax, h, alpha);
    }
    const size_t sp = (size_t)n * Ln.cap;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < sp; e += (size_t)gridDim.x * blockDim.x)
        Ln.sp_id[e] = kLeanEmpty;
    if (Ln.inv_tab)
        for (int d = blockIdx.x * blockDim.x + threadIdx.x; d < Ln.dtab; d += gridDim.x * blockDim.x) {
            const double D = (double)(d > 1 ? d : 1);   // heur_edge's arithmetic for distance d
            double Db = 1.0;
            for (int k = 0; k < beta; ++k) Db = __dmul_rn(Db, D);
            const float h = __double2float_rn(__ddiv_rn(1.0, Db));
            const_cast<float*>(Ln.heur_tab)[d] = h;
            Ln.inv_tab[d] = inv_weight(tmax, h, alpha);
        }
    if (blockIdx.x == 0 && threadIdx.x == 0) Ln.bg[0] = Ln.bg[1] = tmax;
}

__global__ void heur_kernel(const double2* __restrict__ xy, int n, int ld, int beta, float* heur) {
    const int i = blockIdx.y;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ld; c += gridDim.x * blockDim.x)
        heur[(size_t)i * ld + c] = c < n ? heur_edge(xy[i], xy[c], beta) : 1.0f;
}

// Nearest-neighbour tour from city 0 (R3; the initial trail limits, Alg. 1):
// one 1024-thread block; per step every thread takes the closest unvisited city among
// j = tid, tid + 1024, ... as a (d, j) key, the block reduces the key to its minimum (ties
// -> lowest id) and thread 0 moves there.  Visited bits in shared memory (n <= 65535).
constexpr int kNnThreads = 1024;   // upper bound; launched with nn_threads(n)
// Nearest-neighbour tour from city 0, ties -> lowest id (R3; Alg. 1).  Setup
// only, but inside bench.py's end-to-end timing (it was ~1 ms of C2's mmas_create and
// ~170 ms of C5's as a block-wide scan per step).
// Candidate fast path (cl > 0): a candidate row holds the row's cl smallest keys (d, id) in
// ascending order (R10, cand_lists_kernel), and every city off the row has a larger key, so
// when the row of the current city has an unvisited entry the FIRST such entry is the exact
// argmin over all unvisited cities.  Warp 0 alone runs those steps (one row read, a tabu test
// per lane, a ballot); only when the whole row is visited does it wake the block (named
// barrier 1) for the full scan: each thread its cities j = tid, tid + T, ... (ascending, so
// ties keep the lower id), 32-bit warp reductions of (d, id) per warp, named barrier 2, warp 0
// combines.  Without candidate lists every step is a full scan.  The tour length is summed
// over the recorded route at the end (exact int64; the order does not matter).
// Dynamic shared memory: route (n u16, rounded to 16 B), then the candidate table when
// `stage_cand` (n x cl_ld u16), else the rows are read from global memory.
__host__ __device__ constexpr int nn_threads(int n) { return n <= 2048 ? 256 : n <= 8192 ? 512 : 1024; }
__device__ __forceinline__ void nn_bar(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__global__ void __launch_bounds__(kNnThreads) nn_tour_kernel(const double2* __restrict__ xy,
                                                             const short2* __restrict__ xys, int n,
                                                             const uint16_t* __restrict__ cand, int cl, int cl_ld,
                                                             int stage_cand, long long* len_out) {
    extern __shared__ __align__(16) uint16_t nn_smem[];
    __shared__ uint32_t vis[2048];
    __shared__ uint32_t s_d[kNnThreads / 32], s_j[kNnThreads / 32];
    __shared__ int s_cur, s_done;
    __shared__ unsigned long long s_len;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5, T = blockDim.x;
    uint16_t* route = nn_smem;
    uint16_t* s_cand = nn_smem + ((n + 7) & ~7);
    const uint16_t* rows = stage_cand ? s_cand : cand;
    for (int w = tid; w < 2048; w += T) vis[w] = 0u;
    if (stage_cand)
        for (int i = tid; i < n * cl_ld; i += T) s_cand[i] = cand[i];
    if (tid == 0) {
        vis[0] = 1u;
        s_cur = 0;
        s_done = 0;
        s_len = 0ull;
        route[0] = 0;
    }
    __syncthreads();
    // one full-scan step from s_cur (every thread; returns the argmin to warp 0)
    auto full_scan = [&]() -> uint32_t {
        const int cur = s_cur;
        const double2 pc = xy[cur];
        const short2 pcs = xys ? xys[cur] : make_short2(0, 0);
        uint32_t bd = kNone, bj = kNone;
        for (int j = tid; j < n; j += T) {   // ascending j: ties keep the lower id
            if ((vis[j >> 5] >> (j & 31)) & 1u) continue;
            // integral coordinates: the exact 32-bit path (euc2d_int == R12), else fp64
            const uint32_t d = (uint32_t)(xys ? euc2d_int(pcs, xys[j]) : euc2d(pc, xy[j]));
            if (d < bd) {
                bd = d;
                bj = (uint32_t)j;
            }
        }
        uint32_t wd = __reduce_min_sync(kFull, bd);
        uint32_t wj = __reduce_min_sync(kFull, bd == wd ? bj : kNone);
        if (lane == 0) {
            s_d[warp] = wd;
            s_j[warp] = wj;
        }
        nn_bar(2, T);
        if (warp != 0) return kNone;
        const uint32_t d = lane < nw ? s_d[lane] : kNone, jj = lane < nw ? s_j[lane] : kNone;
        wd = __reduce_min_sync(kFull, d);
        return __reduce_min_sync(kFull, d == wd ? jj : kNone);
    };
    if (warp == 0) {
        int cur = 0;
        for (int s = 1; s < n; ++s) {
            uint32_t nxt = kNone;
            for (int k0 = 0; k0 < cl && nxt == kNone; k0 += 32) {   // 32 row entries at a time
                const int k = k0 + lane;
                const uint32_t c = k < cl ? (uint32_t)rows[(size_t)cur * cl_ld + k] : 0u;
                const bool fresh = k < cl && !((vis[c >> 5] >> (c & 31)) & 1u);
                const uint32_t m = __ballot_sync(kFull, fresh);
                if (m) nxt = __shfl_sync(kFull, c, __ffs(m) - 1);
            }
            if (nxt == kNone) {   // the whole row is visited (or no lists): the block scans
                if (lane == 0) s_cur = cur;
                nn_bar(1, T);
                nxt = full_scan();
            }
            MMAS_CHECK(nxt < (uint32_t)n && !((vis[nxt >> 5] >> (nxt & 31)) & 1u));
            __syncwarp();
            if (lane == 0) {
                vis[nxt >> 5] |= 1u << (nxt & 31);
                route[s] = (uint16_t)nxt;
            }
            __syncwarp();
            cur = (int)nxt;
        }
        if (lane == 0) s_done = 1;
        nn_bar(1, T);   // release the helpers
    } else {
        while (true) {
            nn_bar(1, T);
            if (s_done) break;
            full_scan();
        }
    }
    __syncthreads();
    // length over the recorded route (R12 distances, exact in int64)
    long long len = 0;
    for (int s = tid; s < n; s += T) {
        const int a = route[s], b = route[s + 1 < n ? s + 1 : 0];
        len += xys ? (long long)euc2d_int(xys[a], xys[b]) : (long long)euc2d(xy[a], xy[b]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) len += __shfl_down_sync(kFull, len, o);
    if (lane == 0) atomicAdd(&s_len, (unsigned long long)len);
    __syncthreads();
    if (tid == 0) *len_out = (long long)s_len;
}

// tau = tau_max (Alg. 1) and inv_w = 1/choice_info.
// Candidate lists (R10): row i's cl nearest cities by (d, id), self excluded -- one block per
// row, the row's distances cached in shared memory, cl rounds of a block-wide minimum of the
// keys d << 32 | j above the previous round's (keys are unique, so no selection flags).
// Setup only (inside bench.py's end-to-end timing; replaces a host pass that spawned threads).
__global__ void __launch_bounds__(256) cand_lists_kernel(const double2* __restrict__ xy, int n, int cl,
                                                         uint16_t* __restrict__ out, int out_ld) {
    extern __shared__ uint32_t s_d[];   // n distances of the row
    __shared__ unsigned long long s_red[8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
        const double2 pi = xy[i];
        for (int j = tid; j < n; j += blockDim.x) s_d[j] = (uint32_t)euc2d(pi, xy[j]);
        __syncthreads();
        unsigned long long prev = 0ull;
        bool first = true;
        for (int k = 0; k < cl; ++k) {
            unsigned long long best = ~0ull;
            for (int j = tid; j < n; j += blockDim.x) {
                if (j == i) continue;
                const unsigned long long key = ((unsigned long long)s_d[j] << 32) | (uint32_t)j;
                if ((first || key > prev) && key < best) best = key;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const unsigned long long v = __shfl_xor_sync(kFull, best, o);
                best = v < best ? v : best;
            }
            if (lane == 0) s_red[warp] = best;
            __syncthreads();
            best = s_red[0];
            for (int w = 1; w < (int)(blockDim.x >> 5); ++w) best = s_red[w] < best ? s_red[w] : best;
            if (tid == 0) out[(size_t)i * out_ld + k] = (uint16_t)(best & 0xFFFFu);
            prev = best;
            first = false;
            __syncthreads();   // s_red reused next round
        }
    }
}

// The same NN tour for n <= 1024 by one warp (C1, C2): the tabu in registers (lane l holds
// cities l, l + 32, ... as bit k of its word, the layout of the construction kernels' candidate
// test), the candidate rows and the coordinates staged in shared memory.  A candidate step is
// a row read, a shuffle per lane and a ballot; an exhausted row is scanned by the warp alone
// (each lane its own unvisited cities, ascending, then (d, id) by two reductions) instead of
// waking a block.  Dynamic shared memory: route (1024 u16), coordinates (n short2 or double2),
// candidate table (n x cl_ld u16).
__global__ void __launch_bounds__(32) nn_tour_warp_kernel(const double2* __restrict__ xy,
                                                          const short2* __restrict__ xys, int n,
                                                          const uint16_t* __restrict__ cand, int cl, int cl_ld,
                                                          long long* len_out) {
    extern __shared__ __align__(16) unsigned char nnw_smem[];
    uint16_t* route = reinterpret_cast<uint16_t*>(nnw_smem);
    const size_t xy_b = xys ? (size_t)n * 4 : (size_t)n * 16;
    short2* s_xys = reinterpret_cast<short2*>(nnw_smem + 2048);
    double2* s_xy = reinterpret_cast<double2*>(nnw_smem + 2048);
    uint16_t* s_cand = reinterpret_cast<uint16_t*>(nnw_smem + 2048 + ((xy_b + 15) & ~(size_t)15));
    const int lane = threadIdx.x;
    // staging in 16-byte pieces, several in flight per lane (one warp moves ~70 KB for C2: u16
    // element copies took most of the kernel)
    auto stage16 = [&](void* dst, const void* src, size_t bytes) {
        const size_t n16 = bytes / 16;
        uint4* d = reinterpret_cast<uint4*>(dst);
        const uint4* g = reinterpret_cast<const uint4*>(src);
        size_t i = lane;
        for (; i + 96 < n16; i += 128) {
            const uint4 a = __ldg(g + i), b = __ldg(g + i + 32), c = __ldg(g + i + 64), e = __ldg(g + i + 96);
            d[i] = a;
            d[i + 32] = b;
            d[i + 64] = c;
            d[i + 96] = e;
        }
        for (; i < n16; i += 32) d[i] = __ldg(g + i);
        const unsigned char* gs = reinterpret_cast<const unsigned char*>(src);
        unsigned char* ds = reinterpret_cast<unsigned char*>(dst);
        for (size_t b = n16 * 16 + lane; b < bytes; b += 32) ds[b] = gs[b];   // (tail bytes)
    };
    if (xys) stage16(s_xys, xys, (size_t)n * 4);
    else stage16(s_xy, xy, (size_t)n * 16);
    if (cl_ld > 0) stage16(s_cand, cand, (size_t)n * cl_ld * 2);
    uint32_t wt = lane == 0 ? 1u : 0u;   // city 0 visited
    const int cnt = (n - lane + 31) >> 5;   // this lane's cities l + 32 k < n
    const uint32_t mine = cnt >= 32 ? 0xFFFFFFFFu : cnt <= 0 ? 0u : (1u << cnt) - 1u;
    if (lane == 0) route[0] = 0;
    __syncwarp();
    // the row stride and this lane's slot in registers (ptxas otherwise reloads them from the
    // constant bank inside the step chain)
    uint32_t row_ld = (uint32_t)cl_ld, slot_ok = lane < cl ? 1u : 0u;
    uint32_t s_base = (uint32_t)__cvta_generic_to_shared(s_cand) + 2u * (uint32_t)lane;
    asm volatile("" : "+r"(row_ld), "+r"(slot_ok), "+r"(s_base));
    int cur = 0;
    for (int s = 1; s < n; ++s) {
        uint32_t nxt = kNone;
        if (cl <= 32) {   // one row read per step (C1, C2)
            uint32_t c = 0u;
            if (slot_ok) asm volatile("ld.shared.u16 %0, [%1];" : "=r"(c) : "r"(s_base + 2u * (uint32_t)cur * row_ld));
            const bool vis = (__shfl_sync(kFull, wt, (int)(c & 31u)) >> (c >> 5)) & 1u;
            const uint32_t m = __ballot_sync(kFull, slot_ok && !vis);
            if (m) nxt = __shfl_sync(kFull, c, __ffs(m) - 1);
        } else {
            for (int k0 = 0; k0 < cl && nxt == kNone; k0 += 32) {
                const int k = k0 + lane;
                const uint32_t c = k < cl ? (uint32_t)s_cand[cur * cl_ld + k] : 0u;
                const bool vis = (__shfl_sync(kFull, wt, (int)(c & 31u)) >> (c >> 5)) & 1u;
                const uint32_t m = __ballot_sync(kFull, k < cl && !vis);
                if (m) nxt = __shfl_sync(kFull, c, __ffs(m) - 1);
            }
        }
        if (nxt == kNone) {   // the row is exhausted (or no lists): the warp scans
            uint32_t bd = kNone, bj = kNone;
            uint32_t f = ~wt & mine;
            if (xys) {
                const short2 pc = s_xys[cur];
                while (__any_sync(kFull, f != 0u)) {   // four cities per lane per trip (ILP)
                    uint32_t j[4], d[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        j[q] = f ? 32u * (uint32_t)(__ffs(f) - 1) + (uint32_t)lane : kNone;
                        f &= f - 1u;
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        d[q] = j[q] != kNone ? (uint32_t)euc2d_int(pc, s_xys[j[q]]) : kNone;
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (d[q] < bd) { bd = d[q]; bj = j[q]; }   // ascending j: ties keep the lower id
                }
            } else {
                const double2 pc = s_xy[cur];
                while (f) {
                    const uint32_t j = 32u * (uint32_t)(__ffs(f) - 1) + (uint32_t)lane;
                    f &= f - 1u;
                    const uint32_t d = (uint32_t)euc2d(pc, s_xy[j]);
                    if (d < bd) { bd = d; bj = j; }
                }
            }
            const uint32_t wd = __reduce_min_sync(kFull, bd);
            nxt = __reduce_min_sync(kFull, bd == wd ? bj : kNone);
        }
        MMAS_CHECK(nxt < (uint32_t)n);
        if (lane == (int)(nxt & 31u)) wt |= 1u << (nxt >> 5);
        if (lane == 0) route[s] = (uint16_t)nxt;
        cur = (int)nxt;
    }
    __syncwarp();
    long long len = 0;
    for (int s = lane; s < n; s += 32) {
        const int a = route[s], b = route[s + 1 < n ? s + 1 : 0];
        len += xys ? (long long)euc2d_int(s_xys[a], s_xys[b]) : (long long)euc2d(s_xy[a], s_xy[b]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) len += __shfl_down_sync(kFull, len, o);
    if (lane == 0) *len_out = len;
}

// 2-opt neighbour distances d(i, nn[i][q]) (R12) and, for integral coordinates, the packed
// entries nn | d << 16 the 2-opt kernels read (row a8 setup; was a host pass)
__global__ void ls_dist_kernel(const double2* __restrict__ xy, int n, int k, const uint16_t* __restrict__ nn,
                               int32_t* __restrict__ nnd, uint32_t* __restrict__ nnp) {
    const long long total = (long long)n * k;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(e / k);
        const uint32_t j = nn[e];
        MMAS_CHECK(j < (uint32_t)n && j != (uint32_t)i);
        const int32_t d = euc2d(xy[i], xy[j]);
        nnd[e] = d;
        if (nnp) nnp[e] = j | ((uint32_t)d << 16);
    }
}

// The same lists for n <= 1024 by one warp per row: lane l keeps the keys d << 10 | j of its
// cities j = l, l + 32, ... in registers (d < 2^22 for |coordinates| < 2^20 -- else the block
// kernel), and each of the cl rounds takes the warp minimum above the previous one (keys are
// unique, so the (d, id) order is the key order).
constexpr int kCandWarpMaxN = 1024;
__global__ void __launch_bounds__(256) cand_lists_warp_kernel(const double2* __restrict__ xy, int n, int cl,
                                                             uint16_t* __restrict__ out, int out_ld) {
    const int lane = threadIdx.x & 31;
    const int gw = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5), nwarps = (int)((gridDim.x * blockDim.x) >> 5);
    for (int i = gw; i < n; i += nwarps) {
        const double2 pi = xy[i];
        uint32_t key[kCandWarpMaxN / 32];
#pragma unroll
        for (int t = 0; t < kCandWarpMaxN / 32; ++t) {
            const int j = lane + 32 * t;
            key[t] = (j < n && j != i) ? ((uint32_t)euc2d(pi, xy[j]) << 10) | (uint32_t)j : kNone;
        }
        uint32_t prev = 0u;
        for (int k = 0; k < cl; ++k) {
            uint32_t best = kNone;
#pragma unroll
            for (int t = 0; t < kCandWarpMaxN / 32; ++t)
                if ((k == 0 || key[t] > prev) && key[t] < best) best = key[t];
            best = __reduce_min_sync(kFull, best);
            if (lane == 0) out[(size_t)i * out_ld + k] = (uint16_t)(best & 0x3FFu);
            prev = best;
        }
    }
}

__global__ void init_trails_kernel(float* tau, float* inv_w, const float* heur, int n, int ld, int alpha,
                                   const float* scal) {
    const int i = blockIdx.y;
    const float tmax = scal[1];
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ld; c += gridDim.x * blockDim.x) {
        const size_t e = (size_t)i * ld + c;
        tau[e] = tmax;
        inv_w[e] = inv_weight(tmax, heur[e], alpha);
    }
}

__global__ void gather_cand_kernel(const float* inv_w, int n, int ld, const uint16_t* cand_id, float* cand_inv,
                                   int cl) {
    const size_t total = (size_t)n * cl;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
        const size_t i = e / cl;
        cand_inv[e] = inv_w[i * ld + cand_id[e]];
    }
}

// ---- test hooks (mmas_debug_*) ----
__global__ void debug_philox_kernel(const uint32_t* ck, long long count, uint32_t* words, float* logs) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
         i += (long long)gridDim.x * blockDim.x) {
        const uint32_t* p = ck + 6 * i;
        const uint4 x = philox4x32_10(make_uint4(p[0], p[1], p[2], p[3]), PhiloxKey{p[4], p[5]});
        const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
        for (int j = 0; j < 4; ++j) {
            words[4 * i + j] = xs[j];
            logs[4 * i + j] = det_log2(uniform_open(xs[j]));
        }
    }
}

__global__ void debug_log2_kernel(const float* u, long long count, float* out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
         i += (long long)gridDim.x * blockDim.x)
        out[i] = det_log2(u[i]);
}

}  // namespace mmas
