// construct.cuh -- tour construction kernels.
//
// One warp = one ant (the paper's data-parallel mapping at warp granularity,
// P:1076-1082; one warp per ant at cl = 32).  A construction is
// n-1 DEPENDENT selections (Alg. 1), so with ~7 ants per SM the
// kernel is bound by the latency of one step, not by bandwidth or issue.  The
// step is therefore laid out as a short dependency chain:
//
//   cur -> LDS (cand id, 1/w) -> tabu test (SHFL of a register bitmask, or LDS)
//       -> key = log2(u) * (1/w) -> CREDUX.MIN (largest key) -> CREDUX.MIN (lowest id) -> cur
//
// and everything that does not depend on `cur` is moved off it: the random
// keys of a candidate slot come from Philox counter (slot, s>>2, ant, iter)
// (R13), so one Philox call per lane covers four steps, and the call
// for the NEXT four steps is computed in slices interleaved with the current
// four steps (software pipelining), where it fills the latency bubbles.
#pragma once
#include <cstdint>
#include <type_traits>

#include "rng.cuh"

namespace mmas {

// ---- bitmask tabu (Sec. 4.1) ------------------------------------------
// n <= 1024: lane j keeps word j in a register; a test is one SHFL, a mark one OR.
// The same bits are also kept transposed (wt: lane j holds cities j, j+32, j+64, ...,
// city c at bit c>>5 of lane c&31) for the candidate test, whose SHFL then takes c itself
// as the source lane (the shuffle uses its low 5 bits) with no shift before it.
// kLazyW (cl == 32 path): only wt is maintained per step; w, which the fallback scan reads,
// is rebuilt from wt by a warp bit-matrix transpose in prepare() when a scan needs it.
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, int lane) {
    // lane i holds row i of a 32x32 bit matrix; returns column `lane` (bit i = row i's bit)
    const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const int j = 16 >> k;
        const uint32_t m = masks[k];
        const uint32_t y = __shfl_xor_sync(kFull, x, j);
        x = (lane & j) ? (((y >> j) & m) | (x & ~m)) : ((x & m) | ((y & m) << j));
    }
    return x;
}
template <bool kLazyW>
struct RegTabuX {
    uint32_t w, wt;
    __device__ __forceinline__ void init(uint32_t*, int, int) { w = 0u; wt = 0u; }
    // every lane of the warp must call word()/visited() (warp shuffle); kLazyW: after prepare()
    __device__ __forceinline__ uint32_t word(int idx) const { return __shfl_sync(kFull, w, idx); }
    // the calling lane's own word (idx == lane; no shuffle)
    __device__ __forceinline__ uint32_t own(int) const { return w; }
    __device__ __forceinline__ bool visited(uint32_t c) const { return (word((int)(c >> 5)) >> (c & 31)) & 1u; }
    // bit 31 = "c visited" (other bits garbage); lanes may pass any c < 1024
    __device__ __forceinline__ uint32_t top_bit(uint32_t c) const {
        return __shfl_sync(kFull, wt, (int)c) << (~(c >> 5) & 31u);
    }
    __device__ __forceinline__ void mark(uint32_t c, int lane) {
        if (!kLazyW && lane == (int)(c >> 5)) w |= 1u << (c & 31);
        if (lane == (int)(c & 31)) wt |= 1u << (c >> 5);
    }
    __device__ __forceinline__ void unmark(uint32_t c, int lane) {
        if (!kLazyW && lane == (int)(c >> 5)) w &= ~(1u << (c & 31));
        if (lane == (int)(c & 31)) wt &= ~(1u << (c >> 5));
    }
    __device__ __forceinline__ void prepare(int lane) {
        if (kLazyW) w = warp_transpose32(wt, lane);
    }
    __device__ __forceinline__ void sync() {}
};
using RegTabu = RegTabuX<false>;

// (a & ~m) | (b & m) in one LOP3
__device__ __forceinline__ uint32_t bit_select(uint32_t a, uint32_t b, uint32_t m) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0xD8;" : "=r"(d) : "r"(a), "r"(b), "r"(m));
    return d;
}
// any n: ceil(n/32) words per warp in shared memory.
struct SmemTabu {
    uint32_t* t;
    __device__ __forceinline__ void init(uint32_t* base, int nwords, int lane) {
        t = base;
        for (int j = lane; j < nwords; j += 32) t[j] = 0u;
        __syncwarp();
    }
    __device__ __forceinline__ uint32_t word(int idx) const { return t[idx]; }
    __device__ __forceinline__ uint32_t own(int idx) const { return t[idx]; }
    __device__ __forceinline__ bool visited(uint32_t c) const { return (t[c >> 5] >> (c & 31)) & 1u; }
    __device__ __forceinline__ uint32_t top_bit(uint32_t c) const { return t[c >> 5] << (~c & 31u); }
    __device__ __forceinline__ void mark(uint32_t c, int lane) {
        if (lane == 0) t[c >> 5] |= 1u << (c & 31);
    }
    __device__ __forceinline__ void unmark(uint32_t c, int lane) {
        if (lane == 0) t[c >> 5] &= ~(1u << (c & 31));
    }
    __device__ __forceinline__ void prepare(int) {}
    __device__ __forceinline__ void sync() { __syncwarp(); }
};

// ---- Philox in slices (rounds [R0, R1)) for software pipelining ----------------------
// Round keys precomputed once per kernel (warp-uniform: they live in uniform registers).
struct RoundKeys {
    uint32_t k0[10], k1[10];
    __device__ __forceinline__ explicit RoundKeys(PhiloxKey key) {
#pragma unroll
        for (int r = 0; r < 10; ++r) {
            k0[r] = key.k0 + (uint32_t)r * 0x9E3779B9u;
            k1[r] = key.k1 + (uint32_t)r * 0xBB67AE85u;
        }
    }
};

template <int R0, int R1>
__device__ __forceinline__ void philox_rounds(uint4& c, const RoundKeys& rk) {
#pragma unroll
    for (int r = R0; r < R1; ++r) {
        // round keys: base key + r * Weyl constant, uniform (UIADD3 on the uniform datapath)
        const uint32_t k0 = rk.k0[0] + (uint32_t)r * 0x9E3779B9u;
        const uint32_t k1 = rk.k1[0] + (uint32_t)r * 0xBB67AE85u;
        const uint32_t lo0 = 0xD2511F53u * c.x;
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    }
}

// ---------------------------------------------------------------------------
// Scan of ALL unvisited cities from `row` (= inv_w[cur]): the full-row WRS step
// (row a4) and the candidate-list fallback (row a3, R9).  Lane l handles the
// 4-city groups 128t + 4l (a coalesced float4 of inv_w and one Philox per group
// whose word j is city 4g+j's uniform, R13); groups whose four cities are all
// visited are skipped.  Per-lane best with ties to the lower id; the caller
// reduces across the warp.
// ---------------------------------------------------------------------------
// Exact pruning of the key computations.  A city's key
// magnitude is |det_log2(u)| * inv_w >= (1 - u) * log2(e) * inv_w, because -ln u >= 1 - u
// and det_log2 is within 1.61 ulp of log2.  With C = log2(e) deflated by 2^-20 (rounded
// down), |det_log2(u)| >= (1-u) C (1+2^-24)^2/(1-2^-24) on the whole u-grid
// (tests/test_oracle_rng.py, exhaustive).  The scans compare a = fl((1-u) inv_w) with the
// scaled threshold T = fl_up(thr * fl_up(1/C)) >= thr / C: a > T implies
// (1-u) inv_w C > thr / (1+2^-24), hence fl(|det_log2(u)| inv_w) > thr (1+2^-24) > thr, so
// the city can neither win nor tie and its det_log2 is not evaluated.  One FMUL per city.
constexpr float kLog2eLow = 1.4426935911178589f;
constexpr float kInvLog2eLowUp = 0.6931478977203369f;   // fl_up(1 / kLog2eLow)

// One 128-city chunk of the scan: lane l's cities c0 .. c0+3, nib = their visited
// bits (bit j set = visited or beyond n).  Keys are evaluated (in increasing city order)
// only for the unvisited cities whose lower bound does not exceed thr.
// kPrune: per-lane survivor branch (full-row scans: 16+ warps per SM hide its latency);
// kWarpPrune (with kPrune): the warp skips a group's logs only when no lane has a survivor,
// and otherwise evaluates all four logs branch-free (ILP 4: the fallback scans of C3 / C5
// run at a few warps per SM, where a serial per-city branch costs more than it saves)
template <bool kArgmax, bool kPrune, bool kWarpPrune = false>
__device__ __forceinline__ void scan_chunk(float4 iv, int c0, uint32_t nib, uint32_t step, uint32_t ant,
                                           uint32_t iter, PhiloxKey key, uint32_t& best_mag, uint32_t& best_c,
                                           float thr) {
    const float ivs[4] = {iv.x, iv.y, iv.z, iv.w};
    if (kArgmax) {
        // R9 flag: the largest weight = the smallest inv_w (positive floats order as uints)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t mag = ((nib >> j) & 1u) ? kNone : __float_as_uint(ivs[j]);
            if (mag < best_mag) { best_mag = mag; best_c = (uint32_t)(c0 + j); }
        }
    } else if (!kPrune) {
        // branch-free: four independent key chains (the fallback scan of the candidate path,
        // whose few warps per SM need the ILP more than the saved work)
        const uint4 x = philox4x32_10(ctr_city((uint32_t)c0 >> 2, step, ant, iter), key);
        const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float k = __fmul_rn(det_log2(uniform_open(xs[j])), ivs[j]);
            const uint32_t mag = ((nib >> j) & 1u) ? kNone : key_magnitude(k);
            if (mag < best_mag) { best_mag = mag; best_c = (uint32_t)(c0 + j); }
        }
    } else {
        // pruned (thr = the scaled threshold T above): one predicate for "any survivor",
        // the keys of the survivors in a rare branch
        const uint4 x = philox4x32_10(ctr_city((uint32_t)c0 >> 2, step, ant, iter), key);
        const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
        float om[4];
        bool keep[4];
        bool any = false;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            om[j] = one_minus_uniform_open(xs[j]);      // 1 - u, exact on the grid
            keep[j] = ((nib >> j) & 1u) == 0u && !(__fmul_rn(om[j], ivs[j]) > thr);
            any |= keep[j];
        }
        if (kWarpPrune) {
            if (__any_sync(kFull, any)) {
                uint32_t mag[4];
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    mag[j] = keep[j] ? key_magnitude(__fmul_rn(det_log2(__fsub_rn(1.0f, om[j])), ivs[j])) : kNone;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (mag[j] < best_mag) { best_mag = mag[j]; best_c = (uint32_t)(c0 + j); }
            }
        } else if (any) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (keep[j]) {
                    const uint32_t mag = key_magnitude(__fmul_rn(det_log2(__fsub_rn(1.0f, om[j])), ivs[j]));
                    if (mag < best_mag) { best_mag = mag; best_c = (uint32_t)(c0 + j); }
                }
            }
        }
    }
}

// the warp's best magnitude so far as the scaled pruning threshold T = fl_up(thr / C)
// (+inf while nothing is found)
__device__ __forceinline__ float warp_threshold(uint32_t best_mag) {
    const uint32_t b = __reduce_min_sync(kFull, best_mag);
    return b == kNone ? __int_as_float(0x7F800000) : __fmul_ru(__uint_as_float(b), kInvLog2eLowUp);
}

// Visited bits of lane l's four cities c0 .. c0+3 (cities >= n count as visited).
template <class Tabu>
__device__ __forceinline__ uint32_t chunk_nibble(const Tabu& tabu, int c0, int n) {
    const uint32_t word = tabu.word(min(c0, n - 1) >> 5);   // all lanes (RegTabu shuffles)
    if (c0 >= n) return 0xFu;
    uint32_t nib = (word >> (c0 & 31)) & 0xFu;
    if (c0 + 4 > n) nib |= (0xFu << (n - c0)) & 0xFu;
    return nib;
}

// ---------------------------------------------------------------------------
// Scan of ALL unvisited cities from `row` (= inv_w[cur]): the full-row WRS step
// (row a4) and the candidate-list fallback (row a3, R9).  Lane l handles the
// 4-city groups 128t + 4l (a coalesced float4 of inv_w and one Philox per group
// whose word j is city 4g+j's uniform, R13).  Two chunks per trip give two
// independent Philox/log chains; a trip whose 256 cities are all visited is
// skipped by the whole warp at once (no divergence).  Per-lane best with ties to
// the lower id (cities are scanned in increasing order); the caller reduces
// across the warp.
// ---------------------------------------------------------------------------
// kPrefetch (the full-row path, where the scan is the whole step and 16+ warps per SM hide the
// serial pruned key chains): next trip loaded one trip ahead + exact pruning of the keys.
// kPruneFb (candidate-list fallback of the L2-table kernel at >= 16 ant warps per SM, C3):
// exact key pruning against the warp's threshold refreshed every trip, per-lane survivor
// branch (a threshold lagged by a trip, or warp-uniform skipping, measured slower: the
// other warps hide the reduction).  At a few warps per SM with rows loaded from global the
// branch-free scan is faster (C5 streams its rows through shared memory instead).
template <bool kArgmax, bool kPrefetch = false, bool kPruneFb = false, bool kPfPrune = true, class Tabu>
__device__ __forceinline__ void scan_unvisited(const float* __restrict__ row, const Tabu& tabu, int n,
                                               uint32_t step, uint32_t ant, uint32_t iter, PhiloxKey key,
                                               int lane, uint32_t& best_mag, uint32_t& best_c) {
    // pruning threshold (full-row path only: kPrefetch; unused by the argmax flag)
    constexpr bool kLag = kPruneFb && !kArgmax && !kPrefetch;
    float thr = (kPrefetch || kLag) && !kArgmax ? warp_threshold(best_mag) : 0.f;
    auto load_trip = [&](int base, uint32_t& na, uint32_t& nb, float4& iva, float4& ivb) {
        const int ca = base + 4 * lane, cb = ca + 128;
        na = chunk_nibble(tabu, ca, n);
        nb = chunk_nibble(tabu, cb, n);
        iva = na != 0xFu ? __ldg(reinterpret_cast<const float4*>(row + ca)) : make_float4(0.f, 0.f, 0.f, 0.f);
        ivb = nb != 0xFu ? __ldg(reinterpret_cast<const float4*>(row + cb)) : make_float4(0.f, 0.f, 0.f, 0.f);
    };
    if constexpr (kPrefetch) {
        // the next trip's visited bits and inv_w float4s are loaded one trip ahead
        // (full-row path, where the scan is the whole step; costs ~20 registers)
        uint32_t na, nb;
        float4 iva, ivb;
        load_trip(0, na, nb, iva, ivb);
        for (int base = 0; base < n; base += 256) {
            uint32_t na2 = 0xFu, nb2 = 0xFu;
            float4 iva2 = make_float4(0.f, 0.f, 0.f, 0.f), ivb2 = iva2;
            if (base + 256 < n) load_trip(base + 256, na2, nb2, iva2, ivb2);
            if (__any_sync(kFull, (na & nb) != 0xFu)) {
                const int ca = base + 4 * lane;
                scan_chunk<kArgmax, kPrefetch && kPfPrune>(iva, ca, na, step, ant, iter, key, best_mag, best_c, thr);
                scan_chunk<kArgmax, kPrefetch && kPfPrune>(ivb, ca + 128, nb, step, ant, iter, key, best_mag, best_c,
                                                           thr);
                if (!kArgmax && kPfPrune) thr = warp_threshold(best_mag);
            }
            na = na2;
            nb = nb2;
            iva = iva2;
            ivb = ivb2;
        }
    } else {
        for (int base = 0; base < n; base += 256) {
            uint32_t na, nb;
            float4 iva, ivb;
            load_trip(base, na, nb, iva, ivb);
            if (!__any_sync(kFull, (na & nb) != 0xFu)) continue;
            const int ca = base + 4 * lane;
            scan_chunk<kArgmax, kLag, false>(iva, ca, na, step, ant, iter, key, best_mag, best_c, thr);
            scan_chunk<kArgmax, kLag, false>(ivb, ca + 128, nb, step, ant, iter, key, best_mag, best_c, thr);
            if (kLag) thr = warp_threshold(best_mag);
        }
    }
}

// Fallback WRS over all unvisited cities (row a3, R9) with the memory-lean pheromone (R30):
// row cur of inv_w is not stored.  A city off the row's sparse list has the background trail
// b, so its 1 / choice_info is 1 / (b^alpha eta^beta) with eta^beta recomputed from the
// coordinates (heur_edge: the exact value the dense heuristic matrix holds); the few sparse
// trails carry their own.  The sparse cities are hidden from the background scan through the
// tabu (marked, scanned, unmarked), then evaluated with their stored values; every city draws
// the uniform of the dense scan (R13), so the argmax -- ties to the lowest id -- is the dense one.
// (out of line and by value -- it leaves the tabu as it found it -- so the rarely taken lean
// path adds no registers to the construction's step loop)
// phase 1: hide the row's unvisited sparse cities (warp-collective marks, one city at a time);
// bit r of the result: this lane's slot r * 32 + lane was hidden
template <class Tabu>
__device__ __forceinline__ uint32_t lean_hide(const LeanArgs& Ln, int cur, Tabu& tabu, int n, int lane) {
    const uint16_t* ids = Ln.sp_id + (size_t)cur * Ln.cap;
    uint32_t hid = 0;
    tabu.prepare(lane);
    for (int r = 0; r * 32 < Ln.cap; ++r) {
        const uint32_t j = ids[r * 32 + lane];
        const uint32_t jc = j < (uint32_t)n ? j : 0u;
        const bool unvisited = !tabu.visited(jc);   // all lanes (the register tabu shuffles)
        const bool hide = j < (uint32_t)n && unvisited;
        if (hide) hid |= 1u << r;
        for (unsigned m = __ballot_sync(kFull, hide); m; m &= m - 1u) {
            const uint32_t jj = __shfl_sync(kFull, j, __ffs(m) - 1);
            tabu.mark(jj, lane);
        }
        tabu.sync();
    }
    tabu.prepare(lane);
    return hid;
}

// phase 2: the background scan over the trips part, part + nparts, ... (lane l: the 4-city
// groups 128t + 4l, one Philox per group, two groups per trip); with integral coordinates the
// group's four coordinates are one 16-byte load and 1 / choice_info comes from the table by
// distance.  Per-lane minimum in (bm, bc), ascending cities.
template <class Tabu>
__device__ __forceinline__ void lean_scan(const LeanArgs& Ln, const double2* __restrict__ xy, int cur,
                                          const Tabu& tabu, int n, int alpha, uint32_t step, uint32_t ant,
                                          uint32_t iter, PhiloxKey key, int lane, int part, int nparts, uint32_t& bm,
                                          uint32_t& bc) {
    const float b = __ldcg(Ln.bg + Ln.parity);   // the background trail after the last update
    const double2 xc = __ldg(xy + cur);
    const short2 xcs = Ln.xys ? __ldg(Ln.xys + cur) : make_short2(0, 0);
    const float ba = pow_alpha(b, alpha);
    auto group = [&](int c0, uint32_t nib) {
        if (nib == 0xFu) return;
        const uint4 x = philox4x32_10(ctr_city((uint32_t)c0 >> 2, step, ant, iter), key);
        const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
        float iv[4];
        if (Ln.xys) {
            const int4 pk = __ldg(reinterpret_cast<const int4*>(Ln.xys + c0));   // 4 short2 (c0 % 4 == 0)
            const int pv[4] = {pk.x, pk.y, pk.z, pk.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const short2 pq = make_short2((short)(pv[q] & 0xFFFF), (short)(pv[q] >> 16));
                iv[q] = ((nib >> q) & 1u) ? 0.f : __ldg(Ln.inv_tab + euc2d_int(xcs, pq));
            }
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q)
                iv[q] = ((nib >> q) & 1u) ? 0.f
                                          : __fdiv_rn(1.0f, __fmul_rn(ba, heur_edge(xc, __ldg(xy + c0 + q), Ln.beta)));
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if ((nib >> q) & 1u) continue;
            const uint32_t mag = key_magnitude(__fmul_rn(det_log2(uniform_open(xs[q])), iv[q]));
            if (mag < bm) { bm = mag; bc = (uint32_t)(c0 + q); }   // ascending cities: ties keep the lower
        }
    };
    for (int base = 256 * part; base < n; base += 256 * nparts) {
        const int ca = base + 4 * lane, cb = ca + 128;
        const uint32_t na = chunk_nibble(tabu, ca, n), nb = chunk_nibble(tabu, cb, n);
        if (!__any_sync(kFull, (na & nb) != 0xFu)) continue;
        group(ca, na);
        group(cb, nb);
    }
}

// phase 3: unhide the hidden ones and evaluate them with their stored 1 / choice_info
template <class Tabu>
__device__ __forceinline__ void lean_unhide(const LeanArgs& Ln, int cur, Tabu& tabu, uint32_t hid, uint32_t step,
                                            uint32_t ant, uint32_t iter, PhiloxKey key, int lane, uint32_t& bm,
                                            uint32_t& bc) {
    const uint16_t* ids = Ln.sp_id + (size_t)cur * Ln.cap;
    const float* invs = Ln.sp_inv + (size_t)cur * Ln.cap;
    for (int r = 0; r * 32 < Ln.cap; ++r) {
        const uint32_t j = ids[r * 32 + lane];
        const bool h = (hid >> r) & 1u;
        if (h) {
            const uint4 x = philox4x32_10(ctr_city(j >> 2, step, ant, iter), key);
            const uint32_t w = (j & 3u) == 0 ? x.x : (j & 3u) == 1 ? x.y : (j & 3u) == 2 ? x.z : x.w;
            const uint32_t mag = key_magnitude(__fmul_rn(det_log2(uniform_open(w)), invs[r * 32 + lane]));
            if (mag < bm || (mag == bm && j < bc)) { bm = mag; bc = j; }
        }
        for (unsigned m = __ballot_sync(kFull, h); m; m &= m - 1u) {
            const uint32_t jj = __shfl_sync(kFull, j, __ffs(m) - 1);
            tabu.unmark(jj, lane);
        }
        tabu.sync();
    }
}

template <class Tabu>
__device__ __forceinline__ uint32_t lean_fallback(const LeanArgs& Ln, const double2* __restrict__ xy, int cur,
                                                  Tabu& tabu, int n, int alpha, uint32_t step, uint32_t ant,
                                                  uint32_t iter, PhiloxKey key, int lane) {
    const uint32_t hid = lean_hide(Ln, cur, tabu, n, lane);
    uint32_t bm = kNone, bc = kNone;
    lean_scan(Ln, xy, cur, tabu, n, alpha, step, ant, iter, key, lane, 0, 1, bm, bc);
    lean_unhide(Ln, cur, tabu, hid, step, ant, iter, key, lane, bm, bc);
    return warp_select(bm, bc);
}
// Out of line and by value (it leaves the tabu as it found it), for the kernels with a
// 255-register budget (C1, C2), whose step loop's allocation it would otherwise perturb
// (A/B: 0.2259 -> 0.2244 ms); under a 128-register cap the call's saved registers spill, so
// those variants inline it.
template <class Tabu>
__device__ __noinline__ uint32_t lean_fallback_ool(const LeanArgs Ln, const double2* __restrict__ xy, int cur,
                                                   Tabu tabu, int n, int alpha, uint32_t step, uint32_t ant,
                                                   uint32_t iter, PhiloxKey key, int lane) {
    return lean_fallback(Ln, xy, cur, tabu, n, alpha, step, ant, iter, key, lane);
}

// ---------------------------------------------------------------------------
// Lane-compacted fallback (row a3, R9) for the late steps of a tour.  A candidate list is
// exhausted mostly near the end of a construction (C2's driver window: median step 941 of
// 1002, ~6 % of the cities unvisited), where the trip scans above still draw a Philox and a
// key for every 4-city group of the row (~2,900 cycles of the ant's chain at any U).  Here
// each lane takes the unvisited cities of its own tabu bits -- no transpose, list or prefix
// sum: with the register tabu lane l owns cities l, l + 32, l + 64, ... (the transposed word
// wt the candidate test keeps anyway), with the shared-memory tabu the words l, l + 32, ... --
// and evaluates them eight (four, two) at a time: the scattered inv_w loads issued first, then
// independent Philox / log chains (per city the Philox of its group, word c & 3: the uniform
// the dense scan draws, R13).  The result is the same lexicographic (magnitude, city)
// minimum, ties to the lowest id, so the argmax is the dense one bit for bit.  The caller
// takes it at steps with at most `fb_lane_cap` unvisited cities, the trip scan otherwise.
// p ? a : b as one PTX selp (opaque to the compiler's select-to-branch conversion)
__device__ __forceinline__ uint32_t selp_u32(uint32_t a, uint32_t b, bool p) {
    uint32_t r;
    asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\tselp.b32 %0, %1, %2, q;\n\t}"
        : "=r"(r) : "r"(a), "r"(b), "r"((uint32_t)p));
    return r;
}
// det_log2 (rng.cuh, R14) with its range reduction written as selects: the same operations
// on the same values (bit-identical), but no branch, so ptxas interleaves several of them
__device__ __forceinline__ float det_log2_sel(float u) {
    const uint32_t b = __float_as_uint(u);
    const uint32_t mant = b & 0x007FFFFFu;
    const bool hi = mant > 0x003504F3u;
    const int e = (int)(b >> 23) - 127 + (hi ? 1 : 0);
    const uint32_t mb = mant | (hi ? 0x3F000000u : 0x3F800000u);
    const float f = __fsub_rn(__uint_as_float(mb), 1.0f);
    float p = 0.12583690881729126f;
    p = __fmaf_rn(p, f, -0.20726971328258514f);
    p = __fmaf_rn(p, f, 0.21571563184261322f);
    p = __fmaf_rn(p, f, -0.23894482851028442f);
    p = __fmaf_rn(p, f, 0.28791624307632446f);
    p = __fmaf_rn(p, f, -0.3607036769390106f);
    p = __fmaf_rn(p, f, 0.48091062903404236f);
    p = __fmaf_rn(p, f, -0.7213473320007324f);
    p = __fmaf_rn(p, f, 1.4426950216293335f);
    const float ef = __fsub_rn(__int_as_float(0x4B400000 + e), 12582912.0f);
    return __fmaf_rn(f, p, ef);
}

// (checked builds) is city c -- one of this lane's own -- marked in the tabu?
template <bool kLazyW>
__device__ __forceinline__ bool tabu_own_visited(const RegTabuX<kLazyW>& t, uint32_t c, int lane) {
    return (c & 31u) == (uint32_t)lane && ((t.wt >> (c >> 5)) & 1u);
}
__device__ __forceinline__ bool tabu_own_visited(const SmemTabu& t, uint32_t c, int) {
    return (t.t[c >> 5] >> (c & 31)) & 1u;
}
struct LaneCitiesReg {   // register tabu: bit k of ~wt = city 32 k + lane
    uint32_t f;
    int lane;
    __device__ __forceinline__ LaneCitiesReg(uint32_t wt, int n, int l) : lane(l) {
        const int cnt = (n - l + 31) >> 5;   // cities 32 k + l < n
        f = ~wt & (cnt >= 32 ? 0xFFFFFFFFu : cnt <= 0 ? 0u : (1u << cnt) - 1u);
    }
    __device__ __forceinline__ int count() const { return __popc(f); }
    __device__ __forceinline__ uint32_t next() {   // branch-free (kNone when exhausted)
        const uint32_t c = f ? 32u * (uint32_t)(__ffs(f) - 1) + (uint32_t)lane : kNone;
        f &= f - 1u;
        return c;
    }
};
struct LaneCitiesSmem {   // shared-memory tabu: the words lane, lane + 32, ...
    const uint32_t* t;
    int n, nw, wi;
    uint32_t f;
    __device__ __forceinline__ uint32_t free_word(int w) const {
        uint32_t x = ~t[w];
        const int rem = n - (w << 5);
        if (rem < 32) x &= (1u << rem) - 1u;   // cities >= n do not exist
        return x;
    }
    __device__ __forceinline__ LaneCitiesSmem(const SmemTabu& tb, int n_, int lane)
        : t(tb.t), n(n_), nw((n_ + 31) >> 5), wi(lane) {
        f = wi < nw ? free_word(wi) : 0u;
    }
    __device__ __forceinline__ int count() const {
        int c = 0;
        for (int w = wi; w < nw; w += 32) c += __popc(free_word(w));
        return c;
    }
    __device__ __forceinline__ uint32_t next() {
        while (!f) {
            wi += 32;
            if (wi >= nw) return kNone;
            f = free_word(wi);
        }
        const uint32_t b = (uint32_t)(__ffs(f) - 1);
        f &= f - 1u;
        return 32u * (uint32_t)wi + b;
    }
};
template <bool kLazyW>
__device__ __forceinline__ LaneCitiesReg lane_cities(const RegTabuX<kLazyW>& t, int n, int lane) {
    return LaneCitiesReg(t.wt, n, lane);
}
__device__ __forceinline__ LaneCitiesSmem lane_cities(const SmemTabu& t, int n, int lane) {
    return LaneCitiesSmem(t, n, lane);
}

// The per-lane part: (bm, bc) = this lane's minimum over its unvisited cities, 1 / choice_info
// of city c from ivf(c) (a row of inv_w, or the lean pheromone's recomputed background).
// (inlined: out of line measured 1 % slower on C2, the call's ~200-cycle entry)
template <class Tabu, class IvF>
__device__ __forceinline__ void compact_scan(IvF ivf, const Tabu tabu, int n, uint32_t step, uint32_t ant,
                                             uint32_t iter, PhiloxKey key, int lane, uint32_t& bm, uint32_t& bc) {
    const long long t0 = trace_clock();
    auto it = lane_cities(tabu, n, lane);
    // the register tabu counts a lane's cities with one popc; the shared-memory tabu would read
    // every word twice, so its rounds are sized by ballots over the fetched cities instead
    constexpr bool kCount = std::is_same<decltype(it), LaneCitiesReg>::value;
    const uint32_t cnt = kCount ? (uint32_t)it.count() : 0u;
    // K cities per lane at a time, branch-free (a lane with fewer carries kNone), so the K
    // Philox / log chains interleave
    auto eval = [&](auto K, const uint32_t* c, const float* iv) {
        constexpr int k = decltype(K)::value;
        uint32_t mag[k];
#pragma unroll
        for (int j = 0; j < k; ++j) {
            const uint32_t cc = c[j] == kNone ? 0u : c[j];
            const uint4 x = philox4x32_10(ctr_city(cc >> 2, step, ant, iter), key);
            const uint32_t q = cc & 3u;
            // selects in PTX (selp): the compiler would otherwise branch around the unused words
            // and the idle lanes' logs, which serialises the chains
            const uint32_t xw = selp_u32(selp_u32(x.x, x.y, q == 0u), selp_u32(x.z, x.w, q == 2u), q < 2u);
            mag[j] = selp_u32(kNone, key_magnitude(__fmul_rn(det_log2_sel(uniform_open(xw)), iv[j])), c[j] == kNone);
        }
        // a lane's cities ascend (k, then the words, ascending), so a strict "<" keeps the
        // lowest of equal keys (R16)
#pragma unroll
        for (int j = 0; j < k; ++j) {
            const bool take = mag[j] < bm;
            bm = selp_u32(mag[j], bm, take);
            bc = selp_u32(c[j], bc, take);
        }
    };
    // the first round's cities and row loads go out before the warp learns how many rounds
    // it needs (the reduction's latency hides behind the loads)
    uint32_t c[8];
    float iv[8];
    auto fetch = [&]() {
#pragma unroll
        for (int j = 0; j < 8; ++j) c[j] = it.next();
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            MMAS_CHECK(c[j] == kNone || (c[j] < (uint32_t)n && !tabu_own_visited(tabu, c[j], lane)));
            iv[j] = c[j] != kNone ? ivf(c[j]) : 0.f;
        }
    };
    fetch();
    if constexpr (kCount) {
        const int most = (int)__reduce_max_sync(kFull, cnt);
        for (int r = 0;;) {
            // (warp-uniform) 8, 4 or 2 chains: the short tail rounds issue only what they use
            if (r + 4 < most) eval(std::integral_constant<int, 8>{}, c, iv);
            else if (r + 2 < most) eval(std::integral_constant<int, 4>{}, c, iv);
            else eval(std::integral_constant<int, 2>{}, c, iv);
            r += 8;
            if (r >= most) break;
            fetch();
        }
    } else {
        // a lane's fetched cities fill c[0], c[1], ... before kNone
        while (__any_sync(kFull, c[0] != kNone)) {
            if (__any_sync(kFull, c[4] != kNone)) eval(std::integral_constant<int, 8>{}, c, iv);
            else if (__any_sync(kFull, c[2] != kNone)) eval(std::integral_constant<int, 4>{}, c, iv);
            else eval(std::integral_constant<int, 2>{}, c, iv);
            if (!__any_sync(kFull, c[7] != kNone)) break;   // every lane ran out in this round
            fetch();
        }
    }
    const long long t1 = t0;
    trace_compact(lane, t0, t1, trace_clock(), trace_clock());
}
template <class Tabu>
__device__ __forceinline__ uint32_t fallback_compact(const float* __restrict__ row, const Tabu tabu, int n,
                                                  uint32_t step, uint32_t ant, uint32_t iter, PhiloxKey key,
                                                  int lane) {
    uint32_t bm = kNone, bc = kNone;
    compact_scan([row](uint32_t c) { return __ldg(row + c); }, tabu, n, step, ant, iter, key, lane, bm, bc);
    const uint32_t res = warp_select(bm, bc);
    MMAS_CHECK(res < (uint32_t)n);
    return res;
}
// The memory-lean pheromone's fallback (R30) compacted: the row's sparse cities hidden in the
// tabu, every other unvisited city evaluated with the background's 1 / choice_info recomputed
// from the coordinates (the dense value, lean_scan's formula), the sparse ones unhidden and
// evaluated with their stored values -- the same argmax as the dense scan.
template <class Tabu>
__device__ __forceinline__ uint32_t lean_fallback_compact(const LeanArgs& Ln, const double2* __restrict__ xy, int cur,
                                                       Tabu& tabu, int n, int alpha, uint32_t step, uint32_t ant,
                                                       uint32_t iter, PhiloxKey key, int lane) {
    const uint32_t hid = lean_hide(Ln, cur, tabu, n, lane);
    uint32_t bm = kNone, bc = kNone;
    if (Ln.xys) {
        const short2 xcs = __ldg(Ln.xys + cur);
        const short2* __restrict__ xys = Ln.xys;
        const float* __restrict__ tab = Ln.inv_tab;
        compact_scan([=](uint32_t c) { return __ldg(tab + euc2d_int(xcs, __ldg(xys + c))); }, tabu, n, step, ant,
                     iter, key, lane, bm, bc);
    } else {
        const float ba = pow_alpha(__ldcg(Ln.bg + Ln.parity), alpha);
        const double2 xc = __ldg(xy + cur);
        const int beta = Ln.beta;
        compact_scan([=](uint32_t c) { return __fdiv_rn(1.0f, __fmul_rn(ba, heur_edge(xc, __ldg(xy + c), beta))); },
                     tabu, n, step, ant, iter, key, lane, bm, bc);
    }
    lean_unhide(Ln, cur, tabu, hid, step, ant, iter, key, lane, bm, bc);
    const uint32_t res = warp_select(bm, bc);
    MMAS_CHECK(res < (uint32_t)n);
    return res;
}

template <bool kArgmax, class Tabu>
__device__ __noinline__ uint32_t fallback_select(const float* __restrict__ row, const Tabu tabu, int n,
                                                 uint32_t step, uint32_t ant, uint32_t iter, PhiloxKey key,
                                                 int lane) {
    uint32_t bm = kNone, bc = kNone;
    scan_unvisited<kArgmax>(row, tabu, n, step, ant, iter, key, lane, bm, bc);
    return warp_select(bm, bc);
}

// ---- per-ant epilogue: tour length (int64) + local iteration-best key (row a5) ----
__device__ __forceinline__ unsigned long long finish_ant(const ConstructArgs& A, const uint16_t* route, int al,
                                                         uint32_t ant, int lane, long long* lengths = nullptr) {
    long long len = 0;
#pragma unroll 4
    for (int k = lane; k < A.n; k += 32) {
        const int i = route[k];
        const int j = route[(k + 1 < A.n) ? k + 1 : 0];
        len += euc2d(__ldg(A.xy + i), __ldg(A.xy + j));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) len += __shfl_xor_sync(kFull, len, o);
    if (lane == 0) (lengths ? lengths : A.lengths)[al] = len;
    return ((unsigned long long)len << 24) | ant;   // iteration-best key (R8)
}

// Row a7 inside the fused launch (world > 1; called by every thread of the grid's last
// block): the same steps as publish_peers_kernel + wait_peers_kernel + select_best_kernel
// of the split path -- this shard's best record (key, route) into slot `rank` of every
// peer's buffer, a system-wide fence, the flags; then a bounded wait for every peer's flag
// of this iteration and the selection over the gathered records (the local key reset).
__device__ __forceinline__ bool exchange_select_block(const ConstructArgs& A, int lane, int warp) {
    const ExchangeArgs& X = A.X;
    __shared__ unsigned long long s_key;
    if (threadIdx.x == 0) s_key = A.m_local > 0 ? __ldcg(A.best_key) : ~0ull;   // an empty shard never wins
    __syncthreads();
    const unsigned long long key = s_key;
    const int al = (int)(key & 0xFFFFFFu) - A.ant_lo;
    for (int p = 0; p < X.world; ++p) {
        unsigned char* rec = xrecord(X.peers[p], X, (int)X.parity, X.rank);
        if (A.m_local > 0) {
            uint16_t* dst = reinterpret_cast<uint16_t*>(rec + 8);
            for (int k = threadIdx.x; k < A.n; k += blockDim.x) dst[k] = A.routes[(size_t)al * A.ldr + k];
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
    __shared__ unsigned s_lost;
    if (warp == 0) {
        bool lost = false;
        if (lane < X.world) {
            // the flags are written by other devices: acquire at system scope (pairs with the
            // writer's __threadfence_system before its flag store)
            const uint32_t* f = xflag(A.xown, X, (int)X.parity, lane);
            const long long t0 = clock64();
            while (ld_acquire_sys(f) != X.seq) {
                if (clock64() - t0 > X.spin_bound) {
                    atomicOr(A.xerr, kErrPeerTimeout);
                    lost = true;
                    break;
                }
                __nanosleep(200);
            }
        }
        lost = __any_sync(kFull, lost) || ld_volatile_u32(A.xerr) != 0u;
        __threadfence_system();
        // a lost peer: no selection over stale records (and no update, see fused_update)
        if (!lost) {
            SelectArgs S = A.sel;
            S.records = A.xown + (size_t)X.parity * X.world * X.rec_bytes;
            S.count = X.world;
            select_best_warp(S, lane);
        }
        if (lane == 0) {
            *A.done = 0u;
            if (A.m_local > 0) *A.best_key = ~0ull;
            s_lost = lost;
        }
    }
    __syncthreads();
    return s_lost != 0u;
}

// Block epilogue: the block's best key and fallback count reach global memory with
// ONE atomic each (a per-ant global atomic makes ~10^3 same-address atomics queue
// up at the end of the launch).  world == 1: the last block to finish selects the
// iteration best with one warp (row a5; all route writes are fenced first).
__device__ __forceinline__ bool block_finish(const ConstructArgs& A, unsigned long long wbest, long long wfb,
                                             int lane, int warp, bool* aborted = nullptr) {
    __shared__ unsigned long long s_best, s_fb;
    __shared__ unsigned s_last;
    if (threadIdx.x == 0) {
        s_best = ~0ull;
        s_fb = 0ull;
    }
    // (no per-thread fence: the block's route / length writes are ordered before the block
    // barriers, and thread 0's fence before its arrival is cumulative over them)
    __syncthreads();
    if (lane == 0) {
        atomicMin(&s_best, wbest);
        if (wfb) atomicAdd(&s_fb, (unsigned long long)wfb);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (s_best != ~0ull) atomicMin(A.best_key, s_best);
        if (s_fb) atomicAdd(A.fallback_count, s_fb);
        unsigned last = 0;
        if (A.fuse_select) {
            __threadfence();   // release: this block's routes / lengths before its arrival
            last = atomicAdd(A.done, 1u) == gridDim.x - 1u;
            if (last) __threadfence();   // acquire: every block's; bar.sync passes it to the block
        }
        s_last = last;
    }
    __syncthreads();
    const bool last = s_last != 0u;
    if (aborted) *aborted = false;
    if (last && A.xchg) {
        // world > 1 inside the fused launch: the whole last block publishes, waits, selects
        const bool lost = exchange_select_block(A, lane, warp);
        if (aborted) *aborted = lost;
    } else if (last) {
        select_best_block(A.sel);
        if (threadIdx.x == 0) *A.done = 0u;
    }
    return last;
}

// Route staging: lane (s & 31) keeps route[s]; every 32 steps the warp writes a
// coalesced 64-byte segment.
__device__ __forceinline__ void stage_route(uint16_t* route, int s, uint32_t nxt, int lane, uint32_t& stage) {
    if (lane == (s & 31)) stage = nxt;
    if ((s & 31) == 31) route[(s & ~31) + lane] = (uint16_t)stage;
}
__device__ __forceinline__ void flush_route(uint16_t* route, int n, int lane, uint32_t stage) {
    const int last = n - 1;
    if ((last & 31) != 31) {
        const int base = last & ~31;
        if (base + lane <= last) route[base + lane] = (uint16_t)stage;
    }
}

// ---- TMA bulk copy helpers (cp.async.bulk global -> shared, mbarrier completion) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
    }
}

// L2 prefetch of a global range (cp.async.bulk.prefetch.L2; no completion to wait for)
__device__ __forceinline__ void prefetch_l2_bulk(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// this block's 1/gridDim share of [base, base + bytes) (16-byte granules), 32 KB per request
__device__ __forceinline__ void prefetch_l2_share(const void* base, unsigned long long bytes) {
    const unsigned long long granules = bytes >> 4;
    const unsigned long long per = (granules + gridDim.x - 1) / gridDim.x;
    const unsigned long long g0 = per * blockIdx.x, g1 = min(granules, g0 + per);
    for (unsigned long long g = g0; g < g1; g += 2048)
        prefetch_l2_bulk(reinterpret_cast<const unsigned char*>(base) + (g << 4),
                         (uint32_t)(min(g1 - g, 2048ull) << 4));
}

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_gpu(const unsigned int* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ uint32_t lds_u16(uint32_t addr) {
    unsigned short v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ float lds_f32(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}

// smem layout of the candidate-list kernel:
//   [0, 128)                 mbarrier (+ pad)
//   [128, 128+Tinv)          cand_inv  n x cl f32   (smem-table variant)
//   [.., +Tid)               cand_id   n x cl u16   (smem-table variant)
//   [.., + W * 4*nwords)     tabu words (SmemTabu variant)
extern __shared__ __align__(128) unsigned char g_smem[];

// Fallback scan over an HBM-resident row (C5), streamed through shared memory: per warp
// kFbBufs 8 KB chunk buffers (2048 cities = 8 trips) filled by cp.async.bulk, the next
// chunks in flight while the current one is scanned; chunks whose 2048 cities are all
// visited are neither copied nor scanned.  Cities are visited in the same order as
// scan_unvisited (chunks ascending, trips ascending), so the per-lane (key, city) results
// are identical.  Shared memory: the warp's mbarriers at 8 (kFbBufs warp + b), its phase
// bits at 96 + 4 warp, its buffers at fb_off + (kFbBufs warp + b) 8 KB (4 warps per block).
constexpr int kFbChunk = 2048;   // floats per chunk (8 KB)
constexpr int kFbBufs = 2;       // chunks in flight per warp (3 measured the same on C5)
template <class Tabu>
__device__ __forceinline__ void scan_unvisited_staged(const float* __restrict__ row, const Tabu& tabu, int n, int ld,
                                                      uint32_t fb_off, uint32_t step, uint32_t ant, uint32_t iter,
                                                      PhiloxKey key, int lane, int warp, uint32_t& best_mag,
                                                      uint32_t& best_c, int part = 0, int nparts = 1) {
    const int nchunks = (n + kFbChunk - 1) / kFbChunk;   // <= 32 (n < 65536)
    uint32_t need = 0;
    for (int c = part; c < nchunks; c += nparts) {   // (cooperative scans: this warp's chunks)
        bool full = true;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int wi = c * (kFbChunk / 32) + 2 * lane + k;
            if (wi * 32 < n) {
                uint32_t wd = tabu.word(wi);
                const int rem = n - wi * 32;
                if (rem < 32) wd |= ~((1u << rem) - 1u);   // cities >= n count as visited
                full = full && wd == 0xFFFFFFFFu;
            }
        }
        if (!__all_sync(kFull, full)) need |= 1u << c;
    }
    uint64_t* bars = reinterpret_cast<uint64_t*>(g_smem) + kFbBufs * warp;
    uint32_t* phw = reinterpret_cast<uint32_t*>(g_smem + 96) + warp;
    float* bufs = reinterpret_cast<float*>(g_smem + fb_off) + (size_t)warp * kFbBufs * kFbChunk;
    uint32_t ph = *reinterpret_cast<volatile uint32_t*>(phw);
    __syncwarp();
    float thr = warp_threshold(best_mag);
    auto issue = [&](int c, int b) {
        if (lane == 0) {
            fence_proxy_async_smem();   // the buffer's earlier generic reads before the copy
            const uint32_t bytes = (uint32_t)min(kFbChunk, ld - c * kFbChunk) * 4u;   // ld: multiple of 32
            mbar_expect_tx(bars + b, bytes);
            bulk_g2s(smem_u32(bufs + (size_t)b * kFbChunk), row + (size_t)c * kFbChunk, bytes, bars + b);
        }
    };
    int cq[kFbBufs];
#pragma unroll
    for (int b = 0; b < kFbBufs; ++b) {
        cq[b] = -1;
        if (need) {
            cq[b] = __ffs(need) - 1;
            need &= need - 1u;
            issue(cq[b], b);
        }
    }
    for (int b = 0;;) {
        int c = cq[0];
#pragma unroll
        for (int k = 1; k < kFbBufs; ++k)
            if (b == k) c = cq[k];
        if (c < 0) break;
        mbar_wait(bars + b, (ph >> b) & 1u);
        ph ^= 1u << b;
        const float4* buf = reinterpret_cast<const float4*>(bufs + (size_t)b * kFbChunk);
        const int end = min(n, (c + 1) * kFbChunk);
        for (int base = c * kFbChunk; base < end; base += 256) {
            const int ca = base + 4 * lane, cb = ca + 128;
            const uint32_t na = chunk_nibble(tabu, ca, n), nb = chunk_nibble(tabu, cb, n);
            if (!__any_sync(kFull, (na & nb) != 0xFu)) continue;
            const float4 iva = na != 0xFu ? buf[(ca - c * kFbChunk) >> 2] : make_float4(0.f, 0.f, 0.f, 0.f);
            const float4 ivb = nb != 0xFu ? buf[(cb - c * kFbChunk) >> 2] : make_float4(0.f, 0.f, 0.f, 0.f);
            scan_chunk<false, true>(iva, ca, na, step, ant, iter, key, best_mag, best_c, thr);
            scan_chunk<false, true>(ivb, cb, nb, step, ant, iter, key, best_mag, best_c, thr);
            thr = warp_threshold(best_mag);
        }
        __syncwarp();   // every lane is done with this buffer before it is refilled
        int nc = -1;
        if (need) {
            nc = __ffs(need) - 1;
            need &= need - 1u;
            issue(nc, b);
        }
#pragma unroll
        for (int k = 0; k < kFbBufs; ++k)
            if (b == k) cq[k] = nc;
        b = b + 1 == kFbBufs ? 0 : b + 1;
    }
    if (lane == 0) *reinterpret_cast<volatile uint32_t*>(phw) = ph;
    __syncwarp();
}




// ---------------------------------------------------------------------------
// Pheromone update fused into the construction launch (row a6; world == 1, persistent
// shared-memory-table grid, every block resident at once).  Same arithmetic as
// pheromone_update_kernel (update_quad), different schedule:
//   1. a block past its construction no longer needs its candidate table, so each warp
//      TMA-copies its first row of tau and heur into that shared memory while the rest of
//      the grid is still constructing (the update's loads leave the critical path);
//   2. grid barrier: the last block to finish runs the iteration-best selection (row a5,
//      block_finish) and bumps the epoch word; the others spin on it (acquire);
//   3. warp w updates rows w, w + W, ... from shared memory: float4 stores of tau and
//      inv_w, the new inv_w row kept in shared memory for the candidate gather.
// Removes the update launch and its ramp from the iteration.
// Shared memory: [128 + 8w) mbarrier of warp w, [256 + 2w rowbytes) its tau / heur rows.
// ---------------------------------------------------------------------------
__device__ __noinline__ void fused_update(const UpdateArgs U, unsigned int* epoch, bool last_block, bool abort,
                                          uint32_t epoch0, int lane, int warp) {
    const int wpb = (int)(blockDim.x >> 5);
    const int tw = (int)gridDim.x * wpb;
    const uint32_t rowbytes = (uint32_t)U.ld * 4u;
    float* s_tau = reinterpret_cast<float*>(g_smem + 256 + (size_t)warp * 2 * rowbytes);
    float* s_heur = s_tau + U.ld;
    uint64_t* bar = reinterpret_cast<uint64_t*>(g_smem + 128) + warp;
    int i = (int)blockIdx.x * wpb + warp;
    // the table's generic-proxy reads are ordered before the async-proxy writes that reuse it
    fence_proxy_async_smem();
    if (lane == 0) mbar_init(bar, 1);
    __syncwarp();
    auto fetch = [&](int row) {
        if (lane == 0) {
            mbar_expect_tx(bar, 2u * rowbytes);
            bulk_g2s(smem_u32(s_tau), U.tau + (size_t)row * U.ld, rowbytes, bar);
            bulk_g2s(smem_u32(s_heur), U.heur + (size_t)row * U.ld, rowbytes, bar);
        }
    };
    uint32_t cid = 0;
    if (i < U.n) {
        fetch(i);
        if (lane < U.cl) cid = __ldg(U.cand_id + (size_t)i * U.cl + lane);
    }
    // grid barrier (all blocks resident: grid <= SMs, one block each, checked at create).
    // Bounded: a barrier that does not release within spin_bound cycles sets the error word
    // and the block skips the update; the last block releases with the abort bit when its
    // exchange lost a peer (the bit stays set in the epoch word: later launches skip too).
    __shared__ unsigned s_abort;
    __syncthreads();   // the last block's selection warp is done
    if (threadIdx.x == 0) {
        if (last_block) {
            __threadfence();
            atomicAdd(epoch, abort && !(epoch0 & kEpochAbort) ? kEpochAbort + 1u : 1u);
        }
        uint32_t v;
        const long long t0 = clock64();
        bool timeout = false;
        while ((v = ld_acquire_gpu(epoch)) == epoch0) {
            if (clock64() - t0 > U.spin_bound) {
                atomicOr(U.err, kErrGridBarrier);
                timeout = true;
                break;
            }
            __nanosleep(32);
        }
        s_abort = timeout || (v & kEpochAbort) != 0u;
    }
    __syncthreads();
    if (s_abort) {
        // drain this warp's row prefetch before the shared memory goes away
        if (i < U.n) mbar_wait(bar, 0);
        if (blockIdx.x == 0 && threadIdx.x == 0) *U.iter_dev += 1u;
        return;
    }
    trace_mark(4);
    const float tmin = __ldcg(U.scal), tmax = __ldcg(U.scal + 1), delta = __ldcg(U.scal + 2);
    const int n4 = (U.n + 3) >> 2;
    uint32_t phase = 0;
    for (; i < U.n; i += tw) {
        const int si = __ldcg(U.succ + i), pi = __ldcg(U.pred + i);
        float4* trow = reinterpret_cast<float4*>(U.tau + (size_t)i * U.ld);
        float4* wrow = reinterpret_cast<float4*>(U.inv_w + (size_t)i * U.ld);
        mbar_wait(bar, phase);
        phase ^= 1u;
        for (int q = lane; q < n4; q += 32) {
            float4 t = reinterpret_cast<const float4*>(s_tau)[q];
            const float4 h = reinterpret_cast<const float4*>(s_heur)[q];
            const float4 w4 = update_quad(t, h, 4 * q, si, pi, U.rho_f, tmin, tmax, delta, U.alpha);
            trow[q] = t;
            wrow[q] = w4;
            reinterpret_cast<float4*>(s_tau)[q] = w4;   // the new inv_w row, for the gather
        }
        __syncwarp();
        if (lane < U.cl) U.cand_inv[(size_t)i * U.cl + lane] = s_tau[cid];
        __syncwarp();
        if (i + tw < U.n) {
            fence_proxy_async_smem();
            fetch(i + tw);
            if (lane < U.cl) cid = __ldg(U.cand_id + (size_t)(i + tw) * U.cl + lane);
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *U.iter_dev += 1u;
}


// ---------------------------------------------------------------------------
// Paired fallback scans (C5: the L2-table kernel at a few ant warps per SM, rows streamed
// from HBM through shared memory).  A fallback there is ~70 chunk trips on the ant's serial
// chain while the SM idles (~25 % issue active); so the block's warps pair up: the even warp
// of a pair builds an ant, the odd one only helps with its fallbacks.  The ant warp posts
// (current city, step, ant), both meet at the pair's named barrier, each scans every other
// 2048-city chunk with its own buffers, the helper posts its (key, city) minimum, both meet
// again, and the ant warp takes the minimum of the two -- the same argmax, ties to the lowest
// city (each warp's cities ascend; the pairwise minimum is lexicographic).
// ---------------------------------------------------------------------------
struct CoopSlot {
    uint32_t cur, step, ant, done;
    uint32_t mag, city;   // the helper's partial result
};
__device__ __forceinline__ void pair_barrier(int pair) {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + pair), "r"(64) : "memory");
}
__device__ __forceinline__ void warp_best(uint32_t mag, uint32_t city, uint32_t& bmag, uint32_t& bcity) {
    bmag = __reduce_min_sync(kFull, mag);
    bcity = __reduce_min_sync(kFull, mag == bmag ? city : kNone);
}

// ---------------------------------------------------------------------------
// Candidate-list construction (rows a1, a2, a3, a5-local).
// kSlots = ceil(cl/32) candidate slots per lane; kSmemTable: the n x cl
// (1/w, id) table is staged once per block into shared memory by TMA bulk
// copies, else rows are read through L1/L2; kRegTabu: n <= 1024.
// ---------------------------------------------------------------------------
// kWide: up to 16 ant warps per block (large colonies with the shared-memory table; the
// register budget drops to 128), else up to 8
template <int kSlots, bool kSmemTable, bool kRegTabu, bool kFull32, bool kWide = false>
// L2-table variants run 4-warp blocks and need 4 blocks per SM (128 registers) when the
// colony fills the SMs (C3's 3795 ants: 25 warps per SM); with kWide (few ant warps per SM,
// C5) the register budget is left to the compiler
__global__ void __launch_bounds__(kSmemTable ? (kWide ? 512 : 256) : 128, kSmemTable ? 1 : (kWide ? 3 : 4))
    construct_cl_kernel(const ConstructArgs A) {
    // colony (grid.y, R29): its per-colony pointers as locals (a modified copy of the whole
    // argument struct would live in registers through the step loop); the tail takes a copy
    const int col = (int)blockIdx.y;
    const float* __restrict__ c_inv_w = A.inv_w + col * A.cs.nn;
    const float* __restrict__ c_cand_inv = A.cand_inv + col * A.cs.cand;
    uint16_t* __restrict__ c_routes = A.routes + col * A.cs.routes;
    const PhiloxKey c_key = col ? colony_key(A.key, (uint32_t)col) : A.key;
    pdl_wait();
    trace_mark(0);
    static_assert(!kFull32 || kSlots == 1, "kFull32: cl == 32, one slot per lane");
    static_assert(!kWide || kFull32, "kWide: one-slot variants only");
    using Tabu = typename std::conditional<kRegTabu, RegTabuX<kFull32>, SmemTabu>::type;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int n = A.n, cl = A.cl;
    const int nwords = (((n + 31) >> 5) + 3) & ~3;
    uint64_t* bar = reinterpret_cast<uint64_t*>(g_smem);
    const uint32_t tab_off = kSmemTable ? 128u + A.table_bytes_inv + A.table_bytes_id : 128u;

    if (kSmemTable) {
        if (threadIdx.x == 0) {
            mbar_init(bar, 1);
            mbar_expect_tx(bar, A.table_bytes_inv + A.table_bytes_id);
            constexpr uint32_t kChunk = 32768;
            const uint32_t s_base = smem_u32(g_smem);
            for (uint32_t off = 0; off < A.table_bytes_inv; off += kChunk)
                bulk_g2s(s_base + 128u + off, reinterpret_cast<const unsigned char*>(c_cand_inv) + off,
                         min(kChunk, A.table_bytes_inv - off), bar);
            for (uint32_t off = 0; off < A.table_bytes_id; off += kChunk)
                bulk_g2s(s_base + 128u + A.table_bytes_inv + off,
                         reinterpret_cast<const unsigned char*>(A.cand_id) + off,
                         min(kChunk, A.table_bytes_id - off), bar);
        }
    }
    if (threadIdx.x == 0 && A.l2_prefetch_bytes) prefetch_l2_share(c_inv_w, A.l2_prefetch_bytes);
    // 32-bit shared-window addresses of the two tables (plain LDS with a register address)
    uint32_t s_inv = smem_u32(g_smem) + 128u;
    uint32_t s_id = s_inv + A.table_bytes_inv;
    // opaque: keep the addresses in registers (otherwise ptxas re-derives the shared
    // window base with a long-latency S2UR SR_CgaCtaId inside every step)
    asm volatile("" : "+r"(s_inv), "+r"(s_id));
    const RoundKeys rk(c_key);
    const uint32_t id_lane = s_id + 2u * (uint32_t)lane;     // kFull32: slot = lane
    const uint32_t inv_lane = s_inv + 4u * (uint32_t)lane;
    uint32_t* tabu_base = reinterpret_cast<uint32_t*>(g_smem + tab_off) + warp * nwords;
    const uint32_t iter = A.iter_dev[col];
    // grid-barrier generation of the fused update: read before this block can arrive
    const uint32_t epoch0 = (kSmemTable && A.fuse_update) ? ld_acquire_gpu(A.epoch + 2 * col) : 0u;
    if (!kSmemTable && A.fb_row_off) {   // the fallback chunk pipelines (scan_unvisited_staged)
        if (threadIdx.x < 4 * kFbBufs) mbar_init(reinterpret_cast<uint64_t*>(g_smem) + threadIdx.x, 1);
        if (threadIdx.x < 4) reinterpret_cast<uint32_t*>(g_smem + 96)[threadIdx.x] = 0u;
        __syncthreads();
    }
    if (kSmemTable) {
        __syncthreads();   // the barrier is initialised before anyone waits on it
        mbar_wait(bar, 0);
    }
    // paired fallback scans (C5; see CoopSlot): even warp = ant, odd warp = its helper
    constexpr bool kCoop = !kSmemTable && kWide && !kRegTabu;
    __shared__ CoopSlot s_coop[kCoop ? 8 : 1];
    const bool coop = kCoop && A.coop_fb && A.fb_row_off;
    const bool helper = coop && (warp & 1);
    const int pair = warp >> 1;
    const int ant_slot = coop ? pair : warp, ants_per_block = coop ? (A.warps_per_block >> 1) : A.warps_per_block;
    trace_mark(1);
    unsigned long long wbest = ~0ull;
    long long wfb = 0;

    for (int al = blockIdx.x * ants_per_block + ant_slot; !helper && al < A.m_local;
         al += gridDim.x * ants_per_block) {
        const uint32_t ant = (uint32_t)(A.ant_lo + al);
        Tabu tabu;
        tabu.init(tabu_base, nwords, lane);
        // Alg. 1: start node u ~ U{0, n-1} (R13)
        const uint32_t start = __umulhi(philox4x32_10(ctr_start(ant, iter), c_key).x, (uint32_t)n);
        tabu.mark(start, lane);
        tabu.sync();
        uint16_t* route = c_routes + (size_t)al * A.ldr;
        uint32_t stage = (lane == 0) ? start : 0u;
        uint32_t cur = start;
        long long fb = 0;

        // slot uniforms of steps 0..3 (R13: counter (k, s>>2, a, iter), word s&3)
        float L[kSlots][4];
#pragma unroll
        for (int q = 0; q < kSlots; ++q) {
            const uint4 x = philox4x32_10(ctr_slot((uint32_t)(lane + 32 * q), 0u, ant, iter), c_key);
            L[q][0] = det_log2(uniform_open(x.x));
            L[q][1] = det_log2(uniform_open(x.y));
            L[q][2] = det_log2(uniform_open(x.z));
            L[q][3] = det_log2(uniform_open(x.w));
        }

        uint4 nx[kSlots];
        float Ln[kSlots][4];
        // next group's random keys, one slice per step: Philox rounds 0-4, 5-9, then the
        // logs of words 0-1 and 2-3 (off the dependency chain; R13)
        // Each slice is split in two halves (A, B): the step places A behind its table loads
        // and B behind its tabu shuffle, so the in-order issue fills both latency bubbles.
        auto slice_half = [&](auto J, auto H) {
            constexpr int j = decltype(J)::value;
            constexpr int h = decltype(H)::value;
#pragma unroll
            for (int q = 0; q < kSlots; ++q) {
                if (j == 0 && h == 0) philox_rounds<0, 3>(nx[q], rk);
                if (j == 0 && h == 1) philox_rounds<3, 5>(nx[q], rk);
                if (j == 1 && h == 0) philox_rounds<5, 8>(nx[q], rk);
                if (j == 1 && h == 1) philox_rounds<8, 10>(nx[q], rk);
                if (j == 2 && h == 0) Ln[q][0] = det_log2(uniform_open(nx[q].x));
                if (j == 2 && h == 1) Ln[q][1] = det_log2(uniform_open(nx[q].y));
                if (j == 3 && h == 0) Ln[q][2] = det_log2(uniform_open(nx[q].z));
                if (j == 3 && h == 1) Ln[q][3] = det_log2(uniform_open(nx[q].w));
            }
        };
        // Quarter slices for the speculative step, which has four latency windows (table
        // loads, tabu shuffle, and the two reductions): Philox rounds 0-1 | 1-3 | 3-4 | 4-5,
        // 5-6 | 6-8 | 8-9 | 9-10, then each log split in two (det_log2_a / det_log2_b).
        Log2Part lp[kSlots];
        auto slice_q = [&](auto J, auto Q) {
            constexpr int j = decltype(J)::value;
            constexpr int k = decltype(Q)::value;
#pragma unroll
            for (int q = 0; q < kSlots; ++q) {
                if (j == 0 && k == 0) philox_rounds<0, 1>(nx[q], rk);
                if (j == 0 && k == 1) philox_rounds<1, 3>(nx[q], rk);
                if (j == 0 && k == 2) philox_rounds<3, 4>(nx[q], rk);
                if (j == 0 && k == 3) philox_rounds<4, 5>(nx[q], rk);
                if (j == 1 && k == 0) philox_rounds<5, 6>(nx[q], rk);
                if (j == 1 && k == 1) philox_rounds<6, 8>(nx[q], rk);
                if (j == 1 && k == 2) philox_rounds<8, 9>(nx[q], rk);
                if (j == 1 && k == 3) philox_rounds<9, 10>(nx[q], rk);
                if (j >= 2) {
                    const uint32_t w = (j == 2) ? (k < 2 ? nx[q].x : nx[q].y) : (k < 2 ? nx[q].z : nx[q].w);
                    const int slot = 2 * (j - 2) + (k >> 1);
                    if ((k & 1) == 0) lp[q] = det_log2_a(uniform_open(w));
                    else Ln[q][slot] = det_log2_b(lp[q]);
                }
            }
        };
        using Q0 = std::integral_constant<int, 0>;
        using Q1 = std::integral_constant<int, 1>;
        using Q2 = std::integral_constant<int, 2>;
        using Q3 = std::integral_constant<int, 3>;
        using H0 = std::integral_constant<int, 0>;
        using H1 = std::integral_constant<int, 1>;
        using I0 = std::integral_constant<int, 0>;
        using I1 = std::integral_constant<int, 1>;
        using I2 = std::integral_constant<int, 2>;
        using I3 = std::integral_constant<int, 3>;
        auto slice = [&](auto J) {
            slice_half(J, H0{});
            slice_half(J, H1{});
        };
        // Candidate evaluation of the current step (Alg. 3) with the slot key
        // factors Lv: per-lane (value, city) for the warp argmax.  hook_a / hook_b run
        // independent work behind the table loads / the tabu shuffle.
        auto evaluate = [&](const float (&Lv)[kSlots], auto hook_a, auto hook_b, uint32_t& bm, uint32_t& bc) {
            bm = kNone;
            bc = kNone;
            if constexpr (kFull32) {
                // cl == 32: lane k owns slot k.  One IMAD per address; the tabu bit is shifted
                // to bit 31 and merged with the key magnitude (a visited lane's value has bit 31
                // set, so it loses to every unvisited one).
                uint32_t c;
                float iv;
                if (kSmemTable) {
                    c = lds_u16(id_lane + cur * 64u);
                    iv = lds_f32(inv_lane + cur * 128u);
                } else {
                    c = __ldg(A.cand_id + cur * 32u + lane);
                    iv = __ldg(c_cand_inv + cur * 32u + lane);
                }
                hook_a();
                const uint32_t t = tabu.top_bit(c);
                hook_b();
                // bit 31 from the tabu, bits 0-30 the key magnitude
                bm = bit_select(t, __float_as_uint(__fmul_rn(Lv[0], iv)), 0x7FFFFFFFu);
                bc = c;
            } else {
                hook_a();
                hook_b();
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
                        iv = __ldg(c_cand_inv + idx);
                    }
                    const bool vis = tabu.visited(has ? c : cur);
                    const uint32_t mag = vis ? 0x80000000u : key_magnitude(__fmul_rn(Lv[q], iv));
                    if (mag < bm || (mag == bm && c < bc)) {
                        bm = mag;
                        bc = c;
                    }
                }
            }
        };
        auto commit = [&](uint32_t nxt, int s) {
            tabu.mark(nxt, lane);
            stage_route(route, s, nxt, lane, stage);
            tabu.sync();
            cur = nxt;
        };
        // FAST step (compile-time j): returns true, without choosing, when every candidate is
        // visited; the generic path below then redoes the step with the fallback scan
        auto fast_step = [&](auto J, int s) -> bool {
            constexpr int j = decltype(J)::value;
            float Lv[kSlots];
#pragma unroll
            for (int q = 0; q < kSlots; ++q) Lv[q] = L[q][j];
            uint32_t bm, bc;
            evaluate(Lv, [&] { slice_half(J, H0{}); }, [&] { slice_half(J, H1{}); }, bm, bc);
            // argmax (ties -> lowest city id, R16): both reductions back to back
            const uint32_t best = __reduce_min_sync(kFull, bm);
            const uint32_t nxt = __reduce_min_sync(kFull, bm == best ? bc : kNone);
            if (__builtin_expect(best >= 0x80000000u, 0)) return true;
            commit(nxt, s);
            return false;
        };
        // SPECULATIVE step (register tabu): commits its argmax unconditionally and reports
        // whether every candidate was visited (the caller then rolls the group back)
        auto spec_step = [&](auto J, int s, uint32_t& taken) -> bool {
            constexpr int j = decltype(J)::value;
            float Lv[kSlots];
#pragma unroll
            for (int q = 0; q < kSlots; ++q) Lv[q] = L[q][j];
            uint32_t bm, bc;
            evaluate(Lv, [&] { slice_q(J, Q0{}); }, [&] { slice_q(J, Q1{}); }, bm, bc);
            const uint32_t best = __reduce_min_sync(kFull, bm);
            slice_q(J, Q2{});
            const uint32_t nxt = __reduce_min_sync(kFull, bm == best ? bc : kNone);
            slice_q(J, Q3{});
            // every lane holds a real candidate (a visited one has bit 31 set), so nxt is a city
            // id < n even when best >= 2^31 (then it is undone by the caller)
            __builtin_assume(nxt < 65536u);
            commit(nxt, s);
            taken = nxt;
            return best >= 0x80000000u;
        };
        // GENERIC step (runtime j): guards, and the R9 fallback (row a3) inlined ONCE
        // known_fb: the speculative / fast attempt of this step already found every candidate
        // visited (from the same state), so the evaluation is not repeated
        auto generic_step = [&](int j, int s, bool known_fb) {
            uint32_t best = 0x80000000u, nxt = 0u;
            if (!known_fb) {
                float Lv[kSlots];
#pragma unroll
                for (int q = 0; q < kSlots; ++q)
                    Lv[q] = j == 0 ? L[q][0] : j == 1 ? L[q][1] : j == 2 ? L[q][2] : L[q][3];
                uint32_t bm, bc;
                evaluate(Lv, [] {}, [] {}, bm, bc);
                best = __reduce_min_sync(kFull, bm);
                nxt = __reduce_min_sync(kFull, bm == best ? bc : kNone);
            }
            if (best >= 0x80000000u) {   // every candidate visited: R9 fallback
                ++fb;
                const long long t_fb = trace_clock();
                const float* row = c_inv_w + (size_t)cur * A.ld;
                uint32_t fm = kNone, fc = kNone;
                if constexpr (kCoop) {
                    if (coop && A.lean.cand_tau && n - s > A.fb_lane_cap) {
                        // the lean scan, paired (see CoopSlot): hidden sparse cities stay marked in
                        // the ant's shared-memory tabu while both warps scan their trips
                        const uint32_t hid = lean_hide(A.lean, (int)cur, tabu, n, lane);
                        if (lane == 0) {
                            s_coop[pair].cur = cur;
                            s_coop[pair].step = (uint32_t)s;
                            s_coop[pair].ant = ant;
                            s_coop[pair].done = 0u;
                        }
                        pair_barrier(pair);
                        uint32_t bm2 = kNone, bc2 = kNone;
                        lean_scan(A.lean, A.xy, (int)cur, tabu, n, A.alpha, (uint32_t)s, ant, iter, c_key, lane, 0, 2,
                                  bm2, bc2);
                        pair_barrier(pair);   // the helper's partial result is posted
                        const uint32_t m1 = s_coop[pair].mag, c1 = s_coop[pair].city;
                        if (lane == 0 && (m1 < bm2 || (m1 == bm2 && c1 < bc2))) {
                            bm2 = m1;
                            bc2 = c1;
                        }
                        lean_unhide(A.lean, (int)cur, tabu, hid, (uint32_t)s, ant, iter, c_key, lane, bm2, bc2);
                        commit(warp_select(bm2, bc2), s);
                        return;
                    }
                }
                if (A.lean.cand_tau) {
                    // memory-lean pheromone (R30): no inv_w row; the scan recomputes it
                    // late in the tour: compacted, the ant warp alone -- in the L2-table kernels
                    // (C5L, C65KL), not in the 255-register shared-memory-table ones, whose step
                    // loops move by ~1 % with any added code (C2 A/B; their lean rows are short)
                    if constexpr (!(kSmemTable && !kWide)) {
                        if (n - s <= A.fb_lane_cap) {
                            const uint32_t c = lean_fallback_compact(A.lean, A.xy, (int)cur, tabu, n, A.alpha,
                                                                     (uint32_t)s, ant, iter, c_key, lane);
                            trace_fallback(t_fb, lane, n - s);
                            commit(c, s);
                            return;
                        }
                    }
                    tabu.prepare(lane);
                    if constexpr (kSmemTable && !kWide)
                        commit(lean_fallback_ool(A.lean, A.xy, (int)cur, tabu, n, A.alpha, (uint32_t)s, ant, iter, c_key,
                                                 lane),
                               s);
                    else
                        commit(lean_fallback(A.lean, A.xy, (int)cur, tabu, n, A.alpha, (uint32_t)s, ant, iter, c_key,
                                             lane),
                               s);
                    return;
                }
                if (n - s <= A.fb_lane_cap && !A.fallback_argmax) {   // (lean: above)
                    // late in the tour (n - s unvisited cities): each lane evaluates only its own
                    const uint32_t c = fallback_compact(row, tabu, n, (uint32_t)s, ant, iter, c_key, lane);
                    trace_fallback(t_fb, lane, n - s);
                    trace_compact_entry(lane, t_fb);
                    commit(c, s);
                    return;
                }
                tabu.prepare(lane);
                if (A.fallback_argmax)
                    scan_unvisited<true>(row, tabu, n, (uint32_t)s, ant, iter, c_key, lane, fm, fc);
                else if (kCoop && coop) {
                    if (lane == 0) {
                        s_coop[pair].cur = cur;
                        s_coop[pair].step = (uint32_t)s;
                        s_coop[pair].ant = ant;
                        s_coop[pair].done = 0u;
                    }
                    pair_barrier(pair);   // request posted: the helper scans the odd chunks
                    scan_unvisited_staged(row, tabu, n, A.ld, A.fb_row_off, (uint32_t)s, ant, iter, c_key, lane,
                                          warp, fm, fc, 0, 2);
                    uint32_t m0, c0;
                    warp_best(fm, fc, m0, c0);
                    pair_barrier(pair);   // the helper's partial result is posted
                    const uint32_t m1 = s_coop[pair].mag, c1 = s_coop[pair].city;
                    const bool take = m1 < m0 || (m1 == m0 && c1 < c0);
                    fm = take ? m1 : m0;
                    fc = take ? c1 : c0;
                } else if (!kSmemTable && A.fb_row_off) {
                    scan_unvisited_staged(row, tabu, n, A.ld, A.fb_row_off, (uint32_t)s, ant, iter, c_key, lane,
                                          warp, fm, fc);
                } else if (!kSmemTable && A.prune_fallback)
                    scan_unvisited<false, false, !kSmemTable>(row, tabu, n, (uint32_t)s, ant, iter, c_key, lane, fm,
                                                              fc);
                else if (kSmemTable)
                    // the next trip's visited bits and inv_w float4s requested one trip ahead,
                    // keys branch-free (A/B on C2's driver window: 0.2250 -> 0.2201 ms; with the
                    // exact pruning of the full-row scans: 0.2327)
                    scan_unvisited<false, true, false, false>(row, tabu, n, (uint32_t)s, ant, iter, c_key, lane, fm, fc);
                else
                    scan_unvisited<false>(row, tabu, n, (uint32_t)s, ant, iter, c_key, lane, fm, fc);
                nxt = warp_select(fm, fc);
                trace_fallback(t_fb, lane, n - s);
            }
            commit(nxt, s);
        };
        auto slice_rt = [&](int j) {
            if (j == 0) slice(I0{});
            else if (j == 1) slice(I1{});
            else if (j == 2) slice(I2{});
            else slice(I3{});
        };
        auto next_group = [&](int g) {
#pragma unroll
            for (int q = 0; q < kSlots; ++q) nx[q] = ctr_slot((uint32_t)(lane + 32 * q), (uint32_t)(g + 1), ant, iter);
        };
        auto rotate = [&]() {
#pragma unroll
            for (int q = 0; q < kSlots; ++q)
#pragma unroll
                for (int j = 0; j < 4; ++j) L[q][j] = Ln[q][j];
        };
        const int n_groups = (n + 3) / 4;      // groups holding a step s < n
        const int n_full = n / 4;              // groups g < n_full have all four steps < n
        // Groups 1 .. n_full-1 (all four steps real, a next group to prepare) run the FAST
        // path: four straight-line steps with no branch but the fallback exit.  Group 0
        // (s = 0), the ragged tail, and the rest of a group whose fast path hit a fallback
        // run the GENERIC path, which appears once in the loop body.
        int g = 0;
        while (g < n_groups) {
            const long long t_g0 = trace_clock();
            const bool pipeline = g + 1 < n_groups;
            int j0 = 0;
            bool sliced_j0 = false;
            if (pipeline) next_group(g);
            bool sliced_all = false;
            if (g >= 1 && g < n_full && pipeline) {
                if constexpr (kRegTabu) {
                    // SPECULATIVE group: the four steps run as one straight-line block (no
                    // branch between them, so the scheduler can overlap one step's random-key
                    // slices with the next step's chain); a step that needed the fallback is
                    // detected once at the end.  The group is then rolled back to the state
                    // before its FIRST such step jf (tabu: the group's entry words with the steps
                    // before jf re-marked; current city: step jf-1's choice) and the generic path
                    // redoes steps jf..3.  (A hit step's choice is a visited city, so its mark
                    // changed nothing; the route staging of steps >= jf is overwritten by the
                    // redo before the next segment store.)
                    const uint32_t w0 = tabu.w, wt0 = tabu.wt, cur0 = cur;
                    uint32_t t0, t1, t2, t3;
                    const bool h0 = spec_step(I0{}, 4 * g + 0, t0);
                    const bool h1 = spec_step(I1{}, 4 * g + 1, t1);
                    const bool h2 = spec_step(I2{}, 4 * g + 2, t2);
                    const bool h3 = spec_step(I3{}, 4 * g + 3, t3);
                    if (__builtin_expect(!(h0 | h1 | h2 | h3), 1)) {
                        rotate();
                        ++g;
                        trace_group(t_g0, lane, false);
                        continue;
                    }
                    tabu.w = w0;
                    tabu.wt = wt0;
                    cur = cur0;
                    if (!h0) {
                        tabu.mark(t0, lane);
                        cur = t0;
                        j0 = 1;
                        if (!h1) {
                            tabu.mark(t1, lane);
                            cur = t1;
                            j0 = 2;
                            if (!h2) {
                                tabu.mark(t2, lane);
                                cur = t2;
                                j0 = 3;
                            }
                        }
                    }
                    (void)t3;
                    sliced_all = true;   // every slice of this group already ran
                } else {
                    int jf = -1;
                    if (fast_step(I0{}, 4 * g + 0)) jf = 0;
                    else if (fast_step(I1{}, 4 * g + 1)) jf = 1;
                    else if (fast_step(I2{}, 4 * g + 2)) jf = 2;
                    else if (fast_step(I3{}, 4 * g + 3)) jf = 3;
                    if (jf < 0) {
                        rotate();
                        ++g;
                        continue;
                    }
                    j0 = jf;
                    sliced_j0 = true;   // that step's slices ran inside its fast attempt
                }
            }
#pragma unroll 1
            for (int j = j0; j < 4; ++j) {
                if (pipeline && !sliced_all && !(j == j0 && sliced_j0)) slice_rt(j);
                const int s = 4 * g + j;
                if (s > 0 && s < n) generic_step(j, s, j == j0 && (sliced_all || sliced_j0));
            }
            if (pipeline) rotate();
            ++g;
            if (sliced_all || sliced_j0) trace_group(t_g0, lane, true);
        }
        flush_route(route, n, lane, stage);
        __syncwarp();
        if (!A.skip_finish) wbest = min(wbest, finish_ant(A, route, al, ant, lane, A.lengths + (long long)col * A.cs.ants));
        wfb += fb;
        trace_warp_done(warp, lane);
    }
    if constexpr (kCoop) {
        if (coop) {
            if (!helper) {
                if (lane == 0) s_coop[pair].done = 1u;
                pair_barrier(pair);   // release the helper
            } else {
                // the helper: serve the ant warp's fallbacks until it is done
                SmemTabu tv;
                tv.t = reinterpret_cast<uint32_t*>(g_smem + tab_off) + (warp - 1) * nwords;
                while (true) {
                    pair_barrier(pair);
                    if (s_coop[pair].done) break;
                    const uint32_t hcur = s_coop[pair].cur, hs = s_coop[pair].step, hant = s_coop[pair].ant;
                    uint32_t fm = kNone, fc = kNone;
                    if (A.lean.cand_tau)
                        lean_scan(A.lean, A.xy, (int)hcur, tv, n, A.alpha, hs, hant, iter, c_key, lane, 1, 2, fm, fc);
                    else
                        scan_unvisited_staged(c_inv_w + (size_t)hcur * A.ld, tv, n, A.ld, A.fb_row_off, hs, hant, iter,
                                              c_key, lane, warp, fm, fc, 1, 2);
                    uint32_t hm, hc;
                    warp_best(fm, fc, hm, hc);
                    if (lane == 0) {
                        s_coop[pair].mag = hm;
                        s_coop[pair].city = hc;
                    }
                    pair_barrier(pair);
                }
            }
        }
    }
    pdl_trigger();   // this block is done with its ants: let the next kernel's blocks in
    trace_mark(2);
    ConstructArgs At = A;
    if (col) colony_offset(At, col);
    bool aborted;
    const bool last = block_finish(At, wbest, wfb, lane, warp, &aborted);
    trace_mark(3);
    if constexpr (kSmemTable) {
        if (At.fuse_update) fused_update(At.upd, At.epoch, last, aborted, epoch0, lane, warp);
    }
    trace_mark(5);
}

// ---------------------------------------------------------------------------
// Full-row construction (rows a1, a4, a5-local; cl = 0, configuration C4):
// every step scans all unvisited cities (Alg. 3 over the whole row).
// ---------------------------------------------------------------------------
template <bool kRegTabu>
__global__ void __launch_bounds__(128) construct_full_kernel(const ConstructArgs A) {
    // colony (grid.y, R29): per-colony pointers as locals, a colony copy for the tail
    const int col = (int)blockIdx.y;
    const float* __restrict__ c_inv_w = A.inv_w + col * A.cs.nn;
    uint16_t* __restrict__ c_routes = A.routes + col * A.cs.routes;
    const PhiloxKey c_key = col ? colony_key(A.key, (uint32_t)col) : A.key;
    pdl_wait();
    using Tabu = typename std::conditional<kRegTabu, RegTabu, SmemTabu>::type;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int n = A.n;
    const int nwords = (((n + 31) >> 5) + 3) & ~3;
    uint32_t* tabu_base = reinterpret_cast<uint32_t*>(g_smem + 128) + warp * nwords;
    const uint32_t iter = A.iter_dev[col];
    unsigned long long wbest = ~0ull;

    for (int al = blockIdx.x * A.warps_per_block + warp; al < A.m_local; al += gridDim.x * A.warps_per_block) {
        const uint32_t ant = (uint32_t)(A.ant_lo + al);
        Tabu tabu;
        tabu.init(tabu_base, nwords, lane);
        const uint32_t start = __umulhi(philox4x32_10(ctr_start(ant, iter), c_key).x, (uint32_t)n);
        tabu.mark(start, lane);
        tabu.sync();
        uint16_t* route = c_routes + (size_t)al * A.ldr;
        uint32_t stage = (lane == 0) ? start : 0u;
        uint32_t cur = start;
        for (int s = 1; s < n; ++s) {
            uint32_t nxt;
            if (n - s <= A.fb_lane_cap) {
                // late in the tour: each lane evaluates only its own unvisited cities (the
                // candidate-list fallback's compacted scan, same keys, same argmax)
                nxt = fallback_compact(c_inv_w + (size_t)cur * A.ld, tabu, n, (uint32_t)s, ant, iter, c_key, lane);
            } else {
                uint32_t bm = kNone, bc = kNone;
                scan_unvisited<false, true>(c_inv_w + (size_t)cur * A.ld, tabu, n, (uint32_t)s, ant, iter, c_key, lane,
                                            bm, bc);
                nxt = warp_select(bm, bc);
            }
            tabu.mark(nxt, lane);
            stage_route(route, s, nxt, lane, stage);
            tabu.sync();
            cur = nxt;
        }
        flush_route(route, n, lane, stage);
        __syncwarp();
        if (!A.skip_finish) wbest = min(wbest, finish_ant(A, route, al, ant, lane, A.lengths + (long long)col * A.cs.ants));
    }
    pdl_trigger();   // this block is done with its ants: let the next kernel's blocks in
    ConstructArgs At = A;
    if (col) colony_offset(At, col);
    block_finish(At, wbest, 0, lane, warp);
}



// ---------------------------------------------------------------------------
// Full-row construction over the compact tabu (MMAS-WRS-CT, SURVEY NEXT-2,
// DESIGN.md R27; cl = 0 with tabu = COMPACT).  One warp per ant; the CT's
// `entries` (n u16) live in shared memory.  Step s enumerates the
// L = n - s unvisited nodes entries[0..L) (Alg. 3 with l = tabu.length(),
// P:964-994): lane l takes the 4-position groups 128t + 4l, one Philox per group
// (word j = position 4g+j's uniform, counter (0x40000000 | g, s, a, it)), and
// gathers inv_w[cur][v] for the four nodes.  Work per step is L instead of n, so
// a tour costs ~n^2/2 keys instead of n^2 ("direct access to the
// list of nodes to visit").  Keys compare as (magnitude, node), ties -> lowest
// node id (R16), because list order is not node order.
// ---------------------------------------------------------------------------
// Positions >= L get inv_w = +inf: their key is -inf, whose magnitude 0x7F800000 loses
// to every real key (det_log2 < 0 and finite on the u-grid, inv_w finite), and L >= 1
// guarantees a real key in the warp -- so the select needs no position mask.
// Keys are evaluated only for positions whose lower bound does not exceed thr (the exact
// pruning of scan_chunk; +inf padding gives lb = +inf, pruned once thr is finite).
__device__ __forceinline__ void ct_group(uint2 e, float4 iv, int p0, uint32_t step, uint32_t ant, uint32_t iter,
                                         PhiloxKey key, uint32_t& best_mag, uint32_t& best_c, float thr) {
    const uint4 x = philox4x32_10(ctr_city((uint32_t)p0 >> 2, step, ant, iter), key);
    const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
    const float ivs[4] = {iv.x, iv.y, iv.z, iv.w};
    const uint32_t vs[4] = {e.x & 0xFFFFu, e.x >> 16, e.y & 0xFFFFu, e.y >> 16};
    float om[4];
    bool keep[4];
    bool any = false;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        om[j] = one_minus_uniform_open(xs[j]);          // 1 - u, exact on the grid
        keep[j] = !(__fmul_rn(om[j], ivs[j]) > thr);           // thr: scaled threshold T
        any |= keep[j];
    }
    if (any) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (keep[j]) {
                const uint32_t mag = key_magnitude(__fmul_rn(det_log2(__fsub_rn(1.0f, om[j])), ivs[j]));
                // (mag, node) lexicographic minimum
                if ((mag < best_mag) | ((mag == best_mag) & (vs[j] < best_c))) {
                    best_mag = mag;
                    best_c = vs[j];
                }
            }
        }
    }
}

// positions p0 .. p0+3 of the list: their nodes (u16 pairs) and inv_w[cur][node]
// (kChecked: the trip may run past L; positions >= L get +inf)
template <bool kChecked>
__device__ __forceinline__ void ct_load(const uint16_t* ent, const float* __restrict__ row, int p0, int L, uint2& e,
                                        float4& iv) {
    const float inf = __int_as_float(0x7F800000);
    e = *reinterpret_cast<const uint2*>(ent + p0);
    if (kChecked) {
        iv.x = p0 + 0 < L ? __ldg(row + (e.x & 0xFFFFu)) : inf;
        iv.y = p0 + 1 < L ? __ldg(row + (e.x >> 16)) : inf;
        iv.z = p0 + 2 < L ? __ldg(row + (e.y & 0xFFFFu)) : inf;
        iv.w = p0 + 3 < L ? __ldg(row + (e.y >> 16)) : inf;
    } else {
        iv.x = __ldg(row + (e.x & 0xFFFFu));
        iv.y = __ldg(row + (e.x >> 16));
        iv.z = __ldg(row + (e.y & 0xFFFFu));
        iv.w = __ldg(row + (e.y >> 16));
    }
}

// one 256-position trip: lane l's groups base+4l and base+128+4l
__device__ __forceinline__ void ct_trip(const uint2 (&e)[2], const float4 (&iv)[2], int base, int lane, int L,
                                        uint32_t step, uint32_t ant, uint32_t iter, PhiloxKey key,
                                        uint32_t& best_mag, uint32_t& best_c, float& thr) {
    const int pa = base + 4 * lane;
    if (pa < L) ct_group(e[0], iv[0], pa, step, ant, iter, key, best_mag, best_c, thr);
    if (pa + 128 < L) ct_group(e[1], iv[1], pa + 128, step, ant, iter, key, best_mag, best_c, thr);
    thr = warp_threshold(best_mag);
}

__device__ __forceinline__ void ct_load_trip(const uint16_t* ent, const float* __restrict__ row, int base, int lane,
                                             int L, uint2 (&e)[2], float4 (&iv)[2]) {
    if (base + 256 <= L) {   // a full trip (warp-uniform): no per-position bounds
        ct_load<false>(ent, row, base + 4 * lane, L, e[0], iv[0]);
        ct_load<false>(ent, row, base + 128 + 4 * lane, L, e[1], iv[1]);
    } else {
        ct_load<true>(ent, row, base + 4 * lane, L, e[0], iv[0]);
        ct_load<true>(ent, row, base + 128 + 4 * lane, L, e[1], iv[1]);
    }
}

// CT mark(u), by one lane; L = list length before the mark.
__device__ __forceinline__ void ct_mark(uint16_t* ent, int L, int n, uint32_t u) {
    const uint32_t last = (uint32_t)L - 1u;
    const uint32_t t = ent[last];
    const uint32_t iu = u < (uint32_t)L ? u : ent[u];
    if (iu == last) {
        ent[iu] = (uint16_t)n;
    } else {
        ent[iu] = (uint16_t)t;
        ent[t] = (uint16_t)iu;
    }
}

__global__ void __launch_bounds__(128) construct_ct_kernel(const ConstructArgs A) {
    // colony (grid.y, R29): per-colony pointers as locals, a colony copy for the tail
    const int col = (int)blockIdx.y;
    const float* __restrict__ c_inv_w = A.inv_w + col * A.cs.nn;
    uint16_t* __restrict__ c_routes = A.routes + col * A.cs.routes;
    const PhiloxKey c_key = col ? colony_key(A.key, (uint32_t)col) : A.key;
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int n = A.n;
    const int ent_len = (n + 255) & ~255;                 // padded: a trip may read past L
    uint16_t* ent = reinterpret_cast<uint16_t*>(g_smem + 128) + (size_t)warp * ent_len;
    const uint32_t iter = A.iter_dev[col];
    unsigned long long wbest = ~0ull;

    for (int al = blockIdx.x * A.warps_per_block + warp; al < A.m_local; al += gridDim.x * A.warps_per_block) {
        const uint32_t ant = (uint32_t)(A.ant_lo + al);
        for (int i = lane; i < n; i += 32) ent[i] = (uint16_t)i;
        __syncwarp();
        const uint32_t start = __umulhi(philox4x32_10(ctr_start(ant, iter), c_key).x, (uint32_t)n);
        if (lane == 0) ct_mark(ent, n, n, start);
        __syncwarp();
        uint16_t* route = c_routes + (size_t)al * A.ldr;
        uint32_t stage = (lane == 0) ? start : 0u;
        uint32_t cur = start;
        for (int s = 1; s < n; ++s) {
            const int L = n - s;
            const float* row = c_inv_w + (size_t)cur * A.ld;
            uint32_t bm = kNone, bc = kNone;
            // the next trip's list entries and inv_w gathers are loaded one trip ahead
            // (two register sets, loop unrolled by two so no copies are needed)
            uint2 eA[2], eB[2];
            float4 ivA[2], ivB[2];
            float thr = __int_as_float(0x7F800000);
            ct_load_trip(ent, row, 0, lane, L, eA, ivA);
            for (int base = 0; base < L; base += 512) {
                if (base + 256 < L) ct_load_trip(ent, row, base + 256, lane, L, eB, ivB);
                ct_trip(eA, ivA, base, lane, L, (uint32_t)s, ant, iter, c_key, bm, bc, thr);
                if (base + 256 >= L) break;
                if (base + 512 < L) ct_load_trip(ent, row, base + 512, lane, L, eA, ivA);
                ct_trip(eB, ivB, base + 256, lane, L, (uint32_t)s, ant, iter, c_key, bm, bc, thr);
            }
            const uint32_t nxt = warp_select(bm, bc);
            __syncwarp();   // every lane's reads of this step's list before lane 0 rewrites it
            if (lane == 0) ct_mark(ent, L, n, nxt);
            stage_route(route, s, nxt, lane, stage);
            __syncwarp();
            cur = nxt;
        }
        flush_route(route, n, lane, stage);
        __syncwarp();
        if (!A.skip_finish) wbest = min(wbest, finish_ant(A, route, al, ant, lane, A.lengths + (long long)col * A.cs.ants));
    }
    pdl_trigger();   // this block is done with its ants: let the next kernel's blocks in
    ConstructArgs At = A;
    if (col) colony_offset(At, col);
    block_finish(At, wbest, 0, lane, warp);
}

}  // namespace mmas
