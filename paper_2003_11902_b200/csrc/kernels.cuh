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
constexpr uint32_t kNone = 0xFFFFFFFFu;

// TSPLIB EUC_2D (R12): (int)(sqrt(dx*dx + dy*dy) + 0.5) in double.
__device__ __forceinline__ int32_t euc2d(double2 p, double2 q) {
    const double dx = __dsub_rn(p.x, q.x);
    const double dy = __dsub_rn(p.y, q.y);
    const double r = __dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
    return (int32_t)__dadd_rn(r, 0.5);
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
    int warps_per_block;
    uint32_t table_bytes_inv, table_bytes_id;  // smem-table variant: padded table sizes
    uint16_t* __restrict__ routes;          // m_local x ldr
    long long* __restrict__ lengths;        // m_local
    unsigned long long* __restrict__ best_key;       // local min (len << 24 | ant)
    unsigned long long* __restrict__ fallback_count;
};

// ---------------------------------------------------------------------------
// Scan of ALL unvisited cities from `row` (= inv_w[cur]): the full-row WRS step
// (row a4) and the candidate-list fallback (row a3, R9).  Lane l handles the
// 4-city groups 128t + 4l (a coalesced float4 of inv_w and one Philox per group
// whose word j is city 4g+j's uniform, R13); groups whose four cities are all
// visited are skipped.  Per-lane best with ties to the lower id; the caller
// reduces across the warp.
// ---------------------------------------------------------------------------
template <bool kArgmax>
__device__ __forceinline__ void scan_unvisited(const float* __restrict__ row, const uint32_t* tabu, int n,
                                               uint32_t step, uint32_t ant, uint32_t iter, PhiloxKey key,
                                               int lane, uint32_t& best_mag, uint32_t& best_c) {
    for (int base = 0; base < n; base += 128) {
        const int c0 = base + 4 * lane;
        if (c0 >= n) continue;
        uint32_t nib = (tabu[c0 >> 5] >> (c0 & 31)) & 0xFu;
        if (c0 + 4 > n) nib |= (0xFu << (n - c0)) & 0xFu;   // cities >= n count as visited
        if (nib == 0xFu) continue;
        const float4 iv = __ldg(reinterpret_cast<const float4*>(row + c0));
        const float ivs[4] = {iv.x, iv.y, iv.z, iv.w};
        if (kArgmax) {
            // R9 flag: largest weight = smallest inv_w (positive floats order as uints)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if ((nib >> j) & 1u) continue;
                const uint32_t mag = __float_as_uint(ivs[j]);
                if (mag < best_mag) { best_mag = mag; best_c = (uint32_t)(c0 + j); }
            }
        } else {
            const uint4 x = philox4x32_10(ctr_city((uint32_t)c0 >> 2, step, ant, iter), key);
            const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if ((nib >> j) & 1u) continue;
                const float k = __fmul_rn(det_log2(uniform_open(xs[j])), ivs[j]);
                const uint32_t mag = key_magnitude(k);
                if (mag < best_mag) { best_mag = mag; best_c = (uint32_t)(c0 + j); }
            }
        }
    }
}

template <bool kArgmax>
__device__ __noinline__ uint32_t fallback_select(const float* __restrict__ row, const uint32_t* tabu, int n,
                                                 uint32_t step, uint32_t ant, uint32_t iter, PhiloxKey key,
                                                 int lane) {
    uint32_t bm = kNone, bc = kNone;
    scan_unvisited<kArgmax>(row, tabu, n, step, ant, iter, key, lane, bm, bc);
    return warp_select(bm, bc);
}

// ---- per-ant epilogue: tour length (int64) + local iteration-best key (row a5) ----
__device__ __forceinline__ void finish_ant(const ConstructArgs& A, const uint16_t* route, int al, uint32_t ant,
                                           int lane, long long fb) {
    long long len = 0;
    for (int k = lane; k < A.n; k += 32) {
        const int i = route[k];
        const int j = route[(k + 1 < A.n) ? k + 1 : 0];
        len += euc2d(__ldg(A.xy + i), __ldg(A.xy + j));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) len += __shfl_xor_sync(kFull, len, o);
    if (lane == 0) {
        A.lengths[al] = len;
        atomicMin(A.best_key, ((unsigned long long)len << 24) | ant);
        if (fb) atomicAdd(A.fallback_count, (unsigned long long)fb);
    }
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
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
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

// ---------------------------------------------------------------------------
// Candidate-list construction (rows a1, a2, a3, a5-local).  One warp = one ant
// (the paper's data-parallel mapping at warp granularity, with
// one warp per ant at cl = 32 as in P:1469-1472).  kSlots = ceil(cl/32)
// candidate slots per lane.  kSmemTable: the n x cl (inv, id) table is staged
// once per block into shared memory by TMA bulk copies; otherwise rows are read
// through L1/L2.  Tabu: bitmask in shared memory, ceil(n/32) words per warp
// (Sec. 4.1 "bitmask tabu").
// ---------------------------------------------------------------------------
template <int kSlots, bool kSmemTable>
__global__ void __launch_bounds__(512) construct_cl_kernel(ConstructArgs A) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int n = A.n, cl = A.cl;
    const int nwords = (((n + 31) >> 5) + 3) & ~3;

    const float* cinv = A.cand_inv;
    const uint16_t* cid = A.cand_id;
    unsigned char* p = smem;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);  // smem[0..127]: mbarrier (+ pad)
    if (kSmemTable) {
        float* s_inv = reinterpret_cast<float*>(smem + 128);
        uint16_t* s_id = reinterpret_cast<uint16_t*>(smem + 128 + A.table_bytes_inv);
        if (threadIdx.x == 0) {
            mbar_init(bar, 1);
            mbar_expect_tx(bar, A.table_bytes_inv + A.table_bytes_id);
            constexpr uint32_t kChunk = 32768;
            for (uint32_t off = 0; off < A.table_bytes_inv; off += kChunk) {
                const uint32_t sz = min(kChunk, A.table_bytes_inv - off);
                bulk_g2s(reinterpret_cast<unsigned char*>(s_inv) + off,
                         reinterpret_cast<const unsigned char*>(A.cand_inv) + off, sz, bar);
            }
            for (uint32_t off = 0; off < A.table_bytes_id; off += kChunk) {
                const uint32_t sz = min(kChunk, A.table_bytes_id - off);
                bulk_g2s(reinterpret_cast<unsigned char*>(s_id) + off,
                         reinterpret_cast<const unsigned char*>(A.cand_id) + off, sz, bar);
            }
        }
        cinv = s_inv;
        cid = s_id;
        p = smem + 128 + A.table_bytes_inv + A.table_bytes_id;
    } else {
        p = smem + 128;
    }
    uint32_t* tabu = reinterpret_cast<uint32_t*>(p) + warp * nwords;
    const uint32_t iter = *A.iter_dev;
    if (kSmemTable) {
        __syncthreads();  // barrier initialised before anyone waits on it
        mbar_wait(bar, 0);
    }

    for (int al = blockIdx.x * A.warps_per_block + warp; al < A.m_local; al += gridDim.x * A.warps_per_block) {
        const uint32_t ant = (uint32_t)(A.ant_lo + al);
        for (int j = lane; j < nwords; j += 32) tabu[j] = 0u;
        __syncwarp();
        // Alg. 1: start node u ~ U{0, n-1} (R13)
        const uint32_t start = __umulhi(philox4x32_10(ctr_start(ant, iter), A.key).x, (uint32_t)n);
        if (lane == 0) tabu[start >> 5] |= 1u << (start & 31);
        uint16_t* route = A.routes + (size_t)al * A.ldr;
        uint32_t stage = (lane == 0) ? start : 0u;
        uint32_t cur = start;
        long long fb = 0;
        __syncwarp();

        for (int g = 0; 4 * g < n; ++g) {
            // slot uniforms for steps 4g .. 4g+3 (R13: counter (k, s>>2, a, iter), word s&3)
            float L[kSlots][4];
#pragma unroll
            for (int q = 0; q < kSlots; ++q) {
                const uint32_t slot = (uint32_t)(lane + 32 * q);
                const uint4 x = philox4x32_10(ctr_slot(slot, (uint32_t)g, ant, iter), A.key);
                L[q][0] = det_log2(uniform_open(x.x));
                L[q][1] = det_log2(uniform_open(x.y));
                L[q][2] = det_log2(uniform_open(x.z));
                L[q][3] = det_log2(uniform_open(x.w));
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int s = 4 * g + j;
                if (s == 0 || s >= n) continue;
                uint32_t bm = kNone, bc = kNone;
#pragma unroll
                for (int q = 0; q < kSlots; ++q) {
                    const int slot = lane + 32 * q;
                    if (slot < cl) {
                        const uint32_t c = cid[cur * cl + slot];
                        const float iv = cinv[cur * cl + slot];
                        if (!((tabu[c >> 5] >> (c & 31)) & 1u)) {
                            const uint32_t mag = key_magnitude(__fmul_rn(L[q][j], iv));
                            if (mag < bm || (mag == bm && c < bc)) { bm = mag; bc = c; }
                        }
                    }
                }
                uint32_t nxt = warp_select(bm, bc);
                if (nxt == kNone) {  // every candidate visited: R9 fallback (row a3)
                    ++fb;
                    const float* row = A.inv_w + (size_t)cur * A.ld;
                    nxt = A.fallback_argmax
                              ? fallback_select<true>(row, tabu, n, (uint32_t)s, ant, iter, A.key, lane)
                              : fallback_select<false>(row, tabu, n, (uint32_t)s, ant, iter, A.key, lane);
                }
                if (lane == 0) tabu[nxt >> 5] |= 1u << (nxt & 31);
                stage_route(route, s, nxt, lane, stage);
                __syncwarp();
                cur = nxt;
            }
        }
        flush_route(route, n, lane, stage);
        __syncwarp();
        finish_ant(A, route, al, ant, lane, fb);
    }
}

// ---------------------------------------------------------------------------
// Full-row construction (rows a1, a4, a5-local; cl = 0, configuration C4):
// every step scans all unvisited cities (Alg. 3 over the whole row).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) construct_full_kernel(ConstructArgs A) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int n = A.n;
    const int nwords = (((n + 31) >> 5) + 3) & ~3;
    uint32_t* tabu = reinterpret_cast<uint32_t*>(smem + 128) + warp * nwords;
    const uint32_t iter = *A.iter_dev;

    for (int al = blockIdx.x * A.warps_per_block + warp; al < A.m_local; al += gridDim.x * A.warps_per_block) {
        const uint32_t ant = (uint32_t)(A.ant_lo + al);
        for (int j = lane; j < nwords; j += 32) tabu[j] = 0u;
        __syncwarp();
        const uint32_t start = __umulhi(philox4x32_10(ctr_start(ant, iter), A.key).x, (uint32_t)n);
        if (lane == 0) tabu[start >> 5] |= 1u << (start & 31);
        uint16_t* route = A.routes + (size_t)al * A.ldr;
        uint32_t stage = (lane == 0) ? start : 0u;
        uint32_t cur = start;
        __syncwarp();
        for (int s = 1; s < n; ++s) {
            uint32_t bm = kNone, bc = kNone;
            scan_unvisited<false>(A.inv_w + (size_t)cur * A.ld, tabu, n, (uint32_t)s, ant, iter, A.key, lane, bm,
                                  bc);
            const uint32_t nxt = warp_select(bm, bc);
            if (lane == 0) tabu[nxt >> 5] |= 1u << (nxt & 31);
            stage_route(route, s, nxt, lane, stage);
            __syncwarp();
            cur = nxt;
        }
        flush_route(route, n, lane, stage);
        __syncwarp();
        finish_ant(A, route, al, ant, lane, 0);
    }
}

// ---------------------------------------------------------------------------
// Iteration best + global best + limits (row a5; Alg. 1).
// Either from this context's local best key (world == 1) or from `count`
// gathered per-rank records [u64 key][u16 route[n]] (world > 1).
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
};

__global__ void __launch_bounds__(1024) select_best_kernel(SelectArgs S) {
    __shared__ const uint16_t* src;
    __shared__ int improved;
    const int n = S.n;
    if (threadIdx.x == 0) {
        unsigned long long key;
        if (S.records) {
            int bi = 0;
            key = *reinterpret_cast<const unsigned long long*>(S.records);
            for (int r = 1; r < S.count; ++r) {
                const unsigned long long k =
                    *reinterpret_cast<const unsigned long long*>(S.records + (size_t)r * S.rec_bytes);
                if (k < key) { key = k; bi = r; }
            }
            src = reinterpret_cast<const uint16_t*>(S.records + (size_t)bi * S.rec_bytes + 8);
        } else {
            key = *S.local_key;
            src = S.routes + (size_t)((int)(key & 0xFFFFFFu) - S.ant_lo) * S.ldr;
        }
        const long long len = (long long)(key >> 24);
        const long long gbl = *S.gb_len;
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
    }
    __syncthreads();
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        const uint16_t v = src[k];
        S.ib_route[k] = v;
        if (improved) S.gb_route[k] = v;
    }
    __syncthreads();
    const uint16_t* dep = S.deposit_global ? S.gb_route : S.ib_route;
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        const uint16_t i = dep[k];
        const uint16_t j = dep[(k + 1 < n) ? k + 1 : 0];
        S.succ[i] = j;
        S.pred[j] = i;
    }
    __syncthreads();
    if (threadIdx.x == 0 && !S.records) *S.local_key = ~0ull;
}

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
// Pheromone update (row a6; Alg. 1, R1/R4-R6, R22):
//   tau <- min(max(rho tau, tau_min) + Delta [(i,j) in T_dep], tau_max)
//   inv_w <- 1 / (tau^alpha heur);  cand_inv[i][k] <- inv_w[i][cand_id[i][k]]
// One block per row (the paper's evaporation geometry), float4
// streaming; the deposit is the row's succ/pred test, so evaporation and
// deposit fuse into one non-conflicting pass.
// ---------------------------------------------------------------------------
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
    uint32_t* iter_dev;
};

__global__ void __launch_bounds__(256) pheromone_update_kernel(UpdateArgs U) {
    const float tmin = U.scal[0], tmax = U.scal[1], delta = U.scal[2];
    for (int i = blockIdx.x; i < U.n; i += gridDim.x) {
        const int si = U.succ[i], pi = U.pred[i];
        float4* trow = reinterpret_cast<float4*>(U.tau + (size_t)i * U.ld);
        float4* wrow = reinterpret_cast<float4*>(U.inv_w + (size_t)i * U.ld);
        const float4* hrow = reinterpret_cast<const float4*>(U.heur + (size_t)i * U.ld);
        const int n4 = (U.n + 3) >> 2;
        for (int q = threadIdx.x; q < n4; q += blockDim.x) {
            const float4 t = trow[q];
            const float4 h = __ldg(hrow + q);
            float tv[4] = {t.x, t.y, t.z, t.w};
            const float hv[4] = {h.x, h.y, h.z, h.w};
            float wv[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int c = 4 * q + j;
                float v = fmaxf(__fmul_rn(U.rho_f, tv[j]), tmin);
                if (c == si || c == pi) v = __fadd_rn(v, delta);
                v = fminf(v, tmax);
                tv[j] = v;
                wv[j] = inv_weight(v, hv[j], U.alpha);
            }
            trow[q] = make_float4(tv[0], tv[1], tv[2], tv[3]);
            wrow[q] = make_float4(wv[0], wv[1], wv[2], wv[3]);
        }
        if (U.cl > 0) {
            __syncthreads();
            for (int k = threadIdx.x; k < U.cl; k += blockDim.x)
                U.cand_inv[(size_t)i * U.cl + k] = U.inv_w[(size_t)i * U.ld + U.cand_id[(size_t)i * U.cl + k]];
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
__global__ void heur_kernel(const double2* __restrict__ xy, int n, int ld, int beta, float* heur) {
    const int i = blockIdx.y;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ld; c += gridDim.x * blockDim.x) {
        float h = 1.0f;
        if (c < n) {
            const int32_t d = euc2d(xy[i], xy[c]);
            const double D = (double)(d > 1 ? d : 1);
            double Db = 1.0;
            for (int k = 0; k < beta; ++k) Db = __dmul_rn(Db, D);
            h = __double2float_rn(__ddiv_rn(1.0, Db));
        }
        heur[(size_t)i * ld + c] = h;
    }
}

// tau = tau_max (Alg. 1) and inv_w = 1/choice_info.
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
