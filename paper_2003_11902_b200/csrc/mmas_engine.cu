// mmas_engine.cu -- the C ABI (include/mmas.h) and the host-side engine.
//
// One context = one colony shard on one CUDA device and one stream.  Setup
// (row a0) runs once in mmas_create; each iteration is the kernel sequence
//   construct_{cl,full}  ->  select_best  ->  pheromone_update
// with no host synchronisation inside the loop (the iteration counter, the
// limits and the global best live in device memory).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <utility>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/mmas.h"
#include "kernels.cuh"

using namespace mmas;

namespace {

thread_local std::string g_last_error;

int fail(int status, const std::string& msg) {
    g_last_error = msg;
    return status;
}

#define CU(call)                                                                                     \
    do {                                                                                             \
        cudaError_t e_ = (call);                                                                     \
        if (e_ != cudaSuccess)                                                                       \
            return fail(MMAS_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));             \
    } while (0)

inline int round_up(int x, int m) { return (x + m - 1) / m * m; }

// ---- host side of setup (row a0), written from DESIGN.md R3, R10, R12 ----
inline int32_t host_dist(const double* xy, int i, int j) {
    const double dx = xy[2 * i] - xy[2 * j];
    const double dy = xy[2 * i + 1] - xy[2 * j + 1];
    const double r = std::sqrt(dx * dx + dy * dy);   // compiled with -ffp-contract=off
    return (int32_t)(r + 0.5);
}

// cl nearest neighbours of every city by (d, id), self excluded (R10)
void candidate_lists(const double* xy, int n, int cl, std::vector<uint16_t>& out) {
    out.assign((size_t)n * cl, 0);
    unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    auto work = [&](int r0, int r1) {
        std::vector<std::pair<int32_t, int32_t>> buf((size_t)n);
        for (int i = r0; i < r1; ++i) {
            int k = 0;
            for (int j = 0; j < n; ++j)
                if (j != i) buf[k++] = {host_dist(xy, i, j), j};
            std::partial_sort(buf.begin(), buf.begin() + cl, buf.begin() + k);
            for (int q = 0; q < cl; ++q) out[(size_t)i * cl + q] = (uint16_t)buf[q].second;
        }
    };
    std::vector<std::thread> th;
    for (unsigned t = 0; t < hw; ++t) th.emplace_back(work, (int)((int64_t)n * t / hw), (int)((int64_t)n * (t + 1) / hw));
    for (auto& t : th) t.join();
}

// nearest-neighbour tour from city 0, ties -> lowest id; returns its length (R3)
// R2: limits in double, cast to float
void host_limits(double rho, int64_t cost, double factor, float* tmin, float* tmax) {
    const double tx = 1.0 / ((1.0 - rho) * (double)cost);
    double tn = tx * factor;
    if (tn > tx) tn = tx;
    *tmax = (float)tx;
    *tmin = (float)tn;
}

bool is_int_in(double x, int lo, int hi) { return x == std::floor(x) && x >= lo && x <= hi; }

}  // namespace

struct mmas_ctx {
    mmas_config cfg{};
    int n = 0, ld = 0, cl = 0, ldr = 0;
    int cl_ld = 0;   // row stride of the candidate tables: 32 for 0 < cl <= 32 (rows padded with the
                     // row's own city, which is always visited), else cl
    int m = 0, ant_lo = 0, m_local = 0;
    int alpha = 1;
    int device = 0, num_sms = 148, smem_optin = 0, l2_bytes = 0;
    double factor = 0.0;
    int64_t nn_len = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    bool pooled = false;                    // device buffers from the per-device pool (dalloc)
    PhiloxKey key{};
    int rec_bytes = 0;

    // device buffers
    double2* xy = nullptr;
    float *heur = nullptr, *tau = nullptr, *inv_w = nullptr, *cand_inv = nullptr;
    uint16_t* cand_id = nullptr;
    uint16_t* routes = nullptr;
    long long* lengths = nullptr;
    unsigned long long* best_key = nullptr;
    unsigned long long* fallback_count = nullptr;
    uint16_t *ib_route = nullptr, *gb_route = nullptr, *succ = nullptr, *pred = nullptr;
    long long *gb_len = nullptr, *ib_len = nullptr;
    int* ib_ant = nullptr;
    float* scal = nullptr;        // tau_min, tau_max, delta
    uint32_t* iter_dev = nullptr;
    unsigned char* local_record = nullptr;  // world == 1 path of mmas_construct/mmas_update
    unsigned int* done = nullptr;           // fused select: ants finished in the running launch

    // launch plan for construction
    bool smem_table = false;
    bool fuse_update = false;               // world == 1: update fused into the construction launch
    bool fuse_peers = false;                // world > 1: mmas_iterate_exchange as one launch per iteration

    bool reg_tabu = false;   // n <= 1024: tabu words in registers
    bool compact_tabu = false;  // cl == 0 with MMAS_TABU_COMPACT: construct_ct_kernel (R27)
    bool rwm = false;           // MMAS_SELECT_RWM: construct_rwm_kernel (R28)
    int slots = 1;
    int cons_warps = 4, cons_grid = 1;
    bool coop_fb = false;                   // L2-table kernel: paired fallback scans (2 ants + 2 helpers per block)
    size_t cons_smem = 0;
    uint32_t fb_row_off = 0;                // L2-table kernel: fallback row buffer in smem
    int fb_lane_cap = 0;                    // lane-compacted fallback: max unvisited cities per lane (0 = off)
    uint32_t tb_inv = 0, tb_id = 0;

    // memory-lean pheromone (R30): no n x n matrices; candidate trails + sparse rows
    bool lean = false;
    int lean_cap = 0, lean_L = 0;
    float *cand_tau = nullptr, *cand_heur = nullptr, *sp_tau = nullptr, *sp_inv = nullptr, *bg = nullptr;
    uint16_t* sp_id = nullptr;
    short2* lean_xys = nullptr;              // integral coordinates (else null)
    float *heur_tab = nullptr, *inv_tab = nullptr;
    int dtab = 0;

    // concurrent independent colonies (R29): K per-colony copies of the mutable state
    int colonies = 1;
    int view = 0;                           // colony the introspection calls report
    ColonyStride cs{};

    // host mirrors
    int32_t iteration = 0;
    int64_t launches = 0;

    // row a8: 2-opt local search (local_search != 0)
    int ls_k = 0, ls_nwords = 0, ls_coop_smem_max = 0, ls_group_smem_max = 0;
    uint16_t* ls_nn = nullptr;         // n x ls_k neighbour lists
    int32_t* ls_nnd = nullptr;         // n x ls_k: d(a, nn[a][k])
    short2* ls_xys = nullptr;          // integral coordinates (ls_int_xy), else null
    uint32_t* ls_nnp = nullptr;        // ls_int_xy: packed neighbour id | distance << 16
    bool ls_int_xy = false;
    uint16_t *ls_pos = nullptr, *ls_queue = nullptr;
    uint32_t* ls_inq = nullptr;
    unsigned long long* ls_moves = nullptr;

    // peer-memory exchange (row a7 without a collective library; world > 1)
    unsigned char* xbuf = nullptr;            // own buffer: [2][world] records + [2][world] flags
    unsigned char** xpeers_dev = nullptr;     // device array of every rank's (peer-mapped) buffer
    std::vector<void*> xopened;               // IPC mappings to close
    uint32_t* xerr = nullptr;                 // device error word (kErr*): a device-side wait gave up
    long long spin_bound = kSpinBound;        // device-side waits give up after this many cycles
    bool xattached = false;

    // profiling
    bool profiling = false;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    struct Span { cudaEvent_t a, b; int phase; };
    std::vector<Span> spans;
    double acc_ms[4] = {0, 0, 0, 0};
    int64_t acc_iters = 0;
};

namespace {

cudaEvent_t take_event(mmas_ctx* h) {
    if (h->ev_used == h->ev_pool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        h->ev_pool.push_back(e);
    }
    return h->ev_pool[h->ev_used++];
}

// Folds completed spans into the accumulators (synchronises the stream).
void drain_spans(mmas_ctx* h) {
    if (h->spans.empty()) return;
    cudaStreamSynchronize(h->stream);
    for (auto& s : h->spans) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, s.a, s.b);
        h->acc_ms[s.phase] += ms;
    }
    h->spans.clear();
    h->ev_used = 0;
}

struct PhaseScope {
    mmas_ctx* h;
    int phase;
    cudaEvent_t a{};
    PhaseScope(mmas_ctx* hh, int p) : h(hh), phase(p) {
        if (h->profiling) {
            if (h->ev_used + 2 > 4096) drain_spans(h);
            a = take_event(h);
            cudaEventRecord(a, h->stream);
        }
    }
    ~PhaseScope() {
        if (h->profiling) {
            cudaEvent_t b = take_event(h);
            cudaEventRecord(b, h->stream);
            h->spans.push_back({a, b, phase});
        }
    }
};

SelectArgs select_args(mmas_ctx* h, const unsigned char* records, int count) {
    SelectArgs S{};
    S.records = records;
    S.count = count;
    S.rec_bytes = h->rec_bytes;
    S.local_key = h->best_key;
    S.routes = h->routes;
    S.ldr = h->ldr;
    S.ant_lo = h->ant_lo;
    S.n = h->n;
    S.rho = h->cfg.rho;
    S.factor = h->factor;
    S.deposit_global = h->cfg.deposit == MMAS_DEPOSIT_GLOBAL_BEST;
    S.ib_route = h->ib_route;
    S.gb_route = h->gb_route;
    S.gb_len = h->gb_len;
    S.ib_len = h->ib_len;
    S.ib_ant = h->ib_ant;
    S.scal = h->scal;
    S.succ = h->succ;
    S.pred = h->pred;
    S.err = h->xerr;
    S.cs = h->cs;
    return S;
}

UpdateArgs update_args(mmas_ctx* h);

LeanArgs lean_args(mmas_ctx* h) {
    LeanArgs L{};
    if (!h->lean) return L;
    L.cand_tau = h->cand_tau;
    L.cand_heur = h->cand_heur;
    L.sp_id = h->sp_id;
    L.sp_tau = h->sp_tau;
    L.sp_inv = h->sp_inv;
    L.bg = h->bg;
    L.cap = h->lean_cap;
    L.parity = h->iteration & 1;
    L.beta = (int)h->cfg.beta;
    L.xys = h->lean_xys;
    L.heur_tab = h->heur_tab;
    L.inv_tab = h->inv_tab;
    L.dtab = h->dtab;
    return L;
}

ConstructArgs construct_args(mmas_ctx* h, bool fuse_select, bool skip_finish = false) {
    ConstructArgs A{};
    A.fuse_select = fuse_select ? 1 : 0;
    A.skip_finish = skip_finish ? 1 : 0;
    A.done = h->done;
    A.sel = select_args(h, nullptr, 1);
    A.xy = h->xy;
    A.inv_w = h->inv_w;
    A.cand_id = h->cand_id;
    A.cand_inv = h->cand_inv;
    A.iter_dev = h->iter_dev;
    A.key = h->key;
    A.n = h->n;
    A.ld = h->ld;
    A.cl = h->cl_ld;   // padded rows: the kernels see cl_ld slots, the padding is always visited
    A.ldr = h->ldr;
    A.ant_lo = h->ant_lo;
    A.m_local = h->m_local;
    A.fallback_argmax = h->cfg.fallback == MMAS_FALLBACK_ARGMAX;
    // pruned fallback scans where 16+ ant warps per SM hide their reduction latency (C3:
    // 5.78 -> 5.34 ms); the branch-free scan at fewer (C5: 29.4 vs 33.0 ms pruned)
    A.prune_fallback = (long long)h->m_local * h->colonies >= 16ll * h->num_sms;
    A.fb_row_off = h->fb_row_off;
    A.fb_lane_cap = h->fb_lane_cap;
    // candidate-list colonies whose inv_w matrix takes at most half the L2: its fallback rows
    // are prefetched into L2 at launch start (4 MB at pr1002: < 1 us of HBM time); MMAS_L2_PF=0
    // turns it off (A/B)
    {
        static const char* pf = std::getenv("MMAS_L2_PF");
        const unsigned long long bytes = (unsigned long long)h->n * h->ld * sizeof(float);
        A.l2_prefetch_bytes = (h->cl > 0 && !h->rwm && !h->lean && 2 * bytes * h->colonies <= (unsigned long long)h->l2_bytes &&
                               !(pf && pf[0] == '0')) ? bytes : 0ull;
    }
    A.coop_fb = h->coop_fb ? 1 : 0;
    A.warps_per_block = h->cons_warps;
    A.table_bytes_inv = h->tb_inv;
    A.table_bytes_id = h->tb_id;
    A.routes = h->routes;
    A.lengths = h->lengths;
    A.best_key = h->best_key;
    A.fallback_count = h->fallback_count;
    A.tau = h->tau;
    A.heur = h->heur;
    A.alpha = h->alpha;
    A.epoch = h->done + 1;
    A.upd = update_args(h);
    A.xchg = 0;
    A.cs = h->cs;
    A.lean = lean_args(h);
    return A;
}

// Launch with programmatic stream serialisation (PDL): the kernel's blocks may be
// scheduled while the previous kernel on the stream drains; kernels call pdl_wait()
// before reading their predecessor's results.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Raise a kernel's dynamic shared-memory limit to the opt-in maximum (minus its static
// shared memory).  Always the maximum, never the context's own need: the attribute is
// per function and process-wide, so a smaller value set by a later context would break
// the launches of an earlier, larger one.  (Occupancy follows the launch's actual size.)
template <class K>
void allow_max_smem(K* kernel, int optin) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, kernel);
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes);
}

template <int S, bool T, bool R, bool F, bool W = false>
void set_smem_attr(int optin) {
    allow_max_smem(construct_cl_kernel<S, T, R, F, W>, optin);
}

template <int S, bool T, bool R, bool F, bool W = false>
void launch_cl_f(mmas_ctx* h, const ConstructArgs& A) {
    launch_pdl(construct_cl_kernel<S, T, R, F, W>, dim3(h->cons_grid, h->colonies),
               dim3(h->cons_warps * 32), h->cons_smem, h->stream, A);
}

// cl <= 32 (tables padded to 32 slots): one slot per lane; more than 8 ant warps per block
// (large colonies, shared-memory table) take the 16-warp instantiation
template <int S, bool T, bool R>
void launch_cl(mmas_ctx* h, const ConstructArgs& A) {
    if constexpr (S == 1) {
        if constexpr (T) {
            if (h->cons_warps > 8) {
                launch_cl_f<1, T, R, true, true>(h, A);
                return;
            }
        } else {
            // L2 table, fewer than 16 ant warps per SM: the uncapped-register instantiation
            if ((long long)h->m_local * h->colonies < 16ll * h->num_sms) {
                launch_cl_f<1, T, R, true, true>(h, A);
                return;
            }
        }
        launch_cl_f<1, T, R, true>(h, A);
    } else {
        launch_cl_f<S, T, R, false>(h, A);
    }
}

// dispatch over the compile-time variants: slots per lane, table placement, tabu placement
template <bool R>
void launch_cl_r(mmas_ctx* h, const ConstructArgs& A) {
    if (h->smem_table) {
        if (h->slots == 1) launch_cl<1, true, R>(h, A);
        else if (h->slots == 2) launch_cl<2, true, R>(h, A);
        else launch_cl<4, true, R>(h, A);
    } else {
        if (h->slots == 1) launch_cl<1, false, R>(h, A);
        else if (h->slots == 2) launch_cl<2, false, R>(h, A);
        else launch_cl<4, false, R>(h, A);
    }
}

template <bool R>
void set_cl_attrs(int bytes) {
    set_smem_attr<1, true, R, true>(bytes); set_smem_attr<1, false, R, true>(bytes);
    set_smem_attr<1, true, R, true, true>(bytes);
    set_smem_attr<1, false, R, true, true>(bytes);
    set_smem_attr<2, true, R, false>(bytes); set_smem_attr<2, false, R, false>(bytes);
    set_smem_attr<4, true, R, false>(bytes); set_smem_attr<4, false, R, false>(bytes);
}

int launch_two_opt(mmas_ctx* h, bool fuse_select);

// full-row construction (cl == 0): compact-tabu list or bitmask scan; or the roulette wheel
void launch_full(mmas_ctx* h, const ConstructArgs& A) {
    if (h->rwm && h->compact_tabu)
        construct_rwm_kernel<true><<<dim3(h->cons_grid, h->colonies), h->cons_warps * 32, h->cons_smem, h->stream>>>(A);
    else if (h->rwm)
        construct_rwm_kernel<false><<<dim3(h->cons_grid, h->colonies), h->cons_warps * 32, h->cons_smem, h->stream>>>(A);
    else if (h->compact_tabu)
        construct_ct_kernel<<<dim3(h->cons_grid, h->colonies), h->cons_warps * 32, h->cons_smem, h->stream>>>(A);
    else if (h->reg_tabu)
        construct_full_kernel<true><<<dim3(h->cons_grid, h->colonies), h->cons_warps * 32, h->cons_smem, h->stream>>>(A);
    else
        construct_full_kernel<false><<<dim3(h->cons_grid, h->colonies), h->cons_warps * 32, h->cons_smem, h->stream>>>(A);
}

// Construction (rows a1-a4) -- and, with local search on, the 2-opt pass (row a8) that
// then owns the tour lengths and the iteration-best bookkeeping (row a5).
int launch_construct(mmas_ctx* h, bool fuse_select, const ExchangeArgs* xfused = nullptr) {
    if (h->m_local == 0) return MMAS_OK;
    if (h->cfg.local_search) {
        {
            PhaseScope ps(h, 0);
            ConstructArgs A = construct_args(h, false, true);
            if (h->cl == 0 || h->rwm) {
                launch_full(h, A);
            } else if (h->reg_tabu) {
                launch_cl_r<true>(h, A);
            } else {
                launch_cl_r<false>(h, A);
            }
            h->launches++;
            CU(cudaGetLastError());
        }
        return launch_two_opt(h, fuse_select);
    }
    PhaseScope ps(h, 0);
    ConstructArgs A = construct_args(h, fuse_select || xfused != nullptr);
    A.fuse_update = (fuse_select && h->fuse_update) || xfused ? 1 : 0;
    if (xfused) {
        A.xchg = 1;
        A.X = *xfused;
        A.xown = h->xbuf;
        A.xerr = h->xerr;
    }
    if (h->cl == 0 || h->rwm) {
        launch_full(h, A);
    } else if (h->reg_tabu) {
        launch_cl_r<true>(h, A);
    } else {
        launch_cl_r<false>(h, A);
    }
    h->launches++;
    CU(cudaGetLastError());
    return MMAS_OK;
}

int launch_select(mmas_ctx* h, const unsigned char* records, int count) {
    PhaseScope ps(h, 1);
    select_best_kernel<<<dim3(1, h->colonies), 32, 0, h->stream>>>(select_args(h, records, count));
    h->launches++;
    CU(cudaGetLastError());
    return MMAS_OK;
}

int launch_two_opt(mmas_ctx* h, bool fuse_select) {
    PhaseScope ps(h, 3);
    TwoOptArgs T{};
    T.xy = h->xy;
    T.nn = h->ls_nn;
    T.nnd = h->ls_nnd;
    T.xys = h->ls_xys;
    T.nnp = h->ls_nnp;
    T.n = h->n;
    T.K = h->ls_k;
    T.ldr = h->ldr;
    T.m_local = h->m_local;
    T.nwords = h->ls_nwords;
    T.routes = h->routes;
    T.pos = h->ls_pos;
    T.queue = h->ls_queue;
    T.inq = h->ls_inq;
    T.moves = h->ls_moves;
    // route + pos (u16) and the queued bits in shared memory
    const size_t per_ant = (size_t)4 * h->ldr + (size_t)4 * h->ls_nwords;
    // grouped kernel (two_opt.cuh two_opt_group_kernel): coordinates in shared memory, two ants
    // per block.  Opt-in (MMAS_LS_GROUP=1): on C5 its rounds are ~20 % shorter, but two ants per
    // SM instead of three make the local search slower overall (125 -> 151 ms)
    const size_t group_smem = (((size_t)h->n * 4 + 15) & ~(size_t)15) + kLsGroupsMax * per_ant;
    const char* ge = std::getenv("MMAS_LS_GROUP");
    const bool group = h->ls_int_xy && group_smem <= (size_t)h->ls_group_smem_max && ge && ge[0] == '1';
    if (group) {
        T.warps_per_block = kLsGroupsMax * kLsWarps;
        const int grid = std::max(1, (h->m_local + kLsGroupsMax - 1) / kLsGroupsMax);
        launch_pdl(two_opt_group_kernel<kLsGroupsMax>, dim3(grid, h->colonies), dim3(kLsGroupsMax * kLsWarps * 32),
                   group_smem, h->stream, T, construct_args(h, fuse_select));
    } else if (per_ant <= (size_t)h->ls_coop_smem_max) {
        // one block of kLsWarps warps per ant (speculative parallel FIFO, two_opt_coop_kernel)
        T.warps_per_block = kLsWarps;
        if (h->ls_int_xy)
            launch_pdl(two_opt_coop_kernel<true>, dim3(std::max(1, h->m_local), h->colonies), dim3(kLsWarps * 32), per_ant,
                       h->stream, T, construct_args(h, fuse_select));
        else
            launch_pdl(two_opt_coop_kernel<false>, dim3(std::max(1, h->m_local), h->colonies), dim3(kLsWarps * 32), per_ant,
                       h->stream, T, construct_args(h, fuse_select));
    } else {
        T.warps_per_block = 4;
        const int grid = std::max(1, (h->m_local + 3) / 4);
        if (h->ls_int_xy)
            launch_pdl(two_opt_kernel<true>, dim3(grid, h->colonies), dim3(128), 0, h->stream, T, construct_args(h, fuse_select));
        else
            launch_pdl(two_opt_kernel<false>, dim3(grid, h->colonies), dim3(128), 0, h->stream, T, construct_args(h, fuse_select));
    }
    h->launches++;
    CU(cudaGetLastError());
    return MMAS_OK;
}

UpdateArgs update_args(mmas_ctx* h) {
    UpdateArgs U{};
    U.tau = h->tau;
    U.inv_w = h->inv_w;
    U.heur = h->heur;
    U.n = h->n;
    U.ld = h->ld;
    U.alpha = h->alpha;
    U.rho_f = (float)h->cfg.rho;
    U.scal = h->scal;
    U.succ = h->succ;
    U.pred = h->pred;
    U.cand_id = h->cand_id;
    U.cand_inv = h->cand_inv;
    U.cl = h->cl_ld;
    U.iter_dev = h->iter_dev;
    U.err = h->xerr;
    U.spin_bound = h->spin_bound;
    U.cs = h->cs;
    U.lean = lean_args(h);
    U.xy = h->xy;
    U.smem_row = h->cl > 0 && sizeof(float) * (size_t)h->ld <= (size_t)h->smem_optin - 1024;
    return U;
}

int launch_update(mmas_ctx* h) {
    PhaseScope ps(h, 2);
    UpdateArgs U = update_args(h);
    const int threads = 256;
    if (h->lean) {   // one warp per row over the lean representation (R30)
        launch_pdl(lean_update_kernel, dim3((h->n + 7) / 8), dim3(threads), 0, h->stream, U);
        h->launches++;
        CU(cudaGetLastError());
        return MMAS_OK;
    }
    const size_t smem = U.smem_row ? sizeof(float) * (size_t)h->ld : 0;
    launch_pdl(pheromone_update_kernel, dim3(h->n, h->colonies), dim3(threads), smem, h->stream, U);
    h->launches++;
    CU(cudaGetLastError());
    return MMAS_OK;
}

void free_ctx(mmas_ctx* h) {
    if (!h) return;
    if (h->device >= 0) cudaSetDevice(h->device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    void* ptrs[] = {h->xy, h->heur, h->tau, h->inv_w, h->cand_inv, h->cand_id, h->routes, h->lengths,
                    h->best_key, h->fallback_count, h->ib_route, h->gb_route, h->succ, h->pred, h->gb_len,
                    h->ib_len, h->ib_ant, h->scal, h->iter_dev, h->local_record, h->done, h->xerr,
                    h->ls_nn, h->ls_nnd, h->ls_xys, h->ls_nnp, h->ls_pos, h->ls_queue, h->ls_inq, h->ls_moves,
                    h->cand_tau, h->cand_heur, h->sp_id, h->sp_tau, h->sp_inv, h->bg,
                    h->lean_xys, h->heur_tab, h->inv_tab};
    // (pool allocations go back to the pool in stream order; the stream is drained below)
    for (void* p : ptrs)
        if (p) {
            if (h->pooled && h->stream) cudaFreeAsync(p, h->stream);
            else cudaFree(p);
        }
    if (h->stream) cudaStreamSynchronize(h->stream);
    for (void* p : h->xopened) cudaIpcCloseMemHandle(p);
    if (h->xbuf) cudaFree(h->xbuf);
    if (h->xpeers_dev) cudaFree(h->xpeers_dev);
    for (auto e : h->ev_pool) cudaEventDestroy(e);
    if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
    delete h;
}

// Context buffers come from one stream-ordered memory pool per device that keeps what is
// freed (release threshold: unlimited), so creating a colony after another was destroyed maps
// no new memory (mmas_create is inside bench.py's end-to-end timing); MMAS_NO_POOL=1 uses
// plain cudaMalloc.  The peer-exchange buffer stays a cudaMalloc allocation (IPC-exportable).
thread_local cudaStream_t g_alloc_stream = nullptr;   // set by setup() while it allocates
thread_local cudaMemPool_t g_alloc_pool = nullptr;

cudaMemPool_t device_pool(int device) {
    static std::mutex mu;
    static std::vector<cudaMemPool_t> pools;
    if (std::getenv("MMAS_NO_POOL")) return nullptr;
    std::lock_guard<std::mutex> lock(mu);
    if ((int)pools.size() <= device) pools.resize(device + 1, nullptr);
    if (!pools[device]) {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = device;
        cudaMemPool_t pool;
        if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        uint64_t keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        pools[device] = pool;
    }
    return pools[device];
}

template <class T>
int dalloc(T** p, size_t count) {
    const size_t bytes = sizeof(T) * std::max<size_t>(count, 1);
    cudaError_t e = g_alloc_pool ? cudaMallocFromPoolAsync((void**)p, bytes, g_alloc_pool, g_alloc_stream)
                                 : cudaMalloc((void**)p, bytes);
    if (e != cudaSuccess) return fail(MMAS_ENOMEM, std::string("device allocation: ") + cudaGetErrorString(e));
    return MMAS_OK;
}

// The one-launch iteration's grid barrier needs every block of the grid resident at once:
// blocks per SM that fit (registers, shared memory, threads of this instantiation) x SMs >= grid
bool grid_co_resident(mmas_ctx* h) {
    int per_sm = 0;
    cudaError_t e;
    const int threads = h->cons_warps * 32;
    if (h->reg_tabu)
        e = h->cons_warps > 8
                ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, construct_cl_kernel<1, true, true, true, true>, threads, h->cons_smem)
                : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, construct_cl_kernel<1, true, true, true>, threads, h->cons_smem);
    else
        e = h->cons_warps > 8
                ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, construct_cl_kernel<1, true, false, true, true>, threads, h->cons_smem)
                : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, construct_cl_kernel<1, true, false, true>, threads, h->cons_smem);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return (long long)per_sm * h->num_sms >= (long long)h->cons_grid * h->colonies;
}

// MMAS_CREATE_PROFILE=1: host wall time of each setup phase on stderr (the e2e number's
// create share, bench.py)
struct SetupClock {
    bool on = std::getenv("MMAS_CREATE_PROFILE") != nullptr;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now(), t = t0;
    void mark(const char* what, cudaStream_t st) {
        if (!on) return;
        cudaStreamSynchronize(st);
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "mmas_create %-28s %8.3f ms\n", what,
                     std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

int setup(mmas_ctx* h) {
    SetupClock clk;
    const mmas_config& c = h->cfg;
    const int n = c.n;
    if (c.device >= 0) CU(cudaSetDevice(c.device));
    CU(cudaGetDevice(&h->device));
    CU(cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->device));
    CU(cudaDeviceGetAttribute(&h->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device));
    CU(cudaDeviceGetAttribute(&h->l2_bytes, cudaDevAttrL2CacheSize, h->device));
    if (c.stream || c.use_caller_stream) {
        h->stream = (cudaStream_t)c.stream;
    } else {
        CU(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
        h->own_stream = true;
    }
    h->n = n;
    h->ld = round_up(n, 32);
    h->ldr = round_up(n, 32);
    h->cl = c.cand_len;
    h->cl_ld = (h->cl > 0 && h->cl < 32) ? 32 : h->cl;
    h->m = c.n_ants;
    h->alpha = (int)c.alpha;
    h->ant_lo = (int)((int64_t)c.rank * c.n_ants / c.world);
    h->m_local = (int)((int64_t)(c.rank + 1) * c.n_ants / c.world) - h->ant_lo;
    h->key.k0 = (uint32_t)c.seed;
    h->key.k1 = (uint32_t)(c.seed >> 32);
    h->rec_bytes = round_up(8 + 2 * n, 16);
    h->colonies = std::max(1, c.colonies);
    // allocate the context's buffers from the device pool, in this stream's order
    struct PoolScope {
        PoolScope(mmas_ctx* h) {
            g_alloc_pool = device_pool(h->device);
            g_alloc_stream = h->stream;
            h->pooled = g_alloc_pool != nullptr;
        }
        ~PoolScope() {
            g_alloc_pool = nullptr;
            g_alloc_stream = nullptr;
        }
    } pool_scope(h);
    if (const char* sb = std::getenv("MMAS_SPIN_BOUND")) h->spin_bound = std::max(1ll << 10, std::atoll(sb));

    const size_t nn = (size_t)n * h->ld;
    // per-colony strides (R29; kernels shift by blockIdx.y * stride)
    const size_t K = (size_t)h->colonies;
    const size_t ma = (size_t)std::max(h->m_local, 1);
    h->cs.nn = (long long)nn;
    h->cs.cand = (long long)n * h->cl_ld + 64;
    h->cs.routes = (long long)ma * h->ldr;
    h->cs.ants = (int)ma;
    h->cs.vec = h->ldr;
    h->cs.inq = 0;
    int st;
    h->lean = c.pheromone == MMAS_PHEROMONE_LEAN;
    const size_t nn_alloc = h->lean ? 0 : nn;   // lean (R30): no n x n matrices at all
    if ((st = dalloc(&h->xy, n)) || (st = dalloc(&h->heur, nn_alloc)) || (st = dalloc(&h->tau, nn_alloc * K)) ||
        (st = dalloc(&h->inv_w, nn_alloc * K)) || (st = dalloc(&h->cand_inv, (size_t)h->cs.cand * K)) ||
        (st = dalloc(&h->cand_id, (size_t)n * h->cl_ld + 64)) ||
        (st = dalloc(&h->routes, ma * h->ldr * K)) ||
        (st = dalloc(&h->lengths, ma * K)) || (st = dalloc(&h->best_key, K)) ||
        (st = dalloc(&h->fallback_count, 1)) || (st = dalloc(&h->ib_route, (size_t)h->ldr * K)) ||
        (st = dalloc(&h->gb_route, (size_t)h->ldr * K)) ||
        (st = dalloc(&h->succ, (size_t)h->ldr * K)) || (st = dalloc(&h->pred, (size_t)h->ldr * K)) ||
        (st = dalloc(&h->gb_len, K)) || (st = dalloc(&h->ib_len, K)) || (st = dalloc(&h->ib_ant, K)) ||
        (st = dalloc(&h->scal, 4 * K)) || (st = dalloc(&h->iter_dev, K)) ||
        (st = dalloc(&h->local_record, (size_t)h->rec_bytes)) || (st = dalloc(&h->done, 2 * K)) ||
        (st = dalloc(&h->xerr, 1)))
        return st;

    clk.mark("device / stream / allocations", h->stream);
    CU(cudaMemcpyAsync(h->xy, c.coords, sizeof(double) * 2 * n, cudaMemcpyHostToDevice, h->stream));
    CU(cudaMemsetAsync(h->routes, 0, sizeof(uint16_t) * ma * h->ldr * K, h->stream));
    CU(cudaMemsetAsync(h->lengths, 0, sizeof(long long) * ma * K, h->stream));
    CU(cudaMemsetAsync(h->best_key, 0xFF, sizeof(unsigned long long) * K, h->stream));
    CU(cudaMemsetAsync(h->fallback_count, 0, sizeof(unsigned long long), h->stream));
    CU(cudaMemsetAsync(h->gb_len, 0xFF, sizeof(long long) * K, h->stream));   // -1: empty
    CU(cudaMemsetAsync(h->ib_len, 0xFF, sizeof(long long) * K, h->stream));
    CU(cudaMemsetAsync(h->iter_dev, 0, sizeof(uint32_t) * K, h->stream));
    CU(cudaMemsetAsync(h->done, 0, 2 * sizeof(unsigned int) * K, h->stream));
    CU(cudaMemsetAsync(h->xerr, 0, sizeof(uint32_t), h->stream));
    CU(cudaMemsetAsync(h->succ, 0, sizeof(uint16_t) * h->ldr * K, h->stream));
    CU(cudaMemsetAsync(h->pred, 0, sizeof(uint16_t) * h->ldr * K, h->stream));

    // eta^beta (R11, R18)
    if (h->lean) {
        // (lean: computed per edge where needed, heur_edge)
    } else if (is_int_in(c.beta, 0, 8)) {
        dim3 g((h->ld + 255) / 256, n);
        heur_kernel<<<g, 256, 0, h->stream>>>(h->xy, n, h->ld, (int)c.beta, h->heur);
        h->launches++;
        CU(cudaGetLastError());
    } else {
        std::vector<float> hh(nn, 1.0f);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) {
                const int32_t d = host_dist(c.coords, i, j);
                hh[(size_t)i * h->ld + j] = (float)std::pow((double)(d > 1 ? d : 1), -c.beta);
            }
        CU(cudaMemcpyAsync(h->heur, hh.data(), sizeof(float) * nn, cudaMemcpyHostToDevice, h->stream));
        CU(cudaStreamSynchronize(h->stream));
    }

    clk.mark("memsets + eta^beta", h->stream);
    // candidate lists: on the device (cand_lists_kernel) where a row's distances fit in shared
    // memory, else on the host (parallel over rows)
    const bool dev_cand = (size_t)n * 4 <= (size_t)h->smem_optin - 2048 && !std::getenv("MMAS_HOST_CAND");
    if (h->cl > 0 && dev_cand) {
        if (h->cl_ld != h->cl) {   // padding slots: the row's own city (always visited)
            std::vector<uint16_t> padded((size_t)n * h->cl_ld);
            for (int i = 0; i < n; ++i)
                for (int k = 0; k < h->cl_ld; ++k) padded[(size_t)i * h->cl_ld + k] = (uint16_t)i;
            CU(cudaMemcpyAsync(h->cand_id, padded.data(), sizeof(uint16_t) * padded.size(), cudaMemcpyHostToDevice,
                               h->stream));
            CU(cudaStreamSynchronize(h->stream));
        }
        // n <= 1024 with distances < 2^22 (|coordinates| < 2^20): one warp per row, keys in registers
        double cmax = 0.0;
        for (int i = 0; i < 2 * n; ++i) cmax = std::max(cmax, std::fabs(c.coords[i]));
        if (n <= kCandWarpMaxN && cmax < 1048576.0 && !std::getenv("MMAS_CAND_BLOCK")) {
            cand_lists_warp_kernel<<<std::max(1, (n + 7) / 8), 256, 0, h->stream>>>(h->xy, n, h->cl, h->cand_id, h->cl_ld);
        } else {
            cudaFuncSetAttribute(cand_lists_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, h->smem_optin - 2048);
            cand_lists_kernel<<<std::min(n, 8 * h->num_sms), 256, (size_t)n * 4, h->stream>>>(h->xy, n, h->cl,
                                                                                              h->cand_id, h->cl_ld);
        }
        h->launches++;
        CU(cudaGetLastError());
    } else if (h->cl > 0) {
        std::vector<uint16_t> cand;
        candidate_lists(c.coords, n, h->cl, cand);
        if (h->cl_ld != h->cl) {   // pad every row to cl_ld slots with the row's own city
            std::vector<uint16_t> padded((size_t)n * h->cl_ld);
            for (int i = 0; i < n; ++i)
                for (int k = 0; k < h->cl_ld; ++k)
                    padded[(size_t)i * h->cl_ld + k] = k < h->cl ? cand[(size_t)i * h->cl + k] : (uint16_t)i;
            cand.swap(padded);
        }
        CU(cudaMemcpyAsync(h->cand_id, cand.data(), sizeof(uint16_t) * cand.size(), cudaMemcpyHostToDevice,
                           h->stream));
        CU(cudaStreamSynchronize(h->stream));
    }

    // row a8: 2-opt neighbour lists (the 32 nearest) and per-ant scratch
    if (c.local_search) {
        h->ls_k = std::min(32, n - 1);
        h->ls_nwords = (n + 31) / 32;
        std::vector<uint16_t> nnl;
        // the lists and their distances on the device (cand_lists_kernel, ls_dist_kernel) where
        // a row's distances fit in shared memory (C5: was ~80-190 ms on the host), else the host
        const bool dev_ls = dev_cand;
        if (!dev_ls) candidate_lists(c.coords, n, h->ls_k, nnl);
        const size_t nent = (size_t)n * h->ls_k;
        // neighbour distances (exact R12 values; the 2-opt evaluation reads d(a, c) from here)
        std::vector<int32_t> nnd(dev_ls ? 0 : nent);
        if (!dev_ls)
            for (int i = 0; i < n; ++i)
                for (int k = 0; k < h->ls_k; ++k) nnd[(size_t)i * h->ls_k + k] = host_dist(c.coords, i, nnl[(size_t)i * h->ls_k + k]);
        // integral coordinates with |x|, |y| <= 16383: the 2-opt kernels compute distances in
        // 32-bit integer arithmetic (two_opt.cuh euc2d_int; identical results)
        h->ls_int_xy = true;
        std::vector<short2> xys((size_t)n);
        for (int i = 0; i < n && h->ls_int_xy; ++i) {
            const double x = c.coords[2 * i], y = c.coords[2 * i + 1];
            if (x != std::floor(x) || y != std::floor(y) || std::fabs(x) > 16383.0 || std::fabs(y) > 16383.0)
                h->ls_int_xy = false;
            else
                xys[(size_t)i] = make_short2((short)x, (short)y);
        }
        h->cs.inq = (int)(ma * h->ls_nwords);
        if ((st = dalloc(&h->ls_nn, nent)) || (st = dalloc(&h->ls_nnd, nent)) ||
            (st = dalloc(&h->ls_pos, ma * h->ldr * K)) ||
            (st = dalloc(&h->ls_queue, ma * h->ldr * K)) || (st = dalloc(&h->ls_inq, ma * h->ls_nwords * K)) ||
            (st = dalloc(&h->ls_moves, 1)))
            return st;
        if (h->ls_int_xy) {
            if ((st = dalloc(&h->ls_xys, (size_t)n)) || (st = dalloc(&h->ls_nnp, nent))) return st;
            CU(cudaMemcpyAsync(h->ls_xys, xys.data(), sizeof(short2) * n, cudaMemcpyHostToDevice, h->stream));
        }
        if (dev_ls) {
            if (h->cl == h->ls_k && h->cl_ld == h->cl) {   // the same lists (R10): copy them
                CU(cudaMemcpyAsync(h->ls_nn, h->cand_id, sizeof(uint16_t) * nent, cudaMemcpyDeviceToDevice, h->stream));
            } else {
                cudaFuncSetAttribute(cand_lists_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, h->smem_optin - 2048);
                cand_lists_kernel<<<std::min(n, 8 * h->num_sms), 256, (size_t)n * 4, h->stream>>>(h->xy, n, h->ls_k,
                                                                                                  h->ls_nn, h->ls_k);
                h->launches++;
            }
            ls_dist_kernel<<<4 * h->num_sms, 256, 0, h->stream>>>(h->xy, n, h->ls_k, h->ls_nn, h->ls_nnd,
                                                                  h->ls_int_xy ? h->ls_nnp : nullptr);
            h->launches++;
            CU(cudaGetLastError());
            CU(cudaStreamSynchronize(h->stream));   // xys goes out of scope
        } else {
            if (h->ls_int_xy) {
                std::vector<uint32_t> nnp(nent);
                for (size_t e = 0; e < nent; ++e) nnp[e] = (uint32_t)nnl[e] | ((uint32_t)nnd[e] << 16);
                CU(cudaMemcpyAsync(h->ls_nnp, nnp.data(), sizeof(uint32_t) * nnp.size(), cudaMemcpyHostToDevice,
                                   h->stream));
                CU(cudaStreamSynchronize(h->stream));   // the host vectors go out of scope
            }
            CU(cudaMemcpyAsync(h->ls_nnd, nnd.data(), sizeof(int32_t) * nnd.size(), cudaMemcpyHostToDevice, h->stream));
            CU(cudaMemcpyAsync(h->ls_nn, nnl.data(), sizeof(uint16_t) * nnl.size(), cudaMemcpyHostToDevice, h->stream));
        }
        CU(cudaMemsetAsync(h->ls_moves, 0, sizeof(unsigned long long), h->stream));
        CU(cudaStreamSynchronize(h->stream));
    }

    clk.mark("candidate + 2-opt lists", h->stream);
    // initial limits from the NN tour (Alg. 1); F from libm pow (R2)
    {
        // NN tour on the device (one block; the host loop was O(n^2) on one core)
        // (scratch from the context's pool -- dalloc -- not the device's default pool)
        long long* d_len = nullptr;
        if ((st = dalloc(&d_len, 1))) return st;
        // integral coordinates within +-16383: the NN tour's distances in 32-bit arithmetic
        short2* d_xys = nullptr;
        {
            bool integral = true;
            std::vector<short2> xs((size_t)n);
            for (int i = 0; i < n && integral; ++i) {
                const double x = c.coords[2 * i], y = c.coords[2 * i + 1];
                if (x != std::floor(x) || y != std::floor(y) || std::fabs(x) > 16383.0 || std::fabs(y) > 16383.0)
                    integral = false;
                else
                    xs[(size_t)i] = make_short2((short)x, (short)y);
            }
            if (integral) {
                if ((st = dalloc(&d_xys, (size_t)n))) return st;
                CU(cudaMemcpyAsync(d_xys, xs.data(), sizeof(short2) * n, cudaMemcpyHostToDevice, h->stream));
                CU(cudaStreamSynchronize(h->stream));
            }
        }
        clk.mark("NN tour inputs", h->stream);
        {
            // the candidate rows (padded to cl_ld slots with the row's own city, always visited)
            // staged into shared memory next to the route when they fit
            const size_t route_b = (size_t)((n + 7) & ~7) * 2;
            const size_t cand_b = (size_t)n * h->cl_ld * 2;
            const size_t budget = (size_t)h->smem_optin - 16384;   // static: tabu words + partials
            const int stage = h->cl > 0 && route_b + cand_b <= budget;
            const size_t dyn = route_b + (stage ? cand_b : 0);
            // n <= 1024: one warp with the register tabu (nn_tour_warp_kernel), when the route,
            // coordinates and candidate table fit in its shared memory
            const size_t warp_dyn = 2048 + (((size_t)n * (d_xys ? 4 : 16) + 15) & ~(size_t)15) + cand_b;
            if (n <= 1024 && warp_dyn <= budget && !std::getenv("MMAS_NN_BLOCK")) {
                cudaFuncSetAttribute(nn_tour_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)warp_dyn);
                nn_tour_warp_kernel<<<1, 32, warp_dyn, h->stream>>>(h->xy, d_xys, n, h->cl > 0 ? h->cand_id : nullptr,
                                                                    h->cl, h->cl_ld, d_len);
            } else {
                cudaFuncSetAttribute(nn_tour_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
                nn_tour_kernel<<<1, nn_threads(n), dyn, h->stream>>>(h->xy, d_xys, n, h->cl > 0 ? h->cand_id : nullptr,
                                                                     h->cl, h->cl_ld, stage, d_len);
            }
        }
        if (d_xys) CU(h->pooled ? cudaFreeAsync(d_xys, h->stream) : cudaFree(d_xys));
        h->launches++;
        CU(cudaGetLastError());
        long long len = 0;
        CU(cudaMemcpyAsync(&len, d_len, sizeof(len), cudaMemcpyDeviceToHost, h->stream));
        CU(cudaStreamSynchronize(h->stream));
        CU(h->pooled ? cudaFreeAsync(d_len, h->stream) : cudaFree(d_len));
        h->nn_len = len;
    }
    const double pn = std::pow(c.p_best, 1.0 / (double)n);
    h->factor = (1.0 - pn) / (((double)n / 2.0 - 1.0) * pn);
    std::vector<float> lim(4 * K, 0.0f);
    host_limits(c.rho, h->nn_len, h->factor, &lim[0], &lim[1]);
    for (size_t k = 1; k < K; ++k) std::copy(lim.begin(), lim.begin() + 4, lim.begin() + 4 * k);   // same NN tour
    CU(cudaMemcpyAsync(h->scal, lim.data(), sizeof(float) * lim.size(), cudaMemcpyHostToDevice, h->stream));
    if (h->lean) {
        // R30: L = iterations after which a trail without deposits equals tau_min (ratio F =
        // tau_min / tau_max), with margin for the fp32 rounding; <= 2 (L + 1) sparse trails per row
        const double F = std::min(1.0, (double)lim[0] / (double)lim[1]);
        const double rf = (double)(float)c.rho * (1.0 + 1e-6);
        h->lean_L = F >= 1.0 ? 1 : (int)std::ceil(std::log(F * (1.0 - 1e-5)) / std::log(rf)) + 2;
        h->lean_cap = round_up(2 * (h->lean_L + 1), 32);
        const size_t ncl = (size_t)n * h->cl_ld + 64, nsp = (size_t)n * h->lean_cap;
        if ((st = dalloc(&h->cand_tau, ncl)) || (st = dalloc(&h->cand_heur, ncl)) || (st = dalloc(&h->sp_id, nsp)) ||
            (st = dalloc(&h->sp_tau, nsp)) || (st = dalloc(&h->sp_inv, nsp)) || (st = dalloc(&h->bg, 2)))
            return st;
        // integral coordinates within +-16383: 32-bit distances and tables by distance (R30)
        bool integral = true;
        double lo_x = INFINITY, hi_x = -INFINITY, lo_y = INFINITY, hi_y = -INFINITY;
        std::vector<short2> xs((size_t)n);
        for (int i = 0; i < n && integral; ++i) {
            const double x = c.coords[2 * i], y = c.coords[2 * i + 1];
            if (x != std::floor(x) || y != std::floor(y) || std::fabs(x) > 16383.0 || std::fabs(y) > 16383.0)
                integral = false;
            else
                xs[(size_t)i] = make_short2((short)x, (short)y);
            lo_x = std::min(lo_x, x); hi_x = std::max(hi_x, x);
            lo_y = std::min(lo_y, y); hi_y = std::max(hi_y, y);
        }
        if (integral && !std::getenv("MMAS_LEAN_NO_TABLE")) {
            h->dtab = (int)std::ceil(std::sqrt((hi_x - lo_x) * (hi_x - lo_x) + (hi_y - lo_y) * (hi_y - lo_y))) + 2;
            if ((st = dalloc(&h->lean_xys, (size_t)n + 4)) || (st = dalloc(&h->heur_tab, (size_t)h->dtab)) ||
                (st = dalloc(&h->inv_tab, (size_t)h->dtab)))
                return st;
            CU(cudaMemcpyAsync(h->lean_xys, xs.data(), sizeof(short2) * n, cudaMemcpyHostToDevice, h->stream));
            CU(cudaStreamSynchronize(h->stream));   // xs goes out of scope
        }
        lean_init_kernel<<<std::max(1, std::min(4096, (int)((nsp + 255) / 256))), 256, 0, h->stream>>>(
            h->xy, n, h->cl_ld, h->cand_id, (int)c.beta, h->alpha, h->scal, lean_args(h), h->cand_inv);
        h->launches++;
        CU(cudaGetLastError());
    }
    for (size_t k = 0; k < K && !h->lean; ++k) {
        dim3 g((h->ld + 255) / 256, n);
        init_trails_kernel<<<g, 256, 0, h->stream>>>(h->tau + k * nn, h->inv_w + k * nn, h->heur, n, h->ld, h->alpha,
                                                     h->scal);
        h->launches++;
        CU(cudaGetLastError());
        if (h->cl > 0) {
            gather_cand_kernel<<<std::max(1, std::min(4096, (n * h->cl_ld + 255) / 256)), 256, 0, h->stream>>>(
                h->inv_w + k * nn, n, h->ld, h->cand_id, h->cand_inv + k * h->cs.cand, h->cl_ld);
            h->launches++;
            CU(cudaGetLastError());
        }
    }
    CU(cudaStreamSynchronize(h->stream));   // lim goes out of scope

    clk.mark("NN tour kernel + trails", h->stream);
    // ---- construction launch plan ----
    // dynamic shared memory a construction kernel may take: the opt-in limit minus its
    // static shared memory (block_finish's slots; 128 B, reserve 1 KB)
    const size_t cons_dyn_max = (size_t)h->smem_optin - 1024;
    const int nwords = round_up((n + 31) / 32, 4);
    h->reg_tabu = n <= 1024;
    const size_t tabu_bytes = h->reg_tabu ? 0 : (size_t)nwords * 4;
    h->slots = h->cl <= 32 ? 1 : (h->cl <= 64 ? 2 : 4);
    if (h->cfg.selection == MMAS_SELECT_RWM) {
        // roulette wheel: smem bitmask tabu (or CT entries) per ant warp, rows from L2
        h->rwm = true;
        h->compact_tabu = h->cfg.tabu == MMAS_TABU_COMPACT;
        const int words = h->compact_tabu ? (n + 1) / 2 : (n + 31) / 32;
        const size_t per_warp = (size_t)round_up(words, 4) * 4;
        int w = 4;
        while (w > 1 && 128 + (size_t)w * per_warp > cons_dyn_max) --w;
        h->cons_warps = w;
        h->cons_grid = std::max(1, (h->m_local + w - 1) / w);
        h->cons_smem = 128 + (size_t)w * per_warp;
    } else if (h->cl > 0) {
        h->tb_inv = (uint32_t)round_up(n * h->cl_ld * 4, 16);
        h->tb_id = (uint32_t)round_up(n * h->cl_ld * 2, 16);
        const size_t per_warp = tabu_bytes;   // per ant warp: its tabu (shared-memory variant)
        // one block per SM holding the whole table; as many ant warps as needed
        const int wmax = h->slots == 1 ? 16 : 8;   // construct_cl_kernel's launch bounds
        // the SMs are shared out between the colonies (one persistent block per SM each)
        const int sms = std::max(1, h->num_sms / h->colonies);
        int w = std::max(1, std::min(wmax, (h->m_local + sms - 1) / sms));
        if (const char* e = std::getenv("MMAS_CONS_WARPS")) w = std::max(1, std::min(wmax, std::atoi(e)));   // (A/B)
        size_t need = 128 + (size_t)h->tb_inv + h->tb_id + 16 + (size_t)w * per_warp;
        h->smem_table = need <= cons_dyn_max;
        if (h->smem_table) {
            // persistent: at most one block per SM, each loads the table once and loops over
            // its ants (large colonies do not re-stage the table per wave)
            h->cons_warps = w;
            h->cons_grid = std::max(1, std::min(sms, (h->m_local + w - 1) / w));
            h->cons_smem = need;
            // fused update (construct.cuh fused_update): one iteration = one launch.  Needs the
            // whole grid resident (grid <= SMs, one block each), one candidate slot per lane,
            // no exchange or local search between construction and update, and room for each
            // warp's tau + heur rows in the block's shared memory
            const size_t fused_need = 256 + (size_t)w * 2 * 4 * h->ld;
            const bool fusable = !c.local_search && h->slots == 1 && !c.separate_update && !h->lean &&
                                 std::max(need, fused_need) <= cons_dyn_max;
            h->fuse_update = fusable && c.world == 1;
            h->fuse_peers = fusable && c.world > 1 && h->m_local > 0;
            if (fusable) h->cons_smem = std::max(need, fused_need);
        } else {
            h->cons_warps = 4;
            h->cons_grid = std::max(1, (h->m_local + 3) / 4);
            if (const char* e = std::getenv("MMAS_CONS_GRID")) h->cons_grid = std::max(1, std::atoi(e));   // (A/B)
            h->cons_smem = 128 + 16 + 4 * per_warp;
            // per warp kFbBufs 8 KB chunk buffers for the R9 fallback scans over HBM-resident rows
            // (construct.cuh scan_unvisited_staged), when they leave room for two blocks per SM
            const size_t off = (h->cons_smem + 127) & ~(size_t)127;
            const size_t with_row = off + (size_t)h->cons_warps * kFbBufs * 4 * kFbChunk;
            // only where inv_w is not L2-resident (C5: its rows come from HBM; C3's L2-resident
            // rows measured 1.5 % slower with the staging)
            const bool hbm_rows = 4.0 * (double)n * h->ld > 0.75 * (double)h->l2_bytes ||
                                  std::getenv("MMAS_FB_ROW") != nullptr;   // (tests force it on small n)
            if (hbm_rows && 2 * (with_row + 1024) <= (size_t)h->smem_optin && !std::getenv("MMAS_NO_FB_ROW")) {
                h->fb_row_off = (uint32_t)off;
                h->cons_smem = with_row;
                // paired fallback scans (construct.cuh CoopSlot): at fewer than 16 ant warps per SM
                // (the uncapped-register instantiation), n > 1024, one slot per lane, WRS fallback:
                // each block's four warps build two ants, each with a helper for its scans
                // -- only while the paired grid (twice the blocks) is still resident in one wave:
                // C65KL's 32 KB tabus make ~100 KB blocks, 2 per SM, and 400 paired blocks
                // measured 1504 ms against 1256 ms for 200 unpaired ones
                const char* cf = std::getenv("MMAS_COOP_FB");
                h->coop_fb = !(cf && cf[0] == '0') && !h->reg_tabu && h->slots == 1 &&
                             (long long)h->m_local * h->colonies < 16ll * h->num_sms &&
                             c.fallback == MMAS_FALLBACK_WRS;
                if (h->coop_fb && !(cf && cf[0] == '1')) {
                    int per_sm = 0;
                    set_smem_attr<1, false, false, true, true>(h->smem_optin);
                    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, construct_cl_kernel<1, false, false, true, true>,
                                                                      h->cons_warps * 32, with_row) != cudaSuccess) {
                        cudaGetLastError();
                        per_sm = 0;
                    }
                    h->coop_fb = (long long)std::max(1, (h->m_local + 1) / 2) * h->colonies <= (long long)per_sm * h->num_sms;
                }
                if (h->coop_fb) h->cons_grid = std::max(1, (h->m_local + 1) / 2);
            }
        }
    } else if (h->cfg.tabu == MMAS_TABU_COMPACT) {
        // CT entries: n u16 per ant warp, padded to 256 positions (one scan trip)
        h->compact_tabu = true;
        const size_t ent_bytes = (size_t)round_up(n, 256) * 2;
        int w = 4;
        while (w > 1 && 128 + (size_t)w * ent_bytes > cons_dyn_max) --w;
        h->cons_warps = w;
        h->cons_grid = std::max(1, (h->m_local + w - 1) / w);
        h->cons_smem = 128 + (size_t)w * ent_bytes;
    } else {
        h->cons_warps = 4;
        h->cons_grid = std::max(1, (h->m_local + 3) / 4);
        h->cons_smem = 128 + 4 * tabu_bytes;
    }
    if (h->cons_smem > cons_dyn_max)
        return fail(MMAS_EINVAL, "n too large for the shared-memory tabu of one block");
    // lane-compacted fallback scans (construct.cuh fallback_compact / lean_fallback_compact):
    // taken at steps with at most cap unvisited cities.  Measured (A/B):
    // register tabu with rows of more than two 256-city trips (C2) 224 (driver window 0.2286
    // -> 0.2038 ms with the rest of the round's fallback work); one- or two-trip rows (C1) are
    // cheaper to scan whole; the shared-memory tabu with L2-resident rows (C3) 64 (5.13 ->
    // 5.06 ms; 128+ slower: the per-lane word counts); HBM-resident rows (C5, paired scans)
    // n / 8 (construction 18.6 -> 14.7 ms at 2048; 4096: 15.0, 9256: 16.9); the memory-lean
    // pheromone, whose trip scans recompute every background value from the coordinates, n / 2,
    // and every fallback beyond 32768 cities (C5L construction 44 -> 25 ms at 9256, 27.3 at n;
    // C65KL 1256 -> 293 ms per iteration at n, 318 at n / 2, 384 at n / 4).
    // MMAS_FB_COMPACT=<cap> overrides (0 = off; the parity tests force every variant).
    if (h->cl > 0 && !h->rwm) {
        const bool hbm_rows = 4.0 * (double)n * h->ld > 0.75 * (double)h->l2_bytes;
        int cap = h->lean ? (n > 32768 ? n : n / 2)
                          : h->reg_tabu ? (n > 512 && !hbm_rows ? 224 : 0) : (hbm_rows ? n / 8 : 64);
        if (const char* e = std::getenv("MMAS_FB_COMPACT")) cap = std::max(0, std::atoi(e));
        h->fb_lane_cap = cap;
    } else if (h->cl == 0 && !h->rwm && !h->compact_tabu) {
        // full-row construction (construct_full_kernel, C4): the same compacted scan for the
        // last steps of a tour, where the pruned trip scan still draws a Philox per live group
        // (C4 A/B: 27.78 ms at 0, 26.72 at 250 ~ n / 10, 26.83 at 398, 27.77 at 600, 31.9 at 1000)
        int cap = n / 10;
        if (const char* e = std::getenv("MMAS_FB_COMPACT")) cap = std::max(0, std::atoi(e));
        h->fb_lane_cap = cap;
    }
    allow_max_smem(construct_rwm_kernel<false>, h->smem_optin);
    allow_max_smem(construct_rwm_kernel<true>, h->smem_optin);
    if (h->cl > 0) {
        if (h->reg_tabu) set_cl_attrs<true>(h->smem_optin);
        else set_cl_attrs<false>(h->smem_optin);
    } else {
        allow_max_smem(construct_full_kernel<true>, h->smem_optin);
        allow_max_smem(construct_full_kernel<false>, h->smem_optin);
        allow_max_smem(construct_ct_kernel, h->smem_optin);
    }
    {
        cudaFuncAttributes fa{}, fb{};
        cudaFuncGetAttributes(&fa, two_opt_coop_kernel<true>);
        cudaFuncGetAttributes(&fb, two_opt_coop_kernel<false>);
        // dynamic = opt-in limit - static (both instantiations)
        h->ls_coop_smem_max = h->smem_optin - (int)std::max(fa.sharedSizeBytes, fb.sharedSizeBytes);
        cudaFuncSetAttribute(two_opt_coop_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             h->ls_coop_smem_max);
        cudaFuncSetAttribute(two_opt_coop_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             h->ls_coop_smem_max);
        cudaFuncAttributes fg{};
        cudaFuncGetAttributes(&fg, two_opt_group_kernel<kLsGroupsMax>);
        h->ls_group_smem_max = h->smem_optin - (int)fg.sharedSizeBytes;
        cudaFuncSetAttribute(two_opt_group_kernel<kLsGroupsMax>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             h->ls_group_smem_max);
        // experiment (MMAS_LS_CARVEOUT = percent of the unified L1/shared memory given to shared
        // memory): fewer resident 2-opt blocks per SM, but an L1 large enough for the coordinates
        if (const char* co = std::getenv("MMAS_LS_CARVEOUT")) {
            const int pct = std::atoi(co);
            cudaFuncSetAttribute(two_opt_coop_kernel<true>, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
            cudaFuncSetAttribute(two_opt_coop_kernel<false>, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
        }
    }
    allow_max_smem(pheromone_update_kernel, h->smem_optin);
    CU(cudaGetLastError());
    clk.mark("launch plan + attributes", h->stream);
    // the one-launch iteration only where its whole grid fits on the device at once
    if ((h->fuse_update || h->fuse_peers) && !grid_co_resident(h)) h->fuse_update = h->fuse_peers = false;
    clk.mark("co-residency check", h->stream);
    CU(cudaStreamSynchronize(h->stream));
    return MMAS_OK;
}

int validate(const mmas_config* c) {
    if (!c) return fail(MMAS_EINVAL, "config is NULL");
    if (!c->coords) return fail(MMAS_EINVAL, "coords is NULL");
    if (c->n < 3 || c->n >= 65536) return fail(MMAS_EINVAL, "n must satisfy 3 <= n < 65536");
    if (c->n_ants < 1 || c->n_ants >= (1 << 24)) return fail(MMAS_EINVAL, "n_ants must satisfy 1 <= m < 2^24");
    if (c->cand_len < 0 || c->cand_len > c->n - 1 || c->cand_len > 128)
        return fail(MMAS_EINVAL, "cand_len must satisfy 0 <= cl <= min(n-1, 128)");
    if (!(c->rho > 0.0 && c->rho < 1.0)) return fail(MMAS_EINVAL, "rho must satisfy 0 < rho < 1");
    if (!is_int_in(c->alpha, 0, 8)) return fail(MMAS_EINVAL, "alpha must be an integer in [0, 8]");
    if (!(c->beta >= 0.0) || !std::isfinite(c->beta)) return fail(MMAS_EINVAL, "beta must be finite and >= 0");
    if (!(c->p_best > 0.0 && c->p_best < 1.0)) return fail(MMAS_EINVAL, "p_best must satisfy 0 < p < 1");
    if (c->deposit != MMAS_DEPOSIT_ITERATION_BEST && c->deposit != MMAS_DEPOSIT_GLOBAL_BEST)
        return fail(MMAS_EINVAL, "deposit must be MMAS_DEPOSIT_*");
    if (c->fallback != MMAS_FALLBACK_WRS && c->fallback != MMAS_FALLBACK_ARGMAX)
        return fail(MMAS_EINVAL, "fallback must be MMAS_FALLBACK_*");
    if (c->local_search != 0 && c->local_search != 1) return fail(MMAS_EINVAL, "local_search must be 0 or 1");
    if (c->tabu != MMAS_TABU_BITMASK && c->tabu != MMAS_TABU_COMPACT)
        return fail(MMAS_EINVAL, "tabu must be MMAS_TABU_*");
    if (c->tabu == MMAS_TABU_COMPACT && c->cand_len != 0)
        return fail(MMAS_EINVAL, "tabu = MMAS_TABU_COMPACT requires cand_len == 0 (R27)");
    if (c->selection != MMAS_SELECT_WRS && c->selection != MMAS_SELECT_RWM)
        return fail(MMAS_EINVAL, "selection must be MMAS_SELECT_*");
    if (c->selection == MMAS_SELECT_RWM && c->fallback == MMAS_FALLBACK_ARGMAX)
        return fail(MMAS_EINVAL, "selection = MMAS_SELECT_RWM uses the roulette wheel as its fallback (R28)");
    if (c->world < 1 || c->rank < 0 || c->rank >= c->world) return fail(MMAS_EINVAL, "need 0 <= rank < world");
    if (c->colonies < 0 || c->colonies > 65535) return fail(MMAS_EINVAL, "colonies must satisfy 0 <= k <= 65535 (0 = 1)");
    if (c->pheromone != MMAS_PHEROMONE_DENSE && c->pheromone != MMAS_PHEROMONE_LEAN)
        return fail(MMAS_EINVAL, "pheromone must be MMAS_PHEROMONE_*");
    if (c->pheromone == MMAS_PHEROMONE_LEAN &&
        (c->cand_len < 1 || !is_int_in(c->beta, 0, 8) || c->selection != MMAS_SELECT_WRS ||
         c->fallback != MMAS_FALLBACK_WRS || c->colonies > 1))
        return fail(MMAS_EINVAL, "pheromone = MMAS_PHEROMONE_LEAN needs cand_len >= 1, integer beta in [0, 8], WRS "
                                 "selection and fallback, one colony (R30)");
    if (c->colonies > 1 && c->world != 1)
        return fail(MMAS_EINVAL, "concurrent colonies (colonies > 1) need world == 1 (shard independent colonies "
                                 "over ranks instead: each rank its own context)");
    double lo_x = INFINITY, hi_x = -INFINITY, lo_y = INFINITY, hi_y = -INFINITY;
    for (int i = 0; i < c->n; ++i) {
        const double x = c->coords[2 * i], y = c->coords[2 * i + 1];
        if (!std::isfinite(x) || !std::isfinite(y)) return fail(MMAS_EINVAL, "coords must be finite");
        lo_x = std::min(lo_x, x); hi_x = std::max(hi_x, x);
        lo_y = std::min(lo_y, y); hi_y = std::max(hi_y, y);
    }
    // tour length must fit the 40-bit field of the (len << 24 | ant) key
    const double diag = std::sqrt((hi_x - lo_x) * (hi_x - lo_x) + (hi_y - lo_y) * (hi_y - lo_y)) + 1.0;
    if (diag * c->n >= 1099511627776.0 || diag >= 2147483647.0)
        return fail(MMAS_EINVAL, "coordinate range too large: tour lengths must stay below 2^40");
    return MMAS_OK;
}

int check(const mmas_ctx* h) {
    if (!h) return fail(MMAS_EINVAL, "context is NULL");
    return MMAS_OK;
}

}  // namespace

extern "C" {

const char* mmas_last_error(void) { return g_last_error.c_str(); }

void mmas_config_init(mmas_config* cfg) {
    if (!cfg) return;
    std::memset(cfg, 0, sizeof(*cfg));
    cfg->alpha = 1.0;
    cfg->beta = 2.0;
    cfg->rho = 0.5;
    cfg->p_best = 0.01;
    cfg->deposit = MMAS_DEPOSIT_ITERATION_BEST;
    cfg->fallback = MMAS_FALLBACK_WRS;
    cfg->device = -1;
    cfg->rank = 0;
    cfg->world = 1;
}

int mmas_create_ex(const mmas_config* cfg, mmas_ctx** out) {
    g_last_error.clear();
    if (!out) return fail(MMAS_EINVAL, "out is NULL");
    *out = nullptr;
    int st = validate(cfg);
    if (st) return st;
    mmas_ctx* h = new mmas_ctx();
    h->cfg = *cfg;
    h->device = -1;
    st = setup(h);
    if (st) {
        std::string msg = g_last_error;
        free_ctx(h);
        g_last_error = msg;
        return st;
    }
    h->cfg.coords = nullptr;  // not retained
    *out = h;
    return MMAS_OK;
}

mmas_ctx* mmas_create(const double* coords, int32_t n, double alpha, double beta, double rho, int32_t n_ants,
                      int32_t cand_len, uint64_t seed) {
    mmas_config c;
    mmas_config_init(&c);
    c.coords = coords;
    c.n = n;
    c.alpha = alpha;
    c.beta = beta;
    c.rho = rho;
    c.n_ants = n_ants;
    c.cand_len = cand_len;
    c.seed = seed;
    mmas_ctx* h = nullptr;
    return mmas_create_ex(&c, &h) == MMAS_OK ? h : nullptr;
}

int64_t mmas_record_bytes(const mmas_ctx* h) { return h ? h->rec_bytes : fail(MMAS_EINVAL, "context is NULL"); }

static int single_colony(mmas_ctx* h) {
    return h->colonies == 1 ? MMAS_OK
                            : fail(MMAS_ESTATE, "the split / exchange calls serve sharded single colonies (colonies == 1)");
}

int mmas_construct(mmas_ctx* h, void* record_dev) {
    int st = check(h);
    if (st) return st;
    if ((st = single_colony(h))) return st;
    if (!record_dev) return fail(MMAS_EINVAL, "record_dev is NULL");
    CU(cudaSetDevice(h->device));
    if ((st = launch_construct(h, false))) return st;
    if (h->m_local > 0) {
        publish_kernel<<<1, 256, 0, h->stream>>>(h->best_key, h->routes, h->ldr, h->ant_lo, h->n,
                                                 (unsigned char*)record_dev);
        h->launches++;
    } else {
        // empty shard: a record that never wins
        CU(cudaMemsetAsync(record_dev, 0xFF, 8, h->stream));
    }
    CU(cudaGetLastError());
    return MMAS_OK;
}

// ---- peer-memory exchange ----------------------------------------------------------
int64_t mmas_exchange_bytes(const mmas_ctx* h) {
    if (!h) return MMAS_EINVAL;
    return (int64_t)2 * h->cfg.world * h->rec_bytes + (int64_t)2 * h->cfg.world * 4;
}

static int ensure_xbuf(mmas_ctx* h) {
    if (h->xbuf) return MMAS_OK;
    if (h->cfg.world < 2) return fail(MMAS_ESTATE, "the peer exchange needs world > 1");
    CU(cudaSetDevice(h->device));
    const size_t bytes = (size_t)mmas_exchange_bytes(h);
    CU(cudaMalloc(reinterpret_cast<void**>(&h->xbuf), bytes));   // cudaMalloc: IPC-exportable
    CU(cudaMemset(h->xbuf, 0, bytes));
    CU(cudaMalloc(reinterpret_cast<void**>(&h->xpeers_dev), sizeof(unsigned char*) * h->cfg.world));
    return MMAS_OK;
}

int mmas_exchange_buffer(mmas_ctx* h, void** buffer_dev) {
    int st = check(h);
    if (st) return st;
    if (!buffer_dev) return fail(MMAS_EINVAL, "buffer_dev is NULL");
    if ((st = ensure_xbuf(h))) return st;
    *buffer_dev = h->xbuf;
    return MMAS_OK;
}

int mmas_exchange_ipc_handle(mmas_ctx* h, void* handle_out) {
    int st = check(h);
    if (st) return st;
    if (!handle_out) return fail(MMAS_EINVAL, "handle_out is NULL");
    if ((st = ensure_xbuf(h))) return st;
    cudaIpcMemHandle_t hd;
    CU(cudaIpcGetMemHandle(&hd, h->xbuf));
    std::memcpy(handle_out, &hd, sizeof(hd));
    return MMAS_OK;
}

int mmas_exchange_attach(mmas_ctx* h, void* const* peer_buffers) {
    int st = check(h);
    if (st) return st;
    if (!peer_buffers) return fail(MMAS_EINVAL, "peer_buffers is NULL");
    if ((st = ensure_xbuf(h))) return st;
    std::vector<unsigned char*> v((size_t)h->cfg.world);
    for (int p = 0; p < h->cfg.world; ++p) {
        v[p] = p == h->cfg.rank ? h->xbuf : static_cast<unsigned char*>(peer_buffers[p]);
        if (!v[p]) return fail(MMAS_EINVAL, "peer buffer is NULL");
        // a buffer on another device: the exchange kernels store into it and poll its flags
        // over NVLink, which needs peer access from this context's device
        cudaPointerAttributes pa{};
        CU(cudaPointerGetAttributes(&pa, v[p]));
        if (pa.type == cudaMemoryTypeDevice && pa.device != h->device) {
            int can = 0;
            CU(cudaDeviceCanAccessPeer(&can, h->device, pa.device));
            if (!can)
                return fail(MMAS_ECUDA, "device " + std::to_string(h->device) + " cannot access the exchange buffer "
                                        "on device " + std::to_string(pa.device) + " (no peer access)");
            const cudaError_t e = cudaDeviceEnablePeerAccess(pa.device, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
            else if (e != cudaSuccess) return fail(MMAS_ECUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
        }
    }
    CU(cudaMemcpy(h->xpeers_dev, v.data(), sizeof(unsigned char*) * v.size(), cudaMemcpyHostToDevice));
    h->xattached = true;
    return MMAS_OK;
}

int mmas_exchange_open_ipc(mmas_ctx* h, const void* handles) {
    int st = check(h);
    if (st) return st;
    if (!handles) return fail(MMAS_EINVAL, "handles is NULL");
    if ((st = ensure_xbuf(h))) return st;
    std::vector<void*> bufs((size_t)h->cfg.world, nullptr);
    for (int p = 0; p < h->cfg.world; ++p) {
        if (p == h->cfg.rank) continue;
        cudaIpcMemHandle_t hd;
        std::memcpy(&hd, static_cast<const unsigned char*>(handles) + (size_t)p * sizeof(hd), sizeof(hd));
        CU(cudaIpcOpenMemHandle(&bufs[p], hd, cudaIpcMemLazyEnablePeerAccess));
        h->xopened.push_back(bufs[p]);
    }
    return mmas_exchange_attach(h, bufs.data());
}

static ExchangeArgs exchange_args(mmas_ctx* h) {
    ExchangeArgs X{};
    X.peers = h->xpeers_dev;
    X.world = h->cfg.world;
    X.rank = h->cfg.rank;
    X.rec_bytes = h->rec_bytes;
    X.parity = (uint32_t)h->iteration & 1u;
    X.seq = (uint32_t)h->iteration + 1u;
    X.spin_bound = h->spin_bound;
    return X;
}

int mmas_construct_publish(mmas_ctx* h) {
    int st = check(h);
    if (st) return st;
    if (!h->xattached) return fail(MMAS_ESTATE, "attach the peer exchange buffers first");
    CU(cudaSetDevice(h->device));
    if ((st = launch_construct(h, false))) return st;
    launch_pdl(publish_peers_kernel, dim3(1), dim3(256), 0, h->stream, h->best_key,
               static_cast<const uint16_t*>(h->routes), h->ldr, h->ant_lo, h->n, h->m_local, exchange_args(h));
    h->launches++;
    CU(cudaGetLastError());
    return MMAS_OK;
}

int mmas_update_exchange(mmas_ctx* h) {
    int st = check(h);
    if (st) return st;
    if (!h->xattached) return fail(MMAS_ESTATE, "attach the peer exchange buffers first");
    CU(cudaSetDevice(h->device));
    const ExchangeArgs X = exchange_args(h);
    {
        PhaseScope ps(h, 1);
        wait_peers_kernel<<<1, 32, 0, h->stream>>>(h->xbuf, X, h->xerr);
        h->launches++;
        CU(cudaGetLastError());
    }
    if ((st = launch_select(h, h->xbuf + (size_t)X.parity * X.world * X.rec_bytes, X.world))) return st;
    if ((st = launch_update(h))) return st;
    h->iteration++;
    if (h->profiling) h->acc_iters++;
    return MMAS_OK;
}

int mmas_iterate_exchange(mmas_ctx* h, int32_t iters) {
    int st = check(h);
    if (st) return st;
    if (iters < 1) return fail(MMAS_EINVAL, "iters must be >= 1");
    if (!h->xattached) return fail(MMAS_ESTATE, "attach the peer exchange buffers first");
    CU(cudaSetDevice(h->device));
    for (int32_t i = 0; i < iters; ++i) {
        if (h->fuse_peers) {
            // ONE launch: construction, the last block's publish + wait + select, grid
            // barrier, update (construct.cuh exchange_select_block / fused_update)
            const ExchangeArgs X = exchange_args(h);
            if ((st = launch_construct(h, false, &X))) return st;
            h->iteration++;
            if (h->profiling) h->acc_iters++;
        } else if ((st = mmas_construct_publish(h)) || (st = mmas_update_exchange(h))) {
            return st;
        }
    }
    return MMAS_OK;
}

int mmas_device_status(mmas_ctx* h) {
    int st = check(h);
    if (st) return st;
    CU(cudaSetDevice(h->device));
    uint32_t e = 0;
    CU(cudaMemcpyAsync(&e, h->xerr, sizeof(e), cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    if (e & kErrPeerTimeout)
        return fail(MMAS_ETIMEDOUT, "peer exchange timed out waiting for a rank's record; the selection and "
                                    "update have been skipped since (the trails are those of the last complete iteration)");
    if (e & kErrGridBarrier)
        return fail(MMAS_ETIMEDOUT, "the fused launch's grid barrier timed out (a block was not resident); the "
                                    "update has been skipped since");
    return MMAS_OK;
}

int mmas_exchange_status(mmas_ctx* h) { return mmas_device_status(h); }

int mmas_update(mmas_ctx* h, const void* records_dev, int32_t count) {
    int st = check(h);
    if (st) return st;
    if ((st = single_colony(h))) return st;
    if (!records_dev || count < 1) return fail(MMAS_EINVAL, "need records_dev != NULL and count >= 1");
    CU(cudaSetDevice(h->device));
    if ((st = launch_select(h, (const unsigned char*)records_dev, count))) return st;
    if ((st = launch_update(h))) return st;
    h->iteration++;
    if (h->profiling) h->acc_iters++;
    return MMAS_OK;
}

int mmas_iterate(mmas_ctx* h, int32_t iters) {
    int st = check(h);
    if (st) return st;
    if (iters < 1) return fail(MMAS_EINVAL, "iters must be >= 1");
    if (h->cfg.world != 1) return fail(MMAS_ESTATE, "mmas_iterate needs world == 1; use mmas_construct/mmas_update");
    CU(cudaSetDevice(h->device));
    for (int k = 0; k < iters; ++k) {
        // + fused iteration-best selection (and, where eligible, the fused update)
        if ((st = launch_construct(h, true))) return st;
        if (!h->fuse_update && (st = launch_update(h))) return st;
        h->iteration++;
        if (h->profiling) h->acc_iters++;
    }
    return MMAS_OK;
}

int64_t mmas_best_tour(mmas_ctx* h, int32_t* tour_out) {
    int st = check(h);
    if (st) return st;
    if (!tour_out) return fail(MMAS_EINVAL, "tour_out is NULL");
    CU(cudaSetDevice(h->device));
    long long len = -1;
    std::vector<uint16_t> r((size_t)h->n);
    CU(cudaMemcpyAsync(&len, h->gb_len + h->view, sizeof(len), cudaMemcpyDeviceToHost, h->stream));
    CU(cudaMemcpyAsync(r.data(), h->gb_route + (size_t)h->view * h->cs.vec, sizeof(uint16_t) * h->n,
                       cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    if (len < 0) return fail(MMAS_ESTATE, "no global best yet (run at least one iteration)");
    for (int i = 0; i < h->n; ++i) tour_out[i] = r[i];
    return len;
}

int64_t mmas_best_length(mmas_ctx* h) {
    int st = check(h);
    if (st) return st;
    CU(cudaSetDevice(h->device));
    long long len = -1;
    CU(cudaMemcpyAsync(&len, h->gb_len + h->view, sizeof(len), cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    if (len < 0) return fail(MMAS_ESTATE, "no global best yet (run at least one iteration)");
    return len;
}

int mmas_best_length_async(mmas_ctx* h, int64_t* host_dst) {
    int st = check(h);
    if (st) return st;
    if (!host_dst) return fail(MMAS_EINVAL, "host_dst is NULL");
    CU(cudaSetDevice(h->device));
    CU(cudaMemcpyAsync(host_dst, h->gb_len + h->view, sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
    return MMAS_OK;
}

void mmas_destroy(mmas_ctx* h) { free_ctx(h); }

int32_t mmas_n(const mmas_ctx* h) { return h ? h->n : 0; }

int mmas_select_colony(mmas_ctx* h, int32_t colony) {
    int st = check(h);
    if (st) return st;
    if (colony < 0 || colony >= h->colonies) return fail(MMAS_EINVAL, "colony out of range");
    h->view = colony;
    return MMAS_OK;
}

int32_t mmas_colonies(const mmas_ctx* h) { return h ? h->colonies : 0; }
int32_t mmas_iteration(const mmas_ctx* h) { return h ? h->iteration : 0; }

int mmas_get_tours(mmas_ctx* h, int32_t* out, int32_t* first_ant, int32_t* count) {
    int st = check(h);
    if (st) return st;
    if (first_ant) *first_ant = h->ant_lo;
    if (count) *count = h->m_local;
    if (!out) return MMAS_OK;
    CU(cudaSetDevice(h->device));
    std::vector<uint16_t> r((size_t)std::max(h->m_local, 1) * h->ldr);
    CU(cudaMemcpyAsync(r.data(), h->routes + (size_t)h->view * h->cs.routes, sizeof(uint16_t) * r.size(),
                       cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    for (int a = 0; a < h->m_local; ++a)
        for (int k = 0; k < h->n; ++k) out[(size_t)a * h->n + k] = r[(size_t)a * h->ldr + k];
    return MMAS_OK;
}

int mmas_get_lengths(mmas_ctx* h, int64_t* out) {
    int st = check(h);
    if (st) return st;
    if (!out) return fail(MMAS_EINVAL, "out is NULL");
    CU(cudaSetDevice(h->device));
    CU(cudaMemcpyAsync(out, h->lengths + (size_t)h->view * h->cs.ants, sizeof(int64_t) * h->m_local,
                       cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    return MMAS_OK;
}

static int get_matrix(mmas_ctx* h, const float* src, float* out) {
    int st = check(h);
    if (st) return st;
    if (!out) return fail(MMAS_EINVAL, "out is NULL");
    CU(cudaSetDevice(h->device));
    CU(cudaMemcpy2DAsync(out, sizeof(float) * h->n, src, sizeof(float) * h->ld, sizeof(float) * h->n, h->n,
                         cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    return MMAS_OK;
}

// Lean mode (R30): the dense n x n view of tau (which = 0), inv_w (1) or eta^beta (2), expanded
// on the host from the background trail, the candidate trails and the sparse rows; eta^beta
// and the background's 1 / choice_info with the device's arithmetic (R12, R18, R19)
static int lean_expand(mmas_ctx* h, int which, float* out) {
    int st = check(h);
    if (st) return st;
    if (!out) return fail(MMAS_EINVAL, "out is NULL");
    CU(cudaSetDevice(h->device));
    const int n = h->n, cl = h->cl_ld, cap = h->lean_cap;
    std::vector<double> xy(2 * (size_t)n);
    std::vector<uint16_t> cid((size_t)n * cl), sid((size_t)n * cap);
    std::vector<float> cv((size_t)n * cl), sv((size_t)n * cap);
    float bg = 0.f;
    const float* cand_src = which == 0 ? h->cand_tau : which == 1 ? h->cand_inv : h->cand_heur;
    const float* sp_src = which == 0 ? h->sp_tau : h->sp_inv;
    CU(cudaMemcpyAsync(xy.data(), h->xy, sizeof(double) * xy.size(), cudaMemcpyDeviceToHost, h->stream));
    CU(cudaMemcpyAsync(cid.data(), h->cand_id, sizeof(uint16_t) * cid.size(), cudaMemcpyDeviceToHost, h->stream));
    CU(cudaMemcpyAsync(cv.data(), cand_src, sizeof(float) * cv.size(), cudaMemcpyDeviceToHost, h->stream));
    CU(cudaMemcpyAsync(sid.data(), h->sp_id, sizeof(uint16_t) * sid.size(), cudaMemcpyDeviceToHost, h->stream));
    CU(cudaMemcpyAsync(sv.data(), sp_src, sizeof(float) * sv.size(), cudaMemcpyDeviceToHost, h->stream));
    CU(cudaMemcpyAsync(&bg, h->bg + (h->iteration & 1), sizeof(float), cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    const int beta = (int)h->cfg.beta;
    float ba = 1.0f;   // pow_alpha(bg): repeated fp32 multiplication (R17)
    if (h->alpha >= 1) {
        ba = bg;
        for (int k = 1; k < h->alpha; ++k) ba = ba * bg;
    }
    for (int i = 0; i < n; ++i) {
        float* row = out + (size_t)i * n;
        for (int j = 0; j < n; ++j) {
            if (which == 0) {
                row[j] = bg;
                continue;
            }
            const int32_t d = host_dist(xy.data(), i, j);
            double Db = 1.0;
            for (int k = 0; k < beta; ++k) Db = Db * (double)(d > 1 ? d : 1);
            const float heur = (float)(1.0 / Db);
            row[j] = which == 2 ? heur : 1.0f / (ba * heur);
        }
        for (int k = 0; k < cl; ++k) row[cid[(size_t)i * cl + k]] = cv[(size_t)i * cl + k];
        if (which != 2)
            for (int k = 0; k < cap; ++k)
                if (sid[(size_t)i * cap + k] != kLeanEmpty) row[sid[(size_t)i * cap + k]] = sv[(size_t)i * cap + k];
    }
    return MMAS_OK;
}

int mmas_get_pheromone(mmas_ctx* h, float* out) {
    if (h && h->lean) return lean_expand(h, 0, out);
    return get_matrix(h, h ? h->tau + (size_t)h->view * h->cs.nn : nullptr, out);
}
int mmas_get_inv_w(mmas_ctx* h, float* out) {
    if (h && h->lean) return lean_expand(h, 1, out);
    return get_matrix(h, h ? h->inv_w + (size_t)h->view * h->cs.nn : nullptr, out);
}
int mmas_get_heuristic(mmas_ctx* h, float* out) {
    if (h && h->lean) return lean_expand(h, 2, out);
    return get_matrix(h, h ? h->heur : nullptr, out);
}

int64_t mmas_pheromone_bytes(const mmas_ctx* h) {
    if (!h) return MMAS_EINVAL;
    const int64_t ncl = (int64_t)h->n * h->cl_ld;
    if (h->lean)   // candidate trails + eta^beta + 1/w, sparse id + trail + 1/w, tables by distance
        return ncl * 12 + (int64_t)h->n * h->lean_cap * 10 + (int64_t)h->dtab * 8;
    return (int64_t)3 * h->n * h->ld * 4 * h->colonies + ncl * 4 * h->colonies;   // tau, inv_w, heur + cand_inv
}

int mmas_get_candidates(mmas_ctx* h, int32_t* out) {
    int st = check(h);
    if (st) return st;
    if (!out) return fail(MMAS_EINVAL, "out is NULL");
    if (h->cl == 0) return MMAS_OK;
    CU(cudaSetDevice(h->device));
    std::vector<uint16_t> r((size_t)h->n * h->cl_ld);
    CU(cudaMemcpyAsync(r.data(), h->cand_id, sizeof(uint16_t) * r.size(), cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    for (int i = 0; i < h->n; ++i)
        for (int k = 0; k < h->cl; ++k) out[(size_t)i * h->cl + k] = r[(size_t)i * h->cl_ld + k];
    return MMAS_OK;
}

int mmas_get_limits(mmas_ctx* h, float* tau_min, float* tau_max) {
    int st = check(h);
    if (st) return st;
    CU(cudaSetDevice(h->device));
    float s[4];
    CU(cudaMemcpyAsync(s, h->scal + 4 * h->view, sizeof(s), cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    if (tau_min) *tau_min = s[0];
    if (tau_max) *tau_max = s[1];
    return MMAS_OK;
}

int mmas_get_stats(mmas_ctx* h, mmas_stats* out) {
    int st = check(h);
    if (st) return st;
    if (!out) return fail(MMAS_EINVAL, "out is NULL");
    CU(cudaSetDevice(h->device));
    unsigned long long fb = 0;
    CU(cudaMemcpyAsync(&fb, h->fallback_count, sizeof(fb), cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    out->iterations = h->iteration;
    out->fallback_steps = (int64_t)fb;
    out->ant_steps = (int64_t)h->iteration * h->m_local * (h->n - 1) * h->colonies;
    out->ants_local = h->m_local;
    out->first_ant = h->ant_lo;
    out->local_search_moves = 0;
    out->update_fused = (h->fuse_update || h->fuse_peers) ? 1 : 0;
    out->fallback_lane_cap = h->fb_lane_cap;
    if (h->ls_moves) {
        unsigned long long mv = 0;
        CU(cudaMemcpy(&mv, h->ls_moves, sizeof(mv), cudaMemcpyDeviceToHost));
        out->local_search_moves = (int64_t)mv;
    }
    return MMAS_OK;
}

int mmas_profile(mmas_ctx* h, int32_t enable) {
    int st = check(h);
    if (st) return st;
    drain_spans(h);
    h->profiling = enable != 0;
    h->acc_ms[0] = h->acc_ms[1] = h->acc_ms[2] = h->acc_ms[3] = 0.0;
    h->acc_iters = 0;
    return MMAS_OK;
}

int mmas_get_phase_times(mmas_ctx* h, mmas_phase_times* out) {
    int st = check(h);
    if (st) return st;
    if (!out) return fail(MMAS_EINVAL, "out is NULL");
    CU(cudaSetDevice(h->device));
    drain_spans(h);
    out->construct_ms = h->acc_ms[0];
    out->select_ms = h->acc_ms[1];
    out->update_ms = h->acc_ms[2];
    out->local_search_ms = h->acc_ms[3];
    out->iterations = h->acc_iters;
    return MMAS_OK;
}

int mmas_debug_philox(const uint32_t* ctr_key, int64_t count, uint32_t* out_words, float* out_log2) {
    if (count < 0 || (count > 0 && (!ctr_key || !out_words || !out_log2))) return fail(MMAS_EINVAL, "bad arguments");
    if (count == 0) return MMAS_OK;
    uint32_t* d_ck = nullptr;
    uint32_t* d_w = nullptr;
    float* d_l = nullptr;
    int st;
    if ((st = dalloc(&d_ck, 6 * (size_t)count)) || (st = dalloc(&d_w, 4 * (size_t)count)) ||
        (st = dalloc(&d_l, 4 * (size_t)count))) {
        cudaFree(d_ck); cudaFree(d_w); cudaFree(d_l);
        return st;
    }
    cudaMemcpy(d_ck, ctr_key, sizeof(uint32_t) * 6 * count, cudaMemcpyHostToDevice);
    debug_philox_kernel<<<(unsigned)std::min<int64_t>(4096, (count + 255) / 256), 256>>>(d_ck, count, d_w, d_l);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpy(out_words, d_w, sizeof(uint32_t) * 4 * count, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(out_log2, d_l, sizeof(float) * 4 * count, cudaMemcpyDeviceToHost);
    cudaFree(d_ck); cudaFree(d_w); cudaFree(d_l);
    if (e != cudaSuccess) return fail(MMAS_ECUDA, cudaGetErrorString(e));
    return MMAS_OK;
}

int mmas_debug_log2(const float* u, int64_t count, float* out) {
    if (count < 0 || (count > 0 && (!u || !out))) return fail(MMAS_EINVAL, "bad arguments");
    if (count == 0) return MMAS_OK;
    float *d_u = nullptr, *d_o = nullptr;
    int st;
    if ((st = dalloc(&d_u, (size_t)count)) || (st = dalloc(&d_o, (size_t)count))) {
        cudaFree(d_u); cudaFree(d_o);
        return st;
    }
    cudaMemcpy(d_u, u, sizeof(float) * count, cudaMemcpyHostToDevice);
    debug_log2_kernel<<<(unsigned)std::min<int64_t>(8192, (count + 255) / 256), 256>>>(d_u, count, d_o);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpy(out, d_o, sizeof(float) * count, cudaMemcpyDeviceToHost);
    cudaFree(d_u); cudaFree(d_o);
    if (e != cudaSuccess) return fail(MMAS_ECUDA, cudaGetErrorString(e));
    return MMAS_OK;
}

int64_t mmas_kernel_launches(const mmas_ctx* h) { return h ? h->launches : 0; }

void* mmas_stream(const mmas_ctx* h) { return h ? (void*)h->stream : nullptr; }

int mmas_sync(mmas_ctx* h) {
    int st = check(h);
    if (st) return st;
    CU(cudaSetDevice(h->device));
    CU(cudaStreamSynchronize(h->stream));
    return MMAS_OK;
}

// ---- checkpoint / resume ---------------------------------------------------------------
// The colony's whole mutable state is device memory plus the host iteration counter (the
// random numbers are counter-based, R13, so they carry no state): trails and 1/choice_info
// (dense or lean), the candidate 1/w table, limits, global / iteration best, the device
// iteration counters, the last iteration's routes and lengths, the fallback counter.
namespace {
struct StateHeader {
    uint32_t magic, version;
    int32_t n, cl_ld, m, m_local, ant_lo, colonies, lean, lean_cap, dtab, iteration;
    uint64_t seed;
    double alpha, beta, rho, p_best;
    int32_t deposit, fallback, local_search, tabu, selection, world, rank, pad_;
    int64_t payload;
};
constexpr uint32_t kStateMagic = 0x53414D4Du;   // "MMAS"

std::vector<std::pair<void*, size_t>> state_segments(mmas_ctx* h) {
    const size_t K = (size_t)h->colonies, ma = (size_t)std::max(h->m_local, 1);
    const size_t nn = (size_t)h->n * h->ld;
    std::vector<std::pair<void*, size_t>> v;
    auto add = [&](void* p, size_t bytes) {
        if (p && bytes) v.emplace_back(p, bytes);
    };
    if (!h->lean) {
        add(h->tau, nn * K * 4);
        add(h->inv_w, nn * K * 4);
    } else {
        const size_t ncl = (size_t)h->n * h->cl_ld + 64, nsp = (size_t)h->n * h->lean_cap;
        add(h->cand_tau, ncl * 4);
        add(h->sp_id, nsp * 2);
        add(h->sp_tau, nsp * 4);
        add(h->sp_inv, nsp * 4);
        add(h->bg, 2 * 4);
        add(h->inv_tab, (size_t)h->dtab * 4);
    }
    if (h->cl > 0) add(h->cand_inv, (size_t)h->cs.cand * K * 4);
    add(h->scal, 4 * K * 4);
    add(h->gb_route, (size_t)h->ldr * K * 2);
    add(h->ib_route, (size_t)h->ldr * K * 2);
    add(h->gb_len, K * 8);
    add(h->ib_len, K * 8);
    add(h->ib_ant, K * 4);
    add(h->iter_dev, K * 4);
    add(h->routes, ma * h->ldr * K * 2);
    add(h->lengths, ma * K * 8);
    add(h->fallback_count, 8);
    if (h->ls_moves) add(h->ls_moves, 8);
    return v;
}

StateHeader state_header(const mmas_ctx* h, int64_t payload) {
    StateHeader H{};
    H.magic = kStateMagic;
    H.version = 1;
    H.n = h->n;
    H.cl_ld = h->cl_ld;
    H.m = h->m;
    H.m_local = h->m_local;
    H.ant_lo = h->ant_lo;
    H.colonies = h->colonies;
    H.lean = h->lean ? 1 : 0;
    H.lean_cap = h->lean_cap;
    H.dtab = h->dtab;
    H.iteration = h->iteration;
    H.seed = h->cfg.seed;
    H.alpha = h->cfg.alpha;
    H.beta = h->cfg.beta;
    H.rho = h->cfg.rho;
    H.p_best = h->cfg.p_best;
    H.deposit = h->cfg.deposit;
    H.fallback = h->cfg.fallback;
    H.local_search = h->cfg.local_search;
    H.tabu = h->cfg.tabu;
    H.selection = h->cfg.selection;
    H.world = h->cfg.world;
    H.rank = h->cfg.rank;
    H.payload = payload;
    return H;
}
}  // namespace

int64_t mmas_state_bytes(mmas_ctx* h) {
    int st = check(h);
    if (st) return st;
    int64_t total = sizeof(StateHeader);
    for (auto& sgm : state_segments(h)) total += (int64_t)sgm.second;
    return total;
}

int mmas_save_state(mmas_ctx* h, void* host_buf, int64_t bytes) {
    int st = check(h);
    if (st) return st;
    const int64_t need = mmas_state_bytes(h);
    if (!host_buf || bytes < need) return fail(MMAS_EINVAL, "host_buf is NULL or smaller than mmas_state_bytes");
    CU(cudaSetDevice(h->device));
    unsigned char* out = static_cast<unsigned char*>(host_buf);
    const StateHeader H = state_header(h, need - (int64_t)sizeof(StateHeader));
    std::memcpy(out, &H, sizeof(H));
    size_t off = sizeof(H);
    for (auto& sgm : state_segments(h)) {
        CU(cudaMemcpyAsync(out + off, sgm.first, sgm.second, cudaMemcpyDeviceToHost, h->stream));
        off += sgm.second;
    }
    CU(cudaStreamSynchronize(h->stream));
    return MMAS_OK;
}

int mmas_load_state(mmas_ctx* h, const void* host_buf, int64_t bytes) {
    int st = check(h);
    if (st) return st;
    const int64_t need = mmas_state_bytes(h);
    if (!host_buf || bytes < need) return fail(MMAS_EINVAL, "host_buf is NULL or smaller than mmas_state_bytes");
    const unsigned char* in = static_cast<const unsigned char*>(host_buf);
    StateHeader H;
    std::memcpy(&H, in, sizeof(H));
    StateHeader mine = state_header(h, need - (int64_t)sizeof(StateHeader));
    mine.iteration = H.iteration;   // the one field the checkpoint sets
    if (H.magic != kStateMagic || H.version != 1 || std::memcmp(&H, &mine, sizeof(H)) != 0)
        return fail(MMAS_EINVAL, "checkpoint does not match this context (instance size, colony, parameters or rank)");
    CU(cudaSetDevice(h->device));
    CU(cudaStreamSynchronize(h->stream));
    size_t off = sizeof(H);
    for (auto& sgm : state_segments(h)) {
        CU(cudaMemcpyAsync(sgm.first, in + off, sgm.second, cudaMemcpyHostToDevice, h->stream));
        off += sgm.second;
    }
    CU(cudaStreamSynchronize(h->stream));
    h->iteration = H.iteration;
    return MMAS_OK;
}

}  // extern "C"

// Debug: copy the construct_cl_kernel phase timestamps (a -DMMAS_TRACE build; see
// tools/trace_phases.py).  Not part of the documented ABI; MMAS_ESTATE otherwise.
// Debug: fallback-scan cycles (sum, count) since load (a -DMMAS_TRACE build), and reset.
extern "C" int mmas_debug_fb_cycles(unsigned long long* out) {
#ifdef MMAS_TRACE
    if (cudaMemcpyFromSymbol(out, mmas::g_fbcyc, 64 * sizeof(unsigned long long)) != cudaSuccess) return MMAS_ECUDA;
    const unsigned long long z[64] = {};
    if (cudaMemcpyToSymbol(mmas::g_fbcyc, z, sizeof(z)) != cudaSuccess) return MMAS_ECUDA;
    return MMAS_OK;
#else
    (void)out;
    return MMAS_ESTATE;
#endif
}

extern "C" int mmas_debug_trace_warps(unsigned long long* out, int count) {
#ifdef MMAS_TRACE
    if (!out || count < 0 || count > 1024 * 16) return MMAS_EINVAL;
    if (cudaMemcpyFromSymbol(out, mmas::g_trace_w, sizeof(unsigned long long) * count) != cudaSuccess) return MMAS_ECUDA;
    return MMAS_OK;
#else
    (void)out;
    (void)count;
    return MMAS_ESTATE;
#endif
}

extern "C" int mmas_debug_trace(unsigned long long* out, int count) {
#ifdef MMAS_TRACE
    if (!out || count < 0 || count > 1024 * 8) return MMAS_EINVAL;
    if (cudaMemcpyFromSymbol(out, mmas::g_trace, sizeof(unsigned long long) * count) != cudaSuccess) return MMAS_ECUDA;
    return MMAS_OK;
#else
    (void)out;
    (void)count;
    return MMAS_ESTATE;
#endif
}
