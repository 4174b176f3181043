/*
 * mmas.h -- C ABI of the B200-native MAX-MIN Ant System hot path.
 *
 * Implements the per-iteration colony step of Skinderowicz, "Implementing a
 * GPU-based parallel MAX-MIN Ant System" (arXiv 2003.11902): tour construction
 * by weighted reservoir sampling (Sec. 4.2.2, Alg. 3) over
 * candidate lists (Sec. 4.3) with a bitmask tabu (Sec. 4.1,
 * P:806-815), then the MMAS pheromone update (Sec. 2.1, Alg. 1,
 * P:278-325).  The problem statement is the symmetric TSP on a complete graph
 * with TSPLIB EUC_2D distances.  Every numerical
 * convention the paper leaves open is fixed in DESIGN.md Sec. 3 (readings R1-R22);
 * results are bit-identical to the CPU oracle in oracle/.
 *
 * Conventions for every call:
 *  - Plain C types only.  Host pointers unless a parameter says "device".
 *  - Errors: calls returning int return 0 (MMAS_OK) or a negative mmas_status;
 *    calls returning a pointer return NULL.  mmas_last_error() then gives a
 *    thread-local, human-readable message (valid until the next call on this thread).
 *  - A context is bound to one CUDA device and one stream; it is NOT thread-safe.
 *    Use one context per device per process.
 *  - All work is asynchronous with respect to the host unless stated otherwise.
 */
#ifndef MMAS_H
#define MMAS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mmas_ctx mmas_ctx;

typedef enum mmas_status {
    MMAS_OK = 0,
    MMAS_EINVAL = -1, /* invalid argument */
    MMAS_ENOMEM = -2, /* device or host allocation failed */
    MMAS_ECUDA = -3,  /* a CUDA runtime call or kernel failed */
    MMAS_ENCCL = -4,  /* reserved (no collective runs inside the library; the caller's all-gather
                         or the peer-memory exchange below carries row a7) */
    MMAS_ESTATE = -5, /* call not valid in the current state (e.g. no global best yet) */
    MMAS_ETIMEDOUT = -6 /* a bounded device-side wait gave up (a peer's exchange flag, or the fused
                         launch's grid barrier); see mmas_device_status */
} mmas_status;

enum { MMAS_DEPOSIT_ITERATION_BEST = 0, MMAS_DEPOSIT_GLOBAL_BEST = 1 }; /* Alg.1 l.288 / P:332-333 (R7) */
enum { MMAS_FALLBACK_WRS = 0, MMAS_FALLBACK_ARGMAX = 1 };               /* R9 */
/* Tabu of the full-row path (Sec. 4.1, Tab. 1; R27): the bitmask tabu (BT,
 * default, every step scans all n nodes) or the compact tabu (CT, the
 * paper's recommendation without candidate lists P:1998-2001: step s enumerates only
 * the n-s unvisited nodes, and the i-th enumerated node draws the uniform the bitmask
 * scan gives city i -- so the two modes sample the same distribution but different
 * tours).  COMPACT requires cand_len == 0. */
enum { MMAS_TABU_BITMASK = 0, MMAS_TABU_COMPACT = 1 };
/* Node selection (Sec. 4.2, R28): weighted reservoir sampling (WRS, Alg. 3, default) or
 * the parallel roulette wheel (PRWM, Sec. 4.2.1) the paper compares it with --
 * a warp-wide chunked prefix-sum wheel over choice_info = tau^alpha * eta^beta, one
 * uniform per step.  Both follow Eq. (1); they draw different random numbers. */
enum { MMAS_SELECT_WRS = 0, MMAS_SELECT_RWM = 1 };
/* Pheromone storage (the paper's O(n^2) pheromone memory limit, P:1945-1947,
 * and its future work "replacement of the pheromone memory with a more space-efficient
 * alternative").  DENSE (default): tau, eta^beta and 1/choice_info as n x n fp32
 * matrices.  LEAN: no n x n matrix -- the candidate trails (n x cl), one background trail that
 * every never-deposited trail equals, and per row at most 2 (L + 1) other trails
 * (L = ceil(ln(tau_min/tau_max) / ln rho)); the fallback scans recompute eta^beta from the
 * coordinates.  Exactly the same results as DENSE (R30).  LEAN needs cand_len >= 1, integer
 * beta, WRS selection and fallback, colonies <= 1. */
enum { MMAS_PHEROMONE_DENSE = 0, MMAS_PHEROMONE_LEAN = 1 };

/* Full configuration (mmas_config_init() fills the defaults). */
typedef struct mmas_config {
    const double *coords;  /* 2n interleaved x,y (host).  Copied; caller may free after create. */
    int32_t n;             /* cities, 3 <= n < 65536 (u16 ids, Tab. 1 caption P:822-824) */
    double alpha;          /* pheromone exponent (Eq. 1); integer in [0,8] (R17) */
    double beta;           /* heuristic exponent; >= 0 (R18) */
    double rho;            /* retention: evaporation tau <- max(rho tau, tau_min) (R1); 0 < rho < 1 */
    int32_t n_ants;        /* colony size m (global, over all ranks); 1 <= m < 2^24 */
    int32_t cand_len;      /* candidate-list length cl, 0 <= cl <= min(n-1, 128); 0 = full-row WRS */
    uint64_t seed;         /* Philox key (R13) */
    double p_best;         /* trail-limit parameter; default 0.01 */
    int32_t deposit;       /* MMAS_DEPOSIT_*; default iteration best */
    int32_t fallback;      /* MMAS_FALLBACK_*; default WRS over all unvisited */
    int32_t local_search;  /* 1: 2-opt on every route (row a8, Sec. 5.7, R25/R26); default 0 */
    int32_t device;        /* CUDA device ordinal; -1 = current device */
    void *stream;          /* cudaStream_t to run on (see use_caller_stream) */
    int32_t rank, world;   /* ant shard: this context builds global ants [floor(rank*m/world),
                              floor((rank+1)*m/world)) (R21); default 0, 1 */
    int32_t use_caller_stream; /* 1: run on `stream` even when it is NULL (the legacy default
                              stream, e.g. torch's default stream); 0 (default): run on `stream`
                              if non-NULL, else on a non-blocking stream owned by the context */
    int32_t tabu;          /* MMAS_TABU_*; default BITMASK.  COMPACT needs cand_len == 0 (R27) */
    int32_t selection;     /* MMAS_SELECT_*; default WRS (R28) */
    int32_t separate_update; /* 1: always run the pheromone update (row a6) as its own kernel.
                              0 (default): with world == 1, no local search, cand_len <= 32 and the
                              candidate table in shared memory, the update runs inside the
                              construction launch after a grid barrier (same results bit for bit) */
    int32_t colonies;      /* k concurrent independent colonies in this context (the
                              paper's repeated runs P:1143-1145 and colony-size study P:1568-1619).
                              Colony c is a complete MMAS run of n_ants ants with Philox key
                              seed + c (R29): its own trails, choice_info, routes, global best and
                              limits; coordinates, eta^beta and candidate lists are shared.  Every
                              launch runs all k (grid.y = colony).  0 or 1 = one colony (default);
                              k > 1 needs world == 1 and mmas_iterate (not the split / exchange
                              calls).  Introspection reports the colony chosen by mmas_select_colony */
    int32_t pheromone;     /* MMAS_PHEROMONE_*; default DENSE */
} mmas_config;

/* Per-context counters (cumulative since create). */
typedef struct mmas_stats {
    int64_t iterations;       /* completed iterations (== the global iteration counter, R20) */
    int64_t fallback_steps;   /* construction steps that fell back to all unvisited cities (R9), this shard */
    int64_t ant_steps;        /* construction steps taken by this shard's ants */
    int32_t ants_local;       /* ants built by this context per iteration */
    int32_t first_ant;        /* global id of the first of them */
    int64_t local_search_moves; /* improving 2-opt moves applied (row a8), this shard */
    int32_t update_fused;     /* 1: mmas_iterate runs construction + selection + update as ONE
                                 launch (see mmas_config.separate_update) */
    int32_t fallback_lane_cap; /* lane-compacted fallback scans (row a3): a fallback with at most
                                  this many unvisited cities draws keys for the unvisited cities
                                  only (0 = off, a3); env MMAS_FB_COMPACT */
} mmas_stats;

/* Last error message of this thread ("" if none). */
const char *mmas_last_error(void);

/* Fills cfg with defaults (p_best 0.01, iteration-best deposit, WRS fallback,
 * no local search, current device, own stream, rank 0 of 1). */
void mmas_config_init(mmas_config *cfg);

/* Creates a colony and runs setup (row a0): eta^beta, candidate lists, the
 * nearest-neighbour tour and initial limits (Alg. 1),
 * tau = tau_max, inv_w = 1/choice_info.  Synchronous.
 * Returns NULL on error (see mmas_last_error). */
mmas_ctx *mmas_create(const double *coords, int32_t n, double alpha, double beta, double rho,
                      int32_t n_ants, int32_t cand_len, uint64_t seed);

/* As mmas_create with every option; *out receives the context.  Returns mmas_status. */
int mmas_create_ex(const mmas_config *cfg, mmas_ctx **out);

/* Runs `iters` complete MMAS iterations (Alg. 1): construction
 * of every ant's route (a1-a4), iteration/global best and limits (a5),
 * evaporation + deposit + clamp and choice_info refresh (a6).  Single-rank
 * contexts only (world == 1; otherwise MMAS_ESTATE -- use the split calls).
 * Asynchronous. iters >= 1. */
int mmas_iterate(mmas_ctx *h, int32_t iters);

/* ---- split iteration for sharded colonies (world > 1; also valid for world == 1) ----
 * Per iteration:  mmas_construct(h)  ->  caller all-gathers the per-rank records
 * (e.g. torch.distributed.all_gather_into_tensor / ncclAllGather on the same
 * stream)  ->  mmas_update(h, gathered, world).  A record is
 * mmas_record_bytes(h) bytes: uint64 key = (tour_length << 24 | global_ant)
 * followed by the route as n uint16 city ids. */
int64_t mmas_record_bytes(const mmas_ctx *h);

/* Builds this shard's routes and writes its best record into `record_dev`
 * (device pointer, mmas_record_bytes(h) bytes, 8-byte aligned).  Asynchronous. */
int mmas_construct(mmas_ctx *h, void *record_dev);

/* Reads `count` contiguous records at `records_dev` (device), selects the
 * iteration best (min key: shortest, ties -> lowest global ant id, R8), updates
 * the global best and limits, and runs the pheromone update.  Asynchronous. */
int mmas_update(mmas_ctx *h, const void *records_dev, int32_t count);

/* ---- Peer-memory exchange (row a7 without a collective library) ----------------------
 * Instead of mmas_construct -> all-gather -> mmas_update, the ranks can exchange their
 * records through each other's device memory (NVLink P2P stores on an NVSwitch node).
 * Every context owns an exchange buffer of mmas_exchange_bytes(h) bytes ([2][world]
 * records, then [2][world] uint32 flags).  Wire them up once, collectively:
 *   - across processes: mmas_exchange_ipc_handle(h, 64-byte cudaIpcMemHandle out), gather
 *     every rank's handle (world x 64 bytes, rank order) and mmas_exchange_open_ipc(h, all);
 *   - within one process: mmas_exchange_buffer(h, &dev_ptr) on every context and
 *     mmas_exchange_attach(h, ptrs) with the world device pointers in rank order.
 * Then each iteration is mmas_construct_publish(h) (construction; the shard's best record
 * is written into slot `rank` of every buffer and a flag raised in each) followed by
 * mmas_update_exchange(h) (waits on the device until every rank's flag of this iteration
 * is up, selects, updates); mmas_iterate_exchange(h, iters) does both -- as ONE launch
 * per iteration where the context is eligible (mmas_stats.update_fused: candidate table in
 * shared memory, cand_len <= 32, no local search, ants on this rank): the grid's last block
 * publishes, waits for the peers' flags and selects, then every block updates.  That
 * launch spins on the device until every peer has published, so the ranks' launches must
 * run concurrently: one process (or context) per GPU.  Ranks that share ONE GPU must use
 * the split calls (mmas_construct_publish / mmas_update_exchange, or mmas_construct ->
 * all-gather -> mmas_update): a fused grid holds its SMs while it waits, and two of them
 * on one device may not both fit.  mmas_exchange_attach enables peer access to every
 * buffer on another device (MMAS_ECUDA if the devices cannot access each other).
 * Every device-side wait is bounded (~2^34 GPU cycles): a lost peer sets the context's
 * error word, the selection and update are skipped from then on (the replica keeps the
 * trails of the last complete iteration instead of diverging), and mmas_device_status(h) reports
 * MMAS_ETIMEDOUT.  Iteration t uses buffer half t & 1, so ranks stay lockstep without
 * further synchronisation.  All calls are asynchronous except the wiring and
 * mmas_device_status / mmas_exchange_status. */
int64_t mmas_exchange_bytes(const mmas_ctx *h);
int mmas_exchange_buffer(mmas_ctx *h, void **buffer_dev);
int mmas_exchange_ipc_handle(mmas_ctx *h, void *handle_out);
int mmas_exchange_open_ipc(mmas_ctx *h, const void *handles);
int mmas_exchange_attach(mmas_ctx *h, void *const *peer_buffers);
int mmas_construct_publish(mmas_ctx *h);
int mmas_update_exchange(mmas_ctx *h);
int mmas_iterate_exchange(mmas_ctx *h, int32_t iters);
int mmas_exchange_status(mmas_ctx *h);   /* = mmas_device_status */

/* Synchronises the context's stream and reports a device-side failure: MMAS_ETIMEDOUT when a
 * bounded device wait gave up (a peer's exchange flag, or the one-launch iteration's grid
 * barrier, whose blocks must all be resident at once -- checked at create, see
 * mmas_stats.update_fused), else MMAS_OK.  The error is sticky. */
int mmas_device_status(mmas_ctx *h);

/* Synchronises the context's stream and copies the global best route (n city
 * ids, starting at its route[0]) into tour_out (host, n int32, caller-owned).
 * Returns its length (>= 0), or MMAS_ESTATE before the first iteration (gb
 * empty, Alg. 1), or another negative mmas_status. */
int64_t mmas_best_tour(mmas_ctx *h, int32_t *tour_out);

/* Synchronises and returns only the global best length (8-byte read-back), or
 * MMAS_ESTATE before the first iteration. */
int64_t mmas_best_length(mmas_ctx *h);

/* Enqueues, on the context's stream and without synchronising, the copy of the current
 * global best length (int64; -1 while there is none) into `host_dst` (host memory,
 * caller-owned; pinned memory keeps the copy asynchronous).  The value is valid once the
 * stream has reached this point (mmas_sync, or any later synchronising call).  Lets a
 * driver read every iteration's result without a per-iteration host round trip. */
int mmas_best_length_async(mmas_ctx *h, int64_t *host_dst);

/* Frees every device and host resource.  NULL is a no-op. */
void mmas_destroy(mmas_ctx *h);

/* ---- introspection (synchronous; caller-allocated host buffers) ----
 * With the LEAN pheromone, get_pheromone / get_inv_w / get_heuristic expand the dense n x n
 * view on the host (small n only).  With colonies > 1 the calls below (and mmas_best_tour / mmas_best_length[_async]) report
 * colony `colony` of mmas_select_colony (default 0; MMAS_EINVAL if out of range). */
int mmas_select_colony(mmas_ctx *h, int32_t colony);
int32_t mmas_colonies(const mmas_ctx *h);
/* Device bytes of the pheromone state (trails, eta^beta, 1/choice_info, candidate and sparse
 * tables) of every colony. */
int64_t mmas_pheromone_bytes(const mmas_ctx *h);
int32_t mmas_n(const mmas_ctx *h);
int32_t mmas_iteration(const mmas_ctx *h);
/* last iteration's routes of this shard: out has ants_local*n int32 */
int mmas_get_tours(mmas_ctx *h, int32_t *out, int32_t *first_ant, int32_t *count);
int mmas_get_lengths(mmas_ctx *h, int64_t *out);             /* ants_local int64 */
int mmas_get_pheromone(mmas_ctx *h, float *out);             /* n*n float, row-major */
int mmas_get_inv_w(mmas_ctx *h, float *out);                 /* n*n float: 1/choice_info */
int mmas_get_heuristic(mmas_ctx *h, float *out);             /* n*n float: eta^beta */
int mmas_get_candidates(mmas_ctx *h, int32_t *out);          /* n*cl int32 */
int mmas_get_limits(mmas_ctx *h, float *tau_min, float *tau_max);
int mmas_get_stats(mmas_ctx *h, mmas_stats *out);
/* ---- measurement (bench.py) ----
 * With profiling on, the context brackets each phase of every iteration with
 * CUDA events on its own stream and accumulates the device time per phase. */
typedef struct mmas_phase_times {
    double construct_ms;   /* construction kernels (a1-a5 local) */
    double select_ms;      /* iteration/global best + limits (a5) */
    double update_ms;      /* pheromone update kernel (a6) */
    double local_search_ms; /* 2-opt kernel incl. lengths + best (a8 + a5), local_search only */
    int64_t iterations;    /* iterations accumulated */
} mmas_phase_times;
int mmas_profile(mmas_ctx *h, int32_t enable);                   /* resets the accumulators */
int mmas_get_phase_times(mmas_ctx *h, mmas_phase_times *out);    /* synchronises */
/* Number of kernels this context has launched since create (cumulative). */
int64_t mmas_kernel_launches(const mmas_ctx *h);

/* ---- test hooks for the random-key primitives (R13, R14); synchronous, current device ----
 * mmas_debug_philox: for i < count, runs the device Philox4x32-10 on counter
 * ctr_key[6i..6i+3] and key ctr_key[6i+4..6i+5]; writes the 4 output words to
 * out_words[4i..4i+3] and det_log2(uniform(word)) to out_log2[4i..4i+3] (host).
 * mmas_debug_log2: out[i] = device det_log2(u[i]) for normal u[i] > 0 (host arrays). */
int mmas_debug_philox(const uint32_t *ctr_key, int64_t count, uint32_t *out_words, float *out_log2);
int mmas_debug_log2(const float *u, int64_t count, float *out);
/* Measurement tooling of -DMMAS_TRACE builds (tools/trace_phases.py, tools/trace_warps.py,
 * tools/fb_cycles.py); every other build returns MMAS_ESTATE and writes nothing.
 * mmas_debug_trace: %globaltimer stamps, 8 per block (u64, count <= 8192);
 * mmas_debug_trace_warps: the time each ant warp finished its last ant, 16 per block (count <= 16384);
 * mmas_debug_fb_cycles: 64 u64 counters of the fallback scans (kernels.cuh g_fbcyc), then zeroed. */
int mmas_debug_trace(unsigned long long *out, int count);
int mmas_debug_trace_warps(unsigned long long *out, int count);
int mmas_debug_fb_cycles(unsigned long long *out);

/* ---- checkpoint / resume (synchronous; caller-owned host buffer) ----
 * The random numbers are counter-based (keyed by seed, iteration, ant, step, city; R13), so a
 * colony's future is a function of its device state and iteration counter alone:
 * mmas_save_state writes them (a header identifying the instance and parameters, then the
 * trails, 1/choice_info, candidate table, limits, best tours, iteration counters, last
 * routes) into host_buf; mmas_load_state restores them into a context created with the same
 * coordinates and configuration (MMAS_EINVAL if the header does not match), after which
 * iterating continues exactly as the saved colony would have (tested in
 * tests/test_checkpoint_gpu.py).  mmas_state_bytes gives the buffer size. */
int64_t mmas_state_bytes(mmas_ctx *h);
int mmas_save_state(mmas_ctx *h, void *host_buf, int64_t bytes);
int mmas_load_state(mmas_ctx *h, const void *host_buf, int64_t bytes);

/* Device pointer of the stream the context runs on (cudaStream_t). */
void *mmas_stream(const mmas_ctx *h);
/* Synchronises the context's stream. */
int mmas_sync(mmas_ctx *h);

#ifdef __cplusplus
}
#endif
#endif /* MMAS_H */
