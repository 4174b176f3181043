/*
 * oracle/mmas_oracle.c -- plain, slow CPU oracle of the MMAS hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load, call or execute anything under
 * oracle/.  The CUDA product path (paper_2003_11902_b200/) never does, and this
 * file shares no code, header, table or constant generator with it: both sides
 * are written independently from the contract in DESIGN.md ("Oracle contract").
 *
 * Paper: Skinderowicz, "Implementing a GPU-based parallel MAX-MIN Ant System",
 * arXiv 2003.11902.  Citations are PAPER.md lines (P:L) with the section /
 * equation / algorithm they fall in; readings are R-numbers.
 *
 * Compiled with  gcc -O2 -ffp-contract=off -fno-fast-math  (no FMA contraction,
 * no FTZ): every float operation below is one IEEE-754 correctly rounded op.
 *
 * Pins (tests/test_oracle_*.py, -m "not gpu"): Philox KAT vectors (Random123),
 * det_log2 exhaustive vs libm log2, WRS chi-square vs w/sum(w) (Eq. 1),
 * tau limits closed forms, evaporation/deposit worked values, SPEC worked
 * examples for distance / NN tour / candidate lists, brute-force optimum on
 * tiny instances, permutation validity.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_EXPORT __attribute__((visibility("default")))

/* ------------------------------------------------------------------------- */
/* R13: Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11), Random123 constants. */
/* The paper only says "a separate pseudo-random number generator's state needs */
/* to be stored for each thread" (Sec. 4.2.2); we replace it by a  */
/* counter-based generator so both sides can draw the same numbers.            */
/* ------------------------------------------------------------------------- */
ORC_EXPORT void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) {              /* key schedule: bump before rounds 2..10 */
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* R13: uniform in the OPEN interval (0,1) required by A-Res ("u_i is a
 * uniformly chosen number from the range (0, 1)") and by the log key:
 * u = (2*(x>>9)+1) * 2^-24, exactly representable, in [2^-24, 1-2^-24]. */
ORC_EXPORT float orc_uniform(uint32_t x)
{
    uint32_t j = x >> 9;                       /* 23 random bits */
    double num = 2.0 * (double)j + 1.0;        /* odd, < 2^24: exact */
    return (float)(num / 16777216.0);          /* exact */
}

/* R14: deterministic base-2 logarithm replacing __log2f.
 * u = 2^e * m with m in [sqrt(1/2), sqrt(2)); f = m - 1 (exact);
 * log2(u) = e + f * P(f), P of degree 8 evaluated by Horner with fmaf.
 * Coefficients frozen in DESIGN.md (derived by tools/derive_det_log2.py). */
static const float DL2_C[9] = {
    1.4426950216293335f,  -0.7213473320007324f, 0.48091062903404236f,
    -0.3607036769390106f, 0.28791624307632446f, -0.23894482851028442f,
    0.21571563184261322f, -0.20726971328258514f, 0.12583690881729126f,
};

ORC_EXPORT float orc_det_log2(float u)
{
    /* valid for finite normal u > 0 (all values orc_uniform can produce) */
    int e;
    double m = frexp((double)u, &e);           /* u = m * 2^e, m in [0.5, 1) */
    m *= 2.0;                                  /* m in [1, 2) */
    e -= 1;
    if (m > 1.4142135381698608) {              /* > (float)sqrt(2): mantissa bits > 0x3504F3 */
        m *= 0.5;
        e += 1;
    }
    float f = (float)m - 1.0f;                 /* exact (Sterbenz) */
    float p = DL2_C[8];
    for (int i = 7; i >= 0; --i)
        p = fmaf(p, f, DL2_C[i]);
    return fmaf(f, p, (float)e);
}

ORC_EXPORT void orc_det_log2_many(const float *u, float *out, int64_t count)
{
    for (int64_t i = 0; i < count; ++i) out[i] = orc_det_log2(u[i]);
}

/* ------------------------------------------------------------------------- */
/* Problem statement (Sec. 2.1): symmetric TSP on a complete graph,  */
/* d_ij from TSPLIB EUC_2D coordinates: nint(sqrt(dx^2+dy^2)).    */
/* ------------------------------------------------------------------------- */
ORC_EXPORT int32_t orc_dist(const double *xy, int32_t i, int32_t j)
{
    double dx = xy[2 * i] - xy[2 * j];
    double dy = xy[2 * i + 1] - xy[2 * j + 1];
    double r = sqrt(dx * dx + dy * dy);
    return (int32_t)(r + 0.5);                 /* TSPLIB nint: round half up */
}

ORC_EXPORT int64_t orc_tour_length(const double *xy, int32_t n, const int32_t *route)
{
    int64_t len = 0;
    for (int32_t k = 0; k < n; ++k)
        len += orc_dist(xy, route[k], route[(k + 1) % n]);
    return len;
}

/* Nearest-neighbour tour used to initialise the trail limits (P:295-298,
 * P:1142-1143).  R3: start at city 0, ties -> lowest id. Returns its length. */
ORC_EXPORT int64_t orc_nn_tour(const double *xy, int32_t n, int32_t *route)
{
    char *vis = calloc((size_t)n, 1);
    int32_t cur = 0;
    route[0] = 0;
    vis[0] = 1;
    for (int32_t s = 1; s < n; ++s) {
        int32_t best = -1, bestd = 0;
        for (int32_t j = 0; j < n; ++j) {
            if (vis[j]) continue;
            int32_t d = orc_dist(xy, cur, j);
            if (best < 0 || d < bestd) { best = j; bestd = d; }
        }
        route[s] = best;
        vis[best] = 1;
        cur = best;
    }
    free(vis);
    return orc_tour_length(xy, n, route);
}

/* Candidate lists (Sec. 4.3): the cl closest nodes of i.
 * R10: order by (d(i,j), j), i excluded.  Insertion into a sorted list. */
ORC_EXPORT void orc_cand_lists(const double *xy, int32_t n, int32_t cl, int32_t *cand)
{
    int32_t *bd = malloc(sizeof(int32_t) * (size_t)(cl > 0 ? cl : 1));
    for (int32_t i = 0; i < n; ++i) {
        int32_t *row = cand + (size_t)i * cl;
        int32_t cnt = 0;
        for (int32_t j = 0; j < n; ++j) {
            if (j == i) continue;
            int32_t d = orc_dist(xy, i, j);
            /* j is larger than every id already present, so on equal d it goes after */
            if (cnt == cl && d >= bd[cl - 1]) continue;
            int32_t pos = cnt < cl ? cnt : cl - 1;
            while (pos > 0 && bd[pos - 1] > d) {
                bd[pos] = bd[pos - 1];
                row[pos] = row[pos - 1];
                --pos;
            }
            bd[pos] = d;
            row[pos] = j;
            if (cnt < cl) ++cnt;
        }
    }
    free(bd);
}

/* R2 (Stuetzle & Hoos 2000, cited at P:1140-1142): with p = p_best, avg = n/2,
 *   tau_max = 1 / ((1 - rho) C),   tau_min = tau_max (1 - p^(1/n)) / ((avg - 1) p^(1/n)),
 * tau_min clamped to <= tau_max; both computed in double and rounded to float. */
ORC_EXPORT double orc_limits_factor(int32_t n, double p_best)
{
    double pn = pow(p_best, 1.0 / (double)n);
    return (1.0 - pn) / (((double)n / 2.0 - 1.0) * pn);
}

ORC_EXPORT void orc_limits(double rho, int64_t cost, double factor, float *tmin, float *tmax)
{
    double tx = 1.0 / ((1.0 - rho) * (double)cost);
    double tn = tx * factor;
    if (tn > tx) tn = tx;
    *tmax = (float)tx;
    *tmin = (float)tn;
}

/* ------------------------------------------------------------------------- */
/* Colony state                                                               */
/* ------------------------------------------------------------------------- */
typedef struct {
    int32_t n, m, cl;
    double alpha, beta, rho, p_best;
    uint64_t seed;
    int32_t deposit_global;   /* R7: 0 = iteration best (Alg. 1), 1 = global best */
    int32_t fallback_argmax;  /* R9: 0 = WRS over all unvisited (default), 1 = argmax weight */
    int32_t local_search;     /* a8: 2-opt on every route (R25) */
    int32_t nthreads;
    int32_t tabu;             /* R27: 0 = bitmask tabu BT (default), 1 = compact tabu CT (cl = 0 only) */
    int32_t selection;        /* R28: 0 = WRS (Sec. 4.2.2, default), 1 = parallel roulette wheel PRWM (Sec. 4.2.1) */
} orc_params;

typedef struct {
    orc_params p;
    double *xy;
    float *heur, *tau, *inv_w;          /* n x n row-major */
    int32_t *cand;                      /* n x cl */
    int32_t *ls_nn;                     /* n x ls_k: 2-opt neighbour lists (R25) */
    int32_t ls_k;
    int32_t *routes;                    /* m x n, last iteration */
    int64_t *lengths;                   /* m */
    int64_t *fallbacks;                 /* m: fallback steps of each ant, last iteration */
    int32_t *gb_route;
    int64_t gb_len;                     /* -1 = empty (Alg. 1) */
    int32_t *ib_route;
    int64_t ib_len;
    int32_t ib_ant;
    int64_t nn_len;
    double factor;
    float tmin, tmax;
    int32_t iter;                       /* R30: global 0-based iteration counter */
    uint32_t key[2];
} orc_t;

static float pow_alpha(float tau, int32_t a)
{
    /* R17: integer alpha by repeated multiplication (alpha = 1 in every experiment) */
    if (a == 0) return 1.0f;
    float p = tau;
    for (int32_t k = 1; k < a; ++k) p = p * tau;
    return p;
}

static int is_int_in(double x, int lo, int hi)
{
    return x == floor(x) && x >= lo && x <= hi;
}

/* choice_info = tau^alpha * eta^beta, stored as its reciprocal
 * inv_w ("the reciprocal of each weight ... calculated in advance"). */
ORC_EXPORT float orc_inv_w(float tau, float heur, int32_t alpha)
{
    return 1.0f / (pow_alpha(tau, alpha) * heur);
}

/* R11/R18: eta = 1 / max(d, 1); eta^beta built in double, rounded to float.
 * Integer beta in [0, 8]: D^beta by repeated double multiplication; otherwise libm pow. */
ORC_EXPORT float orc_heur(int32_t d, double beta)
{
    double D = (double)(d > 1 ? d : 1);
    if (is_int_in(beta, 0, 8)) {
        double Db = 1.0;
        for (int k = 0; k < (int)beta; ++k) Db = Db * D;
        return (float)(1.0 / Db);
    }
    return (float)pow(D, -beta);
}

static void recompute_inv_w(orc_t *o)
{
    size_t nn = (size_t)o->p.n * o->p.n;
    int32_t a = (int32_t)o->p.alpha;
    for (size_t e = 0; e < nn; ++e)
        o->inv_w[e] = orc_inv_w(o->tau[e], o->heur[e], a);
}

ORC_EXPORT void orc_destroy(orc_t *o)
{
    if (!o) return;
    free(o->xy); free(o->heur); free(o->tau); free(o->inv_w); free(o->cand); free(o->ls_nn);
    free(o->routes); free(o->lengths); free(o->fallbacks);
    free(o->gb_route); free(o->ib_route);
    free(o);
}

ORC_EXPORT orc_t *orc_create(const orc_params *p, const double *coords)
{
    if (p->n < 3 || p->n >= 65536 || p->m < 1 || p->cl < 0 || p->cl > p->n - 1) return NULL;
    if (!(p->rho > 0.0 && p->rho < 1.0)) return NULL;
    if (!is_int_in(p->alpha, 0, 8) || p->beta < 0.0) return NULL;
    if (!(p->p_best > 0.0 && p->p_best < 1.0)) return NULL;
    if (p->tabu < 0 || p->tabu > 1 || (p->tabu == 1 && p->cl != 0)) return NULL;   /* R27 */
    if (p->selection < 0 || p->selection > 1) return NULL;                          /* R28 */
    if (p->selection == 1 && p->fallback_argmax) return NULL;   /* R28: the wheel is its own fallback */
    for (int32_t i = 0; i < 2 * p->n; ++i)
        if (!isfinite(coords[i])) return NULL;

    orc_t *o = calloc(1, sizeof(orc_t));
    o->p = *p;
    if (o->p.nthreads < 1) o->p.nthreads = 1;
    int32_t n = p->n;
    size_t nn = (size_t)n * n;
    o->xy = malloc(sizeof(double) * 2 * (size_t)n);
    memcpy(o->xy, coords, sizeof(double) * 2 * (size_t)n);
    o->heur = malloc(sizeof(float) * nn);
    o->tau = malloc(sizeof(float) * nn);
    o->inv_w = malloc(sizeof(float) * nn);
    o->cand = malloc(sizeof(int32_t) * (size_t)n * (p->cl > 0 ? p->cl : 1));
    o->routes = malloc(sizeof(int32_t) * (size_t)p->m * n);
    o->lengths = calloc((size_t)p->m, sizeof(int64_t));
    o->fallbacks = calloc((size_t)p->m, sizeof(int64_t));
    o->gb_route = malloc(sizeof(int32_t) * n);
    o->ib_route = malloc(sizeof(int32_t) * n);
    o->gb_len = -1;
    o->ib_len = -1;
    o->ib_ant = -1;
    o->key[0] = (uint32_t)p->seed;
    o->key[1] = (uint32_t)(p->seed >> 32);

    /* heuristic matrix eta^beta */
    for (int32_t i = 0; i < n; ++i)
        for (int32_t j = 0; j < n; ++j)
            o->heur[(size_t)i * n + j] = orc_heur(orc_dist(o->xy, i, j), p->beta);
    if (p->cl > 0) orc_cand_lists(o->xy, n, p->cl, o->cand);
    if (p->local_search) {
        /* the 2-opt search is limited to the 32 nearest neighbours */
        o->ls_k = n - 1 < 32 ? n - 1 : 32;
        o->ls_nn = malloc(sizeof(int32_t) * (size_t)n * o->ls_k);
        orc_cand_lists(o->xy, n, o->ls_k, o->ls_nn);
    }

    /* Alg. 1: limits from the NN solution, tau := tau_max. */
    int32_t *nn_route = malloc(sizeof(int32_t) * n);
    o->nn_len = orc_nn_tour(o->xy, n, nn_route);
    free(nn_route);
    o->factor = orc_limits_factor(n, p->p_best);
    orc_limits(p->rho, o->nn_len, o->factor, &o->tmin, &o->tmax);
    for (size_t e = 0; e < nn; ++e) o->tau[e] = o->tmax;
    recompute_inv_w(o);
    return o;
}

/* ------------------------------------------------------------------------- */
/* Node selection: WRS / A-Res with reservoir size 1 (Sec. 4.2.2, Alg. 2       */
/* P:930-948, Alg. 3), log-key form k = (1/w) log2 r.  */
/* argmax over keys, ties -> lowest city id (R16).                             */
/* ------------------------------------------------------------------------- */
static float rng_word(const uint32_t key[2], uint32_t x0, uint32_t x1, uint32_t a, uint32_t it, int w)
{
    uint32_t ctr[4] = {x0, x1, a, it}, out[4];
    orc_philox4x32_10(ctr, key, out);
    return orc_uniform(out[w]);
}

/* One construction step of ant a at step s from node cur.
 * Returns the chosen node; *fell_back = 1 if the candidate list had no
 * unvisited node (R9). */
ORC_EXPORT int32_t orc_select_next(const float *inv_w_row, const int32_t *cand_row, int32_t cl,
                                   const char *visited, int32_t n, int32_t s, uint32_t a,
                                   uint32_t it, const uint32_t key[2], int32_t fallback_argmax,
                                   int32_t *fell_back)
{
    int32_t best = -1;
    float best_key = -INFINITY;
    /* candidate list: slot k uses counter (k, s>>2, a, it), word s&3 (R13) */
    for (int32_t k = 0; k < cl; ++k) {
        int32_t c = cand_row[k];
        if (visited[c]) continue;
        float u = rng_word(key, (uint32_t)k, (uint32_t)s >> 2, a, it, s & 3);
        float kk = orc_det_log2(u) * inv_w_row[c];
        if (best < 0 || kk > best_key || (kk == best_key && c < best)) {
            best = c;
            best_key = kk;
        }
    }
    *fell_back = 0;
    if (best >= 0) return best;
    *fell_back = (cl > 0);
    if (fallback_argmax && cl > 0) {
        /* R9 flag: the unvisited node with the largest weight = smallest inv_w */
        for (int32_t c = 0; c < n; ++c) {
            if (visited[c]) continue;
            if (best < 0 || inv_w_row[c] < inv_w_row[best]) best = c;
        }
        return best;
    }
    /* all unvisited nodes (cl = 0: every step; R9: candidate-list fallback):
     * city c uses counter (0x40000000 | c>>2, s, a, it), word c&3 (R13) */
    for (int32_t c = 0; c < n; ++c) {
        if (visited[c]) continue;
        float u = rng_word(key, 0x40000000u | ((uint32_t)c >> 2), (uint32_t)s, a, it, c & 3);
        float kk = orc_det_log2(u) * inv_w_row[c];
        if (best < 0 || kk > best_key) {   /* ascending c: a tie keeps the lower id */
            best = c;
            best_key = kk;
        }
    }
    return best;
}

/* ------------------------------------------------------------------------- */
/* Compact tabu CT (Sec. 4.1), used by the full-row path (cl = 0,   */
/* the paper's MMAS-WRS-CT, recommended without candidate lists P:1998-2001).  */
/* entries[0..L) is the list of unvisited nodes; a position p >= L holds the   */
/* index of node p if p was relocated into the list, else the sentinel n.      */
/* ------------------------------------------------------------------------- */
ORC_EXPORT void orc_ct_init(int32_t *entries, int32_t *L, int32_t n)
{
    /* "Initially, the entries array contains consecutive numbers from 0 to n-1" */
    for (int32_t i = 0; i < n; ++i) entries[i] = i;
    *L = n;
}

/* mark(u) for an unvisited node u. */
ORC_EXPORT void orc_ct_mark(int32_t *entries, int32_t *L, int32_t n, int32_t u)
{
    /* u < L: u is at its initial position; u >= L: entries[u] is its index */
    int32_t iu = u < *L ? u : entries[u];
    if (iu == *L - 1) {
        entries[iu] = n;                      /* u is the last element: sentinel */
    } else {
        int32_t t = entries[*L - 1];          /* the last element replaces u */
        entries[iu] = t;
        entries[t] = iu;                      /* "the new position of t is saved" */
    }
    *L -= 1;
}

/* One full-row step over the CT (Alg. 3 P:964-994 with l = tabu.length() = L,
 * v = tabu.get_candidate(i) = entries[i]).  R27: the uniform of the i-th
 * enumerated element uses counter (0x40000000 | i>>2, s, a, it), word i&3 --
 * the same counter as the bitmask scan, whose i-th element is city i.
 * argmax key, ties -> lowest node id (R16). */
ORC_EXPORT int32_t orc_select_next_ct(const float *inv_w_row, const int32_t *entries, int32_t L, int32_t s,
                                      uint32_t a, uint32_t it, const uint32_t key[2])
{
    int32_t best = -1;
    float best_key = -INFINITY;
    for (int32_t i = 0; i < L; ++i) {
        int32_t v = entries[i];
        float u = rng_word(key, 0x40000000u | ((uint32_t)i >> 2), (uint32_t)s, a, it, i & 3);
        float kk = orc_det_log2(u) * inv_w_row[v];
        if (best < 0 || kk > best_key || (kk == best_key && v < best)) {
            best = v;
            best_key = kk;
        }
    }
    return best;
}

/* ------------------------------------------------------------------------- */
/* Parallel roulette wheel PRWM (Sec. 4.2.1; reading R28), p = 32.  */
/* Items 0..len-1 with weights w[i] >= 0 (0 = visited).  One stage over items  */
/* [lo, hi): chunk size c = ceil((hi-lo)/p); thread t owns [lo+t c, lo+(t+1)c) */
/* and sums its weights in item order ("computes a sum of the corresponding    */
/* weights"); an inclusive prefix sum of the p chunk sums ("computed in        */
/* parallel": the Hillis-Steele scan, R28); the first stage draws r = u*total  */
/* ("the last thread draws a uniform random number and multiplies it by the    */
/* total"); the winning chunk is the first t with prefix[t] > r; r is reduced  */
/* by the preceding chunks' prefix and the stage repeats on the winning chunk  */
/* until it holds one item ("up to ceil(log_p n) stages").  If rounding leaves */
/* r >= prefix[p-1], the last chunk with a positive sum wins.                  */
/* Returns the selected item, or -1 when every weight is 0.                    */
/* ------------------------------------------------------------------------- */
#define ORC_P 32
ORC_EXPORT int32_t orc_prwm(const float *w, int32_t len, float u)
{
    int32_t lo = 0, hi = len;
    float r = 0.0f;
    int first = 1;
    do {
        int32_t c = (hi - lo + ORC_P - 1) / ORC_P;
        float sum[ORC_P], pre[ORC_P], nxt[ORC_P];
        for (int32_t t = 0; t < ORC_P; ++t) {
            float acc = 0.0f;
            for (int32_t i = lo + t * c; i < lo + (t + 1) * c && i < hi; ++i) acc = acc + w[i];
            sum[t] = acc;
            pre[t] = acc;
        }
        /* Hillis-Steele inclusive scan: log2(p) rounds, pre[t] += pre[t - d] */
        for (int32_t d = 1; d < ORC_P; d *= 2) {
            for (int32_t t = 0; t < ORC_P; ++t) nxt[t] = t >= d ? pre[t] + pre[t - d] : pre[t];
            memcpy(pre, nxt, sizeof(pre));
        }
        if (first) {
            if (pre[ORC_P - 1] == 0.0f) return -1;
            r = u * pre[ORC_P - 1];
            first = 0;
        }
        /* a chunk with a zero sum never wins: with the scan's association its prefix can
         * round above the previous one (R28) */
        int32_t win = -1;
        for (int32_t t = 0; t < ORC_P; ++t)
            if (pre[t] > r && sum[t] > 0.0f) { win = t; break; }
        if (win < 0)
            for (int32_t t = ORC_P - 1; t >= 0; --t)
                if (sum[t] > 0.0f) { win = t; break; }
        if (win > 0) r = r - pre[win - 1];
        lo = lo + win * c;
        hi = lo + c < hi ? lo + c : hi;
    } while (hi - lo > 1);
    return lo;
}

/* weight of edge (i, j) for the roulette wheel: choice_info = tau^alpha * eta^beta */
static float rwm_weight(const orc_t *o, int32_t i, int32_t j)
{
    size_t e = (size_t)i * o->p.n + j;
    return pow_alpha(o->tau[e], (int32_t)o->p.alpha) * o->heur[e];
}

/* One PRWM construction step: candidate list first (cl > 0), else / on fallback
 * all nodes with visited weights 0 (BT) or the CT's list (R27).  One uniform per
 * step: counter (0x20000000, s, a, it), word 0 (R28). */
static int32_t select_next_rwm(const orc_t *o, int32_t cur, const char *vis, const int32_t *entries, int32_t L,
                               int32_t s, uint32_t a, float *wbuf, int32_t *fell_back)
{
    int32_t n = o->p.n, cl = o->p.cl;
    float u = rng_word(o->key, 0x20000000u, (uint32_t)s, a, (uint32_t)o->iter, 0);
    *fell_back = 0;
    if (cl > 0) {
        const int32_t *cand = o->cand + (size_t)cur * cl;
        for (int32_t k = 0; k < cl; ++k) wbuf[k] = vis[cand[k]] ? 0.0f : rwm_weight(o, cur, cand[k]);
        int32_t k = orc_prwm(wbuf, cl, u);
        if (k >= 0) return cand[k];
        *fell_back = 1;
    }
    if (entries) {
        for (int32_t i = 0; i < L; ++i) wbuf[i] = rwm_weight(o, cur, entries[i]);
        return entries[orc_prwm(wbuf, L, u)];
    }
    for (int32_t c = 0; c < n; ++c) wbuf[c] = vis[c] ? 0.0f : rwm_weight(o, cur, c);
    return orc_prwm(wbuf, n, u);
}

/* Start node u ~ U{0, n-1} (Alg. 1): counter (0x80000000, 0, a, it), word 0,
 * start = floor(x * n / 2^32). */
ORC_EXPORT int32_t orc_start_node(int32_t n, uint32_t a, uint32_t it, const uint32_t key[2])
{
    uint32_t ctr[4] = {0x80000000u, 0u, a, it}, out[4];
    orc_philox4x32_10(ctr, key, out);
    return (int32_t)(((uint64_t)out[0] * (uint64_t)n) >> 32);
}

typedef struct {
    orc_t *o;
    int32_t a0, a1;
} orc_job;

/* ------------------------------------------------------------------------- */
/* Row a8: 2-opt local search (Sec. 5.7; Bentley 1992), R25:      */
/*  - neighbour lists: the K = min(32, n-1) nearest nodes by (d, id);          */
/*  - active nodes in a FIFO queue, initially the route in order; a node is in */
/*    the queue at most once ("don't-look bit" clear <=> queued);              */
/*  - for the popped node a: dir = successor, then predecessor; b = dir(a);    */
/*    for k = 0..K-1: c = nn[a][k]; stop at the first d(a,c) >= d(a,b)        */
/*    (Bentley's pruning); d = dir(c); skip c == b or d == a;                  */
/*    gain test  d(a,c) + d(b,d) - d(a,b) - d(c,d) < 0 -> apply the FIRST      */
/*    improving move, enqueue a, b, c, d (in that order, if not queued), and   */
/*    go to the next pop;                                                       */
/*  - a move replaces two edges by (a,c), (b,d): the forward segment between   */
/*    them is reversed, or its complement when that is strictly shorter;       */
/*  - "the search is restarted until no further improvements can be found"     */
/*    (P:1731-1732): when the queue runs empty it is re-seeded with the whole  */
/*    route (in route order) until a full sweep applies no move, so the result */
/*    is a local optimum of the neighbour-restricted move set.                 */
/* ------------------------------------------------------------------------- */

/* Reverse the forward cyclic segment of positions i..j (inclusive); if the
 * complement is strictly shorter, reverse the complement instead. */
ORC_EXPORT void orc_reverse(int32_t *route, int32_t *pos, int32_t n, int32_t i, int32_t j)
{
    int32_t len = (j - i + n) % n + 1;
    if (2 * len > n) {                  /* complement (j+1 .. i-1) is strictly shorter */
        int32_t ni = (j + 1) % n, nj = (i - 1 + n) % n;
        i = ni;
        j = nj;
        len = n - len;
    }
    for (int32_t k = 0; k < len / 2; ++k) {
        int32_t p = (i + k) % n, q = (j - k + n) % n;
        int32_t t = route[p];
        route[p] = route[q];
        route[q] = t;
        pos[route[p]] = p;
        pos[route[q]] = q;
    }
}

ORC_EXPORT int64_t orc_two_opt(const double *xy, int32_t n, const int32_t *nn, int32_t K, int32_t *route,
                               int64_t *moves_out)
{
    int32_t *pos = malloc(sizeof(int32_t) * (size_t)n);
    int32_t *queue = malloc(sizeof(int32_t) * (size_t)n);
    char *inq = malloc((size_t)n);
    for (int32_t i = 0; i < n; ++i) pos[route[i]] = i;
    int64_t delta_total = 0, moves = 0, sweep_moves;
    do {
        for (int32_t i = 0; i < n; ++i) {     /* (re-)seed: every node, in route order */
            queue[i] = route[i];
            inq[route[i]] = 1;
        }
        int32_t head = 0, count = n;
        sweep_moves = 0;
        while (count > 0) {
            int32_t a = queue[head];
            head = (head + 1) % n;
            --count;
            inq[a] = 0;
            int improved = 0;
            for (int dir = 0; dir < 2 && !improved; ++dir) {       /* 0: successor, 1: predecessor */
                int32_t pa = pos[a];
                int32_t b = dir == 0 ? route[(pa + 1) % n] : route[(pa - 1 + n) % n];
                int64_t dab = orc_dist(xy, a, b);
                for (int32_t k = 0; k < K; ++k) {
                    int32_t c = nn[(size_t)a * K + k];
                    int64_t dac = orc_dist(xy, a, c);
                    if (dac >= dab) break;
                    int32_t pc = pos[c];
                    int32_t d = dir == 0 ? route[(pc + 1) % n] : route[(pc - 1 + n) % n];
                    if (c == b || d == a) continue;
                    int64_t delta = dac + orc_dist(xy, b, d) - dab - orc_dist(xy, c, d);
                    if (delta < 0) {
                        if (dir == 0)   /* edges (a,b),(c,d) -> (a,c),(b,d): reverse b .. c */
                            orc_reverse(route, pos, n, pos[b], pos[c]);
                        else            /* edges (b,a),(d,c) -> (b,d),(a,c): reverse a .. d */
                            orc_reverse(route, pos, n, pos[a], pos[d]);
                        int32_t ends[4] = {a, b, c, d};
                        for (int e = 0; e < 4; ++e) {
                            if (!inq[ends[e]]) {
                                queue[(head + count) % n] = ends[e];
                                ++count;
                                inq[ends[e]] = 1;
                            }
                        }
                        delta_total += delta;
                        ++sweep_moves;
                        improved = 1;
                        break;
                    }
                }
            }
        }
        moves += sweep_moves;
    } while (sweep_moves > 0);
    free(pos);
    free(queue);
    free(inq);
    if (moves_out) *moves_out = moves;
    return delta_total;
}

/* Alg. 1: ant a builds its route for the current iteration.
 * Returns the number of fallback steps (R9). */
static int64_t build_route(const orc_t *o, int32_t a, int32_t *route, char *vis)
{
    int32_t n = o->p.n;
    memset(vis, 0, (size_t)n);
    int64_t fb = 0;
    int32_t cur = orc_start_node(n, (uint32_t)a, (uint32_t)o->iter, o->key);
    route[0] = cur;
    vis[cur] = 1;
    if (o->p.selection == 1) {
        /* MMAS-RWM (R28): parallel roulette wheel over the candidate list / BT / CT */
        float *wbuf = malloc(sizeof(float) * (size_t)n);
        int32_t *entries = NULL, L = 0;
        if (o->p.tabu == 1) {
            entries = malloc(sizeof(int32_t) * (size_t)n);
            orc_ct_init(entries, &L, n);
            orc_ct_mark(entries, &L, n, cur);
        }
        for (int32_t s = 1; s < n; ++s) {
            int32_t f;
            int32_t nxt = select_next_rwm(o, cur, vis, entries, L, s, (uint32_t)a, wbuf, &f);
            fb += f;
            if (entries) orc_ct_mark(entries, &L, n, nxt);
            route[s] = nxt;
            vis[nxt] = 1;
            cur = nxt;
        }
        free(wbuf);
        free(entries);
        if (o->p.local_search) orc_two_opt(o->xy, n, o->ls_nn, o->ls_k, route, NULL);
        return fb;
    }
    if (o->p.tabu == 1) {
        /* MMAS-WRS-CT (cl = 0): the list of unvisited nodes is the CT's left part */
        int32_t *entries = malloc(sizeof(int32_t) * (size_t)n), L;
        orc_ct_init(entries, &L, n);
        orc_ct_mark(entries, &L, n, cur);
        for (int32_t s = 1; s < n; ++s) {
            int32_t nxt = orc_select_next_ct(o->inv_w + (size_t)cur * n, entries, L, s, (uint32_t)a,
                                             (uint32_t)o->iter, o->key);
            orc_ct_mark(entries, &L, n, nxt);
            route[s] = nxt;
            cur = nxt;
        }
        free(entries);
        if (o->p.local_search) orc_two_opt(o->xy, n, o->ls_nn, o->ls_k, route, NULL);
        return 0;
    }
    for (int32_t s = 1; s < n; ++s) {
        int32_t f;
        int32_t nxt = orc_select_next(o->inv_w + (size_t)cur * n, o->cand + (size_t)cur * o->p.cl,
                                      o->p.cl, vis, n, s, (uint32_t)a, (uint32_t)o->iter, o->key,
                                      o->p.fallback_argmax, &f);
        fb += f;
        route[s] = nxt;
        vis[nxt] = 1;
        cur = nxt;
    }
    if (o->p.local_search) orc_two_opt(o->xy, n, o->ls_nn, o->ls_k, route, NULL);   /* row a8, R26 */
    return fb;
}

static void *construct_range(void *arg)
{
    orc_job *job = arg;
    orc_t *o = job->o;
    int32_t n = o->p.n;
    char *vis = malloc((size_t)n);
    for (int32_t a = job->a0; a < job->a1; ++a) {
        int32_t *route = o->routes + (size_t)a * n;
        o->fallbacks[a] = build_route(o, a, route, vis);
        o->lengths[a] = orc_tour_length(o->xy, n, route);
    }
    free(vis);
    return NULL;
}

/* One ant's route at the current iteration without advancing the colony (for
 * sampled parity checks at full size).  Returns its length. */
ORC_EXPORT int64_t orc_construct_ant(const orc_t *o, int32_t a, int32_t *route_out, int64_t *fallbacks)
{
    char *vis = malloc((size_t)o->p.n);
    int64_t fb = build_route(o, a, route_out, vis);
    free(vis);
    if (fallbacks) *fallbacks = fb;
    return orc_tour_length(o->xy, o->p.n, route_out);
}

/* Pheromone update, Alg. 1, in the paper's order.
 * 1. evaporation  tau <- max(rho tau, tau_min)            (R1: rho = retention)
 * 2. deposit      tau <- min(tau + Delta, tau_max) on both orientations of every edge
 *    of the deposit route, Delta = (float)(1/cost)        (R5, R6)
 * 3. R4: every trail kept inside [tau_min, tau_max].
 * All n x n entries are processed (the diagonal is never read by construction). */
ORC_EXPORT void orc_update_trails(float *tau, int32_t n, double rho, float tmin, float tmax,
                                  const int32_t *route, int64_t cost)
{
    size_t nn = (size_t)n * n;
    float rho_f = (float)rho;
    for (size_t e = 0; e < nn; ++e) {
        float t = rho_f * tau[e];
        tau[e] = t > tmin ? t : tmin;
    }
    float delta = (float)(1.0 / (double)cost);
    for (int32_t k = 0; k < n; ++k) {
        int32_t i = route[k], j = route[(k + 1) % n];
        float t1 = tau[(size_t)i * n + j] + delta;
        tau[(size_t)i * n + j] = t1 < tmax ? t1 : tmax;
        float t2 = tau[(size_t)j * n + i] + delta;
        tau[(size_t)j * n + i] = t2 < tmax ? t2 : tmax;
    }
    for (size_t e = 0; e < nn; ++e)
        if (tau[e] > tmax) tau[e] = tmax;
}

/* One MMAS iteration: Alg. 1 lines 263-289. */
static void iterate_once(orc_t *o)
{
    int32_t n = o->p.n, m = o->p.m;

    /* lines 266-276: every ant builds a complete route (ants are independent) */
    int32_t T = o->p.nthreads < m ? o->p.nthreads : m;
    pthread_t th[256];
    orc_job jobs[256];
    if (T > 256) T = 256;
    for (int32_t t = 0; t < T; ++t) {
        jobs[t].o = o;
        jobs[t].a0 = (int32_t)((int64_t)m * t / T);
        jobs[t].a1 = (int32_t)((int64_t)m * (t + 1) / T);
    }
    if (T == 1) {
        construct_range(&jobs[0]);
    } else {
        for (int32_t t = 0; t < T; ++t) pthread_create(&th[t], NULL, construct_range, &jobs[t]);
        for (int32_t t = 0; t < T; ++t) pthread_join(th[t], NULL);
    }

    /* line 278: iteration best = shortest route, ties -> lowest ant id (R8) */
    int32_t ib = 0;
    for (int32_t a = 1; a < m; ++a)
        if (o->lengths[a] < o->lengths[ib]) ib = a;
    o->ib_ant = ib;
    o->ib_len = o->lengths[ib];
    memcpy(o->ib_route, o->routes + (size_t)ib * n, sizeof(int32_t) * n);

    /* lines 281-285: global best replaced only by a strictly shorter route; limits from it */
    if (o->gb_len < 0 || o->ib_len < o->gb_len) {
        o->gb_len = o->ib_len;
        memcpy(o->gb_route, o->ib_route, sizeof(int32_t) * n);
        orc_limits(o->p.rho, o->gb_len, o->factor, &o->tmin, &o->tmax);
    }

    /* lines 287-288: evaporation + deposit along the deposit route */
    const int32_t *dep = o->p.deposit_global ? o->gb_route : o->ib_route;
    int64_t dep_len = o->p.deposit_global ? o->gb_len : o->ib_len;
    orc_update_trails(o->tau, n, o->p.rho, o->tmin, o->tmax, dep, dep_len);

    /* choice_info for the next construction */
    recompute_inv_w(o);
    o->iter += 1;
}

ORC_EXPORT int orc_iterate(orc_t *o, int32_t iters)
{
    if (!o || iters < 1) return -1;
    for (int32_t k = 0; k < iters; ++k) iterate_once(o);
    return 0;
}

/* ---- getters (plain copies) ---------------------------------------------- */
ORC_EXPORT int32_t orc_iteration(const orc_t *o) { return o->iter; }
ORC_EXPORT int64_t orc_nn_length(const orc_t *o) { return o->nn_len; }
ORC_EXPORT double orc_factor(const orc_t *o) { return o->factor; }
ORC_EXPORT void orc_get_limits(const orc_t *o, float *tmin, float *tmax) { *tmin = o->tmin; *tmax = o->tmax; }
ORC_EXPORT void orc_get_tours(const orc_t *o, int32_t *out) { memcpy(out, o->routes, sizeof(int32_t) * (size_t)o->p.m * o->p.n); }
ORC_EXPORT void orc_get_lengths(const orc_t *o, int64_t *out) { memcpy(out, o->lengths, sizeof(int64_t) * (size_t)o->p.m); }
ORC_EXPORT void orc_get_fallbacks(const orc_t *o, int64_t *out) { memcpy(out, o->fallbacks, sizeof(int64_t) * (size_t)o->p.m); }
ORC_EXPORT void orc_get_tau(const orc_t *o, float *out) { memcpy(out, o->tau, sizeof(float) * (size_t)o->p.n * o->p.n); }
ORC_EXPORT void orc_get_inv_w(const orc_t *o, float *out) { memcpy(out, o->inv_w, sizeof(float) * (size_t)o->p.n * o->p.n); }
ORC_EXPORT void orc_get_heur(const orc_t *o, float *out) { memcpy(out, o->heur, sizeof(float) * (size_t)o->p.n * o->p.n); }
ORC_EXPORT void orc_get_cand(const orc_t *o, int32_t *out) { memcpy(out, o->cand, sizeof(int32_t) * (size_t)o->p.n * o->p.cl); }
ORC_EXPORT int32_t orc_ib_ant(const orc_t *o) { return o->ib_ant; }
ORC_EXPORT int64_t orc_best_tour(const orc_t *o, int32_t *out)
{
    if (o->gb_len < 0) return -5;
    memcpy(out, o->gb_route, sizeof(int32_t) * o->p.n);
    return o->gb_len;
}
