"""Pins of the oracle's setup, pheromone update and whole MMAS loop (Alg. 1,
P:247-293) against worked examples, closed forms, invariants and brute force."""
import itertools
import math

import numpy as np
import pytest

import oracle
from paper_2003_11902_b200.instances import CONFIGS, make_coords


# ---- setup (row a0) ------------------------------------------------------------
def test_distance_examples():
    # golden/spec_worked_examples.txt dist_345, dist_diag
    c = np.array([[0, 0], [3, 4], [1, 1], [1.5, 2.0]], dtype=np.float64)
    assert oracle.dist(c, 0, 1) == 5
    assert oracle.dist(c, 0, 2) == 1
    assert oracle.dist(c, 0, 3) == 3          # 2.5 rounds half up (TSPLIB nint)


def test_distance_brute_force_symmetry():
    c = make_coords("uniform", 40, 3)
    for i in range(40):
        for j in range(40):
            d = oracle.dist(c, i, j)
            exact = math.hypot(c[i, 0] - c[j, 0], c[i, 1] - c[j, 1])
            assert d == math.floor(exact + 0.5)
            assert d == oracle.dist(c, j, i)


def test_nn_tour_collinear():
    # golden nn_collinear
    c = np.array([[0, 0], [1, 0], [2, 0], [3, 0]], dtype=np.float64)
    r, L = oracle.nn_tour(c)
    assert list(r) == [0, 1, 2, 3] and L == 6


def test_nn_tour_is_greedy_permutation():
    c = make_coords("uniform", 60, 11)
    r, L = oracle.nn_tour(c)
    assert sorted(r) == list(range(60)) and r[0] == 0
    D = np.array([[oracle.dist(c, i, j) for j in range(60)] for i in range(60)])
    seen = {0}
    for k in range(1, 60):
        rest = [j for j in range(60) if j not in seen]
        best = min(rest, key=lambda j: (D[r[k - 1], j], j))
        assert r[k] == best
        seen.add(r[k])
    assert L == sum(D[r[k], r[(k + 1) % 60]] for k in range(60))


def test_candidate_lists_examples_and_sort():
    # golden cand_line
    c = np.array([[0, 0], [1, 0], [2, 0], [10, 0]], dtype=np.float64)
    assert list(oracle.cand_lists(c, 2)[0]) == [1, 2]
    # equilateral-ish tie -> smaller id
    t = np.array([[0, 0], [10, 0], [5, 9], [5, -9]], dtype=np.float64)
    assert [oracle.dist(t, 0, j) for j in (1, 2, 3)] == [10, 10, 10]
    assert list(oracle.cand_lists(t, 2)[0]) == [1, 2]
    # against numpy's lexsort (a library routine) on a clustered instance with many ties
    c = make_coords("d198", 198, 198)
    cl = 16
    got = oracle.cand_lists(c, cl)
    D = np.array([[oracle.dist(c, i, j) for j in range(198)] for i in range(198)])
    for i in range(198):
        ids = np.array([j for j in range(198) if j != i])
        order = np.lexsort((ids, D[i, ids]))
        assert list(got[i]) == list(ids[order[:cl]])


def test_limits_closed_forms():
    # golden tau_max: rho = 0.5, C = 100 -> tau_max = 0.02
    F = oracle.limits_factor(1002, 0.01)
    tmin, tmax = oracle.limits(0.5, 100, F)
    assert tmax == np.float32(0.02)
    # tau_min = tau_max * (1 - p^(1/n)) / ((n/2 - 1) p^(1/n))  (Stuetzle & Hoos)
    for n, approx in ((198, 2.40e-4), (1002, 9.21e-6), (2392, 1.61e-6), (3795, 6.40e-7), (18512, 2.69e-8)):
        assert abs(oracle.limits_factor(n, 0.01) / approx - 1) < 5e-3
    # n <= 5: F > 1, the clamp tau_min <= tau_max applies (SPEC.md S:341's "sanity" claim is false)
    F4 = oracle.limits_factor(4, 0.01)
    assert F4 > 1
    tmin, tmax = oracle.limits(0.5, 4, F4)
    assert tmin == tmax == np.float32(0.5)
    assert oracle.limits_factor(6, 0.01) < 1


def test_choice_info_example():
    # golden choice_info: alpha 1, beta 2, tau 0.02, d 10 -> 2e-4
    w = 1.0 / oracle.inv_w(np.float32(0.02), oracle.heur(10, 2.0), 1)
    assert abs(w - 2e-4) < 1e-10
    # alpha=1, beta=0 -> w = tau; alpha=0, beta=1 -> w = 1/d
    assert oracle.heur(10, 0.0) == 1.0
    assert oracle.inv_w(np.float32(0.25), 1.0, 1) == 4.0
    assert oracle.inv_w(np.float32(0.25), oracle.heur(8, 1.0), 0) == 8.0
    assert oracle.heur(0, 2.0) == 1.0          # R11: eta = 1/max(d, 1)


def test_pow_alpha_fixed_values():
    """R17 (integer alpha by repeated multiplication; Eq. (1) P:228-231 raises tau to alpha):
    with tau a power of two every product is exact, so inv_w = 1/(tau^alpha * eta) has a
    closed form; an off-by-one in the multiplication loop changes it by a factor tau."""
    # tau = 0.5, eta = 1: alpha 2 -> 4, alpha 3 -> 8, alpha 8 -> 256
    assert oracle.inv_w(np.float32(0.5), 1.0, 2) == 4.0
    assert oracle.inv_w(np.float32(0.5), 1.0, 3) == 8.0
    assert oracle.inv_w(np.float32(0.5), 1.0, 8) == 256.0
    # tau = 3 (exact powers 9, 27), eta = 1/4: 1/(9/4) and 1/(27/4) correctly rounded
    assert oracle.inv_w(np.float32(3.0), 0.25, 2) == np.float32(4.0 / 9.0)
    assert oracle.inv_w(np.float32(3.0), 0.25, 3) == np.float32(4.0 / 27.0)
    # a non-representable tau: tau^alpha within 2 ulp (alpha-1 roundings) of the exact power
    t = np.float32(0.013)
    for a in (2, 3):
        exact = 1.0 / (float(t) ** a * 0.5)
        got = oracle.inv_w(t, 0.5, a)
        assert abs(got - exact) <= 3 * np.spacing(np.float32(exact)), (a, got, exact)


def test_heur_fixed_values_beta_3_and_non_integer():
    """R18: eta^beta = 1/max(d,1)^beta, integer beta by repeated double
    multiplication, otherwise libm pow -- closed forms at beta = 3 and beta = 2.5."""
    assert oracle.heur(10, 3.0) == np.float32(1e-3)
    assert oracle.heur(7, 3.0) == np.float32(1.0 / 343.0)
    assert oracle.heur(1000, 3.0) == np.float32(1e-9)
    assert oracle.heur(4, 2.5) == np.float32(1.0 / 32.0)      # 4^2.5 = 32
    assert oracle.heur(9, 2.5) == np.float32(1.0 / 243.0)     # 9^2.5 = 243
    assert oracle.heur(100, 0.5) == np.float32(0.1)           # 100^0.5 = 10
    assert oracle.heur(16, 1.25) == np.float32(1.0 / 32.0)    # 16^1.25 = 32
    assert oracle.heur(0, 2.5) == 1.0                         # R11


# ---- pheromone update (row a6) --------------------------------------------------
def test_update_worked_examples():
    n = 5
    route = [0, 1, 2, 3, 4]
    tau = np.full((n, n), 0.02, dtype=np.float32)
    # golden evaporate then deposit: 0.02 -> 0.01 -> +0.01 at C = 100, clamp at 0.02
    out = oracle.update_trails(tau, 0.5, np.float32(0.001), np.float32(0.02), route, 100)
    on = {(route[k], route[(k + 1) % n]) for k in range(n)}
    on |= {(j, i) for i, j in on}
    for i in range(n):
        for j in range(n):
            expect = np.float32(0.02) if (i, j) in on else np.float32(0.01)
            assert out[i, j] == expect
    # an entry at tau_min stays at tau_min when not deposited
    tau2 = np.full((n, n), 0.001, dtype=np.float32)
    out2 = oracle.update_trails(tau2, 0.5, np.float32(0.001), np.float32(0.02), [0, 1, 2, 3, 4], 10 ** 9)
    assert out2[0, 2] == np.float32(0.001)


def test_update_invariants():
    rng = np.random.default_rng(5)
    n = 23
    tmin, tmax = np.float32(1e-4), np.float32(0.05)
    tau = rng.uniform(1e-4, 0.05, size=(n, n)).astype(np.float32)
    tau = (tau + tau.T) / 2
    route = list(rng.permutation(n))
    cost = 5000
    out = oracle.update_trails(tau, 0.5, tmin, tmax, route, cost)
    # bounds and symmetry
    assert np.all(out >= tmin) and np.all(out <= tmax)
    assert np.array_equal(out, out.T)
    # rho = 0.5 is an exact halving in binary floating point (R1)
    evap = np.maximum(np.float32(0.5) * tau, tmin)
    delta = np.float32(1.0 / cost)
    on = np.zeros((n, n), bool)
    for k in range(n):
        on[route[k], route[(k + 1) % n]] = on[route[(k + 1) % n], route[k]] = True
    assert np.array_equal(out[~on], evap[~on])
    # deposit locality: without clamping the matrix gains exactly 2n Delta, only on tour edges
    big = oracle.update_trails(tau, 0.5, tmin, np.float32(1.0), route, cost)
    gain = big.astype(np.float64) - evap.astype(np.float64)
    assert np.count_nonzero(gain) == 2 * n
    assert abs(gain.sum() - 2 * n * float(delta)) < 2 * n * float(delta) * 1e-5


def test_tau_max_is_the_deposit_fixed_point():
    """tau_max = 1/((1-rho) C) is the limit of tau <- rho tau + 1/C (why Stuetzle &
    Hoos choose it): repeated deposits at a fixed cost converge to it
    from below and are then held there by the clamp."""
    n, C, rho = 6, 40, 0.5
    F = oracle.limits_factor(n, 0.01)
    tmin, tmax = oracle.limits(rho, C, F)
    tau = np.full((n, n), tmin, dtype=np.float32)
    route = list(range(n))
    for _ in range(60):
        tau = oracle.update_trails(tau, rho, tmin, tmax, route, C)
    assert abs(float(tau[0, 1]) - 1.0 / ((1 - rho) * C)) < 1e-6 * tmax
    # repeated evaporation without deposits converges to tau_min
    far = oracle.update_trails(np.full((n, n), tmax, dtype=np.float32), rho, tmin, tmax, [0, 1, 2, 3, 4, 5], 10 ** 15)
    for _ in range(80):
        far = oracle.update_trails(far, rho, tmin, tmax, [0, 1, 2, 3, 4, 5], 10 ** 15)
    assert abs(float(far[0, 2]) - tmin) <= 1e-7 * tmin + 1e-30


# ---- whole loop ------------------------------------------------------------------
def test_colony_routes_are_permutations_and_lengths_exact():
    w = CONFIGS["C1"]
    col = oracle.Colony(w.coords(), w.n_ants, w.cand_len, rho=w.rho, seed=w.mmas_seed)
    col.iterate(3)
    T = col.tours()
    L = col.lengths()
    c = w.coords()
    for a in range(0, w.n_ants, 7):
        assert sorted(T[a]) == list(range(w.n))
        assert L[a] == oracle.tour_length(c, T[a])
        assert L[a] == int(np.floor(np.hypot(*(c[T[a]] - c[np.roll(T[a], -1)]).T) + 0.5).sum())
    # iteration best: shortest, ties -> lowest ant (golden ib_ties)
    assert col.ib_ant == int(np.argmin(L))
    gb, gl = col.best_tour()
    assert gl <= L.min() and sorted(gb) == list(range(w.n))
    tmin, tmax = col.limits()
    tau = col.tau()
    assert tau.min() >= tmin and tau.max() <= tmax


def test_global_best_never_worsens_and_limits_follow_it():
    w = CONFIGS["C1"]
    col = oracle.Colony(w.coords(), w.n_ants, w.cand_len, rho=w.rho, seed=7)
    prev = None
    for _ in range(8):
        col.iterate(1)
        _, gl = col.best_tour()
        assert prev is None or gl <= prev
        prev = gl
        tmin, tmax = col.limits()
        assert tmax == np.float32(1.0 / ((1 - w.rho) * gl))


def test_three_cities_unique_cycle():
    # n = 3 -> every construction yields the unique cycle (perimeter)
    c = np.array([[0, 0], [30, 0], [0, 40]], dtype=np.float64)
    col = oracle.Colony(c, 5, 0, seed=1)
    col.iterate(2)
    assert np.all(col.lengths() == 120)


@pytest.mark.parametrize("cl", [0, 3])
def test_brute_force_optimum_tiny(cl):
    """MMAS on an 8-city instance reaches the optimum found by brute force."""
    c = make_coords("uniform", 8, 99)
    best = None
    for perm in itertools.permutations(range(1, 8)):
        r = (0,) + perm
        L = oracle.tour_length(c, r)
        best = L if best is None or L < best else best
    col = oracle.Colony(c, 8, cl, seed=3)
    col.iterate(60)
    gb, gl = col.best_tour()
    assert gl == best and oracle.tour_length(c, gb) == gl


def test_alpha_beta_zero_first_step_uniform():
    # alpha = beta = 0: every weight is 1, so route[1] is uniform over the n-1 others
    from scipy.stats import chisquare
    c = make_coords("uniform", 6, 5)
    counts = np.zeros((6, 6))
    col = oracle.Colony(c, 3000, 0, alpha=0.0, beta=0.0, seed=11)
    col.iterate(1)
    T = col.tours()
    for r in T:
        counts[r[0], r[1]] += 1
    obs = np.array([counts[i, j] for i in range(6) for j in range(6) if i != j])
    rows = np.array([counts[i].sum() / 5 for i in range(6) for j in range(6) if i != j])
    assert chisquare(obs, rows).pvalue > 1e-3


def test_thread_count_invariance():
    w = CONFIGS["C1"]
    outs = []
    for th in (1, 3, 8):
        col = oracle.Colony(w.coords(), 60, w.cand_len, seed=5, nthreads=th)
        col.iterate(2)
        outs.append((col.tours(), col.tau()))
    for t, p in outs[1:]:
        assert np.array_equal(t, outs[0][0]) and np.array_equal(p, outs[0][1])


def test_rejects_bad_parameters():
    c = make_coords("uniform", 10, 1)
    for kw in (dict(rho=1.0), dict(rho=0.0), dict(cand_len=10), dict(alpha=0.5), dict(n_ants=0)):
        args = dict(n_ants=5, cand_len=3)
        args.update(kw)
        with pytest.raises(ValueError):
            oracle.Colony(c, **args)
