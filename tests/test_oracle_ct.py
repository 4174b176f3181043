"""Pins of the oracle's compact tabu (CT, Sec. 4.1) and of the
full-row WRS step over it (MMAS-WRS-CT, Alg. 3, R27).

The CT is pinned against the paper's other list tabu, the LC of Dawson and
Stewart, written out here as its two arrays: the CT keeps the LC's
list in its left part, so after every mark the two lists must be equal.  The LC
itself is pinned by the paper's worked example.  The sampler over
the CT's list is pinned by Eq. (1) (chi-square), independent of list order.
"""
import itertools

import numpy as np
import pytest
from scipy.stats import chisquare

import oracle
from paper_2003_11902_b200.instances import make_coords

SEED = 42
P_MIN = 1e-3


class _LC:
    """Tabu with list compression: unvisited[0..L), indices[v]."""

    def __init__(self, n):
        self.unvisited = list(range(n))
        self.indices = list(range(n))
        self.L = n

    def mark(self, v):
        # "the visited node is replaced by the last one"; the worked
        # example (indices 7, 6, 5) shows v itself moving to L-1, i.e. a swap
        i, last = self.indices[v], self.L - 1
        t = self.unvisited[last]
        self.unvisited[i], self.unvisited[last] = t, v
        self.indices[t], self.indices[v] = i, last
        self.L -= 1

    def is_visited(self, u):
        return self.indices[u] >= self.L


def test_lc_worked_example():
    # after removing 2, 5, 7 from nodes 0..7 their indices are 7, 6, 5,
    # and n-1-index recovers the visiting order 0, 1, 2
    lc = _LC(8)
    for v in (2, 5, 7):
        lc.mark(v)
    assert [lc.indices[v] for v in (2, 5, 7)] == [7, 6, 5]
    assert [8 - 1 - lc.indices[v] for v in (2, 5, 7)] == [0, 1, 2]
    assert sorted(lc.unvisited[:lc.L]) == [0, 1, 3, 4, 6]


def test_ct_example_two_five_seven():
    # the paper's CT figure removes 2, 5 and 7 from 0..7; the left part
    # must be the LC's list and the right part must locate every relocated node
    e, L = oracle.ct_init(8)
    assert list(e) == list(range(8)) and L == 8
    for v in (2, 5, 7):
        e, L = oracle.ct_mark(e, L, v)
    lc = _LC(8)
    for v in (2, 5, 7):
        lc.mark(v)
    assert L == 5 and list(e[:L]) == lc.unvisited[:5]
    for u in e[:L]:
        iu = u if u < L else e[u]
        assert e[iu] == u


@pytest.mark.parametrize("n,seed", [(2, 0), (3, 1), (8, 2), (37, 3), (200, 4)])
def test_ct_equals_lc_under_random_marks(n, seed):
    rng = np.random.default_rng(seed)
    e, L = oracle.ct_init(n)
    lc = _LC(n)
    visited = set()
    for v in rng.permutation(n):
        e, L = oracle.ct_mark(e, L, int(v))
        lc.mark(int(v))
        visited.add(int(v))
        assert L == n - len(visited) == lc.L
        # the left part is exactly the LC's list (same order), i.e. the unvisited set
        assert list(e[:L]) == lc.unvisited[:L]
        assert set(e[:L].tolist()) == set(range(n)) - visited
        # an unvisited u < L sits at its initial position; an unvisited
        # u >= L was relocated and entries[u] is its index
        for u in range(n):
            if u in visited:
                continue
            iu = u if u < L else e[u]
            assert iu < L and e[iu] == u


def _ct_after(n, marks):
    e, L = oracle.ct_init(n)
    for v in marks:
        e, L = oracle.ct_mark(e, L, v)
    return e, L


def _draw_ct(inv, e, L, s, n_draws):
    counts = {}
    for t in range(n_draws):
        a, it = t % 4096, t // 4096
        c = oracle.select_next_ct(inv, e, L, s, a, it, SEED)
        counts[c] = counts.get(c, 0) + 1
    return counts


def test_ct_sampler_follows_eq1_in_scrambled_list_order():
    # Eq. (1): P(v) = w_v / sum_l w_l over the unvisited set, whatever the
    # order in which the list enumerates it (A-Res: order is arbitrary)
    rng = np.random.default_rng(11)
    n = 12
    w = rng.uniform(0.1, 1.0, size=n)
    inv = (1.0 / w).astype(np.float32)
    e, L = _ct_after(n, [3, 0, 11, 7])          # list order is now scrambled
    assert list(e[:L]) != sorted(e[:L])
    w_eff = 1.0 / inv.astype(np.float64)
    live = sorted(int(v) for v in e[:L])
    probs = {v: w_eff[v] / w_eff[live].sum() for v in live}
    cnt = _draw_ct(inv, e, L, s=4, n_draws=60000)
    assert set(cnt) <= set(live)
    keys = sorted(probs)
    obs = np.array([cnt.get(k, 0) for k in keys], float)
    assert chisquare(obs, np.array([probs[k] for k in keys]) * obs.sum()).pvalue > P_MIN


def test_ct_sampler_single_element_and_equal_weights():
    # a list of one node returns it (Q28); equal weights -> uniform over the list
    n = 9
    inv = np.ones(n, dtype=np.float32)
    e, L = _ct_after(n, [0, 1, 2, 3, 4, 5, 6, 8])
    assert L == 1 and oracle.select_next_ct(inv, e, L, 8, 0, 0, SEED) == 7
    e, L = _ct_after(n, [4, 0])
    cnt = _draw_ct(inv, e, L, s=2, n_draws=28000)
    keys = sorted(int(v) for v in e[:L])
    obs = np.array([cnt.get(k, 0) for k in keys], float)
    assert sum(cnt.values()) == obs.sum()
    assert chisquare(obs).pvalue > P_MIN


def test_ct_keys_use_the_enumeration_index():
    # R27: the i-th list element draws counter (0x40000000 | i>>2, s, a, it) word i&3.
    # With an unscrambled list (only the last node removed) the CT enumerates the
    # cities in id order, so the step equals the bitmask scan's step exactly.
    n = 23
    rng = np.random.default_rng(5)
    inv = rng.uniform(0.5, 4.0, size=n).astype(np.float32)
    e, L = _ct_after(n, [n - 1])
    assert list(e[:L]) == list(range(n - 1))
    vis = [0] * n
    vis[n - 1] = 1
    for a in range(200):
        c_ct = oracle.select_next_ct(inv, e, L, 1, a, 3, SEED)
        c_bt, fb = oracle.select_next(inv, None, vis, 1, a, 3, SEED)
        assert c_ct == c_bt and fb == 0


def test_ct_colony_routes_and_optimum():
    c = make_coords("uniform", 8, 99)
    best = min(oracle.tour_length(c, (0,) + p) for p in itertools.permutations(range(1, 8)))
    col = oracle.Colony(c, 8, 0, seed=3, tabu=1)
    col.iterate(60)
    gb, gl = col.best_tour()
    assert gl == best and oracle.tour_length(c, gb) == gl
    c = make_coords("uniform", 150, 4)
    col = oracle.Colony(c, 40, 0, seed=9, tabu=1)
    col.iterate(2)
    for r, L in zip(col.tours(), col.lengths()):
        assert sorted(r) == list(range(150)) and L == oracle.tour_length(c, r)


def test_ct_alpha_beta_zero_first_step_uniform():
    c = make_coords("uniform", 6, 5)
    counts = np.zeros((6, 6))
    col = oracle.Colony(c, 3000, 0, alpha=0.0, beta=0.0, seed=11, tabu=1)
    col.iterate(1)
    for r in col.tours():
        counts[r[0], r[1]] += 1
    obs = np.array([counts[i, j] for i in range(6) for j in range(6) if i != j])
    rows = np.array([counts[i].sum() / 5 for i in range(6) for j in range(6) if i != j])
    assert chisquare(obs, rows).pvalue > 1e-3


def test_ct_requires_full_row():
    c = make_coords("uniform", 10, 1)
    with pytest.raises(ValueError):
        oracle.Colony(c, 5, 3, tabu=1)
    with pytest.raises(ValueError):
        oracle.Colony(c, 5, 0, tabu=2)
