"""Pins of the oracle's node selection (WRS / A-Res with a reservoir of one,
P:920-961, Alg. 3, log key P:1042-1049) against Eq. (1):
the chosen node must be distributed as w_j / sum_l w_l over the unvisited set.
"""
import itertools

import numpy as np
import pytest
from scipy.stats import chisquare

import oracle

SEED = 42
P_MIN = 1e-3  # significance used by SPEC.md S:281


def _draw(inv_row, cand, visited, s, n_draws, fallback_argmax=0):
    counts = {}
    for t in range(n_draws):
        a, it = t % 4096, t // 4096
        c, _ = oracle.select_next(inv_row, cand, visited, s, a, it, SEED, fallback_argmax)
        counts[c] = counts.get(c, 0) + 1
    return counts


def _chi(counts, probs):
    keys = sorted(probs)
    obs = np.array([counts.get(k, 0) for k in keys], dtype=float)
    assert sum(counts.values()) == obs.sum(), f"selected a node outside the support: {counts}"
    exp = np.array([probs[k] for k in keys]) * obs.sum()
    return chisquare(obs, exp).pvalue


@pytest.mark.parametrize("use_cl", [False, True])
def test_two_nodes_weights_1_3(use_cl):
    # weights (1, 3) -> P(second) = 0.75
    inv = np.array([1.0, 1.0, 1.0 / 3.0], dtype=np.float32)   # node 0 = current (visited)
    vis = [1, 0, 0]
    cand = [1, 2] if use_cl else None
    cnt = _draw(inv, cand, vis, s=1, n_draws=40000)
    assert _chi(cnt, {1: 0.25, 2: 0.75}) > P_MIN
    assert abs(cnt[2] / 40000 - 0.75) < 0.01


@pytest.mark.parametrize("use_cl", [False, True])
def test_weights_1_1_2_4(use_cl):
    # SPEC.md S:241/S:251 style vector: P = w / 8
    w = np.array([1.0, 1.0, 2.0, 4.0])
    inv = np.concatenate([[1.0], 1.0 / w]).astype(np.float32)
    vis = [1, 0, 0, 0, 0]
    cand = [1, 2, 3, 4] if use_cl else None
    cnt = _draw(inv, cand, vis, s=3, n_draws=40000)
    assert _chi(cnt, {j + 1: w[j] / w.sum() for j in range(4)}) > P_MIN


def test_sixteen_weights_both_domains():
    # any weight vector of length <= 16 passes chi-square at 1e-3
    rng = np.random.default_rng(7)
    w = rng.uniform(0.05, 1.0, size=16)
    inv = np.concatenate([[1.0], (1.0 / w)]).astype(np.float32)
    w_eff = 1.0 / inv[1:].astype(np.float64)        # the sampler sees 1/inv_w exactly
    probs = {j + 1: w_eff[j] / w_eff.sum() for j in range(16)}
    vis = [1] + [0] * 16
    for cand in (None, list(range(1, 17))):
        cnt = _draw(inv, cand, vis, s=5, n_draws=60000)
        assert _chi(cnt, probs) > P_MIN


def test_uniform_when_weights_equal():
    # all choice_info equal -> uniform over unvisited nodes
    n = 9
    inv = np.ones(n, dtype=np.float32)
    vis = [0] * n
    vis[0] = vis[4] = 1
    cnt = _draw(inv, None, vis, s=2, n_draws=28000)
    assert _chi(cnt, {j: 1 / 7 for j in range(n) if not vis[j]}) > P_MIN


def test_route_distribution_matches_eq1_product():
    """Whole construction chain on 4 nodes from node 0: P(route) is the product of
    Eq. (1) probabilities over its steps.  Pins the per-step freshness of the
    random keys (counter includes the step) and that visited nodes are excluded."""
    W = np.array([[0, 1, 2, 4], [1, 0, 8, 1], [2, 8, 0, 4], [4, 1, 4, 0]], dtype=np.float64)
    inv = np.where(W > 0, 1.0 / np.where(W > 0, W, 1), 1.0).astype(np.float32)
    probs = {}
    for perm in itertools.permutations([1, 2, 3]):
        p, cur, left = 1.0, 0, {1, 2, 3}
        for nxt in perm:
            p *= W[cur, nxt] / sum(W[cur, l] for l in left)
            left.remove(nxt)
            cur = nxt
        probs[perm] = p
    for use_cl in (False, True):
        counts = {}
        for t in range(30000):
            a, it = t % 4096, t // 4096
            vis = [1, 0, 0, 0]
            cur, route = 0, []
            for s in (1, 2, 3):
                cand = [j for j in range(4) if j != cur] if use_cl else None
                nxt, fb = oracle.select_next(inv[cur], cand, vis, s, a, it, SEED)
                assert vis[nxt] == 0
                vis[nxt] = 1
                route.append(nxt)
                cur = nxt
            counts[tuple(route)] = counts.get(tuple(route), 0) + 1
        assert _chi(counts, probs) > P_MIN


def test_candidate_fallback_to_all_unvisited():
    # R9: all candidates visited -> WRS over every unvisited node (north_star)
    n = 8
    w = np.array([1, 1, 1, 1, 1, 2, 3, 4], dtype=np.float64)
    inv = (1.0 / w).astype(np.float32)
    vis = [1, 1, 1, 1, 0, 0, 0, 0]
    cand = [1, 2, 3]
    cnt = {}
    for t in range(20000):
        c, fb = oracle.select_next(inv, cand, vis, 9, t % 4096, t // 4096, SEED)
        assert fb == 1
        cnt[c] = cnt.get(c, 0) + 1
    tot = w[4:].sum()
    assert _chi(cnt, {j: w[j] / tot for j in range(4, 8)}) > P_MIN


def test_argmax_fallback_flag():
    # candidates all visited, two unvisited with weights 0.1 / 0.9 -> the 0.9 node
    inv = np.array([1.0, 1.0, 1 / 0.1, 1 / 0.9], dtype=np.float32)
    c, fb = oracle.select_next(inv, [1], [1, 1, 0, 0], 2, 0, 0, SEED, fallback_argmax=1)
    assert (c, fb) == (3, 1)
    inv2 = np.array([1.0, 1.0, 1 / 0.9, 1 / 0.1], dtype=np.float32)
    c, fb = oracle.select_next(inv2, [1], [1, 1, 0, 0], 2, 0, 0, SEED, fallback_argmax=1)
    assert (c, fb) == (2, 1)


def _equalising_weight(L1, x, L2):
    """y with fl32(L2*y) == fl32(L1*x), searched around x*L1/L2."""
    target = np.float32(L1) * np.float32(x)
    y = np.float32(float(target) / float(L2))
    for _ in range(200):
        v = np.float32(L2) * y
        if v == target:
            return y
        y = np.nextafter(y, np.float32(np.inf) if v > target else np.float32(-np.inf))
    return None


@pytest.mark.parametrize("use_cl", [False, True])
def test_equal_keys_go_to_lowest_node_id(use_cl):
    """R16: the maximum key wins, ties -> lowest city id, regardless of scan order."""
    found = 0
    s, it = 6, 3
    for a in range(200):
        n = 4
        # the u each node would draw at this step (computed from the RNG contract R13)
        us = {}
        for c in (1, 3):
            if use_cl:
                k = [3, 1].index(c)         # candidate slot of c in cand row [3, 1]
                x = oracle.philox([k, s >> 2, a, it], [SEED, 0])[s & 3]
            else:
                x = oracle.philox([0x40000000 | (c >> 2), s, a, it], [SEED, 0])[c & 3]
            us[c] = oracle.det_log2(oracle.uniform(int(x)))
        y = _equalising_weight(us[3], np.float32(1.0), us[1])
        if y is None:
            continue
        inv = np.array([1.0, y, 1e30, 1.0], dtype=np.float32)
        vis = [1, 0, 1, 0]
        c, _ = oracle.select_next(inv, [3, 1] if use_cl else None, vis, s, a, it, SEED)
        assert c == 1
        found += 1
    assert found > 50
