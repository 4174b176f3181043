"""Pins of the oracle's 2-opt local search (row a8, R25)."""
import itertools

import numpy as np
import pytest

import oracle
from paper_2003_11902_b200.instances import make_coords


def _cycle_key(route):
    """Canonical form of an undirected cycle (rotation and orientation free)."""
    r = list(route)
    i = r.index(0)
    fwd = r[i:] + r[:i]
    bwd = [fwd[0]] + fwd[1:][::-1]
    return tuple(min(fwd, bwd))


def test_reverse_examples():
    # route [0,1,2,3,4], reverse positions 1..3 -> [0,3,2,1,4] (the same cycle;
    # R25 physically reverses the complement when it is strictly shorter)
    r, pos = oracle.reverse([0, 1, 2, 3, 4], 1, 3)
    assert _cycle_key(r) == _cycle_key([0, 3, 2, 1, 4])
    assert list(r) == [4, 1, 2, 3, 0]
    # inner segment shorter -> reversed in place
    r, pos = oracle.reverse([0, 1, 2, 3, 4, 5], 1, 2)
    assert list(r) == [0, 2, 1, 3, 4, 5]
    # equal halves -> the inner segment (tie rule)
    r, pos = oracle.reverse([0, 1, 2, 3], 1, 2)
    assert list(r) == [0, 2, 1, 3]
    # segment wrapping around the end of the array
    r, pos = oracle.reverse([0, 1, 2, 3, 4, 5, 6], 6, 0)
    assert list(r) == [6, 1, 2, 3, 4, 5, 0]
    assert all(pos[r[k]] == k for k in range(7))


def test_pos_invariant_under_random_reversals():
    rng = np.random.default_rng(0)
    n = 37
    r = rng.permutation(n).astype(np.int32)
    for _ in range(1000):
        i, j = rng.integers(0, n, size=2)
        before = _cycle_key(r)
        r2, pos = oracle.reverse(r, int(i), int(j))
        assert sorted(r2) == list(range(n))
        assert all(pos[r2[k]] == k for k in range(n))
        r = r2


def test_crossing_quadrilateral_is_uncrossed():
    # SPEC.md S:513 (convex quadrilateral visited in crossing order) and S:532 (unit-square gain)
    c = np.array([[0, 0], [100, 0], [100, 100], [0, 100]], dtype=np.float64)
    r, d, moves = oracle.two_opt(c, [0, 2, 1, 3])
    assert _cycle_key(r) == _cycle_key([0, 1, 2, 3])
    assert d == 400 - oracle.tour_length(c, [0, 2, 1, 3]) and d < 0 and moves == 1


def test_optimal_tour_is_a_fixed_point():
    c = np.array([[0, 0], [100, 0], [100, 100], [0, 100]], dtype=np.float64)
    r, d, moves = oracle.two_opt(c, [0, 1, 2, 3])
    assert list(r) == [0, 1, 2, 3] and d == 0 and moves == 0


def _no_improving_restricted_move(c, route, K):
    """Full rescan (all nodes, both directions, neighbour-restricted, Bentley-pruned)."""
    n = len(route)
    nn = oracle.cand_lists(c, min(K, n - 1))
    pos = {v: i for i, v in enumerate(route)}
    D = lambda i, j: oracle.dist(c, i, j)
    for a in range(n):
        for dirn in (1, -1):
            b = route[(pos[a] + dirn) % n]
            for cc in nn[a]:
                if D(a, cc) >= D(a, b):
                    break
                d = route[(pos[cc] + dirn) % n]
                if cc == b or d == a:
                    continue
                if D(a, cc) + D(b, d) - D(a, b) - D(cc, d) < 0:
                    return False
    return True


@pytest.mark.parametrize("n,seed", [(7, 1), (9, 2), (10, 3)])
def test_brute_force_bounds_and_local_optimality(n, seed):
    # input >= output >= optimum; output 2-opt-optimal (restricted moves)
    c = make_coords("uniform", n, 500 + seed)
    best = min(oracle.tour_length(c, (0,) + p) for p in itertools.permutations(range(1, n)))
    rng = np.random.default_rng(seed)
    for _ in range(20):
        r0 = rng.permutation(n)
        r, d, _ = oracle.two_opt(c, r0)
        L0, L1 = oracle.tour_length(c, r0), oracle.tour_length(c, r)
        assert sorted(r) == list(range(n))
        assert L1 == L0 + d and best <= L1 <= L0
        assert _no_improving_restricted_move(c, list(r), 32)


def test_local_optimality_on_larger_instance():
    c = make_coords("uniform", 200, 77)
    r0 = np.random.default_rng(5).permutation(200)
    r, d, moves = oracle.two_opt(c, r0)
    assert moves > 50 and d < 0
    assert oracle.tour_length(c, r) == oracle.tour_length(c, r0) + d
    assert _no_improving_restricted_move(c, list(r), 32)


def test_colony_with_local_search_beats_without():
    # Sec. 5.7: LS does the "fine-grained exploitation"; same iterations, better best tour
    c = make_coords("uniform", 120, 9)
    a = oracle.Colony(c, 40, 16, seed=3, local_search=True)
    b = oracle.Colony(c, 40, 16, seed=3, local_search=False)
    a.iterate(5)
    b.iterate(5)
    assert a.best_tour()[1] < b.best_tour()[1]
    for r in a.tours():
        assert _no_improving_restricted_move(c, list(r), 32)
