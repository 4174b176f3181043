"""Pins of the oracle's random-number contract (R13, R14) against
things other than the oracle itself: the Random123 known-answer vectors, the
exact u-grid, libm/numpy log2 over every value the uniform map can produce.
"""
import os

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _kat_rows():
    rows = []
    with open(os.path.join(GOLDEN, "philox4x32_10_kat.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            v = [int(t, 16) for t in line.split()]
            rows.append((v[0:4], v[4:6], v[6:10]))
    return rows


@pytest.mark.parametrize("ctr,key,expect", _kat_rows())
def test_philox_known_answers(ctr, key, expect):
    assert list(oracle.philox(ctr, key)) == expect


def test_uniform_grid_is_exact_and_open():
    # u = (2*(x>>9)+1) 2^-24: the extremes and a mid value, computed from the definition
    assert oracle.uniform(0) == 2.0 ** -24
    assert oracle.uniform(0xFFFFFFFF) == 1.0 - 2.0 ** -24
    assert oracle.uniform(0x1FF) == 2.0 ** -24          # low 9 bits are dropped
    assert oracle.uniform(0x80000000) == (2 * (1 << 22) + 1) * 2.0 ** -24
    rng = np.random.default_rng(1)
    for x in rng.integers(0, 2 ** 32, size=2000, dtype=np.uint64):
        u = oracle.uniform(int(x))
        assert 0.0 < u < 1.0
        k = u * 2 ** 24
        assert k == int(k) and int(k) % 2 == 1


def test_det_log2_exhaustive_against_libm():
    """Every u the uniform map can produce (2^23 values): det_log2 within 2 ulp of
    log2 in double, strictly negative, and non-decreasing in u (A-Res keys,
    P:1042-1049, must be a monotone transform of r)."""
    j = np.arange(1 << 23, dtype=np.float64)
    u64 = (2.0 * j + 1.0) / 2.0 ** 24
    u = u64.astype(np.float32)
    assert np.all(u.astype(np.float64) == u64)
    got = oracle.det_log2_many(u).astype(np.float64)
    ref = np.log2(u64)
    ulp = np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64)
    err = np.abs(got - ref) / ulp
    assert err.max() <= 2.0, err.max()
    assert np.all(got < 0.0)
    assert np.all(np.diff(got) >= 0.0)


def test_det_log2_powers_of_two_exact():
    for e in range(-24, 0):
        assert oracle.det_log2(2.0 ** e) == float(e)
    # SPEC.md S:267-268 (golden/spec_worked_examples.txt wrs_key_w1/w2): key = (1/w) log2 r
    import ctypes
    k1 = np.float32(oracle.det_log2(0.5)) * np.float32(1.0 / 1.0)
    k2 = np.float32(oracle.det_log2(0.5)) * np.float32(1.0 / 2.0)
    assert k1 == -1.0 and k2 == -0.5
    # S:269 monotone in w at fixed r = 0.25
    L = np.float32(oracle.det_log2(0.25))
    assert L * np.float32(1 / 4) > L * np.float32(1 / 2) > L * np.float32(1 / 1)


def test_start_node_uniform():
    """Alg. 1: u ~ U{0, n-1}; chi-square over (ant, iteration) pairs."""
    from scipy.stats import chisquare
    n = 7
    seed = 42
    counts = np.zeros(n)
    for it in range(40):
        for a in range(1000):
            counts[oracle.start_node(n, a, it, seed)] += 1
    assert chisquare(counts).pvalue > 1e-3


def _f32_round_up(x):
    """float64 array -> the smallest float32 >= x (x finite, positive)."""
    f = x.astype(np.float32)
    low = f.astype(np.float64) < x
    f[low] = np.nextafter(f[low], np.float32(np.inf))
    return f


def test_scaled_pruning_threshold_never_prunes_a_tie_or_winner():
    """The GPU scans compare a = fl(fl(1-u) inv) with T = fl_up(thr * K), K = fl_up(1/C)
    (construct.cuh warp_threshold), pruning when a > T.  Safe iff a city whose magnitude
    mag = fl(|det_log2(u)| inv) is <= thr is never pruned; T is monotone in thr, so the
    worst case is thr = mag: a <= fl_up(mag * K) must hold for every u of the grid (all
    2^23, exhaustive) and every inv (a spread of 64 magnitudes per u block)."""
    C = np.float32(1.4426935911178589)
    K = np.float32(0.6931478977203369)
    assert float(K) >= 1.0 / float(C)
    j = np.arange(1 << 23, dtype=np.float64)
    u = ((2.0 * j + 1.0) / 2.0 ** 24).astype(np.float32)
    om = np.float32(1.0) - u
    D = np.abs(oracle.det_log2_many(u))
    rng = np.random.default_rng(1)
    for inv in (10.0 ** rng.uniform(-3, 12, size=64)).astype(np.float32):
        mag = (D * inv).astype(np.float32)                      # fl(|det_log2(u)| inv)
        a = (om * inv).astype(np.float32)                       # fl(fl(1-u) inv)
        T = _f32_round_up(mag.astype(np.float64) * float(K))    # fl_up(mag K)
        assert np.all(a <= T), float(inv)


def test_pruning_lower_bound_holds_on_the_whole_grid():
    """The exact key pruning of the GPU scans skips det_log2
    when lb = fl(fl(1-u) * fl(inv * C)) > thr, C = log2(e)(1 - 2^-20) rounded down.  That is
    safe iff lb <= fl(|det_log2(u)| * inv) for every u of the grid and every inv; with each
    fp32 rounding bounded by 2^-24 it suffices that |det_log2(u)| / ((1-u) C) >=
    (1 + 2^-24)^2 / (1 - 2^-24).  Checked exhaustively on all 2^23 uniforms (the bound
    follows from -ln u >= 1 - u and det_log2's 1.61-ulp accuracy)."""
    C = np.float32(1.4426935911178589)
    assert float(C) <= np.log2(np.e) * (1 - 2.0 ** -20)
    j = np.arange(1 << 23, dtype=np.float64)
    u = ((2.0 * j + 1.0) / 2.0 ** 24).astype(np.float32)
    D = np.abs(oracle.det_log2_many(u).astype(np.float64))
    one_minus_u = (np.float32(1.0) - u).astype(np.float64)      # exact on the grid
    assert np.all(one_minus_u == 1.0 - u.astype(np.float64))
    ratio = D / (one_minus_u * float(C))
    assert ratio.min() >= (1 + 2.0 ** -24) ** 2 / (1 - 2.0 ** -24)
    # and directly in fp32 for a spread of inv_w values (the GPU's exact operation order)
    rng = np.random.default_rng(0)
    sub = rng.choice(1 << 23, size=200000, replace=False)
    inv = (10.0 ** rng.uniform(-3, 12, size=sub.size)).astype(np.float32)
    lb = (np.float32(1.0) - u[sub]) * (inv * C)
    mag = np.abs(oracle.det_log2_many(u[sub]) * inv)
    assert np.all(lb <= mag)
