"""Pins of the oracle's parallel roulette wheel (PRWM, Sec. 4.2.1 P:885-915,
DESIGN.md R28).

With small-integer weights every sum, prefix and difference PRWM forms is exact
in fp32, so PRWM must pick exactly what the textbook sequential roulette wheel
(first item whose running sum exceeds r = u * total) picks -- computed here in
exact rational arithmetic, independent of chunking and scan order.  With real
weights the choice must follow Eq. (1) (chi-square)."""
import itertools
from fractions import Fraction

import numpy as np
import pytest
from scipy.stats import chisquare

import oracle
from paper_2003_11902_b200.instances import make_coords


def _textbook_rwm(w, u):
    """Sequential RWM: r = fl32(u * total); first i with cumsum > r."""
    total = int(sum(w))
    if total == 0:
        return -1
    r = Fraction(float(np.float32(u) * np.float32(total)))
    acc = 0
    for i, x in enumerate(w):
        acc += int(x)
        if acc > r:
            return i
    raise AssertionError("r >= total")


@pytest.mark.parametrize("n", [1, 2, 5, 31, 32, 33, 64, 100, 1002, 1025, 2392])
def test_prwm_equals_sequential_rwm_on_integer_weights(n):
    rng = np.random.default_rng(n)
    w = rng.integers(0, 6, size=n).astype(np.float32)      # zeros = visited nodes
    w[rng.integers(0, n)] = 3.0                            # at least one positive weight
    us = np.concatenate([rng.random(300), [0.0, 1e-7, 0.5, 1 - 2 ** -24]]).astype(np.float32)
    for u in us:
        got = oracle.prwm(w, float(u))
        assert got == _textbook_rwm(w, u), f"n={n} u={u!r}"
        assert w[got] > 0


def test_prwm_every_boundary_of_a_small_wheel():
    # weights 1, 0, 2, 4 (total 7): r crosses each cumulative boundary 1, 3, 7 exactly
    w = np.array([1, 0, 2, 4], dtype=np.float32)
    for k in range(7 * 16):
        u = np.float32(k / (7 * 16))
        assert oracle.prwm(w, float(u)) == _textbook_rwm(w, u)
    assert oracle.prwm(w, 0.0) == 0
    assert oracle.prwm(w, float(np.float32(1 / 7))) == 2       # r = 1 is not > 1: next positive item


def test_prwm_degenerate_inputs():
    assert oracle.prwm(np.zeros(40, np.float32), 0.3) == -1
    w = np.zeros(3000, np.float32)
    w[2999] = 0.25
    assert all(oracle.prwm(w, u) == 2999 for u in (0.0, 0.4, 1 - 2 ** -24))
    assert oracle.prwm(np.array([5.0], np.float32), 0.9) == 0


@pytest.mark.parametrize("n", [17, 700])
def test_prwm_follows_eq1(n):
    rng = np.random.default_rng(3 + n)
    w = rng.uniform(0.05, 1.0, size=n).astype(np.float32)
    w[rng.random(n) < 0.3] = 0.0
    draws = 40000
    us = (np.arange(draws) + 0.5) / draws                   # stratified u: exact quantiles
    counts = np.bincount([oracle.prwm(w, float(u)) for u in us], minlength=n)
    live = w > 0
    assert counts[~live].sum() == 0
    w64 = w[live].astype(np.float64)
    exp = w64 / w64.sum() * draws
    exp *= counts[live].sum() / exp.sum()
    # stratified sampling is much tighter than multinomial; chi-square is conservative
    assert chisquare(counts[live], exp).pvalue > 0.999


def test_rwm_colony_optimum_and_permutations():
    c = make_coords("uniform", 8, 99)
    best = min(oracle.tour_length(c, (0,) + p) for p in itertools.permutations(range(1, 8)))
    for cl, tabu in ((0, 0), (3, 0), (0, 1)):
        col = oracle.Colony(c, 8, cl, seed=3, selection=1, tabu=tabu)
        col.iterate(60)
        gb, gl = col.best_tour()
        assert gl == best and oracle.tour_length(c, gb) == gl
    c = make_coords("uniform", 120, 4)
    col = oracle.Colony(c, 30, 8, seed=9, selection=1)
    col.iterate(2)
    for r, L in zip(col.tours(), col.lengths()):
        assert sorted(r) == list(range(120)) and L == oracle.tour_length(c, r)


def test_rwm_alpha_beta_zero_first_step_uniform():
    c = make_coords("uniform", 6, 5)
    counts = np.zeros((6, 6))
    col = oracle.Colony(c, 3000, 0, alpha=0.0, beta=0.0, seed=11, selection=1)
    col.iterate(1)
    for r in col.tours():
        counts[r[0], r[1]] += 1
    obs = np.array([counts[i, j] for i in range(6) for j in range(6) if i != j])
    rows = np.array([counts[i].sum() / 5 for i in range(6) for j in range(6) if i != j])
    assert chisquare(obs, rows).pvalue > 1e-3


def test_rwm_with_candidate_lists_falls_back():
    c = make_coords("d198", 198, 198)
    col = oracle.Colony(c, 60, 2, seed=3, selection=1)
    col.iterate(1)
    assert col.fallbacks().sum() > 0


def test_rejects_bad_selection():
    with pytest.raises(ValueError):
        oracle.Colony(make_coords("uniform", 10, 1), 5, 3, selection=2)


def _hillis_steele(s):
    """The inclusive scan of R28 (pre[t] += pre[t-d], d = 1, 2, 4, 8, 16) in fp32 -- used
    here only to certify that the input below is adversarial, not to compute a result."""
    p = s.astype(np.float32).copy()
    d = 1
    while d < 32:
        q = p.copy()
        q[d:] = p[d:] + p[:-d]
        p, d = q, 2 * d
    return p


def _adversarial_zero_chunk():
    """32 one-item chunks, item 4 of weight 0 (a visited node), whose scanned prefix
    rounds one ulp ABOVE its predecessor's, and a u whose r = fl(u * total) lands exactly
    on the predecessor's prefix: the rule 'first t with pre[t] > r' alone picks item 4."""
    rng = np.random.default_rng(0)
    for _ in range(100000):
        w = rng.random(32).astype(np.float32)
        w[4] = np.float32(0.0)
        p = _hillis_steele(w)
        if not p[4] > p[3]:
            continue
        total = p[31]
        u0 = np.float32(p[3] / total)
        for k in range(-64, 65):
            u = u0
            for _ in range(abs(k)):
                u = np.nextafter(u, np.float32(2.0 if k > 0 else -1.0), dtype=np.float32)
            if np.float32(u * total) == p[3]:
                return w, u, p
    raise AssertionError("no adversarial input found")


def test_prwm_zero_sum_chunk_never_wins():
    """Eq. (1): a visited node (weight 0) has probability 0.  With the
    Hillis-Steele association (R28) a zero-sum chunk's prefix can round above its
    predecessor's; r on that predecessor's prefix must still not select the zero chunk
    (this input fails under the rule without the positive-sum test of commit c5400dc)."""
    w, u, p = _adversarial_zero_chunk()
    assert p[4] > p[3] and w[4] == 0.0                  # the input is adversarial:
    r = np.float32(u * p[31])
    assert next(t for t in range(32) if p[t] > r) == 4   # the prefix rule alone picks item 4
    got = oracle.prwm(w, float(u))
    assert got != 4 and w[got] > 0
    assert got == 5                                      # the next item whose prefix exceeds r
    # chunked over 64 items (chunk size 2, both items of chunk 4 visited): same story
    w2 = np.repeat(w, 2) / np.float32(2.0)
    w2[8:10] = 0.0
    p2 = _hillis_steele(np.add.reduceat(w2, np.arange(0, 64, 2)))
    if p2[4] > p2[3]:
        got2 = oracle.prwm(w2, float(u))
        assert w2[got2] > 0
