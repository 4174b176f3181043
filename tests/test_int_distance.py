"""The integer EUC_2D path (kernels.cuh euc2d_int: the 2-opt kernels, the NN tour, the lean fallback scans) against the R12 formula.

For integral coordinates with |x|, |y| <= 16383 the kernels compute nint(sqrt(S)),
S = dx^2 + dy^2 < 2^31, as an approximate fp32 sqrt rounded to the nearest integer k0 plus
one integer correction (k^2 + k < S -> k + 1; k^2 - k >= S -> k - 1).  This checks, on the
CPU, that the correction reproduces (int)(sqrt((double)S) + 0.5) -- the oracle's and the
double kernels' formula (R12) -- even when the approximate sqrt is off by several
ulp: exhaustively for S <= 2^22, on random S < 2^31, and at every S next to a half-integer
root (k^2 + k and k^2 + k + 1) up to the largest k."""
import numpy as np


def _nint_double(S):
    return (np.sqrt(S.astype(np.float64)) + 0.5).astype(np.int64)


def _nint_int(S, ulps):
    """euc2d_int's arithmetic with the fp32 sqrt perturbed by `ulps` ulps."""
    r = np.sqrt(S.astype(np.float32))
    for _ in range(abs(ulps)):
        r = np.nextafter(r, np.float32(np.inf) if ulps > 0 else np.float32(-np.inf))
    k = np.rint(r).astype(np.int64)          # __float2int_rn
    S = S.astype(np.int64)
    kk = k * k
    up = kk + k < S
    down = (~up) & (k > 0) & (kk - k >= S)
    return k + up - down


def _check(S):
    want = _nint_double(S)
    for ulps in (-4, -1, 0, 1, 4):
        got = _nint_int(S, ulps)
        bad = np.nonzero(got != want)[0]
        assert bad.size == 0, (ulps, S[bad[:5]], got[bad[:5]], want[bad[:5]])


def test_exhaustive_small_squares():
    _check(np.arange(0, (1 << 22) + 1, dtype=np.int64))


def test_random_large_squares():
    rng = np.random.default_rng(3)
    _check(rng.integers(0, 2 * 32766 ** 2 + 1, size=2_000_000, dtype=np.int64))


def test_next_to_half_integer_roots():
    k = np.arange(1, 46341, dtype=np.int64)
    S = np.concatenate([k * k + k, k * k + k + 1, k * k - k, k * k - k + 1, k * k])
    _check(S[(S >= 0) & (S <= 2 * 32766 ** 2)])


def test_extreme_coordinates_fit_32_bits():
    dx = dy = 2 * 16383
    assert dx * dx + dy * dy < 2 ** 31
