"""The bound the memory-lean pheromone rests on (R30), checked on the oracle's dense
colony: a trail never deposited on equals the background (every diagonal entry is one), and
at any iteration a row holds at most 2 (L + 1) off-candidate trails different from it,
L = ceil(ln F / ln rho) + 2 with F = tau_min / tau_max (each iteration deposits on at most
two edges of a row, and a deposit-free trail reaches tau_min in L steps)."""
import math

import numpy as np
import pytest

import oracle
from paper_2003_11902_b200.instances import make_coords


@pytest.mark.parametrize("n,m,cl,rho,iters", [(120, 30, 8, 0.5, 60), (90, 20, 4, 0.9, 80), (60, 15, 6, 0.2, 40)])
def test_sparse_rows_are_bounded(n, m, cl, rho, iters):
    c = make_coords("uniform", n, 3 * n)
    o = oracle.Colony(c, m, cl, seed=1, rho=rho, nthreads=4)
    tmin, tmax = o.limits()
    F = min(1.0, tmin / tmax)
    L = 1 if F >= 1 else math.ceil(math.log(F * (1 - 1e-5)) / math.log(float(np.float32(rho)) * (1 + 1e-6))) + 2
    cand = o.cand()
    peak = 0
    for _ in range(iters):
        o.iterate(1)
        tau = o.tau()
        bg = np.diag(tau)
        assert np.all(bg == bg[0])                      # the background is one scalar
        off = tau != bg[0]
        off[np.arange(n)[:, None], cand] = False        # candidate trails are stored densely
        rows = off.sum(axis=1)
        peak = max(peak, int(rows.max()))
        assert rows.max() <= 2 * (L + 1)
    assert peak > 0                                      # the sparse rows are exercised
