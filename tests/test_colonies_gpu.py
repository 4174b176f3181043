"""Concurrent independent colonies (R29): a context with k
colonies runs k complete MMAS colonies in every launch (grid.y = colony).  Colony c must be
bit-identical to the CPU oracle's single colony seeded seed + c -- every route, length,
the limits, the global best, tau and inv_w -- on every launch path (fused one-launch
iteration, separate update, L2 table, full row, compact tabu, 2-opt, roulette wheel)."""
import numpy as np
import pytest

import oracle
from paper_2003_11902_b200 import mmas
from paper_2003_11902_b200.instances import CONFIGS, make_coords

from test_parity_gpu import compare_iteration

pytestmark = pytest.mark.gpu


def lockstep_colonies(coords, m, cl, k, iters, seed=5, **kw):
    g = mmas.Colony(coords, m, cl, seed=seed, colonies=k, **kw)
    assert g.colonies == k
    okw = dict(kw)
    okw.pop("separate_update", None)
    os_ = [oracle.Colony(coords, m, cl, seed=seed + c, **okw) for c in range(k)]
    for it in range(iters):
        g.iterate(1)
        for c, o in enumerate(os_):
            o.iterate(1)
            g.select_colony(c)
            compare_iteration(g, o, f"{it} (colony {c})")
    return g, os_


CASES = [
    # (n, m, cl, colonies, iterations, kwargs)
    (130, 40, 16, 3, 3, {}),                                  # fused one-launch iteration
    (130, 40, 16, 3, 3, {"separate_update": True}),
    (97, 30, 8, 2, 3, {"deposit_global": True}),
    (1500, 20, 32, 2, 2, {}),                                 # candidate table beyond smem: L2 table
    (120, 20, 0, 3, 2, {}),                                   # full row, bitmask tabu
    (120, 20, 0, 2, 2, {"tabu": mmas.TABU_COMPACT}),
    (150, 12, 16, 2, 2, {"local_search": True, "rho": 0.7}),  # 2-opt
    (130, 20, 16, 2, 2, {"selection": mmas.SELECT_RWM}),
    (5, 7, 1, 4, 3, {}),                                      # n <= 5 clamp
    (200, 300, 32, 20, 2, {}),                                # 20 colonies: 7 SMs each, several ants per warp
]


@pytest.mark.parametrize("n,m,cl,k,iters,kw", CASES,
                         ids=[f"n{c[0]}-m{c[1]}-cl{c[2]}-k{c[3]}-{'-'.join(c[5])}" for c in CASES])
def test_colonies_equal_independent_oracle_runs(n, m, cl, k, iters, kw):
    lockstep_colonies(make_coords("uniform", n, 700 + n), m, cl, k, iters, **kw)


def test_c2x8_full_size_bit_exact():
    """The C2x8 bench workload in its launch configuration: 8 pr1002-shaped colonies of 1002
    ants, 6 iterations, every colony against its own oracle run."""
    w = CONFIGS["C2x8"]
    g, _ = lockstep_colonies(w.coords(), w.n_ants, w.cand_len, w.colonies, 6, seed=w.mmas_seed, rho=w.rho)
    assert g.stats()["update_fused"] == 1


def test_colony_zero_equals_single_colony_context():
    c = make_coords("uniform", 140, 9)
    a = mmas.Colony(c, 30, 16, seed=11)
    b = mmas.Colony(c, 30, 16, seed=11, colonies=4)
    a.iterate(3)
    b.iterate(3)
    b.select_colony(0)
    assert np.array_equal(a.tours(), b.tours()) and np.array_equal(a.tau(), b.tau())
    assert a.best_tour()[1] == b.best_tour()[1]
    with pytest.raises(mmas.MMASError):
        b.select_colony(4)
    with pytest.raises(mmas.MMASError):
        mmas.Colony(c, 30, 16, colonies=2, rank=0, world=2)
