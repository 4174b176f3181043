"""Checkpoint / resume: a colony saved after k iterations and loaded into a
fresh context with the same coordinates and configuration continues exactly as the saved
one would have -- every route, length, the limits, the global best, tau and inv_w -- and
both equal the CPU oracle run straight through (the random numbers are counter-based, R13,
so the device state and the iteration counter are the whole state)."""
import numpy as np
import pytest

import oracle
from paper_2003_11902_b200 import mmas
from paper_2003_11902_b200.instances import CONFIGS, make_coords

from test_parity_gpu import compare_iteration

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,m,cl,kw", [
    (198, 60, 16, {}),                                        # fused one-launch iteration
    (150, 30, 16, {"separate_update": True}),
    (120, 20, 0, {"tabu": mmas.TABU_COMPACT}),
    (150, 12, 16, {"local_search": True, "rho": 0.7}),
    (130, 40, 8, {"pheromone": mmas.PHEROMONE_LEAN}),
    (1500, 20, 32, {}),                                       # L2 table
], ids=["fused", "separate", "ct", "two-opt", "lean", "l2-table"])
def test_resume_equals_uninterrupted_and_oracle(n, m, cl, kw):
    c = make_coords("uniform", n, 900 + n)
    a = mmas.Colony(c, m, cl, seed=21, **kw)
    a.iterate(4)
    state = a.save_state()
    b = mmas.Colony(c, m, cl, seed=21, **kw)
    b.load_state(state)
    assert b.iteration == 4
    okw = {k: v for k, v in kw.items() if k not in ("separate_update", "pheromone")}
    o = oracle.Colony(c, m, cl, seed=21, **okw)
    o.iterate(4)
    compare_iteration(b, o, "restored")
    for it in range(4, 8):
        a.iterate(1)
        b.iterate(1)
        o.iterate(1)
        compare_iteration(b, o, it)
        assert np.array_equal(a.tours(), b.tours())


def test_resume_colonies():
    w = CONFIGS["C1"]
    c = w.coords()
    a = mmas.Colony(c, 64, w.cand_len, seed=3, colonies=3)
    a.iterate(3)
    b = mmas.Colony(c, 64, w.cand_len, seed=3, colonies=3)
    b.load_state(a.save_state())
    a.iterate(2)
    b.iterate(2)
    for col in range(3):
        a.select_colony(col)
        b.select_colony(col)
        assert np.array_equal(a.tours(), b.tours()) and np.array_equal(a.tau(), b.tau())
        assert a.best_tour()[1] == b.best_tour()[1]


def test_checkpoint_of_another_configuration_is_rejected():
    c = make_coords("uniform", 120, 5)
    a = mmas.Colony(c, 30, 16, seed=1)
    a.iterate(2)
    st = a.save_state()
    for kw in ({"seed": 2}, {"rho": 0.7}, {"n_ants": 31}):
        args = dict(seed=1)
        m = kw.pop("n_ants", 30)
        args.update(kw)
        b = mmas.Colony(c, m, 16, **args)
        with pytest.raises(mmas.MMASError):
            b.load_state(st)
    with pytest.raises(mmas.MMASError):
        mmas.Colony(c, 30, 16, seed=1).load_state(st[:100])
