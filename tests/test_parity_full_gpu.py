"""Full-size parity (SURVEY.md Sec. 8(d) "oracle parity iterations"): every config at
BASELINE.json's sizes, in the launch configuration bench.py times, compared with the CPU
oracle element by element over whole iterations of Alg. 1 -- every ant's
route, every length, the limits, the global best and the full tau / inv_w matrices.

  C2  the bench workload: iterations 0-29 (the driver's 5 warm-up + 20 timed steps and
      more) every iteration, then both sides on to iteration 400 with a full comparison
      every 50 iterations (the steady-state regime of the 1000-iteration run)
  C3  5 iterations (clustered, cl 32 + fallbacks)
  C4  3 iterations (full row, bitmask tabu) and 3 with the compact tabu (NEXT-2)
  C5  2 iterations (cl 32 + 2-opt, n = 18512: three 1.37 GB matrices per side)
"""
import gc

import numpy as np
import pytest

import oracle
from paper_2003_11902_b200 import mmas
from paper_2003_11902_b200.instances import CONFIGS

from test_parity_gpu import compare_iteration, compare_setup

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    assert torch.cuda.is_available(), "-m gpu tests need a CUDA device"
    mmas.lib()


def _pair(cfg, **kw):
    w = CONFIGS[cfg]
    c = w.coords()
    args = dict(seed=w.mmas_seed, rho=w.rho, **kw)
    g = mmas.Colony(c, w.n_ants, w.cand_len, **args)
    o = oracle.Colony(c, w.n_ants, w.cand_len, **args)
    return w, g, o


def test_c2_driver_window_and_steady_state():
    w, g, o = _pair("C2")
    assert g.stats()["update_fused"] == 1           # bench.py's launch configuration
    compare_setup(g, o)
    for it in range(30):
        g.iterate(1)
        o.iterate(1)
        compare_iteration(g, o, it)
    fb_window = g.stats()["fallback_steps"]
    assert fb_window > 0                            # the driver's window has fallbacks
    for it in range(30, 400, 10):
        g.iterate(10)
        o.iterate(10)
        if (it + 10) % 50 == 0:
            compare_iteration(g, o, it + 9)
    assert g.iteration == o.iteration == 400


@pytest.mark.parametrize("cfg,iters,kw", [("C3", 5, {}), ("C4", 3, {}),
                                          ("C4", 3, {"tabu": mmas.TABU_COMPACT})],
                         ids=["C3", "C4", "C4CT"])
def test_full_size_lockstep(cfg, iters, kw):
    w, g, o = _pair(cfg, **kw)
    compare_setup(g, o)
    for it in range(iters):
        g.iterate(1)
        o.iterate(1)
        compare_iteration(g, o, it)
    if cfg == "C3":
        assert g.stats()["fallback_steps"] > 0


def test_c5_two_iterations_with_two_opt():
    """d18512-shaped, cl 32 + 2-opt, 800 ants: both full iterations (construction, 2-opt
    of every route, best, update) compared with the oracle.  The n^2 matrices are
    compared one at a time to bound host memory (~6 GB peak)."""
    w, g, o = _pair("C5", local_search=True)
    assert g.limits() == o.limits()
    assert np.array_equal(g.cand(), o.cand())
    for it in range(2):
        g.iterate(1)
        o.iterate(1)
        gt, ot = g.tours(), o.tours()
        bad = np.where((gt != ot).any(axis=1))[0]
        assert len(bad) == 0, f"iteration {it}: {len(bad)} routes differ (first ant {bad[:1]})"
        del gt, ot
        assert np.array_equal(g.lengths(), o.lengths())
        assert g.limits() == o.limits()
        gb, gl = g.best_tour()
        ob, ol = o.best_tour()
        assert gl == ol and np.array_equal(gb, ob)
        for fn in ("tau", "inv_w"):
            a, b = getattr(g, fn)(), getattr(o, fn)()
            assert np.array_equal(a, b), f"iteration {it}: {fn}"
            del a, b
            gc.collect()
    assert g.stats()["local_search_moves"] > 0
