"""GPU parity of the lane-compacted fallback (row a3, R9; construct.cuh fallback_compact).

When every candidate of the current city is visited, Alg. 3 draws a key for
every unvisited city and takes the largest.  Late in a tour each lane of the ant's warp
evaluates only the unvisited cities of its own tabu bits; the trip scans over the whole row
remain for fallbacks with more than `cap` unvisited cities.  Both must give
the oracle's choice bit for bit on every kernel variant: MMAS_FB_COMPACT forces the cap
(0: trip scans only; >= n: the compacted scan for every fallback; small: a mix within one
tour)."""
import pytest

from paper_2003_11902_b200.instances import make_coords

from test_parity_gpu import lockstep

pytestmark = pytest.mark.gpu

# (label, coords recipe, n, ants, cl, iterations, extra env)
KERNELS = [
    ("smem-table-regtabu", "uniform", 1002, 64, 8, 3, {}),      # C2's kernel (n <= 1024)
    ("smem-table-ragged", "uniform", 67, 40, 5, 4, {}),
    ("smem-table-smemtabu", "uniform", 1025, 40, 8, 2, {}),     # 33 tabu words
    ("l2-table", "fl3795", 1500, 40, 32, 2, {}),                # table beyond shared memory
    ("l2-table-staged-coop", "fl3795", 1300, 40, 4, 2, {"MMAS_FB_ROW": "1"}),   # C5's paired path
]
CAPS = [("trip-only", lambda n: 0), ("compact-always", lambda n: n), ("mixed", lambda n: n // 3)]


@pytest.mark.parametrize("cap_name,cap", CAPS, ids=[c[0] for c in CAPS])
@pytest.mark.parametrize("label,recipe,n,m,cl,iters,env", KERNELS, ids=[k[0] for k in KERNELS])
def test_compacted_fallback_bit_exact(label, recipe, n, m, cl, iters, env, cap_name, cap, monkeypatch):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    monkeypatch.setenv("MMAS_FB_COMPACT", str(cap(n)))
    c = make_coords(recipe, n, 900 + n)
    g, o = lockstep(c, m, cl, iters, seed=31 + n)
    st = g.stats()
    assert st["fallback_steps"] > 0
    assert st["fallback_lane_cap"] == cap(n)


def test_compacted_fallback_pruned_l2_kernel(monkeypatch):
    """The 16-warps-per-SM L2-table kernel (pruned trip scans otherwise): 2400 ants, cl = 4,
    most steps fall back; the compacted scan at the steps with at most 400 unvisited cities."""
    monkeypatch.setenv("MMAS_FB_COMPACT", "400")
    c = make_coords("fl3795", 1300, 21)
    g, o = lockstep(c, 2400, 4, 1, seed=13)
    assert g.stats()["fallback_steps"] > 100000
    assert g.stats()["fallback_lane_cap"] == 400


def test_compacted_fallback_colonies(monkeypatch):
    """Concurrent colonies (grid.y) take the compacted scan with their own colony's rows."""
    import oracle
    from paper_2003_11902_b200 import mmas
    from test_parity_gpu import compare_iteration
    monkeypatch.setenv("MMAS_FB_COMPACT", "40")
    c = make_coords("uniform", 130, 77)
    g = mmas.Colony(c, 40, 6, seed=5, colonies=3)
    os_ = [oracle.Colony(c, 40, 6, seed=5 + k) for k in range(3)]
    for it in range(3):
        g.iterate(1)
        for k, o in enumerate(os_):
            o.iterate(1)
            g.select_colony(k)
            compare_iteration(g, o, f"{it} (colony {k})")
    assert g.stats()["fallback_lane_cap"] == 40


def test_default_cap_is_set_for_c2():
    """bench.py's C2 launch (pr1002-shaped, cl 32): the compacted scan is on with the default
    cap (224 unvisited cities: register tabu, L2-resident rows); off for C1 (one-trip rows)."""
    from paper_2003_11902_b200 import mmas
    from paper_2003_11902_b200.instances import CONFIGS
    w = CONFIGS["C2"]
    g = mmas.Colony(w.coords(), w.n_ants, w.cand_len, rho=w.rho, seed=w.mmas_seed)
    assert g.stats()["fallback_lane_cap"] == 224
    w = CONFIGS["C1"]
    g = mmas.Colony(w.coords(), w.n_ants, w.cand_len, rho=w.rho, seed=w.mmas_seed)
    assert g.stats()["fallback_lane_cap"] == 0


@pytest.mark.parametrize("cap_name,cap", CAPS, ids=[c[0] for c in CAPS])
@pytest.mark.parametrize("n,m", [(300, 40), (1100, 16)], ids=["regtabu", "smemtabu"])
def test_full_row_compacted_steps_bit_exact(n, m, cap_name, cap, monkeypatch):
    """Full-row construction (cl = 0, construct_full_kernel): the last steps of a tour take the
    compacted scan (default n / 10 unvisited cities); every variant against the oracle."""
    monkeypatch.setenv("MMAS_FB_COMPACT", str(cap(n)))
    c = make_coords("uniform", n, 1300 + n)
    g, o = lockstep(c, m, 0, 2, seed=5 + n)
    assert g.stats()["fallback_lane_cap"] == cap(n)
