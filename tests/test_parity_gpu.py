"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element
by element on the same seeded inputs.  Tours, lengths, candidate lists and
limits must be bit-exact; pheromone / inv_w are compared bit-exactly too (the
north_star tolerance is 1e-6 relative; the contract makes them exact)."""
import numpy as np
import pytest

import oracle
from paper_2003_11902_b200 import mmas
from paper_2003_11902_b200.instances import CONFIGS, make_coords

pytestmark = pytest.mark.gpu
RTOL_TAU = 1e-6   # north_star: "to 1e-6 relative for pheromone values"


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    assert torch.cuda.is_available(), "-m gpu tests need a CUDA device"
    mmas.lib()


def assert_matrix(g, o, what):
    if not np.array_equal(g, o):
        diff = np.abs(g.astype(np.float64) - o.astype(np.float64)) / np.maximum(np.abs(o.astype(np.float64)), 1e-300)
        i = np.unravel_index(np.argmax(diff), diff.shape)
        assert diff.max() <= RTOL_TAU, f"{what}: max rel diff {diff.max()} at {i}: gpu {g[i]} oracle {o[i]}"
        pytest.fail(f"{what}: not bit-exact (max rel diff {diff.max()} within tolerance, but the contract is exact)")


def compare_setup(g, o):
    assert_matrix(g.heur(), o.heur(), "heuristic")
    assert_matrix(g.inv_w(), o.inv_w(), "inv_w (setup)")
    assert_matrix(g.tau(), o.tau(), "tau (setup)")
    assert g.limits() == o.limits()
    if o.cl > 0:
        assert np.array_equal(g.cand(), o.cand())


def compare_iteration(g, o, it):
    gt, ot = g.tours(), o.tours()
    if not np.array_equal(gt, ot):
        bad = np.where((gt != ot).any(axis=1))[0]
        a = bad[0]
        k = int(np.argmax(gt[a] != ot[a]))
        pytest.fail(f"iteration {it}: {len(bad)} ants differ; ant {a} first at step {k}: gpu {gt[a][k]} oracle {ot[a][k]}")
    assert np.array_equal(g.lengths(), o.lengths()), f"iteration {it}: lengths"
    assert g.limits() == o.limits(), f"iteration {it}: limits"
    gb, gl = g.best_tour()
    ob, ol = o.best_tour()
    assert gl == ol and np.array_equal(gb, ob), f"iteration {it}: global best"
    assert_matrix(g.tau(), o.tau(), f"tau after iteration {it}")
    assert_matrix(g.inv_w(), o.inv_w(), f"inv_w after iteration {it}")


def lockstep(coords, m, cl, iters, seed=42, **kw):
    g = mmas.Colony(coords, m, cl, seed=seed, **kw)
    o = oracle.Colony(coords, m, cl, seed=seed, **kw)
    compare_setup(g, o)
    for it in range(iters):
        g.iterate(1)
        o.iterate(1)
        compare_iteration(g, o, it)
    return g, o


# ---- primitives -------------------------------------------------------------------
def test_device_philox_matches_kat_and_oracle():
    kat = [(0, 0, 0, 0, 0, 0), (0xFFFFFFFF,) * 6, (0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344, 0xA4093822, 0x299F31D0)]
    expect = [[0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8], [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD],
              [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]]
    w, _ = mmas.debug_philox(np.array(kat, dtype=np.uint32))
    assert w.tolist() == expect
    rng = np.random.default_rng(3)
    ck = rng.integers(0, 2 ** 32, size=(4000, 6), dtype=np.uint64).astype(np.uint32)
    w, logs = mmas.debug_philox(ck)
    for i in range(0, 4000, 37):
        ow = oracle.philox(ck[i, :4], ck[i, 4:])
        assert list(w[i]) == list(ow)
        for j in range(4):
            assert logs[i, j] == np.float32(oracle.det_log2(oracle.uniform(int(ow[j]))))


def test_device_det_log2_exhaustive_bitwise():
    j = np.arange(1 << 23, dtype=np.float64)
    u = ((2.0 * j + 1.0) / 2.0 ** 24).astype(np.float32)
    assert np.array_equal(mmas.debug_log2(u).view(np.uint32), oracle.det_log2_many(u).view(np.uint32))


# ---- whole iterations ---------------------------------------------------------------
def test_c1_all_50_iterations_bit_exact():
    w = CONFIGS["C1"]
    lockstep(w.coords(), w.n_ants, w.cand_len, w.iterations, seed=w.mmas_seed, rho=w.rho)


CASES = [
    # (n, m, cl, iterations, kwargs)   -- ragged sizes, edge cases, every kernel variant
    (3, 1, 0, 3, {}),
    (3, 4, 2, 3, {}),
    (4, 3, 3, 3, {}),                          # n <= 5: tau_min clamped to tau_max
    (5, 7, 1, 4, {}),
    (33, 33, 0, 3, {}),                        # full row, ragged tail of a 128-city chunk
    (67, 40, 5, 4, {}),
    (130, 70, 16, 4, {}),
    (130, 70, 32, 4, {}),
    (129, 31, 1, 3, {}),                       # cl = 1: fallback at most steps
    (200, 37, 40, 3, {}),                      # 2 slots per lane
    (150, 20, 100, 3, {}),                     # 4 slots per lane
    (97, 50, 8, 4, {"fallback_argmax": True}),
    (97, 50, 8, 4, {"deposit_global": True}),
    (64, 20, 10, 3, {"alpha": 2.0, "beta": 3.0}),
    (64, 20, 10, 3, {"alpha": 0.0, "beta": 1.0}),
    (80, 20, 12, 3, {"beta": 2.5}),            # non-integer beta: host libm pow (R18)
    (90, 25, 12, 3, {"rho": 0.9, "p_best": 0.05}),
    (1025, 12, 32, 2, {}),                     # n > 1024: 33 tabu words
    (1500, 20, 32, 2, {}),                     # candidate table > shared memory: L2 variant
    (300, 300, 0, 2, {}),                      # full row, many ants
]


@pytest.mark.parametrize("n,m,cl,iters,kw", CASES, ids=[f"n{c[0]}-m{c[1]}-cl{c[2]}-{'-'.join(c[4])}" for c in CASES])
def test_small_cases_bit_exact(n, m, cl, iters, kw):
    lockstep(make_coords("uniform", n, 1000 + n), m, cl, iters, seed=7 + n, **kw)


def test_clustered_instance_with_fallbacks():
    c = make_coords("fl3795", 600, 5)
    g, o = lockstep(c, 60, 8, 3, seed=9)
    assert g.stats()["fallback_steps"] > 0


def test_pruned_fallback_scan_bit_exact():
    """The L2-table kernel at >= 16 ant warps per SM takes the pruned (lagged-threshold)
    fallback scan (construct.cuh scan_unvisited kLagPrune): table too large for shared
    memory (n = 1300, cl padded to 32 slots), 2400 ants, cl = 4 on a clustered instance so
    most steps fall back."""
    c = make_coords("fl3795", 1300, 21)
    g, o = lockstep(c, 2400, 4, 1, seed=13)
    assert g.stats()["fallback_steps"] > 100000


@pytest.mark.parametrize("m", [40, 2400], ids=["few-warps-uncapped", "16-warps-pruned"])
def test_staged_fallback_rows_bit_exact(m, monkeypatch):
    """Fallback scans over an inv_w row staged into the block's shared memory by one TMA copy
    (construct.cuh stage_fallback_row; on by default only where inv_w is not L2-resident,
    forced here with MMAS_FB_ROW): L2-table kernel (n = 1300), cl = 4 on a clustered
    instance, both the low-occupancy (uncapped registers) and the pruned 16-warp variants."""
    monkeypatch.setenv("MMAS_FB_ROW", "1")
    c = make_coords("fl3795", 1300, 23)
    g, o = lockstep(c, m, 4, 2, seed=17)
    assert g.stats()["fallback_steps"] > 1000


def test_fallback_counter_matches_oracle():
    c = make_coords("d198", 198, 198)
    g = mmas.Colony(c, 120, 4, seed=3)
    o = oracle.Colony(c, 120, 4, seed=3)
    tot = 0
    for _ in range(3):
        g.iterate(1)
        o.iterate(1)
        tot += int(o.fallbacks().sum())
    assert tot > 0 and g.stats()["fallback_steps"] == tot


# ---- identities of the contract -----------------------------------------------------
def test_resume_identity():
    """R20: iterate(2); iterate(3) == iterate(5)."""
    c = make_coords("uniform", 150, 4)
    a = mmas.Colony(c, 40, 16, seed=5)
    b = mmas.Colony(c, 40, 16, seed=5)
    a.iterate(2)
    a.iterate(3)
    b.iterate(5)
    assert np.array_equal(a.tours(), b.tours()) and np.array_equal(a.tau(), b.tau())
    assert a.iteration == b.iteration == 5


def test_split_calls_equal_iterate():
    import torch
    c = make_coords("uniform", 120, 8)
    a = mmas.Colony(c, 30, 16, seed=2)
    s = torch.cuda.current_stream().cuda_stream
    b = mmas.Colony(c, 30, 16, seed=2, stream=s)
    rec = torch.zeros(b.record_bytes, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        a.iterate(1)
        b.construct(rec.data_ptr())
        b.update(rec.data_ptr(), 1)
    assert np.array_equal(a.tours(), b.tours()) and np.array_equal(a.tau(), b.tau())
    assert a.best_tour()[1] == b.best_tour()[1]


@pytest.mark.parametrize("world,m", [(2, 43), (3, 43), (5, 43), (4, 3)])
def test_sharded_colony_equals_oracle(world, m):
    """R21 / Alg. 1 select_shortest: ants sharded over `world` contexts (one
    GPU here; one per GPU in production) with their records gathered give the oracle's
    unsharded colony bit for bit -- every route, length, the global best, limits, tau and
    inv_w on every replica; (4, 3) leaves rank 0 without ants (its record never wins)."""
    import torch
    c = make_coords("uniform", 140, 12)
    cl = 16
    s = torch.cuda.current_stream().cuda_stream
    o = oracle.Colony(c, m, cl, seed=4)
    shards = [mmas.Colony(c, m, cl, seed=4, stream=s, rank=r, world=world) for r in range(world)]
    rb = shards[0].record_bytes
    recs = torch.zeros(world * rb, dtype=torch.uint8, device="cuda")
    for it in range(4):
        o.iterate(1)
        for r, sh in enumerate(shards):
            sh.construct(recs.data_ptr() + r * rb)
        for sh in shards:
            sh.update(recs.data_ptr(), world)
        compare_shards(shards, o, it)


def compare_shards(shards, o, it):
    """Every shard's routes/lengths against the oracle's ants of that shard; every
    replica's limits, global best, tau and inv_w against the oracle's."""
    ot, ol = o.tours(), o.lengths()
    for sh in shards:
        first, count = sh.shard()
        assert np.array_equal(sh.tours(), ot[first:first + count]), f"iteration {it}: rank {sh.rank} routes"
        assert np.array_equal(sh.lengths(), ol[first:first + count]), f"iteration {it}: rank {sh.rank} lengths"
        assert sh.limits() == o.limits(), f"iteration {it}: rank {sh.rank} limits"
        gb, gl = sh.best_tour()
        ob, obl = o.best_tour()
        assert gl == obl and np.array_equal(gb, ob), f"iteration {it}: rank {sh.rank} global best"
        assert_matrix(sh.tau(), o.tau(), f"rank {sh.rank} tau after iteration {it}")
        assert_matrix(sh.inv_w(), o.inv_w(), f"rank {sh.rank} inv_w after iteration {it}")


def test_best_tour_before_first_iteration_is_estate():
    g = mmas.Colony(make_coords("uniform", 20, 1), 5, 4)
    assert g.best_tour() == (None, None)
    with pytest.raises(mmas.MMASError):
        g.iterate(0)


def test_profiling_accumulates_phase_times():
    w = CONFIGS["C1"]
    g = mmas.Colony(w.coords(), w.n_ants, w.cand_len)
    g.profile(True)
    n0 = g.kernel_launches
    g.iterate(5)
    t = g.phase_times()
    assert g.stats()["update_fused"] == 1   # C1: the update runs inside the construction launch
    assert t["iterations"] == 5 and t["construct_ms"] > 0 and t["update_ms"] == 0
    assert g.kernel_launches - n0 == 5      # one launch per iteration: construct + select + update
    s = mmas.Colony(w.coords(), w.n_ants, w.cand_len, separate_update=True)
    s.profile(True)
    n0 = s.kernel_launches
    s.iterate(5)
    t = s.phase_times()
    assert s.stats()["update_fused"] == 0
    assert t["iterations"] == 5 and t["construct_ms"] > 0 and t["update_ms"] > 0
    assert s.kernel_launches - n0 == 10     # construct (+ fused select) and update per iteration


# ---- the update fused into the construction launch (construct.cuh fused_update) --------
FUSE_CASES = [
    # (n, m, cl, iterations, kwargs)
    (198, 198, 16, 4, {}),                     # C1 shape: one row per warp
    (600, 20, 16, 3, {}),                      # 20 warps for 600 rows: 30 rows per warp (mbarrier phases)
    (1002, 1002, 32, 3, {}),                   # the bench workload's launch configuration
    (1025, 40, 32, 2, {}),                     # n > 1024: shared-memory tabu, ragged float4 tail
    (130, 2400, 32, 2, {}),                    # 16 ant warps per block, several ants per warp
    (97, 50, 8, 3, {"deposit_global": True}),
    (97, 50, 8, 3, {"fallback_argmax": True}),
    (90, 25, 12, 3, {"rho": 0.9, "p_best": 0.05}),
    (64, 20, 10, 3, {"alpha": 2.0, "beta": 3.0}),
    (5, 7, 1, 3, {}),                          # n <= 5: tau_min clamped to tau_max
]


@pytest.mark.parametrize("n,m,cl,iters,kw", FUSE_CASES,
                         ids=[f"n{c[0]}-m{c[1]}-cl{c[2]}-{'-'.join(c[4])}" for c in FUSE_CASES])
def test_fused_update_equals_separate_kernel(n, m, cl, iters, kw):
    """One launch per iteration (grid barrier + update from TMA-prefetched rows) gives the
    separate update kernel's results bit for bit, and both the oracle's."""
    c = make_coords("uniform", n, 500 + n)
    f = mmas.Colony(c, m, cl, seed=11, **kw)
    s = mmas.Colony(c, m, cl, seed=11, separate_update=True, **kw)
    o = oracle.Colony(c, m, cl, seed=11, **kw)
    assert f.stats()["update_fused"] == 1 and s.stats()["update_fused"] == 0
    for it in range(iters):
        f.iterate(1)
        s.iterate(1)
        o.iterate(1)
        compare_iteration(f, o, it)
        assert np.array_equal(f.tau(), s.tau()) and np.array_equal(f.inv_w(), s.inv_w())
        assert np.array_equal(f.tours(), s.tours())
    assert f.iteration == s.iteration == iters


def test_fused_update_not_used_where_ineligible():
    """Local search, cl > 32, L2-table colonies and empty shards keep the separate update
    kernel (world > 1 shards with ants fuse mmas_iterate_exchange, test_exchange_gpu.py)."""
    c = make_coords("uniform", 200, 3)
    assert mmas.Colony(c, 40, 16, rank=0, world=2).stats()["update_fused"] == 1
    assert mmas.Colony(c, 3, 16, rank=0, world=4).stats()["update_fused"] == 0   # no ants on rank 0
    assert mmas.Colony(c, 10, 16, local_search=True).stats()["update_fused"] == 0
    assert mmas.Colony(c, 40, 40).stats()["update_fused"] == 0
    assert mmas.Colony(make_coords("uniform", 1500, 3), 20, 32).stats()["update_fused"] == 0


# ---- row a8: 2-opt local search ------------------------------------------------------
LS_CASES = [
    (12, 5, 4, 3),
    (60, 20, 8, 3),
    (150, 37, 16, 3),
    (300, 40, 32, 2),
    (130, 25, 0, 2),      # full-row construction + 2-opt
    (1100, 12, 32, 2),    # n > 1024 (shared-memory tabu), ragged n
]


@pytest.mark.parametrize("n,m,cl,iters", LS_CASES, ids=[f"n{c[0]}-m{c[1]}-cl{c[2]}" for c in LS_CASES])
def test_two_opt_bit_exact(n, m, cl, iters):
    lockstep(make_coords("uniform", n, 3000 + n), m, cl, iters, seed=11 + n, local_search=True, rho=0.7)


@pytest.mark.parametrize("n,m,cl,iters", [(300, 21, 32, 2), (1100, 9, 32, 2), (60, 5, 8, 3)],
                         ids=["n300-odd-ants", "n1100", "n60"])
def test_two_opt_grouped_kernel_bit_exact(n, m, cl, iters, monkeypatch):
    """The grouped 2-opt kernel (coordinates in shared memory, two ants per block, one named
    barrier per ant; opt-in with MMAS_LS_GROUP=1): lockstep with the oracle, including an odd
    ant count (one group of the last block idle)."""
    monkeypatch.setenv("MMAS_LS_GROUP", "1")
    lockstep(make_coords("uniform", n, 5000 + n), m, cl, iters, seed=9 + n, local_search=True, rho=0.7)


@pytest.mark.parametrize("n,m,cl", [(300, 20, 32), (150, 20, 16)], ids=["cl32", "cl16"])
def test_two_opt_host_built_lists_bit_exact(n, m, cl, monkeypatch):
    """The candidate and 2-opt neighbour lists (and the neighbour distances) built on the host
    (the path for rows whose distances exceed shared memory, n > ~57k; forced here with
    MMAS_HOST_CAND) equal the device-built ones: lockstep with the oracle."""
    monkeypatch.setenv("MMAS_HOST_CAND", "1")
    lockstep(make_coords("uniform", n, 4000 + n), m, cl, 2, seed=3 + n, local_search=True, rho=0.7)


@pytest.mark.parametrize("shift,scale", [(0.25, 1.0), (0.0, 3.0)], ids=["fractional", "beyond-16383"])
def test_two_opt_bit_exact_double_distance_path(shift, scale):
    """Coordinates that are not integers, or exceed |x| <= 16383, take the 2-opt kernels'
    double EUC_2D path (two_opt.cuh Pts<false>); integral ones the 32-bit path."""
    c = make_coords("uniform", 150, 77) * scale + shift
    if scale > 1:
        c[:, 0] += 20000.0
    lockstep(c, 30, 16, 2, seed=5, local_search=True, rho=0.7)


# ---- maximum size (u16 ids: n = 65535) --------------------------------------------
def test_maximum_n_properties():
    """n = 65535 (the largest n with u16 city ids; 3 x 17 GB n^2 matrices in
    HBM): one iteration with cl = 32 and fallbacks; properties that hold at any size --
    every route a permutation, lengths equal to the EUC_2D sum recomputed here, the
    global best is the shortest route, trails inside the limits."""
    n, m = 65535, 16
    c = make_coords("uniform", n, 65535)
    g = mmas.Colony(c, m, 32, seed=3)
    g.iterate(1)
    T, L = g.tours(), g.lengths()
    assert np.all(np.sort(T, axis=1) == np.arange(n))
    for a in range(m):
        p = c[T[a]]
        d = np.floor(np.sqrt(((p - np.roll(p, -1, axis=0)) ** 2).sum(axis=1)) + 0.5).astype(np.int64)
        assert L[a] == d.sum()
    gb, gl = g.best_tour()
    assert gl == L.min() and np.array_equal(gb, T[int(np.argmin(L))])
    assert g.stats()["fallback_steps"] > 0
    tmin, tmax = g.limits()
    assert tmax == np.float32(1.0 / ((1.0 - 0.5) * gl))


def test_best_length_async_matches_sync_reads():
    import torch
    c = make_coords("uniform", 100, 4)
    g = mmas.Colony(c, 20, 8, seed=2)
    buf = torch.full((6,), -7, dtype=torch.int64).pin_memory()
    g.best_length_async(buf.data_ptr())           # before the first iteration: -1
    for k in range(5):
        g.iterate(1)
        g.best_length_async(buf.data_ptr() + 8 * (k + 1))
    g.sync()
    vals = buf.numpy().tolist()
    assert vals[0] == -1
    assert vals[-1] == g.best_length() == g.best_tour()[1]
    assert all(a >= b for a, b in zip(vals[1:], vals[2:]))


# ---- setup: the NN tour (Alg. 1, R3) behind the limits ---------------------------
@pytest.mark.parametrize("n,cl", [(300, 16), (1024, 32), (1025, 8)], ids=["n300", "n1024", "n1025"])
def test_candidate_lists_block_and_warp_kernels(n, cl, monkeypatch):
    """The candidate lists (R10: the cl nearest by (d, id)) of the warp-per-row kernel (n <= 1024,
    the default) and of the block kernel (MMAS_CAND_BLOCK=1) equal the oracle's."""
    c = make_coords("uniform", n, 700 + n)
    o = oracle.Colony(c, 4, cl, seed=1)
    assert np.array_equal(mmas.Colony(c, 4, cl, seed=1).cand(), o.cand())
    monkeypatch.setenv("MMAS_CAND_BLOCK", "1")
    assert np.array_equal(mmas.Colony(c, 4, cl, seed=1).cand(), o.cand())


@pytest.mark.parametrize("block", [False, True], ids=["warp-kernel", "block-kernel"])
@pytest.mark.parametrize("n,cl,frac", [(198, 16, False), (1002, 32, False), (300, 0, False), (257, 8, True)],
                         ids=["d198", "pr1002", "no-lists", "fractional"])
def test_nn_tour_limits_equal_oracle(n, cl, frac, block, monkeypatch):
    """tau_max = 1 / ((1 - rho) L_nn): the NN tour length of the one-warp kernel (n <= 1024,
    register tabu) and of the block kernel (MMAS_NN_BLOCK=1) equal the oracle's, with the
    candidate fast path (cl > 0), without lists, and with fractional coordinates (fp64 path)."""
    if block:
        monkeypatch.setenv("MMAS_NN_BLOCK", "1")
    c = make_coords("uniform", n, 600 + n) + (0.375 if frac else 0.0)
    g = mmas.Colony(c, 8, cl, seed=1)
    o = oracle.Colony(c, 8, cl, seed=1)
    assert g.limits() == o.limits()
    assert o.nn_length == oracle.nn_tour(c)[1]
