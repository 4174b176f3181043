"""GPU parity of the full-row path over the compact tabu (MMAS-WRS-CT, SURVEY
NEXT-2, R27): construct_ct_kernel through the C ABI against the
oracle's CT, bit-exact, at ragged small sizes and at C4's full size (sampled)."""
import numpy as np
import pytest

import oracle
from paper_2003_11902_b200 import mmas
from paper_2003_11902_b200.instances import CONFIGS, make_coords

from test_parity_gpu import lockstep

pytestmark = pytest.mark.gpu
CT = mmas.TABU_COMPACT

CT_CASES = [
    # (n, m, iterations, kwargs) -- list lengths around the 128/256-position trips
    (3, 1, 3, {}),
    (3, 4, 3, {}),
    (4, 3, 3, {}),
    (5, 7, 4, {}),
    (33, 33, 3, {}),
    (128, 9, 3, {}),
    (129, 9, 3, {}),
    (255, 10, 2, {}),
    (256, 11, 2, {}),
    (257, 12, 2, {}),
    (300, 300, 2, {}),                      # many ants: several warps and blocks
    (513, 40, 2, {}),
    (97, 50, 3, {"deposit_global": True}),
    (64, 20, 3, {"alpha": 2.0, "beta": 3.0}),
    (64, 20, 3, {"alpha": 0.0, "beta": 0.0}),   # equal weights: ties broken by node id only via keys
    (90, 25, 3, {"rho": 0.9, "p_best": 0.05}),
    (1025, 12, 2, {}),
    (2100, 6, 1, {}),
]


@pytest.mark.parametrize("n,m,iters,kw", CT_CASES, ids=[f"n{c[0]}-m{c[1]}-{'-'.join(c[3])}" for c in CT_CASES])
def test_ct_small_cases_bit_exact(n, m, iters, kw):
    lockstep(make_coords("uniform", n, 5000 + n), m, 0, iters, seed=13 + n, tabu=CT, **kw)


def test_ct_clustered_bit_exact():
    lockstep(make_coords("fl3795", 400, 6), 50, 0, 3, seed=3, tabu=CT)


def test_ct_with_two_opt_bit_exact():
    lockstep(make_coords("uniform", 260, 77), 30, 0, 2, seed=5, tabu=CT, local_search=True, rho=0.7)


def test_ct_and_bitmask_differ_but_both_valid():
    # R27: same distribution, different draws -> different tours, both permutations
    c = make_coords("uniform", 200, 3)
    a = mmas.Colony(c, 40, 0, seed=1, tabu=CT)
    b = mmas.Colony(c, 40, 0, seed=1)
    a.iterate(1)
    b.iterate(1)
    Ta, Tb = a.tours(), b.tours()
    assert not np.array_equal(Ta, Tb)
    assert np.all(Ta[:, 0] == Tb[:, 0])          # the start city draw is shared (R13)
    for T in (Ta, Tb):
        assert np.all(np.sort(T, axis=1) == np.arange(200))


def test_ct_c4_full_size_sampled_ants():
    """C4 (pr2392-shaped, full row, 2392 ants) with the compact tabu, in the launch
    configuration bench.py uses for --tabu compact: sampled ants vs the oracle."""
    w = CONFIGS["C4"]
    c = w.coords()
    g = mmas.Colony(c, w.n_ants, 0, seed=w.mmas_seed, rho=w.rho, tabu=CT)
    o = oracle.Colony(c, w.n_ants, 0, seed=w.mmas_seed, rho=w.rho, nthreads=8, tabu=CT)
    g.iterate(1)
    T, L = g.tours(), g.lengths()
    rng = np.random.default_rng(1)
    for a in sorted(set([0, w.n_ants - 1] + list(rng.integers(0, w.n_ants, size=4)))):
        r, l, _ = o.construct_ant(int(a))
        assert np.array_equal(T[a], r), f"ant {a}"
        assert L[a] == l
    assert np.all(np.sort(T, axis=1) == np.arange(w.n))
    gb, gl = g.best_tour()
    assert gl == L.min() and oracle.tour_length(c, gb) == gl


def test_ct_sharded_identical_to_single():
    import torch
    c = make_coords("uniform", 150, 12)
    m, world = 29, 3
    s = torch.cuda.current_stream().cuda_stream
    ref = mmas.Colony(c, m, 0, seed=4, tabu=CT)
    shards = [mmas.Colony(c, m, 0, seed=4, stream=s, rank=r, world=world, tabu=CT) for r in range(world)]
    rb = shards[0].record_bytes
    recs = torch.zeros(world * rb, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        ref.iterate(1)
        for r, sh in enumerate(shards):
            sh.construct(recs.data_ptr() + r * rb)
        for sh in shards:
            sh.update(recs.data_ptr(), world)
        assert np.array_equal(np.concatenate([sh.tours() for sh in shards]), ref.tours())
        for sh in shards:
            assert np.array_equal(sh.tau(), ref.tau())


def test_ct_global_best_resume_and_padding_sizes():
    """Deposit of the global best, resume identity, and list lengths that end exactly on /
    just past the 512-position unrolled trip pair."""
    c = make_coords("uniform", 120, 8)
    lockstep(c, 25, 0, 3, seed=3, tabu=CT, deposit_global=True)
    a = mmas.Colony(c, 25, 0, seed=5, tabu=CT)
    b = mmas.Colony(c, 25, 0, seed=5, tabu=CT)
    a.iterate(1)
    a.iterate(2)
    b.iterate(3)
    assert np.array_equal(a.tours(), b.tours()) and np.array_equal(a.tau(), b.tau())
    for n in (512, 513, 769):
        lockstep(make_coords("uniform", n, 90 + n), 6, 0, 1, seed=n, tabu=CT)
