"""GPU parity of the parallel roulette wheel construction (PRWM, Sec. 4.2.1,
SURVEY NEXT-1, R28): construct_rwm_kernel through the C ABI against
the oracle, bit-exact (the fp32 chunk sums, Hillis-Steele scan, r = u*total and
the chunk descent are the same operations in the same order on both sides)."""
import numpy as np
import pytest

import oracle
from paper_2003_11902_b200 import mmas
from paper_2003_11902_b200.instances import CONFIGS, make_coords

from test_parity_gpu import lockstep

pytestmark = pytest.mark.gpu
RWM, CT = mmas.SELECT_RWM, mmas.TABU_COMPACT

RWM_CASES = [
    # (n, m, cl, iterations, kwargs)
    (3, 2, 0, 3, {}),
    (4, 3, 1, 3, {}),
    (5, 7, 0, 3, {"tabu": CT}),
    (33, 20, 0, 3, {}),
    (33, 20, 0, 3, {"tabu": CT}),
    (100, 30, 5, 3, {}),
    (130, 40, 16, 3, {}),
    (130, 40, 32, 3, {}),
    (200, 25, 40, 2, {}),                     # 2 candidates per lane in the first stage
    (150, 20, 100, 2, {}),
    (97, 50, 8, 3, {"deposit_global": True}),
    (64, 20, 10, 3, {"alpha": 2.0, "beta": 3.0}),
    (64, 20, 0, 3, {"alpha": 0.0, "beta": 0.0}),
    (1025, 10, 0, 2, {}),                     # 3 stages: chunk 33, then 2, then 1
    (1025, 10, 32, 2, {}),
    (2100, 6, 0, 1, {"tabu": CT}),
]


@pytest.mark.parametrize("n,m,cl,iters,kw", RWM_CASES,
                         ids=[f"n{c[0]}-m{c[1]}-cl{c[2]}-{'-'.join(c[4])}" for c in RWM_CASES])
def test_rwm_small_cases_bit_exact(n, m, cl, iters, kw):
    lockstep(make_coords("uniform", n, 7000 + n), m, cl, iters, seed=17 + n, selection=RWM, **kw)


def test_rwm_fallbacks_counted_and_bit_exact():
    c = make_coords("d198", 198, 198)
    g, o = lockstep(c, 60, 3, 3, seed=3, selection=RWM)
    assert g.stats()["fallback_steps"] > 0


def test_rwm_with_two_opt_bit_exact():
    lockstep(make_coords("uniform", 220, 5), 20, 16, 2, seed=8, selection=RWM, local_search=True, rho=0.7)


@pytest.mark.parametrize("cfg,kw", [("C2", {}), ("C4", {"tabu": CT})])
def test_rwm_full_size_sampled_ants(cfg, kw):
    """pr1002-shaped with cl 32 (the paper's MMAS-RWM-BT with CL) and pr2392-shaped
    full row over the CT (MMAS-RWM-CT) at full size: sampled ants vs the oracle."""
    w = CONFIGS[cfg]
    c = w.coords()
    g = mmas.Colony(c, w.n_ants, w.cand_len, seed=w.mmas_seed, rho=w.rho, selection=RWM, **kw)
    o = oracle.Colony(c, w.n_ants, w.cand_len, seed=w.mmas_seed, rho=w.rho, nthreads=8, selection=RWM, **kw)
    g.iterate(1)
    T, L = g.tours(), g.lengths()
    rng = np.random.default_rng(2)
    for a in sorted(set([0, w.n_ants - 1] + list(rng.integers(0, w.n_ants, size=4)))):
        r, l, _ = o.construct_ant(int(a))
        assert np.array_equal(T[a], r), f"ant {a}"
        assert L[a] == l
    assert np.all(np.sort(T, axis=1) == np.arange(w.n))


def test_rwm_sharded_identical_to_single():
    """R21 with the roulette wheel: shards with gathered records == one context."""
    import torch
    c = make_coords("uniform", 130, 21)
    m, world, cl = 37, 3, 12
    s = torch.cuda.current_stream().cuda_stream
    ref = mmas.Colony(c, m, cl, seed=6, selection=RWM)
    shards = [mmas.Colony(c, m, cl, seed=6, stream=s, rank=r, world=world, selection=RWM) for r in range(world)]
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


def test_rwm_global_best_deposit_and_resume():
    c = make_coords("uniform", 90, 31)
    lockstep(c, 20, 0, 3, seed=2, selection=RWM, tabu=CT, deposit_global=True)
    a = mmas.Colony(c, 20, 8, seed=4, selection=RWM)
    b = mmas.Colony(c, 20, 8, seed=4, selection=RWM)
    a.iterate(2)
    a.iterate(2)
    b.iterate(4)
    assert np.array_equal(a.tours(), b.tours()) and np.array_equal(a.tau(), b.tau())
