"""Small runs of every launch path for compute-sanitizer:

    compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} python tools/sanitize_runs.py MODE

MODE: fused (one launch per iteration: construction + grid barrier + update), separate (the
two-kernel path), exchange (two shards in one process on their own streams, the fused
peer-exchange launch), split (two shards, construct_publish / update_exchange), full (cl = 0
bitmask + compact tabu), ls (2-opt), rwm (roulette wheel), compact (the lane-compacted fallback
scan on three kernel variants).  d198-shaped C1 colony (smaller
for the slow tools), 2 iterations; results compared with the oracle, so a run that the tool
perturbs still has to be right."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (test infrastructure: checks the sanitised run)
from paper_2003_11902_b200 import mmas  # noqa: E402
from paper_2003_11902_b200.instances import CONFIGS, make_coords  # noqa: E402


def check(shards, o, what):
    ot = o.tours()
    for sh in shards:
        f, c = sh.shard()
        assert np.array_equal(sh.tours(), ot[f:f + c]), what
        assert np.array_equal(sh.tau(), o.tau()), what
    print(what, "ok")


def main(mode):
    import torch
    w = CONFIGS["C1"]
    c = w.coords()
    m, cl = 64, w.cand_len
    if mode in ("fused", "separate"):
        g = mmas.Colony(c, m, cl, seed=3, separate_update=(mode == "separate"))
        assert g.stats()["update_fused"] == (mode == "fused")
        o = oracle.Colony(c, m, cl, seed=3)
        for it in range(2):
            g.iterate(1)
            o.iterate(1)
            check([g], o, f"{mode} iteration {it}")
        g.status()
    elif mode in ("exchange", "split"):
        streams = [torch.cuda.Stream() for _ in range(2)]
        sh = [mmas.Colony(c, m, cl, seed=3, rank=r, world=2, stream=streams[r].cuda_stream) for r in range(2)]
        bufs = [s.exchange_buffer() for s in sh]
        for s in sh:
            s.exchange_attach(bufs)
        o = oracle.Colony(c, m, cl, seed=3)
        for it in range(2):
            o.iterate(1)
            if mode == "exchange":
                for s in sh:
                    s.iterate_exchange(1)
            else:
                for s in sh:
                    s.construct_publish()
                for s in sh:
                    s.update_exchange()
            for s in sh:
                s.sync()
            check(sh, o, f"{mode} iteration {it}")
        for s in sh:
            s.status()
    elif mode == "full":
        cc = make_coords("uniform", 150, 3)
        for tabu in (mmas.TABU_BITMASK, mmas.TABU_COMPACT):
            g = mmas.Colony(cc, 32, 0, seed=3, tabu=tabu)
            o = oracle.Colony(cc, 32, 0, seed=3, tabu=tabu)
            for it in range(2):
                g.iterate(1)
                o.iterate(1)
                check([g], o, f"full tabu={tabu} iteration {it}")
    elif mode == "ls":
        cc = make_coords("uniform", 150, 4)
        g = mmas.Colony(cc, 16, 16, seed=3, local_search=True, rho=0.7)
        o = oracle.Colony(cc, 16, 16, seed=3, local_search=True, rho=0.7)
        for it in range(2):
            g.iterate(1)
            o.iterate(1)
            check([g], o, f"2-opt iteration {it}")
    elif mode == "compact":
        # the lane-compacted fallback scan on the register-tabu, shared-memory-tabu and
        # L2-table kernels (forced for every fallback); the NN tour and list kernels run in
        # every mode's setup
        os.environ["MMAS_FB_COMPACT"] = "4096"
        for n, mm, cl in ((700, 24, 6), (1100, 16, 6), (1500, 16, 32)):
            cc = make_coords("fl3795", n, 7)
            g = mmas.Colony(cc, mm, cl, seed=3)
            o = oracle.Colony(cc, mm, cl, seed=3)
            assert g.stats()["fallback_lane_cap"] == 4096
            for it in range(2):
                g.iterate(1)
                o.iterate(1)
                check([g], o, f"compact n={n} iteration {it}")
    elif mode == "rwm":
        g = mmas.Colony(c, 32, cl, seed=3, selection=mmas.SELECT_RWM)
        o = oracle.Colony(c, 32, cl, seed=3, selection=1)
        for it in range(2):
            g.iterate(1)
            o.iterate(1)
            check([g], o, f"rwm iteration {it}")
    else:
        raise SystemExit(f"unknown mode {mode}")


if __name__ == "__main__":
    main(sys.argv[1])
