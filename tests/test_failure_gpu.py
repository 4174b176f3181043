"""Failure paths of the device-side waits (SURVEY.md Sec. 5 "failure detection"): a rank
whose peer never publishes must not hang the GPU nor select over stale records.  With a
short spin bound (MMAS_SPIN_BOUND, cycles, read at create) the wait gives up, the context's
error word is set, mmas_device_status reports MMAS_ETIMEDOUT, and the selection + update
are skipped from then on: the trails stay those of the last complete iteration."""
import numpy as np
import pytest
import torch

from paper_2003_11902_b200 import mmas
from paper_2003_11902_b200.instances import make_coords

pytestmark = pytest.mark.gpu


def _lonely_rank(monkeypatch, m, cl):
    monkeypatch.setenv("MMAS_SPIN_BOUND", str(1 << 22))   # ~2 ms
    c = make_coords("uniform", 150, 31)
    streams = [torch.cuda.Stream() for _ in range(2)]
    sh = [mmas.Colony(c, m, cl, seed=2, rank=r, world=2, stream=streams[r].cuda_stream) for r in range(2)]
    bufs = [s.exchange_buffer() for s in sh]
    for s in sh:
        s.exchange_attach(bufs)
    return sh


@pytest.mark.parametrize("fused", [True, False], ids=["one-launch", "split"])
def test_lost_peer_times_out_and_skips_the_update(monkeypatch, fused):
    sh = _lonely_rank(monkeypatch, 40, 16)
    r0 = sh[0]
    assert r0.stats()["update_fused"] == 1
    tau0, inv0, lim0 = r0.tau(), r0.inv_w(), r0.limits()
    r0.status()                                     # healthy before
    for _ in range(2):                              # rank 1 never publishes
        if fused:
            r0.iterate_exchange(1)
        else:
            r0.construct_publish()
            r0.update_exchange()
    r0.sync()
    with pytest.raises(mmas.MMASError) as e:
        r0.status()
    assert e.value.status == mmas.MMAS_ETIMEDOUT
    with pytest.raises(mmas.MMASError):
        r0.exchange_status()
    # no selection, no update: trails, inv_w, limits untouched; no global best
    assert np.array_equal(r0.tau(), tau0) and np.array_equal(r0.inv_w(), inv0)
    assert r0.limits() == lim0
    assert r0.best_tour() == (None, None)
    sh[1].status()                                  # the idle rank saw nothing wrong


def test_healthy_contexts_report_ok():
    c = make_coords("uniform", 120, 4)
    for kw in ({}, {"separate_update": True}, {"local_search": True}):
        g = mmas.Colony(c, 20, 8, seed=1, **kw)
        g.iterate(3)
        g.status()
