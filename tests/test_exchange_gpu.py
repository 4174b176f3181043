"""The peer-memory exchange (row a7 without a collective library, include/mmas.h):
shards publish their best record straight into every rank's device buffer and wait on
device flags.  Checked against the CPU oracle's unsharded colony (Alg. 1 select_shortest,
P:278-285, R21), bit for bit on every replica: in one process (buffers attached by
pointer, every shard's construction enqueued before any update) and across two processes
on one GPU (CUDA IPC handles, concurrent device-side waits)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
from paper_2003_11902_b200 import mmas
from paper_2003_11902_b200.instances import make_coords

from test_parity_gpu import compare_shards

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world,m,cl", [(2, 40, 16), (3, 43, 0), (4, 3, 8)])
def test_in_process_peer_exchange_equals_oracle(world, m, cl):
    c = make_coords("uniform", 150, 17)
    s = torch.cuda.current_stream().cuda_stream
    ref = oracle.Colony(c, m, cl, seed=8)
    shards = [mmas.Colony(c, m, cl, seed=8, stream=s, rank=r, world=world) for r in range(world)]
    bufs = [sh.exchange_buffer() for sh in shards]
    for sh in shards:
        sh.exchange_attach(bufs)
    for it in range(5):
        ref.iterate(1)
        for sh in shards:
            sh.construct_publish()
        for sh in shards:
            sh.update_exchange()
        compare_shards(shards, ref, it)
    for sh in shards:
        sh.exchange_status()


@pytest.mark.parametrize("world,m,cl,kw", [(2, 40, 16, {}), (3, 43, 8, {}), (2, 30, 8, {"deposit_global": True})])
def test_in_process_fused_exchange_iteration_equals_oracle(world, m, cl, kw):
    """mmas_iterate_exchange as ONE launch per iteration (construct.cuh
    exchange_select_block: the grid's last block publishes, waits on the device flags and
    selects; then the fused update).  The shards run on their own streams so their
    launches overlap on the one GPU (each grid is a few small blocks), as they would on
    separate GPUs."""
    c = make_coords("uniform", 150, 19)
    ref = oracle.Colony(c, m, cl, seed=6, **kw)
    streams = [torch.cuda.Stream() for _ in range(world)]
    shards = [mmas.Colony(c, m, cl, seed=6, stream=streams[r].cuda_stream, rank=r, world=world, **kw)
              for r in range(world)]
    assert all(sh.stats()["update_fused"] == 1 for sh in shards)
    bufs = [sh.exchange_buffer() for sh in shards]
    for sh in shards:
        sh.exchange_attach(bufs)
    for it in range(4):
        ref.iterate(1)
        for sh in shards:
            sh.iterate_exchange(1)
        for sh in shards:
            sh.sync()
            sh.exchange_status()
        compare_shards(shards, ref, it)


def _free_port():
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    p = sk.getsockname()[1]
    sk.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2003_11902_b200.parallel import PeerShardedColony
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        col = PeerShardedColony(make_coords("uniform", 120, 5), 30, 16, seed=3)
        col.iterate(4)
        col.colony.exchange_status()
        gb, gl = col.best_tour()
        q.put((rank, col.colony.tours(), col.colony.lengths(), col.colony.tau(), col.colony.inv_w(),
               col.colony.limits(), gb, gl))
        dist.barrier()
        col.close()
    finally:
        dist.destroy_process_group()


def test_two_processes_ipc_peer_exchange_equals_oracle():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref = oracle.Colony(make_coords("uniform", 120, 5), 30, 16, seed=3)
    ref.iterate(4)
    assert np.array_equal(np.concatenate([o[1] for o in out]), ref.tours())
    assert np.array_equal(np.concatenate([o[2] for o in out]), ref.lengths())
    ob, ol = ref.best_tour()
    for o in out:
        assert np.array_equal(o[3], ref.tau()) and np.array_equal(o[4], ref.inv_w())
        assert o[5] == ref.limits() and o[7] == ol and np.array_equal(o[6], ob)
