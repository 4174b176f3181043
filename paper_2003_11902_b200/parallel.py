"""Ant-sharded colonies over torch.distributed (row a7).

Each rank (one process per GPU) holds a replica of tau / inv_w / candidate
tables and builds the global ants [floor(r*m/G), floor((r+1)*m/G)) (DESIGN.md
R21).  The one exchange per iteration is an all-gather of every rank's best
record (u64 key = len << 24 | global ant, then the route): after it, every rank
selects the same iteration best on the device and applies the same update, so
the replicas stay bit-identical without a broadcast or host round trip.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import mmas


def shard_range(rank: int, world: int, m: int):
    """Global ant ids built by `rank` (the same formula mmas_create_ex uses)."""
    return (rank * m) // world, ((rank + 1) * m) // world


def exchange_records(local: torch.Tensor, gathered: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather every rank's record into `gathered` (world * record bytes)."""
    dist.all_gather_into_tensor(gathered, local, group=group)
    return gathered


class ShardedColony:
    """One rank's share of a colony; call iterate() on every rank collectively."""

    def __init__(self, coords, n_ants, cand_len, group=None, **kw):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        dev = torch.cuda.current_device()
        stream = torch.cuda.current_stream(dev).cuda_stream
        self.colony = mmas.Colony(coords, n_ants, cand_len, device=dev, stream=stream,
                                  rank=self.rank, world=self.world, **kw)
        rb = self.colony.record_bytes
        self.local = torch.zeros(rb, dtype=torch.uint8, device="cuda")
        self.gathered = torch.zeros(self.world * rb, dtype=torch.uint8, device="cuda")

    def iterate(self, iters: int = 1):
        for _ in range(iters):
            self.colony.construct(self.local.data_ptr())
            exchange_records(self.local, self.gathered, self.group)
            self.colony.update(self.gathered.data_ptr(), self.world)

    def best_tour(self):
        return self.colony.best_tour()

    def close(self):
        self.colony.close()


class PeerShardedColony:
    """One rank's share of a colony whose per-iteration exchange goes through the ranks'
    device memory instead of a collective: CUDA IPC handles of every rank's exchange buffer
    are all-gathered once (torch.distributed, any backend), then each iteration is
    construct + peer publish + device-side wait + update (mmas_iterate_exchange)."""

    def __init__(self, coords, n_ants, cand_len, group=None, **kw):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        dev = torch.cuda.current_device()
        stream = torch.cuda.current_stream(dev).cuda_stream
        self.colony = mmas.Colony(coords, n_ants, cand_len, device=dev, stream=stream,
                                  rank=self.rank, world=self.world, **kw)
        mine = self.colony.exchange_ipc_handle()
        handles = [None] * self.world
        dist.all_gather_object(handles, mine, group=group)
        self.colony.exchange_open_ipc(handles)
        dist.barrier(group=group)

    def iterate(self, iters: int = 1, check: bool = True):
        """`iters` iterations; with check (default) synchronises once at the end and raises if
        a peer's record did not arrive (the device-side wait is bounded, mmas_status)."""
        self.colony.iterate_exchange(iters)
        if check:
            self.colony.status()

    def best_tour(self):
        return self.colony.best_tour()

    def close(self):
        self.colony.close()
