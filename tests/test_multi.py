"""CPU, world_size 2 over gloo: the multi-GPU frame-mode host logic of bench.py —
disjoint, covering shards and max-over-ranks timing (no data-path collective)."""
from __future__ import annotations

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, ws: int, port: int, per_gpu: int, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import bench
    import torch
    mine = list(bench.shard(rank, ws, per_gpu))
    gathered = [None] * ws
    dist.all_gather_object(gathered, mine)
    t = bench.allreduce_max(1.0 + rank, ws)  # rank-local durations 1.0, 2.0 -> max 2.0
    if rank == 0:
        q.put((gathered, t))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("ws,per_gpu", [(2, 4), (2, 128)])
def test_frame_sharding_and_max_timing(ws, per_gpu):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, per_gpu, q)) for r in range(ws)]
    for p in procs:
        p.start()
    gathered, t = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    flat = [i for part in gathered for i in part]
    assert sorted(flat) == list(range(ws * per_gpu))  # disjoint and covering
    assert t == 2.0
