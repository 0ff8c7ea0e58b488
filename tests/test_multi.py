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


def _solve_worker(rank: int, ws: int, port: int, per_rank: int, q):
    """One frame-mode rank: solve this rank's shard of pairs (bench.shard, seeds 1610 + global index) with the
    CPU checker, then gather every rank's grids to rank 0 (the driver's only cross-rank traffic is the timing
    max; the gather here is the test's)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import numpy as np

    import bench
    from paper_1610_07159_b200 import build, synthetic
    from paper_1610_07159_b200.hwflow import EnergyParams, SolveSchedule, Solver
    solver = Solver(build.ORACLE_LIB)
    S = SolveSchedule(levels=2, grid_step=8, pcg_iters=3, subdomain_px=0)
    pairs = bench.shard(rank, ws, per_rank)
    frames = np.stack([synthetic.webcam_pair(i, 64, 48)[0] for i in pairs])
    outs, _ = solver.solve_batch(frames, EnergyParams(), S, outputs=("grid_total",))
    mine = (list(pairs), [o.grid_total for o in outs])
    gathered = [None] * ws
    dist.all_gather_object(gathered, mine)
    if rank == 0:
        q.put(gathered)
    dist.barrier()
    dist.destroy_process_group()


def test_frame_mode_ranks_solve_their_shards():
    """world_size 2: every rank solves only its own pairs, and the union equals one process solving them all."""
    import numpy as np

    from paper_1610_07159_b200 import build, synthetic
    from paper_1610_07159_b200.hwflow import EnergyParams, SolveSchedule, Solver
    ws, per_rank = 2, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_solve_worker, args=(r, ws, port, per_rank, q)) for r in range(ws)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    S = SolveSchedule(levels=2, grid_step=8, pcg_iters=3, subdomain_px=0)
    whole, _ = Solver(build.ORACLE_LIB).solve_batch(
        np.stack([synthetic.webcam_pair(i, 64, 48)[0] for i in range(ws * per_rank)]), EnergyParams(), S,
        outputs=("grid_total",))
    seen = set()
    for idx, grids in gathered:
        assert not seen & set(idx)
        seen |= set(idx)
        for i, g in zip(idx, grids):
            assert np.array_equal(g, whole[i].grid_total)
    assert seen == set(range(ws * per_rank))
