"""Strip-split solve of one frame pair (SURVEY.md §8e, 4K mode; include/hwflow_split.h).

-m "not gpu": the split driver (paper_1610_07159_b200/split.py) with the oracle restatement
(oracle/split.cpp). First with in-process ranks (LocalComm), then with world_size 2 and 3
gloo processes (TorchComm). The result must be bitwise identical to the unsplit oracle
solve. The oracle poisons every published row a rank should not know, so a missing halo
exchange fails.
-m gpu: the device split (csrc/split.cu) with in-process ranks sharing one context, against
the unsplit device solve. The ranks are stepped by the host, and no kernel waits on
another rank. Also the NCCL path with world_size 1. The unsplit solve runs the small levels'
PCG in one CTA per pair (k_pcg_fused) while the split runs the per-phase kernels, so the
bitwise comparisons also pin the fused kernel to the per-phase arithmetic.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1610_07159_b200 import synthetic
from paper_1610_07159_b200.capi import DTYPE_U8
from paper_1610_07159_b200.hwflow import EnergyParams, SolveSchedule
from paper_1610_07159_b200.split import LocalComm, SplitGraph, SplitRank, solve_split

SCHED = SolveSchedule(levels=3, grid_step=4, gn_per_level=[2, 2, 2], pcg_iters=4, patch_iters=3, subdomain_px=16)
GSCHED = SolveSchedule(levels=3, grid_step=4, gn_per_level=[2, 2, 2], pcg_iters=4, subdomain_px=0)  # global PCG
MODES = {"schwarz": SCHED, "global": GSCHED}


def _frames(w=128, h=96, seed=0):
    return synthetic.webcam_pair(seed, w, h)[0]


def _unsplit(solver, imgs, sched, params=None):
    (r,), (st,) = solver.solve_batch(imgs[None], params or EnergyParams(), sched)
    return r, st


def _assert_same(split, ref, energy_rtol):
    (r, st), (r0, st0) = split, ref
    assert np.array_equal(r.grid_total, r0.grid_total)
    assert np.array_equal(r.vis4, r0.vis4)
    assert np.array_equal(r.s, r0.s) and np.array_equal(r.disparity, r0.disparity)
    for a, b in zip(st.energy_before + st.energy_after, st0.energy_before + st0.energy_after):
        assert np.allclose(a, b, rtol=energy_rtol, atol=0.0)


@pytest.mark.parametrize("mode", ["schwarz", "global"])
@pytest.mark.parametrize("world", [1, 2, 3, 5])
def test_split_local_matches_unsplit_oracle(oracle, world, mode):
    imgs = _frames()
    ref = _unsplit(oracle, imgs, MODES[mode])
    ranks = [SplitRank(oracle, 128, 96, DTYPE_U8, EnergyParams(), MODES[mode], None, r, world) for r in range(world)]
    owned = [r.rows[0][:2] for r in ranks]
    assert owned[0][0] == 0 and owned[-1][1] == 25 and all(a[1] == b[0] for a, b in zip(owned, owned[1:]))
    outs = solve_split(ranks, LocalComm(), imgs)
    for out in outs:
        _assert_same(out, ref, 1e-12 if world > 1 else 0.0)


class _NoHalo(LocalComm):
    def halo(self, ranks, level, name):
        pass


class _NoPartials(LocalComm):
    def allgather_rows(self, ranks, level, name):
        if name != "pcg_part":
            super().allgather_rows(ranks, level, name)


@pytest.mark.parametrize("mode,comm", [("schwarz", _NoHalo), ("global", _NoHalo), ("global", _NoPartials)])
def test_split_detects_a_missing_exchange(oracle, mode, comm):
    imgs = _frames()
    ref = _unsplit(oracle, imgs, MODES[mode])
    ranks = [SplitRank(oracle, 128, 96, DTYPE_U8, EnergyParams(), MODES[mode], None, r, 2) for r in range(2)]
    try:
        (r, _), _ = solve_split(ranks, comm(), imgs)
        assert not np.array_equal(r.grid_total, ref[0].grid_total)
    except Exception as e:  # NaN from a poisoned row reaching a divergence check
        assert "diverg" in str(e).lower() or "non-finite" in str(e).lower() or "pcg" in str(e).lower()


def test_split_global_mode_rejects_sweeps(oracle):
    from paper_1610_07159_b200.capi import InvalidArgument
    r = SplitRank(oracle, 128, 96, DTYPE_U8, EnergyParams(), GSCHED, None, 0, 2)
    with pytest.raises(InvalidArgument, match="Schwarz"):
        r.sweep(0, 0)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, ws: int, port: int, q, mode: str = "schwarz"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        from paper_1610_07159_b200 import build
        from paper_1610_07159_b200.hwflow import Solver
        from paper_1610_07159_b200.split import TorchComm
        solver = Solver(build.ORACLE_LIB)
        me = SplitRank(solver, 128, 96, DTYPE_U8, EnergyParams(), MODES[mode], None, rank, ws)
        ((r, st),) = solve_split([me], TorchComm(me), _frames())
        q.put((rank, r.grid_total, r.vis4, st.energy_before, st.energy_after))
    finally:
        dist.barrier()
        dist.destroy_process_group()


@pytest.mark.parametrize("ws,mode", [(2, "schwarz"), (3, "schwarz"), (2, "global"), (3, "global")])
def test_split_gloo_ranks_match_unsplit_oracle(oracle, ws, mode):
    ref = _unsplit(oracle, _frames(), MODES[mode])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q, mode)) for r in range(ws)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(ws)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, grid, vis, eb, ea in got:  # every rank ends with the full, identical result
        assert np.array_equal(grid, ref[0].grid_total)
        assert np.array_equal(vis, ref[0].vis4)
        for a, b in zip(eb + ea, ref[1].energy_before + ref[1].energy_after):
            assert np.allclose(a, b, rtol=1e-12, atol=0.0)


# ---------------------------------------------------------------- device
@pytest.mark.gpu
@pytest.mark.parametrize("w,h,world,sched", [
    (128, 96, 2, SCHED),
    (640, 480, 3, SolveSchedule(levels=4, grid_step=8, pcg_iters=5, patch_iters=5, subdomain_px=16)),
    (3840, 2160, 4, SolveSchedule(levels=5, grid_step=4, gn_per_level=[1, 1, 2, 2, 2], pcg_iters=5,
                                  patch_iters=5, subdomain_px=16)),
    (128, 96, 2, GSCHED),
    (640, 480, 3, SolveSchedule(levels=4, grid_step=8, pcg_iters=5, subdomain_px=0)),
    (3840, 2160, 4, SolveSchedule(levels=5, grid_step=4, gn_per_level=[1, 1, 2, 2, 2], pcg_iters=5,
                                  subdomain_px=0)),
])
def test_split_device_matches_unsplit_device(device, w, h, world, sched):
    imgs = _frames(w, h, seed=3)
    ref = _unsplit(device, imgs, sched)
    ranks = [SplitRank(device, w, h, DTYPE_U8, EnergyParams(), sched, None, r, world) for r in range(world)]
    for out in solve_split(ranks, LocalComm(), imgs):
        _assert_same(out, ref, 1e-12)
    for r in ranks:
        r.close()


@pytest.mark.gpu
@pytest.mark.parametrize("w,h,world,sched", [
    (128, 96, 2, GSCHED),
    (640, 480, 3, SolveSchedule(levels=4, grid_step=8, pcg_iters=5, subdomain_px=0)),
    (640, 480, 2, SolveSchedule(levels=4, grid_step=8, pcg_iters=5, patch_iters=5, subdomain_px=16)),
])
def test_split_graph_matches_unsplit_device(device, w, h, world, sched):
    """SplitGraph: every rank's steps and the exchanges captured into one CUDA graph (no host code between PCG
    phases); two different frames replayed through the same graph, each bitwise the unsplit solve."""
    ranks = [SplitRank(device, w, h, DTYPE_U8, EnergyParams(), sched, None, r, world) for r in range(world)]
    g = SplitGraph(ranks, LocalComm(), _frames(w, h, seed=3))
    for seed in (3, 4):
        imgs = _frames(w, h, seed=seed)
        ref = _unsplit(device, imgs, sched)
        for out in g(imgs):
            _assert_same(out, ref, 1e-12)
    for r in ranks:
        r.close()


def _nccl_worker(port: int, q, mode: str = "schwarz", graph: bool = False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        from paper_1610_07159_b200 import build
        from paper_1610_07159_b200.hwflow import Solver
        from paper_1610_07159_b200.split import TorchComm
        solver = Solver(build.CUDA_LIB)
        me = SplitRank(solver, 128, 96, DTYPE_U8, EnergyParams(), MODES[mode], None, 0, 1)
        if graph:  # the NCCL collectives captured in the CUDA graph with the library's kernels
            ((r, st),) = SplitGraph([me], TorchComm(me), _frames())(_frames())
        else:
            ((r, st),) = solve_split([me], TorchComm(me), _frames())
        q.put((r.grid_total, r.vis4))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("mode,graph", [("schwarz", False), ("global", False), ("global", True)])
def test_split_nccl_single_rank(device, mode, graph):
    ref = _unsplit(device, _frames(), MODES[mode])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(_free_port(), q, mode, graph))
    p.start()
    grid, vis = q.get(timeout=300)
    p.join(timeout=60)
    assert p.exitcode == 0
    assert np.array_equal(grid, ref[0].grid_total) and np.array_equal(vis, ref[0].vis4)


def _nccl_multi_worker(rank: int, ws: int, port: int, q, mode: str, graph: bool):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=ws)
    try:
        from paper_1610_07159_b200 import build
        from paper_1610_07159_b200.hwflow import Solver
        from paper_1610_07159_b200.split import TorchComm
        solver = Solver(build.CUDA_LIB)
        me = SplitRank(solver, 640, 480, DTYPE_U8, EnergyParams(), MODES_640[mode], None, rank, ws)
        imgs = _frames(640, 480, seed=3)
        if graph:
            ((r, st),) = SplitGraph([me], TorchComm(me), imgs)(imgs)
        else:
            ((r, st),) = solve_split([me], TorchComm(me), imgs)
        q.put((rank, r.grid_total, r.vis4, st.energy_after))
        me.close()
    finally:
        dist.barrier()
        dist.destroy_process_group()


MODES_640 = {"schwarz": SolveSchedule(levels=4, grid_step=8, pcg_iters=5, patch_iters=5, subdomain_px=16),
             "global": SolveSchedule(levels=4, grid_step=8, pcg_iters=5, subdomain_px=0)}


@pytest.mark.gpu
@pytest.mark.parametrize("ws", [2, 4])
@pytest.mark.parametrize("mode,graph", [("schwarz", False), ("global", False), ("global", True)])
def test_split_nccl_multi_gpu(device, ws, mode, graph):
    """One rank per GPU over NCCL (the halo P2P and the partial all-gathers cross devices), bitwise the unsplit
    solve on every rank. Needs ws GPUs; skipped on the 1-GPU boxes this project is measured on."""
    import torch
    if torch.cuda.device_count() < ws:
        pytest.skip(f"needs {ws} GPUs, found {torch.cuda.device_count()}")
    imgs = _frames(640, 480, seed=3)
    ref = _unsplit(device, imgs, MODES_640[mode])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_nccl_multi_worker, args=(r, ws, port, q, mode, graph)) for r in range(ws)]
    for p in procs:
        p.start()
    got = [q.get(timeout=600) for _ in range(ws)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for _, grid, vis, ea in got:
        assert np.array_equal(grid, ref[0].grid_total) and np.array_equal(vis, ref[0].vis4)
        assert np.allclose(ea, ref[1].energy_after, rtol=1e-12, atol=0.0)
