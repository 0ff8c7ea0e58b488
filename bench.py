#!/usr/bin/env python
"""Throughput of the per-frame-pair halfway-domain scene-flow solve on B200.

Workload (BASELINE.json configs[1], the real-time case; cfg4 sharding for N>1):
640x480 synthetic textured stereo pairs (t, t+1) with known constant flow,
4-level pyramid, 8 px warp grid, the paper's iteration schedule (GN 2,2,5,5
finest-first, 5 PCG iterations) with the reference's global PCG solver
(pcg_solve, subdomain_px = 0), live preset. A step = one solve of a batch of
B independent frame pairs per GPU (weak scaling: B fixed per GPU; pairs are
sharded across ranks with no collective — frame mode).

The reference's Schwarz mode (--mode schwarz: 5 PCG x 5 sweeps over 16 px
subdomains, i.e. 2x2-node blocks at this grid step) is an additive block-Jacobi
iteration that diverges on this configuration: the energy grows every
Gauss-Newton step and the solved flow is hundreds of pixels off. The device
reproduces that bit for bit (tests/test_gpu_parity.py), but it is not a
meaningful headline; it is reported under other_configs with its flow error.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl ours|reference]

value = pairs/s with inputs resident in HBM (graph replays); e2e = pairs/s
through hwf_solve_batch from pinned host buffers (H2D of the u8 frames and D2H
of the finest warp grid + visibility inside the timed region).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "frame-pairs/s (640x480, full pyramid)"
UNIT = "frame-pairs/s"
W_, H_ = 640, 480


def schedule(mode: str):
    from paper_1610_07159_b200.hwflow import SolveSchedule
    return SolveSchedule(levels=4, grid_step=8, pcg_iters=5, patch_iters=5,
                         subdomain_px=16 if mode == "schwarz" else 0, boundary_px=2)


def workload_desc(mode: str) -> str:
    solve = "5 PCG x 5 Schwarz sweeps (16 px subdomains)" if mode == "schwarz" else "5 global PCG iterations"
    return f"cfg2: 640x480 pairs, 4-level pyramid, 8 px warp grid, GN 2,2,5,5, {solve}, live preset"


def extra_configs(dev, lib, h, C, capi, reps: int = 5) -> dict:
    """The other BASELINE.json shapes on this GPU, device-resident replays (not the headline):
    cfg3 1920x1080 occluder + illumination change, 5 levels, 8 px grid, batch 4;
    cfg5 3840x2160 single frame pair, 5 levels, 4 px grid (north_star: >= 30 Hz);
    cfg1 (BASELINE configs[0]) 320x240, 3 levels, fixed 5 GN x 10 PCG in global mode, batch 128;
    SURVEY §8f rank 3 at cfg2 scale, batch 32: stereo-only (active_fields = s, global PCG; the
    reference's Schwarz mode hits pAp <= 0 on it) and the stereo-hq preset with the epipolar term on
    (w_epi = 0.5, rectified-rig F)."""
    from paper_1610_07159_b200 import synthetic
    from paper_1610_07159_b200.hwflow import EnergyParams, SolveSchedule
    out = {}
    F_rect = np.array([[0.0, 0.0, 0.0], [0.0, 0.0, -1.0], [0.0, 1.0, 0.0]])  # x_0^T F x_1 = y_1 - y_0
    web = [synthetic.webcam_truth(i) for i in range(128)]
    cases = [("cfg3_1920x1080_batch4", lambda: np.stack([synthetic.valgaerts_pair(i)[0] for i in range(4)]),
              SolveSchedule(levels=5, grid_step=8, pcg_iters=5, subdomain_px=0), EnergyParams(), None,
              [synthetic.valgaerts_pair(i, 8, 8)[1] for i in range(4)]),
             ("cfg5_3840x2160_single_frame", lambda: synthetic.uhd_pair(0)[0][None],
              SolveSchedule(levels=5, grid_step=4, pcg_iters=5, subdomain_px=0), EnergyParams(), None,
              [synthetic.uhd_pair(0, 8, 8)[1]]),
             ("cfg1_320x240_5gn_10pcg_global_batch128",
              lambda: np.stack([synthetic.constant_pair(320, 240, seed=1610 + i)[0] for i in range(128)]),
              SolveSchedule(levels=3, grid_step=8, gn_per_level=[5, 5, 5], pcg_iters=10, subdomain_px=0),
              EnergyParams(), None, [synthetic.constant_pair(8, 8)[1]] * 128),
             ("cfg2_paper_schwarz_16px_batch128", lambda: make_frames(128, 0),
              SolveSchedule(levels=4, grid_step=8, pcg_iters=5, patch_iters=5, subdomain_px=16), EnergyParams(), None,
              web),
             ("cfg2_stereo_only_global_pcg_batch32", lambda: make_frames(32, 0),
              SolveSchedule(levels=4, grid_step=8, pcg_iters=5, subdomain_px=0, active_fields=1), EnergyParams(),
              None, web[:32]),
             ("cfg2_stereo_hq_epipolar_batch32", lambda: make_frames(32, 0),
              SolveSchedule(levels=4, grid_step=8, pcg_iters=5, subdomain_px=0), EnergyParams.preset("stereo-hq"),
              F_rect, web[:32])]
    for name, frames_fn, sched, params, F, truth in cases:
        frames = frames_fn()
        n = frames.shape[0]
        err = None
        try:
            outs, _ = dev.solve_batch(frames, params, sched, F, outputs=("grid_total",))
            err = synthetic.flow_error(np.stack([o.grid_total for o in outs]), truth)
            status = "ok"
        except capi.SolverDivergence:
            status = "diverged-flag"
        import torch
        stream = torch.cuda.ExternalStream(lib.hwf_stream(h))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        lib.hwf_run_device(h)
        e0.record(stream)
        for _ in range(reps):
            lib.hwf_run_device(h)
        e1.record(stream)
        e1.synchronize()
        lib.hwf_sync(h, None)
        ms = e0.elapsed_time(e1) / reps
        out[name] = {"pairs": n, "ms_per_step": ms, "pairs_per_s": 1000.0 * n / ms,
                     "solver_status": status, "launches_per_step": lib.hwf_launch_count(h), "flow_error": err}
    # live sequences, each step warm-started from the previous frame's device-resident
    # hierarchy (hwf_solve_batch_seq; states ping-pong), 16 parallel sequences of 640x480, host in/out; global
    # PCG (the reference's Schwarz mode diverges on these noise-free constant-velocity scenes, as in the tests)
    # (frames 0 and 1 are untimed: the cold start and the first warm start build their plans)
    nseq, steps = 16, 6
    per_seq = [synthetic.sequence_pairs(steps, W_, H_, seed=1610 + i) for i in range(nseq)]
    frames = [np.ascontiguousarray(np.stack([per_seq[i][k] for i in range(nseq)])) for k in range(steps)]
    S = SolveSchedule(levels=4, grid_step=8, pcg_iters=5, subdomain_px=0)
    st = [dev.new_state(nseq, W_, H_, S), dev.new_state(nseq, W_, H_, S)]
    status = "ok"
    try:
        dev.solve_batch_seq(frames[0], EnergyParams(), S, None, st[0], outputs=("grid_total",))
        dev.solve_batch_seq(frames[1], EnergyParams(), S, st[0], st[1], outputs=("grid_total",))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k in range(2, len(frames)):
            dev.solve_batch_seq(frames[k], EnergyParams(), S, st[(k - 1) % 2], st[k % 2], outputs=("grid_total",))
        dt = (time.perf_counter() - t0) / (len(frames) - 2)
    except capi.SolverDivergence:
        status, dt = "diverged-flag", float("nan")
    out["cfg2_sequence_warm_start_global_pcg_16x"] = {"pairs": nseq, "ms_per_step": 1000.0 * dt,
                                           "pairs_per_s": nseq / dt if dt == dt else None,
                                           "solver_status": status,
                                           "note": "wall clock per step incl. H2D of u8 frames and D2H of the grid"}
    return out


def make_frames(n: int, first: int) -> np.ndarray:
    from paper_1610_07159_b200 import synthetic
    return np.stack([synthetic.webcam_pair(first + i, W_, H_)[0] for i in range(n)])


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d.get("hbm_gbs", 6650.0), "src": "measured"}
    return {"hbm_gbs": 6650.0, "src": "fallback"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx, self.all_rows, self.proc = gpu_index, [], None
        self.t0 = self.t1 = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            deadline = time.time() + 3.0  # wait until the sampler is live
            while not self.all_rows and time.time() < deadline:
                time.sleep(0.02)
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.all_rows.append((time.time(), [x.strip() for x in line.split(",")]))

    def start(self):
        self.t0 = time.time()

    def stop(self):
        self.t1 = time.time()
        time.sleep(0.15)

    @property
    def rows(self):
        t0, t1 = self.t0 or 0.0, self.t1 or 1e30
        inside = [r for t, r in self.all_rows if t0 <= t <= t1 + 0.1]
        return inside or [r for _, r in self.all_rows[-3:]]

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 4 + i and r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def cpu_baseline(steps: int, warmup: int, mode: str, threads: int | None = None) -> dict:
    """The reference's CPU path (oracle/_ref: reference sources + SPEC-restated hierarchy),
    all host threads (or `threads`), one cfg2 pair per step. Falls back to the oracle port."""
    from paper_1610_07159_b200 import build
    from paper_1610_07159_b200.hwflow import EnergyParams, Solver
    lib, kind = (build.REF_LIB, "reference") if build.REF_LIB.exists() else (build.ORACLE_LIB, "port")
    if not lib.exists():
        build.build_oracle()
    cpu = Solver(lib)
    cores = threads or os.cpu_count() or 1
    sched = schedule(mode)
    sched.threads = cores
    frames = make_frames(max(steps, 1), 0)
    for i in range(warmup):
        cpu.run_scene_flow(frames[i % len(frames)], EnergyParams(), sched)
    t0 = time.perf_counter()
    for i in range(steps):
        cpu.run_scene_flow(frames[i % len(frames)], EnergyParams(), sched)
    dt = time.perf_counter() - t0
    return {"value": steps / dt, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"{steps} cfg2 pairs (640x480, {workload_desc(mode).split(', ', 1)[1]}), one per step, "
                      f"threads={cores}, after {warmup} warm-up pairs", "seconds": dt}


def e2e_flowresult(dev, lib, h, frames_np, pc, sc, steps, ws, ok, batch: int = 64) -> dict:
    """The reference's full output contract end to end: every pair returns the dense FlowResult
    (geometry.hpp:26-37: s, m, d and disparity per pixel as f64, vis4) plus the finest grid, through the streaming
    public API from/to pinned host memory (two batches in flight, each slot with its own device buffers). This is
    what the CPU reference arm produces per pair (hwflow.py run_scene_flow), so it is the like-for-like e2e
    number. `batch` pairs per step (64: 1.1 GB of results per step, pinned twice); it is PCIe-bound."""
    import ctypes as C

    import torch

    from paper_1610_07159_b200 import capi
    from paper_1610_07159_b200.capi import DTYPE_U8, Frame4C, ResultC, StatsC
    from paper_1610_07159_b200.hwflow import grid_dims
    Bd = min(batch, frames_np.shape[0])
    N = W_ * H_
    gw, gh = grid_dims(W_, H_, 8)
    G = gw * gh
    host_in = torch.from_numpy(np.ascontiguousarray(frames_np[:Bd])).pin_memory()
    per = {"s": 2 * N, "m": 2 * N, "d": 2 * N, "disparity": N, "grid_total": 6 * G}
    slots = [{k: torch.empty((Bd, v), dtype=torch.float64).pin_memory() for k, v in per.items()} for _ in range(2)]
    vis = [torch.empty((Bd, N), dtype=torch.uint8).pin_memory() for _ in range(2)]
    fr = (Frame4C * Bd)()
    res = [(ResultC * Bd)() for _ in range(2)]
    for i in range(Bd):
        fr[i].width, fr[i].height, fr[i].dtype = W_, H_, DTYPE_U8
        for e in range(4):
            fr[i].plane[e] = host_in.data_ptr() + (4 * i + e) * N
        for k in range(2):
            for name, t in slots[k].items():
                setattr(res[k][i], name, C.cast(t.data_ptr() + i * t.shape[1] * 8, capi._dp))
            res[k][i].vis4 = C.cast(vis[k].data_ptr() + i * N, capi._u8p)
    stats = [(StatsC * Bd)() for _ in range(2)]

    def run(n):
        for i in range(n):
            ok(lib.hwf_submit_batch(h, Bd, fr, C.byref(pc), C.byref(sc), capi.dptr(None), res[i % 2], stats[i % 2]))
            if i >= 1:
                ok(lib.hwf_wait(h))
        ok(lib.hwf_wait(h))

    run(3)  # plan build + both slots' graphs
    torch.cuda.synchronize()
    barrier(ws)
    t0 = time.perf_counter()
    run(steps)
    t1 = time.perf_counter()
    barrier(ws)
    sec = allreduce_max(t1 - t0, ws)
    d2h = Bd * (8 * (7 * N + 6 * G) + N)
    return {"value": ws * Bd * steps / sec, "unit": UNIT, "pairs_per_step": Bd, "h2d_bytes_per_step": Bd * 4 * N,
            "d2h_bytes_per_step": d2h, "d2h_gbs": d2h * steps / sec / 1e9,
            "note": "dense FlowResult (s, m, d, disparity f64 + vis4) + grid per pair, streaming API, pinned host memory"}


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        import torch
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return ws, rank, local


def shard(rank: int, ws: int, per_gpu: int) -> range:
    """Frame mode: rank r owns global pairs [r*B, (r+1)*B); no collective."""
    return range(rank * per_gpu, (rank + 1) * per_gpu)


def allreduce_max(x: float, ws: int) -> float:
    """Max over ranks of a device-timed duration (the only cross-rank traffic)."""
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws: int):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def run_reference(args, ws, rank):
    if rank != 0:
        return
    cb = cpu_baseline(args.steps, args.warmup, args.mode)
    line = {"metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000.0 / cb["value"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_desc(args.mode), "pairs_per_step": 1}, "impl": "reference",
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args, ws, rank, local):
    import torch

    from paper_1610_07159_b200 import build, capi
    from paper_1610_07159_b200.capi import DTYPE_U8, Frame4C, ResultC, StatsC, dptr, u8ptr
    from paper_1610_07159_b200.hwflow import EnergyParams, Solver, grid_dims

    torch.cuda.set_device(local)
    if not build.CUDA_LIB.exists():
        build.build_cuda()
    dev = Solver(build.CUDA_LIB, device=local)
    lib, h = dev.lib, dev.ctx.h
    B = args.batch
    P, S = EnergyParams(), schedule(args.mode)
    pc, sc = P.to_c(), S.to_c()
    N = W_ * H_
    gw, gh = grid_dims(W_, H_, S.grid_step)
    G = gw * gh

    # inputs: B distinct pairs for this rank (seeds 1610 + global pair index), pinned host copy
    pairs = shard(rank, ws, B)
    frames_np = make_frames(B, pairs.start)
    host_in = torch.from_numpy(frames_np).pin_memory()
    # two result slots (the streaming API keeps two batches in flight)
    host_grid = [torch.empty((B, G, 6), dtype=torch.float64).pin_memory() for _ in range(2)]
    host_vis = [torch.empty((B, H_, W_), dtype=torch.uint8).pin_memory() for _ in range(2)]
    fr = (Frame4C * B)()
    res = [(ResultC * B)() for _ in range(2)]
    base = host_in.data_ptr()
    for i in range(B):
        fr[i].width, fr[i].height, fr[i].dtype = W_, H_, DTYPE_U8
        for e in range(4):
            fr[i].plane[e] = base + (4 * i + e) * N
        for k in range(2):
            res[k][i].grid_total = C.cast(host_grid[k].data_ptr() + i * G * 6 * 8, capi._dp)
            res[k][i].vis4 = C.cast(host_vis[k].data_ptr() + i * N, capi._u8p)
    stats = [(StatsC * B)() for _ in range(2)]

    lib.hwf_set_profiling(h, 0)  # the timed replays carry no timing events (in-graph events cost ~0.5%)
    d_in, d_grid = C.c_void_p(), C.c_void_p()
    dev.ctx.check(lib.hwf_prepare_device(h, B, W_, H_, DTYPE_U8, C.byref(pc), C.byref(sc), dptr(None),
                                         C.byref(d_in), C.byref(d_grid)))

    def ok(rc):
        if rc not in (capi.HWF_OK, capi.HWF_EDIVERGED):  # divergence is the reference's own behaviour; reported
            dev.ctx.check(rc)
        return rc

    def e2e_step():
        return ok(lib.hwf_solve_batch(h, B, fr, C.byref(pc), C.byref(sc), dptr(None), res[0], stats[0]))

    def e2e_stream(steps):
        """steps batches through hwf_submit_batch/hwf_wait: every step uploads its u8 frames from
        pinned host memory and downloads its finest grid + visibility; transfers of neighbouring
        steps overlap the current step's device solve."""
        for i in range(steps):
            ok(lib.hwf_submit_batch(h, B, fr, C.byref(pc), C.byref(sc), dptr(None), res[i % 2], stats[i % 2]))
            if i >= 1:
                ok(lib.hwf_wait(h))
        ok(lib.hwf_wait(h))

    # warm-up (also fills the plan's device input buffer with this rank's frames)
    for _ in range(args.warmup):
        rc_div = e2e_step()
    stream = torch.cuda.ExternalStream(lib.hwf_stream(h))
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    # ---- value: device-resident replays -------------------------------------------
    barrier(ws)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        clk.start()
        ev0.record(stream)
        for _ in range(args.steps):
            dev.ctx.check(lib.hwf_run_device(h))
        ev1.record(stream)
        ev1.synchronize()
        clk.stop()
    torch.cuda.synchronize()
    barrier(ws)
    ms_total = allreduce_max(ev0.elapsed_time(ev1), ws)
    ms_per_step = ms_total / args.steps
    value = ws * B * args.steps / (ms_total / 1000.0)
    rc_sync = lib.hwf_sync(h, stats[0])

    # kernel and GN-iteration timings: the same plan rebuilt with CUDA events inside the graph (around every
    # k_pixel<LIN> launch and every GN iteration), one untimed replay after its inputs are uploaded
    lib.hwf_set_profiling(h, 1)
    dev.ctx.check(lib.hwf_prepare_device(h, B, W_, H_, DTYPE_U8, C.byref(pc), C.byref(sc), dptr(None),
                                         C.byref(d_in), C.byref(d_grid)))
    e2e_step()
    dev.ctx.check(lib.hwf_run_device(h))
    lib.hwf_sync(h, None)
    cap = 64
    kms, kbytes = (C.c_double * cap)(), (C.c_double * cap)()
    nk = lib.hwf_pixel_kernel_times(h, cap, kms, kbytes)
    launches_k = [(kms[i], kbytes[i]) for i in range(max(nk, 0))]
    pk_ms = sum(t for t, _ in launches_k)  # all k_pixel<LIN> launches of the last timed replay
    big = max((b for _, b in launches_k), default=0.0)
    l0 = [(t, b) for t, b in launches_k if b == big]  # the finest-level (dominant) launches
    l0_ms = sum(t for t, _ in l0) / max(len(l0), 1)
    pk = peaks()
    achieved = big / (l0_ms / 1000.0) / 1e9 if l0_ms > 0 else 0.0  # per launch, algorithmic bytes
    traffic, prof = None, {}
    tf = ROOT / "profiles" / "pixel_traffic.json"
    if tf.exists():  # ncu --set full capture at B=128; DRAM bytes scale with the batch
        prof = json.loads(tf.read_text())
        v = prof.get("dram_bytes_per_launch_L0")
        traffic = v * B / prof.get("batch", 128) if v is not None else None
    # per Gauss-Newton iteration (linearisation + PCG) of the last timed replay, CUDA events inside the graph
    gms, glv = (C.c_double * cap)(), (C.c_int * cap)()
    ng = lib.hwf_gn_iteration_times(h, cap, gms, glv)
    gn_iter = {}
    for i in range(max(ng, 0)):
        gn_iter.setdefault(f"L{glv[i]}", []).append(gms[i])
    gn_iter = {k: {"iters": len(v), "batch_ms": sum(v) / len(v), "per_pair_us": 1000.0 * sum(v) / len(v) / B}
               for k, v in sorted(gn_iter.items())}
    launches = lib.hwf_launch_count(h)
    lib.hwf_set_profiling(h, 0)  # e2e and the side measurements build their own plans, without timing events
    # FP64 roofline of the same kernel: FP64 flops per launch from the committed ncu capture (scaled by the batch),
    # over this run's CUDA-event launch time, against the builder-measured DFMA peak (profiles/fp64_peak.json)
    fp64 = None
    if prof.get("fp64_flop_per_launch_L0"):
        flop = prof["fp64_flop_per_launch_L0"] * B / prof.get("batch", 128)
        inst = sum(prof["fp64_inst_per_launch_L0"].values()) * B / prof.get("batch", 128)
        fpk = json.loads((ROOT / "profiles" / "fp64_peak.json").read_text())
        ach = flop / (l0_ms / 1000.0) / 1e12 if l0_ms > 0 else 0.0
        inst_peak = fpk["dadd_inst_per_s"]  # FP64 pipe issue ceiling (64 lanes / clk / SM)
        fp64 = {"achieved": ach, "peak": fpk["fp64_tflops"], "unit": "TFLOP/s", "frac": ach / fpk["fp64_tflops"],
                "pipe_inst_frac": inst / (l0_ms / 1000.0) / inst_peak if l0_ms > 0 else None,
                "flop_per_launch": flop, "peak_src": "profiles/fp64_peak.json (builder-measured DFMA, tools/fp64_peak.cu)"}

    # ---- e2e: through the public C-ABI from pinned host buffers ---------------------
    barrier(ws)
    torch.cuda.synchronize()
    e2e_stream(2)  # warm the streaming slots (second graph capture)
    torch.cuda.synchronize()
    barrier(ws)
    t0 = time.perf_counter()
    e2e_stream(args.steps)
    t1 = time.perf_counter()
    barrier(ws)
    e2e_s = allreduce_max(t1 - t0, ws)
    e2e_value = ws * B * args.steps / e2e_s

    from paper_1610_07159_b200 import synthetic
    flow_err = synthetic.flow_error(host_grid[(args.steps - 1) % 2].numpy(),
                                    [synthetic.webcam_truth(i) for i in range(pairs.start, pairs.start + B)])
    gn_total = sum(S.gn_for_level(l) for l in range(4))
    e2e_fr = None if args.no_flowresult else e2e_flowresult(dev, lib, h, frames_np, pc, sc, args.steps, ws, ok)
    extra = extra_configs(dev, lib, h, C, capi) if (rank == 0 and ws == 1 and not args.no_extra) else None
    if rank == 0:
        cb = cpu_baseline(max(1, min(3, args.steps)), 1, args.mode) if ws == 1 and not args.no_cpu else None
        cb1 = cpu_baseline(1, 0, args.mode, threads=1) if ws == 1 and not args.no_cpu else None
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_desc(args.mode), "pairs_per_gpu_per_step": B,
                       "global_pairs_per_step": ws * B, "parallelism": f"frame-sharded x{ws} (no collective)",
                       "l2": "no flush: per-step working set > 3 GB >> 126 MB L2"},
            "ms_per_gn_iter": ms_per_step / gn_total / B,  # whole step per pair per GN iteration (amortised)
            "gn_iter_by_level": gn_iter,  # measured: one GN iteration (linearise + solve) of the B-pair batch
            "hbm_gbs": achieved,  # dominant kernel, algorithmic bytes / CUDA-event time
            # the whole pipeline against SURVEY.md §8(d)'s streaming model of cfg2 (~271 MB and ~3.45 GFLOP per pair):
            # the HBM-bound and FP64-bound pair rates, and this run's fraction of each
            "pipeline_model": {"bytes_per_pair": 271e6, "flop_per_pair": 3.45e9,
                               "hbm_pairs_per_s": pk["hbm_gbs"] * 1e9 / 271e6,
                               "hbm_frac": value * 271e6 / (pk["hbm_gbs"] * 1e9) / ws if pk["hbm_gbs"] else None,
                               "fp64_pairs_per_s": (fp64["peak"] * 1e12 / 3.45e9) if fp64 else None,
                               "fp64_frac": (value / ws * 3.45e9 / (fp64["peak"] * 1e12)) if fp64 else None,
                               "src": "SURVEY.md §8(d) streaming model; peaks: MEASURED_PEAKS.json hbm_gbs, "
                                      "profiles/fp64_peak.json"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / pk["hbm_gbs"] if pk["hbm_gbs"] else None, "traffic": traffic,
                         "kernel": "k_pixel<LIN,U8> (fused data term + cell reduction), finest level, u8 frames sampled directly",
                         "peak_src": pk["src"], "algorithmic_bytes_per_launch": big, "ms_per_launch": l0_ms,
                         "launches_per_step": nk, "share_of_step": pk_ms / ms_per_step if ms_per_step else None,
                         # not HBM-bound: the limiter and pipe utilisations of the same kernel from the committed
                         # ncu --set full capture (profiles/pixel_traffic.json)
                         "limiter": prof.get("limiter"), "fp64_pipe_frac": prof.get("fp64_pipe_frac"),
                         "l1_lsu_frac": prof.get("l1_lsu_frac"), "issue_slots_frac": prof.get("issue_slots_frac"),
                         "fp64": fp64},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": B * 4 * N,
                    "d2h_bytes_per_step": B * (G * 6 * 8 + N)},
            "e2e_flowresult": e2e_fr,
            "gpu_launches": launches * args.steps,
            "clocks": clk.summary(),
            "solver_status": "diverged-flag" if (rc_sync == capi.HWF_EDIVERGED or rc_div == capi.HWF_EDIVERGED) else "ok",
            # finest warp-grid nodes of the last e2e step against the synthetic ground truth (the live preset
            # damps motion updates hard, m_m = 100, so m converges slowly; s is the recovered stereo flow)
            "flow_error": flow_err,
        }
        if cb:
            line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
            line["cpu_baseline"]["single_thread"] = {k: cb1[k] for k in ("value", "cores", "sample")}
        if extra:
            line["other_configs"] = extra
        print(json.dumps(line), flush=True)


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` without a launcher: re-exec this script under torch.distributed.run with N local ranks
    (one process per GPU, rendezvous on 127.0.0.1), the same way the driver launches it. Rank 0 prints the line.
    NCCL's communicator lines (NCCL_DEBUG=INFO, INIT subsystem) go to stderr so the rank count can be checked."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def dry_run(args):
    """--dry: the multi-rank plumbing without a GPU (gloo): every rank reports its frame-mode shard; rank 0
    gathers them and prints one JSON line (tests/test_bench.py)."""
    import torch.distributed as dist
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if ws > 1:
        dist.init_process_group("gloo")
    sh = shard(rank, ws, args.batch)
    mine = [rank, sh.start, sh.stop, os.getpid()]
    allv = [mine]
    if ws > 1:
        allv = [None] * ws
        dist.all_gather_object(allv, mine)
    t = allreduce_max(float(rank + 1), ws)
    if rank == 0:
        print(json.dumps({"dry": True, "n_gpus": ws, "ranks": allv, "max_over_ranks": t}), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=256,
                    help="frame pairs per GPU per step (256 = BASELINE cfg4's pair count at N = 1)")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--mode", choices=["schwarz", "global"], default="global")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-extra", action="store_true", help="skip the cfg3/cfg5 side measurements")
    ap.add_argument("--no-flowresult", action="store_true", help="skip the dense-FlowResult e2e leg")
    ap.add_argument("--dry", action="store_true", help="multi-rank plumbing only (gloo, no GPU work)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(spawn_ranks(args.gpus))
    if args.dry:
        dry_run(args)
        return
    ws, rank, local = (1, 0, 0)
    if args.impl == "reference":
        ws = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        run_reference(args, ws, rank)
        return
    ws, rank, local = dist_init()
    if ws != args.gpus and rank == 0:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}; reporting n_gpus={ws}", file=sys.stderr)
    run_ours(args, ws, rank, local)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
