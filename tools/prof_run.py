"""Profiling driver: W warm-up replays then R timed replays of the cfg2 batch graph.

    python tools/prof_run.py --batch 8 --warmup 2 --runs 1
Used under `ncu` (launch list / --set full). Prints launches per replay.
"""
import argparse
import ctypes as C
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from bench import make_frames, schedule  # noqa: E402
from paper_1610_07159_b200 import build, capi  # noqa: E402
from paper_1610_07159_b200.hwflow import EnergyParams, Solver  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--runs", type=int, default=1)
ap.add_argument("--mode", default="schwarz")
ap.add_argument("--profiling", action="store_true", help="plans with in-graph k_pixel<LIN> timing events")
ap.add_argument("--lib", default=None, help="library to load (A/B variants, tools/ab.py)")
a = ap.parse_args()

dev = Solver(a.lib or build.CUDA_LIB)
if a.profiling:
    dev.lib.hwf_set_profiling(dev.ctx.h, 1)
frames = make_frames(a.batch, 0)
P, S = EnergyParams(), schedule(a.mode)
outs, _ = None, None
try:
    dev.solve_batch(frames, P, S, outputs=("grid_total",))
except capi.SolverDivergence as e:
    print("divergence flag (reference behaviour):", str(e)[:200])
lib, h = dev.lib, dev.ctx.h
for _ in range(a.warmup):
    dev.ctx.check(lib.hwf_run_device(h))
lib.hwf_sync(h, None)
t = time.perf_counter()
for _ in range(a.runs):
    dev.ctx.check(lib.hwf_run_device(h))
lib.hwf_sync(h, None)
dt = time.perf_counter() - t
line = f"launches_per_replay={lib.hwf_launch_count(h)} batch={a.batch} ms_per_replay={1000 * dt / max(a.runs, 1):.3f}"
if a.profiling:  # k_pixel<LIN> launches of the last replay (in-graph events)
    kms, kb = (C.c_double * 64)(), (C.c_double * 64)()
    nk = lib.hwf_pixel_kernel_times(h, 64, kms, kb)
    big = max(kb[i] for i in range(nk))
    l0 = [kms[i] for i in range(nk) if kb[i] == big]
    line += f" pixel_lin_ms={sum(kms[i] for i in range(nk)):.3f} pixel_lin_L0_ms_per_launch={sum(l0) / len(l0):.3f}"
print(line)
