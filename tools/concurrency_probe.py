"""Probe: do two half-batch pipelines overlap usefully when run concurrently (two contexts,
two streams) compared with one full-batch pipeline? Prints ms per 128 pairs for both."""
import ctypes as C
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from bench import make_frames, schedule  # noqa: E402
from paper_1610_07159_b200 import build, capi  # noqa: E402
from paper_1610_07159_b200.hwflow import EnergyParams, Solver  # noqa: E402


def ready(n, first):
    dev = Solver(build.CUDA_LIB)
    try:
        dev.solve_batch(make_frames(n, first), EnergyParams(), schedule("schwarz"), outputs=("grid_total",))
    except capi.SolverDivergence:
        pass
    return dev


def timed(devs, reps):
    for d in devs:
        d.lib.hwf_run_device(d.ctx.h)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        for d in devs:
            d.lib.hwf_run_device(d.ctx.h)
    for d in devs:
        d.lib.hwf_sync(d.ctx.h, None)
    return 1000 * (time.perf_counter() - t) / reps


one = [ready(128, 0)]
print("one B=128 ctx      ms/128 pairs:", round(timed(one, 10), 2))
del one
two = [ready(64, 0), ready(64, 64)]
print("two B=64 ctx (conc) ms/128 pairs:", round(timed(two, 10), 2))
