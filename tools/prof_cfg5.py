"""Profiling driver for cfg5 (3840x2160, step 4, 5 levels): one solve to build the plan, then replays."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import time  # noqa: E402

from paper_1610_07159_b200 import build, capi, synthetic  # noqa: E402
from paper_1610_07159_b200.hwflow import EnergyParams, SolveSchedule, Solver  # noqa: E402

runs = int(sys.argv[1]) if len(sys.argv) > 1 else 3
dev = Solver(build.CUDA_LIB)
S = SolveSchedule(levels=5, grid_step=4, pcg_iters=5, patch_iters=5)
try:
    dev.solve_batch(synthetic.uhd_pair(0)[0][None], EnergyParams(), S, outputs=("grid_total",))
except capi.SolverDivergence:
    pass
lib, h = dev.lib, dev.ctx.h
t = time.perf_counter()
for _ in range(runs):
    lib.hwf_run_device(h)
lib.hwf_sync(h, None)
print(f"cfg5 ms/frame {1000 * (time.perf_counter() - t) / max(runs, 1):.2f}")
