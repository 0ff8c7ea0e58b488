"""Profiling driver for cfg5 (3840x2160, step 4, 5 levels): one solve to build the plan, then replays.

    python tools/prof_cfg5.py [runs] [schwarz|global]
Also prints the median node error of the solved flow against the known constant flow."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import time  # noqa: E402

import numpy as np  # noqa: E402

from paper_1610_07159_b200 import build, capi, synthetic  # noqa: E402
from paper_1610_07159_b200.hwflow import EnergyParams, SolveSchedule, Solver  # noqa: E402

runs = int(sys.argv[1]) if len(sys.argv) > 1 else 3
dev = Solver(build.CUDA_LIB)
mode = sys.argv[2] if len(sys.argv) > 2 else "schwarz"
S = SolveSchedule(levels=5, grid_step=4, pcg_iters=5, patch_iters=5, subdomain_px=16 if mode == "schwarz" else 0)
imgs, gt = synthetic.uhd_pair(0)
try:
    (r,), _ = dev.solve_batch(imgs[None], EnergyParams(), S, outputs=("grid_total",))
    G = r.grid_total
    es = np.hypot(G[:, 0] - gt["s"][0], G[:, 1] - gt["s"][1])
    em = np.hypot(G[:, 2] - gt["m"][0], G[:, 3] - gt["m"][1])
    print(f"{mode}: node error median s {np.median(es):.4f} px, m {np.median(em):.4f} px")
except capi.SolverDivergence as e:
    print(f"{mode}: divergence flag: {e}")
lib, h = dev.lib, dev.ctx.h
t = time.perf_counter()
for _ in range(runs):
    lib.hwf_run_device(h)
lib.hwf_sync(h, None)
print(f"cfg5 ms/frame {1000 * (time.perf_counter() - t) / max(runs, 1):.2f}")
