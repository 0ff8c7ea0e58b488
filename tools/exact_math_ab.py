"""Verdict item: does correctly rounded math (HWF_EXACT_MATH: sqrt and divisions as the reference) bring the device
within 1e-3 px of the reference build at the ill-conditioned full cfg1 / cfg3 schedules? Prints per-node summaries
of |device - reference| for the default and the exact-math library (golden grids: tests/golden/ref_headline.npz)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1610_07159_b200 import synthetic  # noqa: E402
from paper_1610_07159_b200.hwflow import EnergyParams, SolveSchedule, Solver  # noqa: E402

g = dict(np.load(ROOT / "tests" / "golden" / "ref_headline.npz"))
cases = {"cfg1_full": (synthetic.constant_pair(320, 240)[0],
                       SolveSchedule(levels=3, grid_step=8, gn_per_level=[5], pcg_iters=10, subdomain_px=0)),
         "cfg3": (synthetic.valgaerts_pair(0)[0], SolveSchedule(levels=5, grid_step=8, pcg_iters=5, subdomain_px=0))}
for name in ("base", "exact"):
    lib = ROOT / "paper_1610_07159_b200" / "lib" / ("libhwflow_cuda.so" if name == "base" else "variants/exact/libhwflow_cuda.so")
    dev = Solver(lib)
    for tag, (imgs, S) in cases.items():
        (r,), _ = dev.solve_batch(imgs[None], EnergyParams(), S, outputs=("grid_total",))
        d = np.abs(r.grid_total - g[f"{tag}_grid"]).max(1)
        print(f"{name:6s} {tag:10s} max {d.max():.3e} p99 {np.percentile(d, 99):.2e} p50 {np.median(d):.2e} "
              f"nodes>1e-3 {(d > 1e-3).sum()}", flush=True)
    dev.close()
