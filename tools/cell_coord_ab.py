"""The round-1 'branch-free cell_coord moved acceptance 5 to 0.35 px' note, re-run.

    python tools/ab.py build cc1=HWF_CELL_COORD=1 cc2=HWF_CELL_COORD=2 cc3=HWF_CELL_COORD=3   # here
    python tools/cell_coord_ab.py base cc1 cc2 cc3                                              # on the GPU box

Variants of image.cpp:19-31 cell_coord (csrc/device.cuh):
  base  the branchy form;
  cc1   the same function with selects (NaN -> i0 = 0, f = NaN, as the branches give);
  cc2   clamp-first with fmin/fmax (a NaN coordinate becomes cell 0 with f = 0);
  cc3   the cell clamped but not the fraction (f = v - i0 extrapolates beyond the border).
For SPEC acceptance 5 (tests/test_gpu_accuracy.py: 256x256, 5 levels, step 8, global PCG, s = shift/2) and the cfg2
headline golden pair 0, prints max |device - oracle| over the finest grid and the 90th-percentile stereo error.
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_1610_07159_b200 import build, synthetic  # noqa: E402
from paper_1610_07159_b200.hwflow import EnergyParams, SolveSchedule, Solver  # noqa: E402


def main():
    oracle = Solver(build.ORACLE_LIB)
    S = SolveSchedule(levels=5, grid_step=8, subdomain_px=0)
    cases = [(shift, synthetic.render_pair(256, 256, s=(shift / 2, 0.0), seed=5)) for shift in (2.0, 8.0, 16.0)]
    refs = [oracle.run_scene_flow(imgs, EnergyParams(), S)[0] for _, imgs in cases]
    for name in sys.argv[1:]:
        lib = ROOT / "paper_1610_07159_b200" / "lib" / ("libhwflow_cuda.so" if name == "base" else f"variants/{name}/libhwflow_cuda.so")
        dev = Solver(str(lib))
        for (shift, imgs), ro in zip(cases, refs):
            (r,), _ = dev.solve_batch(imgs[None], EnergyParams(), S)
            e = np.hypot(r.s[..., 0] - shift / 2, r.s[..., 1])[16:-16, 16:-16]
            d = np.abs(r.grid_total - ro.grid_total)
            print(f"{name:5s} shift {shift:4.1f}: max|dev-oracle| {d.max():.3e} px at node {np.unravel_index(d.argmax(), d.shape)}, "
                  f"p90 stereo error {np.percentile(e, 90):.3f} px, finite {np.isfinite(r.grid_total).all()}", flush=True)
        dev.close()


if __name__ == "__main__":
    main()
