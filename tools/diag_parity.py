"""Diagnostic: growth of device-vs-oracle differences along the GN schedule (cfg1, global PCG)."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1610_07159_b200 import build, synthetic
from paper_1610_07159_b200.hwflow import EnergyParams, SolveSchedule, Solver
dev, orc = Solver(build.CUDA_LIB), Solver(build.ORACLE_LIB)
ref = Solver(build.REF_LIB) if build.REF_LIB.exists() else None
imgs, gt = synthetic.constant_pair(320, 240)
for levels, gns in ((1, range(1, 8)), (3, [[5, 5, 1], [5, 5, 3], [5, 2], [5, 5, 5], [5]])):
    for g in gns:
        gl = [g] if isinstance(g, int) else g
        S = SolveSchedule(levels=levels, grid_step=8, gn_per_level=gl, pcg_iters=10, subdomain_px=0)
        (a,), (sa,) = dev.solve_batch(imgs[None], EnergyParams(), S)
        b, sb = orc.run_scene_flow(imgs, EnergyParams(), S)
        d = np.abs(a.grid_total - b.grid_total)
        line = f"L={levels} gn={gl} max={d.max():.2e} med={np.median(d):.2e} at node {np.unravel_index(d.argmax(), d.shape)} vis_agree={(a.vis4 == b.vis4).mean():.6f} dE={abs(sa.final_energy()-sb.final_energy())/sb.final_energy():.1e}"
        if ref is not None:
            c, _ = ref.run_scene_flow(imgs, EnergyParams(), S)
            line += f" | port-vs-ref max={np.abs(c.grid_total - b.grid_total).max():.2e}"
        print(line, flush=True)
