"""Diagnostic: Algorithm 1 driven through the stage seams on two libraries in lock step (tests/lockstep.py).
Prints, per level and GN iteration, how far their deltas, outlier bits W and node weights are apart — to find
where two faithful builds of the reference part ways.

    python tools/hier_trace.py [--a ref|port|cuda] [--b ref|port|cuda] [--cfg cfg1|cfg2|cfg3|cfg5] [--sync]

Without --sync both run free (the accumulated divergence); with --sync b is re-seeded from a's state before
every iteration, so each line is one iteration's own divergence. profiles/r2_parity_*.txt hold the outputs.
"""
from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from lockstep import lockstep  # noqa: E402

from paper_1610_07159_b200 import build, synthetic  # noqa: E402
from paper_1610_07159_b200.hwflow import EnergyParams, SolveSchedule, Solver  # noqa: E402

LIBS = {"ref": lambda: build.REF_LIB, "port": lambda: build.ORACLE_LIB, "cuda": lambda: build.CUDA_LIB}


def case(cfg: str):
    if cfg == "cfg1":
        return synthetic.constant_pair(320, 240)[0], SolveSchedule(levels=3, grid_step=8, gn_per_level=[5],
                                                                   pcg_iters=10, subdomain_px=0)
    if cfg == "cfg2":
        return synthetic.webcam_pair(0)[0], SolveSchedule(levels=4, grid_step=8, pcg_iters=5, subdomain_px=0)
    if cfg == "cfg3":
        return synthetic.valgaerts_pair(0)[0], SolveSchedule(levels=5, grid_step=8, pcg_iters=5, subdomain_px=0)
    return synthetic.uhd_pair(0)[0], SolveSchedule(levels=5, grid_step=4, pcg_iters=5, subdomain_px=0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--a", default="ref")
    ap.add_argument("--b", default="port")
    ap.add_argument("--cfg", default="cfg1")
    ap.add_argument("--sync", action="store_true")
    args = ap.parse_args()
    imgs, S = case(args.cfg)
    import os
    S.threads = os.cpu_count() or 1
    print(f"# {args.a} vs {args.b}, {args.cfg}, {'lock-step (synced every iteration)' if args.sync else 'free-running'}")

    def on_iter(l, it, A, B, ea, eb):
        gw = A.dims[l][2]
        d = np.abs(A.delta - B.delta)
        k = np.unravel_index(d.argmax(), d.shape)
        wf = int((A.W != B.W).sum())
        print(f"L{l} gn {it}: |ddelta| max {d.max():.2e} med {np.median(d):.2e} at node ({k[0] % gw},{k[0] // gw}) "
              f"field {k[1]}  W flips {wf}  |dnw| {np.abs(A.nw - B.nw).max():.1e}  E_after {ea[1]:.9g} / {eb[1]:.9g}",
              flush=True)

    def on_level(l, A, B):
        print(f"L{l} end: occlusion flips {int((A.vis_prev != B.vis_prev).sum())}"
              + (f"  |dillum| {np.abs(A.hm_prev - B.hm_prev).max():.1e}" if l > 0 else ""), flush=True)

    A, B = lockstep(Solver(LIBS[args.a]()), Solver(LIBS[args.b]()), imgs, S, EnergyParams(), sync=args.sync,
                    on_iter=on_iter, on_level=on_level)
    print(f"final |dtotal| max {np.abs(A.total_prev - B.total_prev).max():.3e}")


if __name__ == "__main__":
    main()
