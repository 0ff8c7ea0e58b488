"""Diagnostic: the reference's own reproducibility envelope vs the device's deviation from it.

For a configuration, runs the reference build (oracle/_ref) on the u8 frames and on K copies of the same frames
as f64 with a random half of the pixels nudged by one ulp (np.nextafter), the oracle port, and (when a GPU is
present) the device. Prints per-node statistics of |x - ref| (max over the 6 fields) for each, and how many nodes
exceed env + 1e-3 px where env is the per-node max over the perturbed runs.

    python tools/parity_envelope.py [--cfg cfg1|cfg2|cfg3|cfg5] [--k 4] [--out gpurun_out/env_cfg1.npz]
"""
from __future__ import annotations

import argparse
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
from hier_trace import case  # noqa: E402

from paper_1610_07159_b200 import build  # noqa: E402
from paper_1610_07159_b200.hwflow import EnergyParams, Solver  # noqa: E402


def ulp_perturbed(imgs: np.ndarray, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    f = imgs.astype(np.float64) / 255.0
    return np.where(rng.random(f.shape) < 0.5, np.nextafter(f, 2.0), f)


def stats(tag, d, env=None):
    q = np.percentile(d, [50, 99])
    s = f"{tag:>10}: max {d.max():.3e} p99 {q[1]:.2e} p50 {q[0]:.2e} nodes>1e-3 {int((d > 1e-3).sum())}"
    if env is not None:
        s += f" | exceeds env+1e-3: {int((d > env + 1e-3).sum())}, exceeds 2env+1e-3: {int((d > 2 * env + 1e-3).sum())}"
    print(s, flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="cfg1")
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    imgs, S = case(args.cfg)
    S.threads = os.cpu_count() or 1
    P = EnergyParams()
    ref = Solver(build.REF_LIB)
    r0, s0 = ref.run_scene_flow(imgs, P, S)
    pert = []
    for k in range(args.k):
        rk, _ = ref.run_scene_flow(ulp_perturbed(imgs, k), P, S)
        pert.append(np.abs(rk.grid_total - r0.grid_total).max(1))
    env = np.max(pert, axis=0) if pert else np.zeros(r0.grid_total.shape[0])
    print(f"# {args.cfg}: per-node |x - ref| (px), env = max over {args.k} one-ulp input perturbations of the reference")
    for k, d in enumerate(pert):
        others = np.max([p for j, p in enumerate(pert) if j != k], axis=0) if len(pert) > 1 else None
        stats(f"ref+ulp{k}", d, others)
    q, _ = Solver(build.ORACLE_LIB).run_scene_flow(imgs, P, S)
    dq = np.abs(q.grid_total - r0.grid_total).max(1)
    stats("port", dq, env)
    out = {"ref": r0.grid_total, "env": env, "port": dq}
    try:
        import torch
        if torch.cuda.is_available():
            dev = Solver(build.CUDA_LIB)
            (a,), (sa,) = dev.solve_batch(imgs[None], P, S)
            dd = np.abs(a.grid_total - r0.grid_total).max(1)
            stats("device", dd, env)
            print(f"    device energy rel {abs(sa.final_energy() - s0.final_energy()) / s0.final_energy():.2e}")
            out["device"] = dd
    except ImportError:
        pass
    if args.out:
        np.savez_compressed(args.out, **out)


if __name__ == "__main__":
    main()
