"""Generate golden vectors from the REFERENCE itself (oracle/_ref/libhwflow_ref.so:
/root/reference/proj/src/*.cpp compiled verbatim against oracle/eigen_shim).

    python tests/golden/make_golden.py

Writes tests/golden/ref_small.npz. Run in the build container (it needs
oracle/_ref, built by `make -C oracle` where /root/reference exists); the npz is
committed so the CPU and GPU test suites can pin the oracle and the device
library without the reference tree.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from paper_1610_07159_b200.hwflow import EnergyParams, LevelState, SolveSchedule, Solver, grid_dims  # noqa: E402
from paper_1610_07159_b200 import synthetic  # noqa: E402


def level_case(seed: int, w: int, h: int, step: int):
    rng = np.random.default_rng(seed)
    imgs = synthetic.render_pair(w, h, s=(1.0, 0.2), m=(0.5, -0.3), seed=seed, dtype=np.float64)
    gw, gh = grid_dims(w, h, step)
    return dict(
        images=imgs,
        total=rng.normal(0, 0.5, (gw * gh, 6)),
        delta=rng.normal(0, 0.2, (gw * gh, 6)),
        vis4=rng.integers(0, 16, (h, w)).astype(np.uint8),
        outlier=(rng.random((h, w)) > 0.2).astype(np.uint8),
        node_w=rng.uniform(1, 100, gw * gh),
        illum=rng.normal(0, 0.02, (4, h, w)),
        F=np.array([[0, 0, 0], [0, 0, -1], [0, 1, 0.0]]),
        step=np.int64(step),
    )


def main() -> None:
    ref = Solver(ROOT / "oracle" / "_ref" / "libhwflow_ref.so")
    assert ref.backend == "reference"
    out: dict[str, np.ndarray] = {}
    # pyramid (image.cpp:100-122): odd sizes exercise partial blocks
    rng = np.random.default_rng(7)
    pimg = rng.integers(0, 256, (4, 13, 11)).astype(np.uint8)
    out["pyr_in"] = pimg
    for l, lev in enumerate(ref.build_pyramid(pimg, 4)):
        out[f"pyr_L{l}"] = lev
    # one level, all terms on (facial preset has w_epi > 0)
    c = level_case(11, 24, 20, 4)
    for k, v in c.items():
        out[f"lv_{k}"] = v
    lv = LevelState(c["images"], int(c["step"]), c["total"], c["delta"], c["vis4"], c["outlier"], c["node_w"],
                    c["illum"], c["F"])
    for pname in ("live", "facial"):
        P = EnergyParams.preset(pname)
        e, R = ref.energy(lv, P, residuals=True)
        out[f"E_{pname}"] = np.array([e.photo, e.grad, e.smooth, e.epi, e.mag, e.total, e.residual_count])
        out[f"R_{pname}"] = R
        W, nw = ref.refresh_weights(lv, P)
        out[f"W_{pname}"], out[f"nw_{pname}"] = W, nw
        b, r, p = ref.build_normal_system(lv, P, 7, 0.0)
        out[f"blocks_{pname}"], out[f"rhs_{pname}"], out[f"pre_{pname}"] = b, r, p
    b, r, _ = ref.build_normal_system(lv, EnergyParams(), 1, 0.25)  # stereo-only + LM
    out["blocks_s_lm"], out["rhs_s_lm"] = b, r
    gw, gh = grid_dims(24, 20, 4)
    x, tr = ref.pcg_solve(gw, gh, out["blocks_live"], out["rhs_live"], 10, trace=True)
    out["pcg_x"], out["pcg_trace"] = x, tr
    out["schwarz_x"] = ref.schwarz_iterate(gw, gh, 4, out["blocks_live"], out["rhs_live"], 3, 4)
    # Gauss-Newton level (solver.cpp:484-532), both solve modes
    g = level_case(5, 40, 32, 8)
    gw, gh = grid_dims(40, 32, 8)
    lv2 = LevelState(g["images"], 8, np.zeros((gw * gh, 6)), np.zeros((gw * gh, 6)))
    out["gn_images"] = g["images"]
    for mode, sub in (("schwarz", 16), ("global", 0)):
        S = SolveSchedule(levels=1, grid_step=8, pcg_iters=5, patch_iters=5, subdomain_px=sub)
        d, W, nw, eb, ea = ref.gauss_newton(lv2, np.zeros((gw * gh, 6)), EnergyParams(), S, 3)
        out[f"gn_{mode}_delta"], out[f"gn_{mode}_W"], out[f"gn_{mode}_nw"] = d, W, nw
        out[f"gn_{mode}_eb"], out[f"gn_{mode}_ea"] = eb, ea
    # full cfg1 solves (Algorithm 1 with the reference's own gauss_newton), for the
    # end-to-end reproducibility bar: the reference is ill-conditioned on the full
    # schedule, so its own build and the oracle port differ by ~1e-2 px there.
    port = Solver(ROOT / "oracle" / "_build" / "libhwflow_oracle.so")
    imgs, _ = synthetic.constant_pair(320, 240)
    out["cfg1_images"] = imgs
    for tag, gl in (("full", [5]), ("short", [5, 5, 3])):
        S = SolveSchedule(levels=3, grid_step=8, gn_per_level=gl, pcg_iters=10, subdomain_px=0)
        r, st = ref.run_scene_flow(imgs, EnergyParams(), S)
        q, _ = port.run_scene_flow(imgs, EnergyParams(), S)
        out[f"cfg1_{tag}_grid"], out[f"cfg1_{tag}_vis4"] = r.grid_total, r.vis4
        out[f"cfg1_{tag}_E"] = np.array(st.final_energy())
        out[f"cfg1_{tag}_port_vs_ref"] = np.array(np.abs(q.grid_total - r.grid_total).max())
    path = ROOT / "tests" / "golden" / "ref_small.npz"
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({path.stat().st_size} bytes, {len(out)} arrays)")


if __name__ == "__main__":
    main()
