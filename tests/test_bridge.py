"""GPU: the reference-side bridge (include/hwflow_bridge.hpp) executed.

oracle/_ref/bridge_demo is a program written against the reference's own C++ API (hwflow::Image, WarpGrid,
PixelWeights, EnergyContext, SolveSchedule; /root/reference/proj/include/hwflow/*.hpp), linked with the
reference's sources (CPU, compiled verbatim by oracle/Makefile) and with libhwflow_cuda.so. It calls
hwflow::gauss_newton / build_pyramid on the CPU and hwflow::b200::gauss_newton / build_pyramid /
run_scene_flow on the B200 with the same value types (oracle/bridge_demo.cpp). It is built in the build
container (it needs the reference headers) and travels to the GPU box with the tree.
"""
from __future__ import annotations

import json
import subprocess

import numpy as np
import pytest

from paper_1610_07159_b200 import build
from paper_1610_07159_b200.hwflow import EnergyParams, SolveSchedule

pytestmark = pytest.mark.gpu

DEMO = build.ORACLE_DIR / "_ref" / "bridge_demo"


def test_bridge_runs_reference_api_on_device(oracle, tmp_path):
    if not DEMO.exists():
        pytest.skip("oracle/_ref/bridge_demo not built (needs /root/reference at build time)")
    out = tmp_path / "flow.bin"
    r = subprocess.run([str(DEMO), str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["pyramid_bit_exact"] is True  # image.cpp:100-122,177-185
    # gauss_newton (solver.cpp:484-532), 3 GN x 5 global PCG, reference value types on both sides
    assert d["gn_delta_max"] < 1e-9 and d["gn_energy_rel"] < 1e-9 and d["gn_node_w_rel"] < 1e-9
    assert d["gn_W_exact"] is True
    assert d["pcg_trace_shape"] is True and d["pcg_trace_rel"] < 1e-8  # SolveSchedule::pcg_trace (solver.cpp:508-513)
    # SolverDivergence (core.hpp:19) / std::invalid_argument (energy.cpp:43-50) thrown where the reference throws
    assert d["divergence_dev"] == d["divergence_ref"], d
    assert d["invalid_ref"] == 2 and d["invalid_dev"] == 2
    # assemble_jacobian (solver.cpp:247-314) with the negate_field hook: the reference's triplets, in order
    assert d["jacobian_same_entries"] is True and d["jacobian_nnz"] > 0 and d["jacobian_rel"] < 1e-9
    # run_scene_flow through the bridge vs the oracle's Algorithm 1 on the same images
    w, h = d["solve_width"], d["solve_height"]
    N = w * h
    raw = out.read_bytes()
    imgs = np.frombuffer(raw, np.float64, 4 * N).reshape(4, h, w)
    f = np.frombuffer(raw, np.float64, 7 * N, offset=8 * 4 * N)
    s, m, dd, disp = f[:2 * N].reshape(h, w, 2), f[2 * N:4 * N].reshape(h, w, 2), f[4 * N:6 * N].reshape(h, w, 2), f[6 * N:]
    vis = np.frombuffer(raw, np.uint8, N, offset=8 * 11 * N).reshape(h, w)
    S = SolveSchedule(levels=3, grid_step=8, subdomain_px=0, pcg_iters=5)
    q, st = oracle.run_scene_flow(imgs, EnergyParams(), S)
    assert d["finest_gn_iters"] == len(st.energy_after[0])
    assert np.abs(s - q.s).max() < 1e-3 and np.abs(m - q.m).max() < 1e-3 and np.abs(dd - q.d).max() < 1e-3
    assert np.abs(disp.reshape(h, w) - q.disparity).max() < 2e-3
    assert np.array_equal(vis, q.vis4)
