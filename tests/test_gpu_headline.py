"""GPU: the schedules bench.py reports, end to end and in lock step, against the reference.

End to end (against tests/golden/ref_headline.npz, made by tests/golden/make_golden_headline.py from the
reference build, oracle/_ref):
- cfg2 headline (bench.py: 640x480, 4 levels, 8 px grid, GN 2,2,5,5, 5 global PCG, live preset), four pairs
  embedded in a 256-pair batch (bench.py's batch): grid within 1e-3 px (north_star), disparity within 2e-3 px,
  every per-level energy within 1e-4 relative, visibility masks bit-exact.
- cfg1 full (BASELINE configs[0]), cfg3 and cfg5 at bench.py's schedules: on these schedules the reference's
  full-step Gauss-Newton (solver.cpp:484-532) amplifies one-ulp differences by ~1e12 at a few nodes, so the
  reference is not reproducible to 1e-3 px against ITSELF (a one-ulp change of its input images moves its
  output by up to 9e-3 px at cfg1 and 6e-2 px at cfg3; profiles/r2_parity_notes.md). The device must
  deviate from the reference no more than the reference deviates from itself: each summary of the per-node
  deviation (max, p99, p50, count > 1e-3 px) at most the largest over 8 one-ulp input perturbations of the
  reference (and the oracle port); at cfg1 also per node, |dev - ref| <= env + 1e-3 px with env the per-node
  max of those excursions. Energies within 1e-4 relative everywhere.

Lock step (tests/lockstep.py, against the oracle port, which tests/test_oracle.py pins to the reference in lock
step at 1e-12): at EVERY level and GN iteration of the full schedules, device and oracle are handed the same
state and take one iteration; the device's delta must be within 1e-9 px, W bit-exact, node weights and
energies within 1e-9 relative; occlusion masks bit-exact and illumination maps within 1e-12 on the same flows.
This is the schedule-length-independent statement of parity.
"""
from __future__ import annotations

import numpy as np
import pytest

from lockstep import lockstep
from paper_1610_07159_b200 import synthetic
from paper_1610_07159_b200.hwflow import EnergyParams, SolveSchedule, grid_dims

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gold():
    from pathlib import Path
    return dict(np.load(Path(__file__).parent / "golden" / "ref_headline.npz"))


def headline_schedule():
    import bench
    return bench.schedule("global")


def interp_grid(grid: np.ndarray, w: int, h: int, step: int) -> np.ndarray:
    """WarpGrid::interpolate (warp_grid.cpp:41-65) of a (G, 6) grid at every pixel: (h, w, 6)."""
    gw, gh = grid_dims(w, h, step)
    g = grid.reshape(gh, gw, 6)
    u, v = np.arange(w) / step, np.arange(h) / step
    a0 = np.clip(np.floor(u).astype(int), 0, gw - 2)
    b0 = np.clip(np.floor(v).astype(int), 0, gh - 2)
    fu = np.clip(u - a0, 0.0, 1.0)[None, :, None]
    fv = np.clip(v - b0, 0.0, 1.0)[:, None, None]
    B0, A0 = np.meshgrid(b0, a0, indexing="ij")
    return ((1 - fu) * (1 - fv) * g[B0, A0] + fu * (1 - fv) * g[B0, A0 + 1] + (1 - fu) * fv * g[B0 + 1, A0]
            + fu * fv * g[B0 + 1, A0 + 1])


def flat(st):
    return (np.concatenate([np.array(e) for e in st.energy_before]),
            np.concatenate([np.array(e) for e in st.energy_after]))


SLOTS = (0, 85, 170, 255)


def test_cfg2_headline_schedule_batch256(device, gold):
    """bench.py's exact workload: 256 pairs per batch, the golden pairs at four slots, the other 252 slots
    distinct pairs (x-rolled copies) so a cross-pair indexing error would show."""
    S = headline_schedule()
    pairs = [synthetic.webcam_pair(i)[0] for i in range(4)]
    frames = np.empty((256, 4, 480, 640), np.uint8)
    for k in range(256):
        frames[k] = np.roll(pairs[k % 4], 1 + k // 4, axis=2)
    for i, k in enumerate(SLOTS):
        frames[k] = pairs[i]
    res, st = device.solve_batch(frames, EnergyParams(), S, outputs=("grid_total", "vis4"))
    for i, k in enumerate(SLOTS):
        d = np.abs(res[k].grid_total - gold[f"cfg2_{i}_grid"])
        assert d.max() < 1e-3, (i, d.max())
        assert np.array_equal(res[k].vis4, gold[f"cfg2_{i}_vis4"]), (i, int((res[k].vis4 != gold[f"cfg2_{i}_vis4"]).sum()))
        eb, ea = flat(st[k])
        np.testing.assert_allclose(eb, gold[f"cfg2_{i}_eb"], rtol=1e-4)
        np.testing.assert_allclose(ea, gold[f"cfg2_{i}_ea"], rtol=1e-4)
    # the same four pairs alone (B = 4): bitwise the batch-256 results (determinism contract), with the dense
    # FlowResult (geometry.hpp:26-37) checked against WarpGrid::interpolate of the reference grid
    small, _ = device.solve_batch(np.stack(pairs), EnergyParams(), S)
    for i, k in enumerate(SLOTS):
        assert np.array_equal(small[i].grid_total, res[k].grid_total)
        ref_px = interp_grid(gold[f"cfg2_{i}_grid"], 640, 480, 8)
        assert np.abs(small[i].disparity - 2.0 * ref_px[..., 0]).max() < 2e-3
        assert np.abs(small[i].s - ref_px[..., 0:2]).max() < 1e-3
        assert np.abs(small[i].m - ref_px[..., 2:4]).max() < 1e-3
        assert np.abs(small[i].d - ref_px[..., 4:6]).max() < 1e-3


STAT_NAMES = ("max", "p99", "p50", "nodes>1e-3")


def dev_stats(d: np.ndarray) -> np.ndarray:
    return np.array([d.max(), np.percentile(d, 99), np.percentile(d, 50), (d > 1e-3).sum()])


def _within_reference_distribution(gold, tag, d):
    """The device's per-node deviation from the reference, summarised as max / p99 / p50 / count > 1e-3 px,
    is no larger than the largest the reference itself shows under one-ulp input perturbations
    (tests/golden/make_golden_headline.py, K draws) or against the oracle port."""
    draws = np.vstack([gold[f"{tag}_draw_stats"], gold[f"{tag}_port_stats"][None]])
    mine, worst = dev_stats(d), draws.max(0)
    for name, a, b in zip(STAT_NAMES, mine, worst):
        assert a <= b, (tag, name, a, b, draws)
    return mine


def _solve_and_energies(device, gold, tag, imgs, S):
    (r,), (s,) = device.solve_batch(imgs[None], EnergyParams(), S, outputs=("grid_total",))
    eb, ea = flat(s)
    np.testing.assert_allclose(eb, gold[f"{tag}_eb"], rtol=1e-4)
    np.testing.assert_allclose(ea, gold[f"{tag}_ea"], rtol=1e-4)
    return r.grid_total


def test_cfg1_full_schedule_within_reference_envelope(device, gold):
    """BASELINE configs[0] (cfg1, 3 levels x 5 GN x 10 PCG): per node |dev - ref| <= env + 1e-3 px, env the
    per-node max of the reference's own one-ulp excursions and the port's deviation; and in distribution."""
    imgs = synthetic.constant_pair(320, 240)[0]
    S = SolveSchedule(levels=3, grid_step=8, gn_per_level=[5], pcg_iters=10, subdomain_px=0)
    g = _solve_and_energies(device, gold, "cfg1_full", imgs, S)
    d = np.abs(g - gold["cfg1_full_grid"]).max(1)
    env = gold["cfg1_full_env"].astype(np.float64)
    bad = np.flatnonzero(d > env + 1e-3)
    assert bad.size == 0, (bad[:8], d[bad[:8]], env[bad[:8]])
    _within_reference_distribution(gold, "cfg1_full", d)


def test_cfg3_bench_schedule_within_reference_distribution(device, gold):
    imgs = synthetic.valgaerts_pair(0)[0]
    S = SolveSchedule(levels=5, grid_step=8, pcg_iters=5, subdomain_px=0)
    g = _solve_and_energies(device, gold, "cfg3", imgs, S)
    _within_reference_distribution(gold, "cfg3", np.abs(g - gold["cfg3_grid"]).max(1))


def test_cfg5_bench_schedule_within_reference_distribution(device, gold, request):
    """cfg5 (3840x2160, 4 px grid, 5 levels, GN 2,2,5,5,5): energies vs the golden within 1e-4; the grid (25 MB,
    not committed) against the reference build run here when it is present (oracle/_ref travels with the tree
    from the build container)."""
    import os
    imgs = synthetic.uhd_pair(0)[0]
    S = SolveSchedule(levels=5, grid_step=4, pcg_iters=5, subdomain_px=0)
    g = _solve_and_energies(device, gold, "cfg5", imgs, S)
    from paper_1610_07159_b200 import build
    if not build.REF_LIB.exists():
        pytest.skip("oracle/_ref absent: energies checked, grid not")
    reference = request.getfixturevalue("reference")
    S.threads = os.cpu_count() or 1
    r, _ = reference.run_scene_flow(imgs, EnergyParams(), S)
    _within_reference_distribution(gold, "cfg5", np.abs(g - r.grid_total).max(1))


# ---- lock step over the full schedules ---------------------------------------------------------
LOCKSTEP_CASES = {
    "cfg1_full": lambda: (synthetic.constant_pair(320, 240)[0],
                          SolveSchedule(levels=3, grid_step=8, gn_per_level=[5], pcg_iters=10, subdomain_px=0)),
    "cfg2_headline": lambda: (synthetic.webcam_pair(1)[0], headline_schedule()),
    "cfg3": lambda: (synthetic.valgaerts_pair(0)[0], SolveSchedule(levels=5, grid_step=8, pcg_iters=5,
                                                                   subdomain_px=0)),
    "cfg5": lambda: (synthetic.uhd_pair(0)[0], SolveSchedule(levels=5, grid_step=4, pcg_iters=5, subdomain_px=0)),
}


@pytest.mark.parametrize("case", list(LOCKSTEP_CASES))
def test_lockstep_every_gn_iteration(device, oracle, case):
    import os
    imgs, S = LOCKSTEP_CASES[case]()
    S.threads = os.cpu_count() or 1
    worst = {"delta": 0.0, "nw": 0.0, "E": 0.0}

    def on_iter(l, it, A, B, ea, eb):
        scale = max(1.0, float(np.abs(A.delta).max()))
        d = float(np.abs(A.delta - B.delta).max())
        worst["delta"] = max(worst["delta"], d)
        assert d < 1e-9 * scale, (l, it, d)
        assert np.array_equal(A.W, B.W), (l, it, int((A.W != B.W).sum()))
        nwr = float((np.abs(A.nw - B.nw) / A.nw).max())
        worst["nw"] = max(worst["nw"], nwr)
        assert nwr < 1e-9, (l, it, nwr)
        for x, y in zip(ea, eb):
            worst["E"] = max(worst["E"], abs(x - y) / abs(x))
            assert y == pytest.approx(x, rel=1e-9), (l, it)

    def on_level(l, A, B):
        assert np.array_equal(A.vis_prev, B.vis_prev), (l, int((A.vis_prev != B.vis_prev).sum()))
        if l > 0:
            assert np.abs(A.hm_prev - B.hm_prev).max() < 1e-12, l

    # a = oracle (the state both are handed), b = device
    lockstep(oracle, device, imgs, S, EnergyParams(), sync=True, on_iter=on_iter, on_level=on_level)
    print(case, worst)
