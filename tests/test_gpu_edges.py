"""GPU: ragged and extreme inputs against the oracle (SURVEY.md §4 edge cases).

Covered here:
  - tiny images (2×2, 3×5);
  - one-pixel-thin and very wide images;
  - odd sizes;
  - grid steps 1, 3, 5, 7, 16 and 32, which exercise the general (non-fast) cell-reduction path;
  - ragged last cells;
  - Schwarz tiles from 1 node to 8×8 nodes;
  - level auto-reduction;
  - invalid inputs (the reference's std::invalid_argument cases) reported as HWF_EINVAL.
Tolerances as in test_gpu_parity.py.
"""
from __future__ import annotations

import numpy as np
import pytest

from paper_1610_07159_b200 import synthetic
from paper_1610_07159_b200.capi import InvalidArgument
from paper_1610_07159_b200.hwflow import EnergyParams, LevelState, SolveSchedule, grid_dims

pytestmark = pytest.mark.gpu

STAGE_RTOL = 1e-9
FLOW_TOL_PX = 1e-3
ENERGY_RTOL = 1e-4

# (65, 49, 8) and (641, 481, 8): (w - 1) and (h - 1) divisible by the step, so the last cell holds step + 1
# pixels and the last k_pixel tiles are 17 x 17 (the largest tile that keeps the 27-product records)
SHAPES = [(2, 2, 1), (3, 5, 1), (17, 13, 3), (41, 9, 5), (200, 3, 7), (65, 33, 16), (70, 70, 32), (5, 120, 2),
          (1, 9, 2), (9, 1, 4), (65, 49, 8), (641, 481, 8)]


def _level(seed, w, h, step):
    rng = np.random.default_rng(seed)
    imgs = rng.random((4, h, w))
    gw, gh = grid_dims(w, h, step)
    return LevelState(imgs, step, rng.normal(0, 0.7, (gw * gh, 6)), rng.normal(0, 0.2, (gw * gh, 6)),
                      rng.integers(0, 16, (h, w)).astype(np.uint8), (rng.random((h, w)) > 0.15).astype(np.uint8),
                      rng.uniform(1, 100, gw * gh), rng.normal(0, 0.02, (4, h, w)),
                      np.array([[0, 0, 0], [0, 0, -1], [0, 1, 0.0]]))


@pytest.mark.parametrize("w,h,step", SHAPES)
def test_stage_seams_on_ragged_shapes(device, oracle, w, h, step):
    lv = _level(w * 1000 + h * 10 + step, w, h, step)
    for P in (EnergyParams(), EnergyParams.preset("facial")):
        a, ra = device.energy(lv, P, residuals=True)
        b, rb = oracle.energy(lv, P, residuals=True)
        for k in ("photo", "grad", "smooth", "epi", "mag", "total"):
            assert getattr(a, k) == pytest.approx(getattr(b, k), rel=STAGE_RTOL, abs=1e-12), k
        np.testing.assert_allclose(ra, rb, rtol=STAGE_RTOL, atol=1e-12)
        Wa, na = device.refresh_weights(lv, P)
        Wb, nb = oracle.refresh_weights(lv, P)
        assert np.array_equal(Wa, Wb)
        np.testing.assert_allclose(na, nb, rtol=1e-9)
        ba, rha, pa = device.build_normal_system(lv, P, 7, 0.1)
        bb, rhb, pb = oracle.build_normal_system(lv, P, 7, 0.1)
        np.testing.assert_allclose(ba, bb, rtol=0, atol=STAGE_RTOL * max(np.abs(bb).max(), 1e-300))
        np.testing.assert_allclose(rha, rhb, rtol=0, atol=STAGE_RTOL * max(np.abs(rhb).max(), 1e-300))
        np.testing.assert_allclose(pa, pb, rtol=1e-7, atol=1e-12 * max(np.abs(pb).max(), 1e-300))


@pytest.mark.parametrize("w,h,step,sub", [(18, 14, 1, 0), (33, 17, 3, 0), (100, 20, 5, 0), (65, 49, 8, 0),
                                          (47, 61, 2, 16),
                                          (47, 61, 3, 16), (96, 64, 4, 8), (96, 64, 16, 16), (130, 70, 32, 16)])
def test_solve_on_ragged_shapes(device, oracle, w, h, step, sub):
    imgs = synthetic.render_pair(w, h, s=(1.5, 0.0), m=(0.5, 0.25), seed=w + h, dtype=np.float64)
    S = SolveSchedule(levels=3, grid_step=step, gn_per_level=[2, 2, 2], pcg_iters=6, patch_iters=3,
                      subdomain_px=sub)
    (ra,), (sa,) = device.solve_batch(imgs[None], EnergyParams(), S)
    rb, sb = oracle.run_scene_flow(imgs, EnergyParams(), S)
    assert len(sa.energy_after) == len(sb.energy_after)
    assert np.abs(ra.grid_total - rb.grid_total).max() < FLOW_TOL_PX
    for l in range(len(sb.energy_after)):
        np.testing.assert_allclose(sa.energy_after[l], sb.energy_after[l], rtol=ENERGY_RTOL)
    assert (ra.vis4 == rb.vis4).mean() > 0.999


def test_invalid_inputs_are_einval(device):
    imgs = synthetic.constant_pair(32, 24)[0]
    P, S = EnergyParams(), SolveSchedule(levels=2, grid_step=8)
    bad = [
        (imgs[None], EnergyParams(w_reg=-1.0), S, None, "weights"),                       # energy.cpp:43-50
        (imgs[None], EnergyParams(eps_huber=0.0), S, None, "eps_huber"),
        (imgs[None], EnergyParams.preset("facial"), S, None, "fundamental"),              # energy.cpp:171
        (imgs[None], P, SolveSchedule(levels=2, grid_step=0), None, "grid_step"),         # warp_grid.cpp:10
        (imgs[None], P, SolveSchedule(levels=2, grid_step=33), None, "grid_step"),
        (imgs[None], P, SolveSchedule(levels=2, grid_step=1, subdomain_px=16), None, "subdomain"),
        (imgs[None], P, SolveSchedule(levels=2, grid_step=8, pcg_iters=-1), None, "negative"),
        (imgs[None], P, SolveSchedule(levels=0, grid_step=8), None, "level"),             # image.cpp:178
        (np.zeros((1, 4, 0, 5), np.uint8), P, S, None, "dims"),                            # image.cpp:101
    ]
    for frames, params, sched, F, what in bad:
        with pytest.raises(InvalidArgument):
            device.solve_batch(frames, params, sched, F)
    (r,), _ = device.solve_batch(imgs[None], P, S)  # the context is still usable afterwards
    assert np.isfinite(r.grid_total).all()


def test_c_abi_nulls_and_limits(device):
    """C-level argument checks (the reference's std::invalid_argument cases) and the schedule maxima."""
    import ctypes as C

    from paper_1610_07159_b200 import capi
    lib, h = device.lib, device.ctx.h
    imgs = synthetic.constant_pair(32, 24)[0]
    P, S = EnergyParams().to_c(), SolveSchedule(levels=2, grid_step=8).to_c()
    fr = capi.Frame4C()
    fr.width, fr.height, fr.dtype = 32, 24, capi.DTYPE_U8
    keep = np.ascontiguousarray(imgs)
    for e in range(4):
        fr.plane[e] = keep[e].ctypes.data
    out = capi.ResultC()
    st = capi.StatsC()
    assert lib.hwf_solve_pair(h, None, C.byref(P), C.byref(S), None, C.byref(out), C.byref(st)) == capi.HWF_EINVAL
    assert lib.hwf_solve_pair(h, C.byref(fr), None, C.byref(S), None, C.byref(out), C.byref(st)) == capi.HWF_EINVAL
    assert lib.hwf_solve_pair(h, C.byref(fr), C.byref(P), None, None, C.byref(out), C.byref(st)) == capi.HWF_EINVAL
    fr.plane[2] = None
    assert lib.hwf_solve_pair(h, C.byref(fr), C.byref(P), C.byref(S), None, C.byref(out), C.byref(st)) == capi.HWF_EINVAL
    assert "plane" in lib.hwf_last_error(h).decode()
    fr.plane[2] = keep[2].ctypes.data
    S_many = SolveSchedule(levels=2, grid_step=8, gn_per_level=[33]).to_c()
    assert lib.hwf_solve_pair(h, C.byref(fr), C.byref(P), C.byref(S_many), None, C.byref(out), C.byref(st)) == capi.HWF_EINVAL
    # the maxima themselves run: 8 levels requested (auto-reduced), 32 GN iterations at a level
    S_max = SolveSchedule(levels=8, grid_step=8, gn_per_level=[32, 1], pcg_iters=2, subdomain_px=0).to_c()
    g = np.empty((5 * 4, 6))
    out.grid_total = g.ctypes.data_as(capi._dp)
    assert lib.hwf_solve_pair(h, C.byref(fr), C.byref(P), C.byref(S_max), None, C.byref(out), C.byref(st)) in (
        capi.HWF_OK, capi.HWF_EDIVERGED)
    assert st.levels_used >= 1 and st.gn_iters[0] == 32


@pytest.mark.parametrize("step,w,h", [(16, 120, 88), (32, 200, 136), (12, 97, 61)])
def test_linearize_large_and_odd_steps_match_oracle(device, oracle, step, w, h):
    """hwf_linearize at grid steps >= 16 (k_pixel's 14-double operand-pair records instead of the 27 products: a tile
    is one cell of up to 33 x 33 pixels) and at a non-power-of-two step (the correctly rounded x / step), through
    the thread-per-node assembly: blocks, rhs and preconditioner against the oracle."""
    rng = np.random.default_rng(step)
    imgs = synthetic.render_pair(w, h, s=(1.2, 0.2), m=(0.5, -0.4), seed=step, dtype=np.float64)
    gw, gh = grid_dims(w, h, step)
    lv = LevelState(imgs, step, rng.normal(0, 0.6, (gw * gh, 6)), rng.normal(0, 0.2, (gw * gh, 6)),
                    rng.integers(0, 16, (h, w)).astype(np.uint8), (rng.random((h, w)) > 0.1).astype(np.uint8),
                    rng.uniform(1, 100, gw * gh), rng.normal(0, 0.02, (4, h, w)),
                    np.array([[0, 0, 0], [0, 0, -1], [0, 1, 0.0]]))  # rectified rig (the facial preset's epipolar term)
    for preset in ("live", "facial"):
        P = EnergyParams.preset(preset)
        a, b = device.build_normal_system(lv, P), oracle.build_normal_system(lv, P)
        for x, y in zip(a, b):
            np.testing.assert_allclose(x, y, rtol=STAGE_RTOL, atol=STAGE_RTOL * np.abs(y).max())
