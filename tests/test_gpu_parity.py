"""GPU: device (libhwflow_cuda.so, sm_100a) vs the CPU oracle through the C-ABI.

Tolerances (BASELINE.json north_star): pyramid and occlusion masks bit-exact;
per-node flow within 1e-3 px max-abs after a fixed GN x PCG schedule; final
energy within 1e-4 relative. Stage seams are checked tighter (FP64 on both
sides, differing only in summation order): 1e-9 relative unless stated.
"""
from __future__ import annotations

import numpy as np
import pytest

from paper_1610_07159_b200 import synthetic
from paper_1610_07159_b200.hwflow import EnergyParams, LevelState, SolveSchedule, SolverDivergence, grid_dims

pytestmark = pytest.mark.gpu

FLOW_TOL_PX = 1e-3
ENERGY_RTOL = 1e-4
STAGE_RTOL = 1e-9


def _golden_level(g, **over):
    kw = dict(images=g["lv_images"], grid_step=int(g["lv_step"]), total=g["lv_total"], delta=g["lv_delta"],
              vis4=g["lv_vis4"], outlier=g["lv_outlier"], node_w=g["lv_node_w"], illum=g["lv_illum"],
              fundamental=g["lv_F"])
    kw.update(over)
    return LevelState(**kw)


def _random_level(seed, w, h, step, illum=True):
    rng = np.random.default_rng(seed)
    imgs = synthetic.render_pair(w, h, s=(1.0, 0.3), m=(0.4, -0.6), seed=seed, dtype=np.float64)
    gw, gh = grid_dims(w, h, step)
    return LevelState(imgs, step, rng.normal(0, 0.7, (gw * gh, 6)), rng.normal(0, 0.2, (gw * gh, 6)),
                      rng.integers(0, 16, (h, w)).astype(np.uint8), (rng.random((h, w)) > 0.15).astype(np.uint8),
                      rng.uniform(1, 100, gw * gh), rng.normal(0, 0.02, (4, h, w)) if illum else None,
                      np.array([[0, 0, 0], [0, 0, -1], [0, 1, 0.0]]))


# ---- pyramid: bit-exact -------------------------------------------------------------
def test_pyramid_bit_exact(device, oracle, golden):
    for l, lev in enumerate(device.build_pyramid(golden["pyr_in"], 4)):
        assert np.array_equal(lev, golden[f"pyr_L{l}"]), l
    rng = np.random.default_rng(3)
    for shape in ((4, 480, 640), (4, 37, 53), (4, 1, 9)):
        im = rng.integers(0, 256, shape).astype(np.uint8)
        for a, b in zip(device.build_pyramid(im, 4), oracle.build_pyramid(im, 4)):
            assert np.array_equal(a, b)
    f = rng.normal(0.5, 0.4, (4, 31, 17))  # F64 input: clamped to [0,1]
    for a, b in zip(device.build_pyramid(f, 3), oracle.build_pyramid(f, 3)):
        assert np.array_equal(a, b)


# ---- energy / weights / linearization ------------------------------------------------
@pytest.mark.parametrize("preset", ["live", "facial", "stereo-hq"])
def test_energy_matches_oracle(device, oracle, golden, preset):
    P = EnergyParams.preset(preset)
    for lv in (_golden_level(golden), _random_level(2, 70, 45, 8), _random_level(4, 33, 29, 2, illum=False)):
        a, _ = device.energy(lv, P)
        b, _ = oracle.energy(lv, P)
        for k in ("photo", "grad", "smooth", "epi", "mag", "total"):
            assert getattr(a, k) == pytest.approx(getattr(b, k), rel=STAGE_RTOL, abs=1e-12), k
        assert a.residual_count == b.residual_count


def test_refresh_weights_match_oracle(device, oracle, golden):
    for lv in (_golden_level(golden), _random_level(5, 64, 40, 8), _random_level(6, 35, 21, 4)):
        for P in (EnergyParams(), EnergyParams.preset("facial")):
            Wa, na = device.refresh_weights(lv, P)
            Wb, nb = oracle.refresh_weights(lv, P)
            assert np.array_equal(Wa, Wb)
            np.testing.assert_allclose(na, nb, rtol=1e-9)


@pytest.mark.parametrize("active,lm", [(7, 0.0), (1, 0.0), (5, 0.3)])
def test_linearize_matches_oracle(device, oracle, golden, active, lm):
    for lv in (_golden_level(golden), _random_level(8, 50, 34, 8), _random_level(9, 27, 19, 2)):
        for P in (EnergyParams(), EnergyParams.preset("stereo-hq")):
            ba, ra, pa = device.build_normal_system(lv, P, active, lm)
            bb, rb, pb = oracle.build_normal_system(lv, P, active, lm)
            np.testing.assert_allclose(ba, bb, rtol=0, atol=STAGE_RTOL * np.abs(bb).max())
            np.testing.assert_allclose(ra, rb, rtol=0, atol=STAGE_RTOL * np.abs(rb).max())
            np.testing.assert_allclose(pa, pb, rtol=1e-7, atol=1e-12 * np.abs(pb).max())


def test_pcg_and_schwarz_match_reference_golden(device, golden):
    gw, gh = grid_dims(24, 20, 4)
    x, tr = device.pcg_solve(gw, gh, golden["blocks_live"], golden["rhs_live"], 10, trace=True)
    np.testing.assert_allclose(x, golden["pcg_x"], rtol=0, atol=1e-9 * np.abs(golden["pcg_x"]).max())
    np.testing.assert_allclose(tr, golden["pcg_trace"], rtol=1e-8)
    xs = device.schwarz_iterate(gw, gh, 4, golden["blocks_live"], golden["rhs_live"], 3, 4)
    np.testing.assert_allclose(xs, golden["schwarz_x"], rtol=0, atol=1e-9 * np.abs(golden["schwarz_x"]).max())


def test_schwarz_step8_and_global_match_oracle(device, oracle):
    lv = _random_level(12, 96, 64, 8)
    b, r, _ = oracle.build_normal_system(lv, EnergyParams())
    gw, gh = grid_dims(96, 64, 8)
    for pi, ki in ((1, 5), (5, 5), (3, 10)):
        xa = device.schwarz_iterate(gw, gh, 8, b, r, pi, ki)
        xb = oracle.schwarz_iterate(gw, gh, 8, b, r, pi, ki)
        np.testing.assert_allclose(xa, xb, rtol=0, atol=1e-9 * np.abs(xb).max())
    xa = device.pcg_solve(gw, gh, b, r, 25)
    xb = oracle.pcg_solve(gw, gh, b, r, 25)
    np.testing.assert_allclose(xa, xb, rtol=0, atol=1e-9 * np.abs(xb).max())


@pytest.mark.parametrize("mode,sub", [("schwarz", 16), ("global", 0)])
def test_gauss_newton_level_matches_reference_golden(device, golden, mode, sub):
    gw, gh = grid_dims(40, 32, 8)
    lv = LevelState(golden["gn_images"], 8, np.zeros((gw * gh, 6)), np.zeros((gw * gh, 6)))
    S = SolveSchedule(levels=1, grid_step=8, pcg_iters=5, patch_iters=5, subdomain_px=sub)
    d, W, nw, eb, ea = device.gauss_newton(lv, np.zeros((gw * gh, 6)), EnergyParams(), S, 3)
    assert np.abs(d - golden[f"gn_{mode}_delta"]).max() < FLOW_TOL_PX
    assert np.array_equal(W, golden[f"gn_{mode}_W"])
    np.testing.assert_allclose(eb, golden[f"gn_{mode}_eb"], rtol=ENERGY_RTOL)
    np.testing.assert_allclose(ea, golden[f"gn_{mode}_ea"], rtol=ENERGY_RTOL)


def test_gauss_newton_pcg_trace_matches_oracle(device, oracle, golden):
    """SolveSchedule::pcg_trace in global mode (solver.cpp:508-513) through hwf_gn_level_trace."""
    gw, gh = grid_dims(40, 32, 8)
    lv = LevelState(golden["gn_images"], 8, np.zeros((gw * gh, 6)), np.zeros((gw * gh, 6)))
    S = SolveSchedule(levels=1, grid_step=8, pcg_iters=5, subdomain_px=0)
    a = device.gauss_newton(lv, np.zeros((gw * gh, 6)), EnergyParams(), S, 3, pcg_trace=True)
    b = oracle.gauss_newton(lv, np.zeros((gw * gh, 6)), EnergyParams(), S, 3, pcg_trace=True)
    np.testing.assert_allclose(a[5], b[5], rtol=1e-6)  # norms after 3 GN iterations of an ill-conditioned level
    np.testing.assert_allclose(a[5][0], b[5][0], rtol=1e-9)


# ---- occlusion (bit-exact on identical input flows), illumination, prolongation --------
def _wavy_total(seed, w, h, step, amp):
    rng = np.random.default_rng(seed)
    gw, gh = grid_dims(w, h, step)
    t = rng.normal(0, amp, (gw * gh, 6))
    t[:, 0] += 3.0
    return t


def test_occlusion_bit_exact(device, oracle):
    for seed, (w, h, step, amp) in enumerate(((64, 48, 8, 0.8), (100, 61, 4, 1.5), (33, 17, 2, 0.6), (640, 480, 8, 2.0))):
        t = _wavy_total(seed, w, h, step, amp)
        va = device.compute_occlusion_maps(w, h, step, t)
        vb = oracle.compute_occlusion_maps(w, h, step, t)
        assert np.array_equal(va, vb)
        assert (va != 0x0F).any()  # the case actually occludes something
    gw, gh = grid_dims(21, 13, 4)
    assert np.all(device.compute_occlusion_maps(21, 13, 4, np.zeros((gw * gh, 6))) == 0x0F)


def test_occlusion_two_layer_scene(device, oracle):
    # foreground band with larger disparity: background beside it is occluded in one camera
    w, h, step = 96, 64, 4
    gw, gh = grid_dims(w, h, step)
    t = np.zeros((gw * gh, 6))
    t[:, 0] = 1.0
    a = np.arange(gw * gh) % gw
    t[(a >= 10) & (a <= 14), 0] = 5.0
    va, vb = device.compute_occlusion_maps(w, h, step, t), oracle.compute_occlusion_maps(w, h, step, t)
    assert np.array_equal(va, vb)
    assert ((va & 0b0101) != 0b0101).any() or ((va & 0b1010) != 0b1010).any()


def test_illumination_matches_oracle(device, oracle):
    lv = _random_level(21, 80, 60, 8)
    vis = oracle.compute_occlusion_maps(80, 60, 8, lv.total)
    ha = device.compute_illumination_maps(lv.images, 8, lv.total, vis)
    hb = oracle.compute_illumination_maps(lv.images, 8, lv.total, vis)
    np.testing.assert_allclose(ha, hb, rtol=0, atol=1e-12)


@pytest.mark.parametrize("w,h,step", [(97, 61, 8), (23, 17, 4), (330, 20, 8), (161, 9, 2)])
def test_illumination_ragged_widths(device, oracle, w, h, step):
    """The windowed blur (160-wide row segments, 8-row column windows) on widths and heights that are not multiples
    of either, including rows shorter than the 10 px radius."""
    lv = _random_level(w + h, w, h, step)
    vis = oracle.compute_occlusion_maps(w, h, step, lv.total)
    ha = device.compute_illumination_maps(lv.images, step, lv.total, vis)
    hb = oracle.compute_illumination_maps(lv.images, step, lv.total, vis)
    np.testing.assert_allclose(ha, hb, rtol=0, atol=1e-12)


@pytest.mark.parametrize("wc,hc,wf,hf,step", [(40, 30, 80, 60, 8), (21, 11, 41, 21, 4), (3, 2, 5, 3, 2),
                                             (160, 120, 320, 240, 8), (1, 7, 2, 13, 1)])
def test_mask_prolongation_bit_exact(device, oracle, wc, hc, wf, hf, step):
    """Masks alone (the pipeline's k_prolong_vis: 4 pixels per thread, the quarter-weight vote as bitwise ops), on
    fine widths that are not multiples of 4 and single-column coarse levels."""
    rng = np.random.default_rng(wc * 7 + hf)
    gwc, ghc = grid_dims(wc, hc, step)
    tc = rng.normal(0, 2, (gwc * ghc, 6))
    vc = rng.integers(0, 16, (hc, wc)).astype(np.uint8)
    a = device.prolongate(wc, hc, wf, hf, step, tc, vc, None)
    b = oracle.prolongate(wc, hc, wf, hf, step, tc, vc, None)
    for x, y in zip(a, b):
        if x is not None or y is not None:
            assert np.array_equal(x, y)


def test_prolongation_bit_exact(device, oracle):
    rng = np.random.default_rng(2)
    for (wc, hc, wf, hf, step) in ((40, 30, 80, 60, 8), (21, 11, 41, 21, 4), (160, 120, 320, 240, 8)):
        gwc, ghc = grid_dims(wc, hc, step)
        tc = rng.normal(0, 2, (gwc * ghc, 6))
        vc = rng.integers(0, 16, (hc, wc)).astype(np.uint8)
        hm = rng.normal(0, 0.1, (2, hc, wc))
        a = device.prolongate(wc, hc, wf, hf, step, tc, vc, hm)
        b = oracle.prolongate(wc, hc, wf, hf, step, tc, vc, hm)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)


# ---- Algorithm 1 end to end -------------------------------------------------------
def _check_solve(device, oracle, imgs, P, S, F=None):
    (ra,), (sa,) = device.solve_batch(imgs[None], P, S, F)
    rb, sb = oracle.run_scene_flow(imgs, P, S, F)
    assert np.abs(ra.grid_total - rb.grid_total).max() < FLOW_TOL_PX
    assert np.abs(ra.disparity - rb.disparity).max() < 2 * FLOW_TOL_PX
    for l in range(len(sb.energy_after)):
        np.testing.assert_allclose(sa.energy_before[l], sb.energy_before[l], rtol=ENERGY_RTOL)
        np.testing.assert_allclose(sa.energy_after[l], sb.energy_after[l], rtol=ENERGY_RTOL)
    agree = (ra.vis4 == rb.vis4).mean()
    assert agree > 0.999, agree  # masks bit-exact on identical flows; flows differ by <1e-3 px here
    return ra, sa


def test_solve_cfg1_global_pcg(device, oracle, golden):
    """cfg1 (320x240, 3 levels, 8 px grid, 10 PCG) over 13 GN iterations: <= 1e-3 px vs the oracle
    AND vs the reference build's own output (golden)."""
    imgs, gt = synthetic.constant_pair(320, 240)
    assert np.array_equal(imgs, golden["cfg1_images"])
    S = SolveSchedule(levels=3, grid_step=8, gn_per_level=[5, 5, 3], pcg_iters=10, subdomain_px=0)
    r, s = _check_solve(device, oracle, imgs, EnergyParams(), S)
    assert np.abs(r.grid_total - golden["cfg1_short_grid"]).max() < FLOW_TOL_PX
    assert s.final_energy() == pytest.approx(float(golden["cfg1_short_E"]), rel=ENERGY_RTOL)
    assert abs(np.median(r.s[..., 0]) - gt["s"][0]) < 0.25


def test_solve_short_schwarz_schedule(device, oracle):
    imgs, _ = synthetic.webcam_pair(3, 160, 120)
    S = SolveSchedule(levels=3, grid_step=8, gn_per_level=[1, 1, 2], pcg_iters=5, patch_iters=5, subdomain_px=16)
    _check_solve(device, oracle, imgs, EnergyParams(), S)


def test_solve_epipolar_and_stereo_only(device, oracle):
    imgs, _ = synthetic.constant_pair(96, 64)
    F = np.array([[0, 0, 0], [0, 0, -1], [0, 1, 0.0]])
    S = SolveSchedule(levels=2, grid_step=4, gn_per_level=[2], pcg_iters=6, subdomain_px=0, lm_lambda=0.1)
    _check_solve(device, oracle, imgs, EnergyParams.preset("facial"), S, F)
    S1 = SolveSchedule(levels=2, grid_step=8, gn_per_level=[2], pcg_iters=6, subdomain_px=0, active_fields=1,
                       coarse_s_offset=(0.5, 0.0))
    r, _ = _check_solve(device, oracle, imgs, EnergyParams(), S1)
    assert np.abs(r.grid_total[:, 2:]).max() == 0.0  # m, d pinned (solver.cpp:218-220)


@pytest.mark.parametrize("mode", ["stereo_only", "stereo_hq_epipolar"])
def test_cfg2_scale_stereo_modes(device, oracle, mode):
    """SURVEY §8f rank 3 at cfg2 scale (640x480, 4 levels, 8 px grid): stereo-only (active_fields = s,
    solver.cpp:27-31, 213-226; global PCG) and the stereo-hq preset with the epipolar term (w_epi = 0.5 > 0,
    energy.cpp:168-192; Schwarz mode) against the oracle."""
    imgs = synthetic.webcam_pair(5)[0]
    F = np.array([[0, 0, 0], [0, 0, -1], [0, 1, 0.0]])
    if mode == "stereo_only":  # global PCG: the reference's Schwarz mode hits pAp <= 0 here (oracle too)
        S = SolveSchedule(levels=4, grid_step=8, gn_per_level=[1, 1, 2, 2], pcg_iters=5, subdomain_px=0,
                          active_fields=1)
        r, _ = _check_solve(device, oracle, imgs, EnergyParams(), S)
        assert np.abs(r.grid_total[:, 2:]).max() == 0.0
    else:
        S = SolveSchedule(levels=4, grid_step=8, gn_per_level=[1, 1, 2, 2], pcg_iters=5, patch_iters=5)
        _check_solve(device, oracle, imgs, EnergyParams.preset("stereo-hq"), S, F)


@pytest.mark.parametrize("sub", [16, 0])
def test_batch_is_bitwise_independent(device, sub):
    """Schwarz sweeps and the global PCG (fixed tile-order dots) give every pair the same bits alone
    or inside a batch."""
    frames = np.stack([synthetic.webcam_pair(i, 128, 96)[0] for i in range(3)])
    S = SolveSchedule(levels=3, grid_step=8, pcg_iters=5, patch_iters=5, subdomain_px=sub)
    batch, _ = device.solve_batch(frames, EnergyParams(), S)
    for i in range(3):
        (single,), _ = device.solve_batch(frames[i:i + 1], EnergyParams(), S)
        assert np.array_equal(single.grid_total, batch[i].grid_total)
        assert np.array_equal(single.vis4, batch[i].vis4)
    again, _ = device.solve_batch(frames, EnergyParams(), S)
    assert all(np.array_equal(a.grid_total, b.grid_total) for a, b in zip(batch, again))


@pytest.mark.parametrize("w,h", [(128, 96), (131, 97)])
def test_u8_finest_level_matches_f64_frames(device, w, h):
    """The finest level of u8 frames is sampled from the bytes in the integer domain (k_pixel<*, U8>); the f64
    path samples the correctly rounded k/255 planes (k_pyr_in, k_pack). The two differ only by the rounding of
    the interpolation (a few ulps per sample), so the solves agree to round-off: grids within 1e-9 px, masks
    bit-exact, energies within 1e-12 relative."""
    frames = np.stack([synthetic.webcam_pair(i, w, h)[0] for i in range(2)])
    frames[0, 2, :, :7] = 255  # saturated border columns
    frames[1, 1, -3:, :] = 0
    f64 = frames.astype(np.float64) / 255.0
    for S in (SolveSchedule(levels=3, grid_step=8, pcg_iters=5, patch_iters=5),
              SolveSchedule(levels=2, grid_step=4, gn_per_level=[3, 2], pcg_iters=6, subdomain_px=0,
                            coarse_s_offset=(2.5, -1.0))):
        a, sa = device.solve_batch(frames, EnergyParams(), S)
        b, sb = device.solve_batch(f64, EnergyParams(), S)
        for x, y, u, v in zip(a, b, sa, sb):
            assert np.abs(x.grid_total - y.grid_total).max() < 1e-9
            assert np.array_equal(x.vis4, y.vis4)
            for eu, ev in zip(u.energy_after, v.energy_after):
                np.testing.assert_allclose(eu, ev, rtol=1e-12)


def test_cfg2_full_size_properties(device):
    """BASELINE cfg2 shape on a batch: finite, deterministic, identity scene stationary."""
    frames = np.stack([synthetic.webcam_pair(i)[0] for i in range(4)])
    S = SolveSchedule(levels=4, grid_step=8, pcg_iters=5, patch_iters=5, subdomain_px=16)
    res, st = device.solve_batch(frames, EnergyParams(), S, outputs=("grid_total", "vis4"))
    for r, s in zip(res, st):
        assert np.isfinite(r.grid_total).all()
        assert len(s.energy_after) == 4 and [len(e) for e in s.energy_after] == [2, 2, 5, 5]
    ident = np.stack([np.repeat(frames[0, :1], 4, axis=0)])  # four identical images
    (r,), (s,) = device.solve_batch(ident, EnergyParams(), SolveSchedule(levels=4, grid_step=8, subdomain_px=0))
    assert np.abs(r.grid_total).max() < 1e-6  # SPEC.md:348 stationarity
    assert np.all(r.vis4 == 0x0F)


def test_divergence_is_reported(device):
    imgs, _ = synthetic.constant_pair(64, 48)
    P = EnergyParams(m_s=0.0, m_m=0.0, m_d=0.0, w_reg=0.0)  # no Tikhonov: J^T J singular on flat regions
    imgs = np.zeros_like(imgs)
    S = SolveSchedule(levels=1, grid_step=8, gn_per_level=[1], pcg_iters=5, subdomain_px=0)
    try:
        device.solve_batch(imgs[None], P, S)
    except SolverDivergence:
        pass  # reported, not aborted
    with pytest.raises(ValueError):
        device.solve_batch(imgs[None], EnergyParams.preset("facial"), S)  # w_epi > 0 without F


# ---- the other BASELINE.json shapes ----------------------------------------------
def test_cfg3_occluder_and_illumination_change(device, oracle):
    """cfg3: 1920x1080, 5 levels, foreground square with +6 px extra disparity, right camera +0.05,
    t+1 gain x1.05 (short GN schedule so the CPU oracle stays fast)."""
    imgs, gt = synthetic.valgaerts_pair(0)
    S = SolveSchedule(levels=5, grid_step=8, gn_per_level=[1, 1, 2], pcg_iters=5, patch_iters=5, threads=16)
    r, s = _check_solve(device, oracle, imgs, EnergyParams(), S)
    assert (r.vis4 != 0x0F).any()  # the occluder produces occlusion
    assert np.isfinite(r.grid_total).all()


def test_cfg5_uhd_step4_general_schwarz_tiles(device, oracle):
    """cfg5: 3840x2160, 4 px grid -> 4x4-node subdomains (the general Schwarz team path)."""
    imgs, _ = synthetic.uhd_pair(0)
    S = SolveSchedule(levels=5, grid_step=4, gn_per_level=[1], pcg_iters=5, patch_iters=3, threads=16)
    _check_solve(device, oracle, imgs, EnergyParams(), S)


# ---- temporal propagation -----------------------------------------
def test_propagation_bit_exact(device, oracle):
    rng = np.random.default_rng(5)
    for (w, h, step) in ((64, 48, 8), (101, 77, 4)):
        gw, gh = grid_dims(w, h, step)
        d, t = rng.normal(0, 1, (gw * gh, 6)), rng.normal(0, 3, (gw * gh, 6))
        assert np.array_equal(device.propagate_temporal(w, h, step, d, t), oracle.propagate_temporal(w, h, step, d, t))


def test_sequence_matches_oracle(device, oracle):
    """Two independent 3-frame sequences advanced together (one device batch per frame)."""
    seqs = [synthetic.sequence_pairs(3, 128, 96, s=(1.5, 0.0), v=v, seed=1700 + i) for i, v in
            enumerate(((2.0, 1.0), (-1.0, 0.5)))]
    # global PCG: the reference's step-8 Schwarz mode diverges, which would
    # turn this propagation test into a test of amplified round-off
    S = SolveSchedule(levels=3, grid_step=8, gn_per_level=[2, 2, 3], pcg_iters=8, subdomain_px=0)
    P = EnergyParams()
    dst = [device.new_state(2, 128, 96, S) for _ in range(2)]
    ost = [[oracle.new_state(1, 128, 96, S) for _ in range(2)] for _ in range(2)]
    dprev, oprev = None, [None, None]
    for k in range(3):
        frames = np.stack([seqs[0][k], seqs[1][k]])
        ra, sa = device.solve_batch_seq(frames, P, S, dprev, dst[k % 2])
        dprev = dst[k % 2]
        for i in range(2):
            (rb,), (sb,) = oracle.solve_batch_seq(frames[i:i + 1], P, S, oprev[i], ost[i][k % 2])
            oprev[i] = ost[i][k % 2]
            assert np.abs(ra[i].grid_total - rb.grid_total).max() < FLOW_TOL_PX
            np.testing.assert_allclose(sa[i].energy_after[0], sb.energy_after[0], rtol=ENERGY_RTOL)
            da, ta = dprev.read(i)
            db, tb = oprev[i].read(0)
            for l in range(len(da)):
                assert np.abs(ta[l] - tb[l]).max() < FLOW_TOL_PX


def test_streaming_submit_wait_matches_sync(device):
    """hwf_submit_batch/hwf_wait (two batches in flight, transfers overlapping compute) return
    exactly what hwf_solve_batch returns."""
    import ctypes as C
    from paper_1610_07159_b200 import capi
    frames = [np.stack([synthetic.webcam_pair(4 * k + i, 128, 96)[0] for i in range(4)]) for k in range(3)]
    S = SolveSchedule(levels=3, grid_step=8, pcg_iters=5, patch_iters=5)
    P = EnergyParams()
    ref = [device.solve_batch(f, P, S, outputs=("grid_total", "vis4")) for f in frames]
    lib, h = device.lib, device.ctx.h
    gw, gh = grid_dims(128, 96, 8)
    keep, outs = [], []
    pc, sc = P.to_c(), S.to_c()
    for k, f in enumerate(frames):
        fr = (capi.Frame4C * 4)()
        res = (capi.ResultC * 4)()
        st = (capi.StatsC * 4)()
        grids = np.empty((4, gw * gh, 6))
        vis = np.empty((4, 96, 128), np.uint8)
        for i in range(4):
            fr[i].width, fr[i].height, fr[i].dtype = 128, 96, capi.DTYPE_U8
            for e in range(4):
                fr[i].plane[e] = f[i, e].ctypes.data
            res[i].grid_total = capi.dptr(grids[i])
            res[i].vis4 = capi.u8ptr(vis[i])
        keep.append((fr, res, st, grids, vis, f))
        device.ctx.check(lib.hwf_submit_batch(h, 4, fr, C.byref(pc), C.byref(sc), capi.dptr(None), res, st))
        if k >= 1:
            device.ctx.check(lib.hwf_wait(h))
    device.ctx.check(lib.hwf_wait(h))
    for k in range(3):
        (_, _, st, grids, vis, _) = keep[k]
        outs_ref, stats_ref = ref[k]
        for i in range(4):
            assert np.array_equal(grids[i], outs_ref[i].grid_total)
            assert np.array_equal(vis[i], outs_ref[i].vis4)
            assert st[i].energy_after[0][1] == stats_ref[i].energy_after[0][1]


def test_streaming_dense_flowresult_matches_sync(device):
    """The streaming API with the reference's full FlowResult (geometry.hpp:26-37: s, m, d, disparity, vis4 per
    pixel, plus the grid): four batches, two in flight, each slot writing its own dense buffers; every field
    bitwise what hwf_solve_batch returns."""
    import ctypes as C
    from paper_1610_07159_b200 import capi
    w, h, n = 96, 72, 3
    frames = [np.stack([synthetic.webcam_pair(3 * k + i, w, h)[0] for i in range(n)]) for k in range(4)]
    S = SolveSchedule(levels=3, grid_step=8, pcg_iters=5, subdomain_px=0)
    P = EnergyParams()
    ref = [device.solve_batch(f, P, S)[0] for f in frames]
    lib, hh = device.lib, device.ctx.h
    gw, gh = grid_dims(w, h, 8)
    pc, sc = P.to_c(), S.to_c()
    keep = []
    for k, f in enumerate(frames):
        fr, res, st = (capi.Frame4C * n)(), (capi.ResultC * n)(), (capi.StatsC * n)()
        o = {"s": np.empty((n, h, w, 2)), "m": np.empty((n, h, w, 2)), "d": np.empty((n, h, w, 2)),
             "disparity": np.empty((n, h, w)), "vis4": np.empty((n, h, w), np.uint8), "grid_total": np.empty((n, gw * gh, 6))}
        for i in range(n):
            fr[i].width, fr[i].height, fr[i].dtype = w, h, capi.DTYPE_U8
            for e in range(4):
                fr[i].plane[e] = f[i, e].ctypes.data
            res[i].s, res[i].m, res[i].d = capi.dptr(o["s"][i]), capi.dptr(o["m"][i]), capi.dptr(o["d"][i])
            res[i].disparity, res[i].grid_total = capi.dptr(o["disparity"][i]), capi.dptr(o["grid_total"][i])
            res[i].vis4 = capi.u8ptr(o["vis4"][i])
        keep.append((fr, res, st, o, f))
        device.ctx.check(lib.hwf_submit_batch(hh, n, fr, C.byref(pc), C.byref(sc), capi.dptr(None), res, st))
        if k >= 1:
            device.ctx.check(lib.hwf_wait(hh))
    device.ctx.check(lib.hwf_wait(hh))
    for k in range(4):
        o = keep[k][3]
        for i in range(n):
            for name in ("s", "m", "d", "disparity", "vis4", "grid_total"):
                assert np.array_equal(o[name][i], getattr(ref[k][i], name)), (k, i, name)


def test_residual_vector_matches_oracle(device, oracle, golden):
    """assemble_residuals (energy.cpp:208-228): the stacked R, M = 2N + 14G entries."""
    for P in (EnergyParams(), EnergyParams.preset("facial")):
        lv = _golden_level(golden)
        ea, Ra = device.energy(lv, P, residuals=True)
        eb, Rb = oracle.energy(lv, P, residuals=True)
        assert Ra.size == Rb.size == ea.residual_count
        np.testing.assert_allclose(Ra, Rb, rtol=1e-9, atol=1e-13)
        assert (Ra ** 2).sum() == pytest.approx(ea.total, rel=1e-9)  # |R|^2 = E (SPEC acceptance 2)


def _fd_jacobian_check(solver, lv, P, picks, h=1e-7):
    """rhs = -J^T r must equal -(1/2) dE/dx by central differences of E(total, delta) with
    W, V and w_i frozen (SPEC acceptance 1 through the blocked assembly)."""
    _, rhs, _ = solver.build_normal_system(lv, P, 7, 0.0)
    errs = []
    for (k, c) in picks:
        e = []
        for sgn in (1.0, -1.0):
            t, d = lv.total.copy(), lv.delta.copy()
            t[k, c] += sgn * h
            d[k, c] += sgn * h
            lv2 = LevelState(lv.images, lv.grid_step, t, d, lv.vis4, lv.outlier, lv.node_w, lv.illum, lv.fundamental)
            e.append(solver.energy(lv2, P)[0].total)
        fd = -(e[0] - e[1]) / (2 * h) / 2.0
        errs.append(abs(fd - rhs[6 * k + c]) / max(abs(rhs[6 * k + c]), 1e-3 * np.abs(rhs).max()))
    return np.array(errs)


def test_jacobian_finite_differences(device, oracle):
    rng = np.random.default_rng(11)
    lv = _random_level(31, 40, 32, 4)
    G = lv.total.shape[0]
    picks = [(int(rng.integers(G)), int(rng.integers(6))) for _ in range(24)]
    for s in (device, oracle):
        errs = _fd_jacobian_check(s, lv, EnergyParams.preset("facial"), picks)
        assert np.median(errs) < 1e-5 and (errs < 1e-3).mean() >= 0.9, errs


@pytest.mark.parametrize("gw,gh", [(3, 2), (32, 16), (33, 17)])  # fused (<= 16 tiles, system in smem), fused, per-phase
def test_pcg_device_edge_cases_match_oracle(device, oracle, gw, gh):
    """hwf_pcg on both device paths (k_pcg_fused for <= 16 tiles per pair, the per-phase kernels above): SPEC.md:330-331
    identity / diagonal systems solve in one iteration, a zero rhs returns x = 0 with a zero trace (solver.cpp:334-338),
    a random SPD system matches the oracle with its trace, and an indefinite one raises SolverDivergence as the
    oracle does (pAp <= 0, solver.cpp:344-346)."""
    G = gw * gh
    rng = np.random.default_rng(gw * 100 + gh)
    b = rng.normal(size=6 * G)
    blocks = np.zeros((G, 9, 6, 6))
    blocks[:, 4] = np.eye(6)
    np.testing.assert_allclose(device.pcg_solve(gw, gh, blocks, b, 1), b, rtol=1e-14)
    blocks[:, 4] = np.diag(np.arange(1.0, 7.0))
    np.testing.assert_allclose(device.pcg_solve(gw, gh, blocks, b, 1), b / np.tile(np.arange(1.0, 7.0), G), rtol=1e-13)
    x, tr = device.pcg_solve(gw, gh, blocks, np.zeros(6 * G), 4, trace=True)
    assert not x.any() and not np.asarray(tr).any()
    # SPD: diagonally dominant, with symmetric coupling blocks (every block of this system is a sum of a a' J J^T, and
    # the device keeps 21 packed entries per block), mirrored as NormalSystem stores them
    spd = np.zeros((G, 9, 6, 6))
    for n in range(G):
        a, bb = n % gw, n // gw
        spd[n, 4] = np.eye(6) * 40.0 + 0.5 * (lambda m: m + m.T)(rng.normal(size=(6, 6)))
        for s9 in (5, 6, 7, 8):  # forward slots; the backward ones mirror them
            dx, dy = s9 % 3 - 1, s9 // 3 - 1
            if 0 <= a + dx < gw and bb + dy < gh:
                m = (lambda r: 0.5 * (r + r.T))(rng.normal(size=(6, 6)))
                spd[n, s9] = m
                spd[n + dy * gw + dx, 8 - s9] = m.T
    xd, td = device.pcg_solve(gw, gh, spd, b, 6, trace=True)
    xo, to = oracle.pcg_solve(gw, gh, spd, b, 6, trace=True)
    np.testing.assert_allclose(xd, xo, rtol=1e-10, atol=1e-12 * np.abs(xo).max())
    np.testing.assert_allclose(td, to, rtol=1e-10)
    bad = spd.copy()
    bad[:, 4] = -np.eye(6) * 40.0  # negative definite diagonal: the first p.Ap is negative
    for solver in (oracle, device):
        with pytest.raises(SolverDivergence):
            solver.pcg_solve(gw, gh, bad, b, 6)
