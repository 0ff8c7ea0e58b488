"""CPU: pin the oracle restatement against the reference's own outputs
(tests/golden/ref_small.npz, made by oracle/_ref from /root/reference/proj/src)
and against SPEC.md's worked examples; plus port-vs-reference live checks
where oracle/_ref is present."""
from __future__ import annotations

import numpy as np
import pytest

from paper_1610_07159_b200 import synthetic
from paper_1610_07159_b200.hwflow import EnergyParams, LevelState, SolveSchedule, grid_dims


def _level(g, **over):
    kw = dict(images=g["lv_images"], grid_step=int(g["lv_step"]), total=g["lv_total"], delta=g["lv_delta"],
              vis4=g["lv_vis4"], outlier=g["lv_outlier"], node_w=g["lv_node_w"], illum=g["lv_illum"],
              fundamental=g["lv_F"])
    kw.update(over)
    return LevelState(**kw)


# ---- golden vectors from the reference build --------------------------------------
def test_pyramid_bit_exact_vs_reference(oracle, golden):
    pyr = oracle.build_pyramid(golden["pyr_in"], 4)
    for l, lev in enumerate(pyr):
        assert np.array_equal(lev, golden[f"pyr_L{l}"]), l


@pytest.mark.parametrize("preset", ["live", "facial"])
def test_energy_vs_reference(oracle, golden, preset):
    e, R = oracle.energy(_level(golden), EnergyParams.preset(preset), residuals=True)
    ref = golden[f"E_{preset}"]
    got = np.array([e.photo, e.grad, e.smooth, e.epi, e.mag, e.total, e.residual_count])
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=0)
    np.testing.assert_allclose(R, golden[f"R_{preset}"], rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("preset", ["live", "facial"])
def test_refresh_and_linearize_vs_reference(oracle, golden, preset):
    P = EnergyParams.preset(preset)
    lv = _level(golden)
    W, nw = oracle.refresh_weights(lv, P)
    assert np.array_equal(W, golden[f"W_{preset}"])
    np.testing.assert_allclose(nw, golden[f"nw_{preset}"], rtol=1e-12)
    b, r, p = oracle.build_normal_system(lv, P, 7, 0.0)
    scale = np.abs(golden[f"blocks_{preset}"]).max()
    np.testing.assert_allclose(b, golden[f"blocks_{preset}"], rtol=0, atol=1e-12 * scale)
    np.testing.assert_allclose(r, golden[f"rhs_{preset}"], rtol=0, atol=1e-12 * np.abs(golden[f"rhs_{preset}"]).max())
    np.testing.assert_allclose(p, golden[f"pre_{preset}"], rtol=1e-10, atol=1e-14)


def test_linearize_stereo_only_lm_vs_reference(oracle, golden):
    b, r, _ = oracle.build_normal_system(_level(golden), EnergyParams(), 1, 0.25)
    np.testing.assert_allclose(b, golden["blocks_s_lm"], rtol=0, atol=1e-12 * np.abs(golden["blocks_s_lm"]).max())
    np.testing.assert_allclose(r, golden["rhs_s_lm"], rtol=0, atol=1e-12 * np.abs(golden["rhs_s_lm"]).max())


def test_pcg_and_schwarz_vs_reference(oracle, golden):
    gw, gh = grid_dims(24, 20, 4)
    x, tr = oracle.pcg_solve(gw, gh, golden["blocks_live"], golden["rhs_live"], 10, trace=True)
    np.testing.assert_allclose(x, golden["pcg_x"], rtol=0, atol=1e-10 * np.abs(golden["pcg_x"]).max())
    np.testing.assert_allclose(tr, golden["pcg_trace"], rtol=1e-9)
    xs = oracle.schwarz_iterate(gw, gh, 4, golden["blocks_live"], golden["rhs_live"], 3, 4)
    np.testing.assert_allclose(xs, golden["schwarz_x"], rtol=0, atol=1e-10 * np.abs(golden["schwarz_x"]).max())


@pytest.mark.parametrize("mode,sub", [("schwarz", 16), ("global", 0)])
def test_gauss_newton_vs_reference(oracle, golden, mode, sub):
    gw, gh = grid_dims(40, 32, 8)
    lv = LevelState(golden["gn_images"], 8, np.zeros((gw * gh, 6)), np.zeros((gw * gh, 6)))
    S = SolveSchedule(levels=1, grid_step=8, pcg_iters=5, patch_iters=5, subdomain_px=sub)
    d, W, nw, eb, ea = oracle.gauss_newton(lv, np.zeros((gw * gh, 6)), EnergyParams(), S, 3)
    np.testing.assert_allclose(d, golden[f"gn_{mode}_delta"], rtol=0, atol=1e-9)
    assert np.array_equal(W, golden[f"gn_{mode}_W"])
    np.testing.assert_allclose(eb, golden[f"gn_{mode}_eb"], rtol=1e-10)
    np.testing.assert_allclose(ea, golden[f"gn_{mode}_ea"], rtol=1e-10)


# ---- live port-vs-reference on fresh random inputs (skips without oracle/_ref) -----
def test_port_matches_reference_random(oracle, reference):
    rng = np.random.default_rng(123)
    for w, h, step in ((17, 13, 2), (32, 32, 4), (45, 31, 8)):
        imgs = rng.random((4, h, w))
        gw, gh = grid_dims(w, h, step)
        lv = LevelState(imgs, step, rng.normal(0, 1, (gw * gh, 6)), rng.normal(0, 0.3, (gw * gh, 6)),
                        rng.integers(0, 16, (h, w)).astype(np.uint8))
        for P in (EnergyParams(), EnergyParams.preset("stereo-hq")):
            lv.fundamental = np.array([[0, 0, 0], [0, 0, -1], [0, 1, 0.0]])
            a, _ = oracle.energy(lv, P)
            b, _ = reference.energy(lv, P)
            assert a.total == pytest.approx(b.total, rel=1e-12)
            ba, ra, _ = oracle.build_normal_system(lv, P)
            bb, rb, _ = reference.build_normal_system(lv, P)
            np.testing.assert_allclose(ba, bb, rtol=0, atol=1e-12 * np.abs(bb).max())
            np.testing.assert_allclose(ra, rb, rtol=0, atol=1e-12 * np.abs(rb).max())


def test_full_solve_port_matches_reference(oracle, reference):
    imgs, _ = synthetic.constant_pair(96, 72)
    S = SolveSchedule(levels=3, grid_step=8, gn_per_level=[3], pcg_iters=6, patch_iters=3, subdomain_px=0)
    a, sa = oracle.run_scene_flow(imgs, EnergyParams(), S)
    b, sb = reference.run_scene_flow(imgs, EnergyParams(), S)
    np.testing.assert_allclose(a.grid_total, b.grid_total, rtol=0, atol=1e-9)
    assert np.array_equal(a.vis4, b.vis4)
    assert sa.final_energy() == pytest.approx(sb.final_energy(), rel=1e-9)


# ---- SPEC.md worked examples (the reference ships no tests) -----------------------
def test_spec_residual_count(oracle):
    for w, h, step in ((4, 4, 2), (17, 13, 2), (32, 32, 4)):
        gw, gh = grid_dims(w, h, step)
        lv = LevelState(np.zeros((4, h, w)), step, np.zeros((gw * gh, 6)), np.zeros((gw * gh, 6)))
        e, R = oracle.energy(lv, EnergyParams(), residuals=True)
        assert e.residual_count == 2 * w * h + 14 * gw * gh == R.size
    gw, gh = grid_dims(4, 4, 2)
    assert 2 * 16 + 14 * gw * gh == 158


def test_spec_huber_floor_identity_scene(oracle):
    # identical constant images, zero flow, all visible: |R|^2 = N*6*eps*(w_photo + w_grad)
    h, w, step = 8, 8, 2
    gw, gh = grid_dims(w, h, step)
    lv = LevelState(np.full((4, h, w), 0.5), step, np.zeros((gw * gh, 6)), np.zeros((gw * gh, 6)))
    P = EnergyParams(w_grad=1.0)
    e, R = oracle.energy(lv, P, residuals=True)
    assert R[0] == pytest.approx(np.sqrt(6 * 0.001), rel=1e-12)  # 0.0775
    assert e.total == pytest.approx(2 * w * h * 6 * 0.001, rel=1e-12)


def test_spec_single_check_photo(oracle):
    # one visible check with d_0 = 0.3 -> sqrt(Phi(0.3)) ~= 0.5477
    h, w = 4, 4
    imgs = np.zeros((4, h, w))
    imgs[1] = 0.3
    gw, gh = grid_dims(w, h, 2)
    vis = np.full((h, w), 0b0011, np.uint8)  # images 0 and 1 -> only check 0 (1,0)
    lv = LevelState(imgs, 2, np.zeros((gw * gh, 6)), np.zeros((gw * gh, 6)), vis4=vis)
    _, R = oracle.energy(lv, EnergyParams(), residuals=True)
    assert R[0] == pytest.approx(np.sqrt(np.sqrt(0.09 + 1e-6)), rel=1e-12)


def test_spec_smooth_and_mag_examples(oracle):
    # two-node grid g^s = (0,0),(2,0), unit weights -> s-x residual 2; m_s=4, delta s=(3,0) -> 6 (:261)
    h, w = 1, 3
    lv_total = np.zeros((2 * 2, 6))
    lv_total[1, 0] = 2.0
    lv_total[3, 0] = 2.0
    P = EnergyParams(w_s=1.0, w_m=1.0, w_d=1.0, m_s=4.0)
    delta = np.zeros((4, 6))
    delta[0, 0] = 3.0
    lv = LevelState(np.zeros((4, h, w)), 2, lv_total, delta)
    _, R = oracle.energy(lv, P, residuals=True)
    N, G = 3, 4
    assert R[2 * N + 0] == pytest.approx(2.0)       # node 0 smooth s_x
    assert R[2 * N + 8 * G + 0] == pytest.approx(6.0)  # node 0 mag s_x


def test_spec_pyramid_examples(oracle):
    im = np.zeros((4, 2, 2))
    im[:, 1, :] = 1.0  # [0,0,1,1] -> 0.5
    assert np.all(oracle.build_pyramid(im, 2)[1] == 0.5)
    cb = (np.indices((4, 4)).sum(0) % 2).astype(float)
    assert np.all(oracle.build_pyramid(np.stack([cb] * 4), 2)[1] == 0.5)


def test_spec_pcg_identity_and_dense(oracle):
    gw, gh = 3, 2
    G = gw * gh
    blocks = np.zeros((G, 9, 6, 6))
    blocks[:, 4] = np.eye(6)
    b = np.arange(6 * G, dtype=float) + 1.0
    x = oracle.pcg_solve(gw, gh, blocks, b, 1)  # identity, 1 iteration -> x = b
    np.testing.assert_allclose(x, b, rtol=1e-14)
    blocks[:, 4] = np.diag(np.arange(1.0, 7.0))  # diagonal -> exact in 1 iteration
    x = oracle.pcg_solve(gw, gh, blocks, b, 1)
    np.testing.assert_allclose(x, b / np.tile(np.arange(1.0, 7.0), G), rtol=1e-13)


def test_spec_schwarz_degenerate_tiling_equals_global(oracle, golden):
    # one subdomain covering the whole grid, patch_iters = 1 -> identical to global PCG
    gw, gh = grid_dims(24, 20, 4)
    xg = oracle.pcg_solve(gw, gh, golden["blocks_live"], golden["rhs_live"], 4)
    xs = oracle.schwarz_iterate(gw, gh, 4, golden["blocks_live"], golden["rhs_live"], 1, 4, tile_px=1024)
    np.testing.assert_allclose(xs, xg, rtol=0, atol=1e-12 * np.abs(xg).max())


def test_spec_occlusion_zero_flow_all_visible(oracle):
    for w, h, step in ((9, 7, 2), (33, 17, 8)):
        gw, gh = grid_dims(w, h, step)
        v = oracle.compute_occlusion_maps(w, h, step, np.zeros((gw * gh, 6)))
        assert np.all(v == 0x0F)


def test_spec_prolongation_constant_flow(oracle):
    gwc, ghc = grid_dims(20, 15, 4)
    tc = np.tile(np.array([0.5, -0.25, 1.0, 2.0, 0.0, -1.0]), (gwc * ghc, 1))
    base, vf, hf = oracle.prolongate(20, 15, 40, 30, 4, tc, np.full((15, 20), 0x0F, np.uint8), np.zeros((2, 15, 20)))
    np.testing.assert_allclose(base, 2 * np.tile(tc[0], (base.shape[0], 1)))
    assert np.all(vf == 0x0F)


def test_spec_illumination_constant_offset(oracle):
    # right image = left + 0.1 -> L_{0,t} ~ +0.05
    h, w, step = 32, 40, 8
    rng = np.random.default_rng(0)
    base = rng.random((h, w)) * 0.5
    imgs = np.stack([base, base + 0.1, base, base + 0.1])
    gw, gh = grid_dims(w, h, step)
    hm = oracle.compute_illumination_maps(imgs, step, np.zeros((gw * gh, 6)), np.full((h, w), 0x0F, np.uint8))
    np.testing.assert_allclose(hm, 0.05, rtol=1e-12)


def test_validation_errors(oracle):
    bad = EnergyParams(w_photo=-1.0)
    imgs, _ = synthetic.constant_pair(32, 24)
    with pytest.raises(ValueError):
        oracle.run_scene_flow(imgs, bad, SolveSchedule(levels=1, grid_step=8))
    with pytest.raises(ValueError):  # w_epi > 0 without F (energy.cpp:170-171)
        oracle.run_scene_flow(imgs, EnergyParams.preset("facial"), SolveSchedule(levels=1, grid_step=8))


# ---- temporal propagation -----------------------------------------
def test_spec_propagation_examples(oracle):
    w, h, step = 40, 32, 4
    gw, gh = grid_dims(w, h, step)
    rng = np.random.default_rng(0)
    d = rng.normal(0, 1, (gw * gh, 6))
    t = np.zeros((gw * gh, 6))
    np.testing.assert_array_equal(oracle.propagate_temporal(w, h, step, d, t), d)  # zero motion -> identity
    c = np.tile(np.array([0.3, -0.2, 0.1, 0.4, -0.5, 0.6]), (gw * gh, 1))
    t[:, 2], t[:, 3] = 0.75, -0.5  # constant motion on constant fields -> unchanged where in coverage
    out = oracle.propagate_temporal(w, h, step, c, t)
    a, b = np.arange(gw * gh) % gw, np.arange(gw * gh) // gw
    inside = (a * step - 1.5 >= 0) & (b * step + 1.0 <= (gh - 1) * step)
    np.testing.assert_allclose(out[inside], c[inside], rtol=1e-15)
    assert np.all(out[~inside] == 0.0)  # pulled from outside the lattice -> zero


def test_sequence_propagation_lowers_initial_energy(oracle):
    """SPEC acceptance 12: 3-frame constant-velocity sequence — the initial energy of frame 3
    with propagation is below the initial energy with zero init."""
    pairs = synthetic.sequence_pairs(3, 96, 72, s=(1.0, 0.0), v=(2.0, 1.0))
    S = SolveSchedule(levels=3, grid_step=8, gn_per_level=[2], pcg_iters=8, subdomain_px=0)
    P = EnergyParams()
    st = [oracle.new_state(1, 96, 72, S) for _ in range(2)]
    prev = None
    for k in range(3):
        (r,), (s,) = oracle.solve_batch_seq(pairs[k][None], P, S, prev, st[k % 2])
        prev = st[k % 2]
    (_,), (cold,) = oracle.solve_batch(pairs[2][None], P, S)
    assert s.energy_before[0][0] < cold.energy_before[0][0]


def test_jacobian_finite_differences_oracle():
    """CPU-only variant of the SPEC acceptance-1 check on the oracle (the GPU test repeats it on the device)."""
    import importlib
    from paper_1610_07159_b200 import build
    from paper_1610_07159_b200.hwflow import Solver
    gp = importlib.import_module("test_gpu_parity")
    orc = Solver(build.ORACLE_LIB)
    rng = np.random.default_rng(11)
    lv = gp._random_level(31, 40, 32, 4)
    G = lv.total.shape[0]
    picks = [(int(rng.integers(G)), int(rng.integers(6))) for _ in range(24)]
    errs = gp._fd_jacobian_check(orc, lv, EnergyParams.preset("facial"), picks)
    assert np.median(errs) < 1e-5 and (errs < 1e-3).mean() >= 0.9, errs


def test_gn_pcg_trace_port_matches_reference(oracle, reference, golden):
    """SolveSchedule::pcg_trace (solver.hpp:28, solver.cpp:508-513): one PCG residual-norm trace per GN
    iteration in global mode; the restatement against the reference build."""
    gw, gh = grid_dims(40, 32, 8)
    lv = LevelState(golden["gn_images"], 8, np.zeros((gw * gh, 6)), np.zeros((gw * gh, 6)))
    S = SolveSchedule(levels=1, grid_step=8, pcg_iters=5, subdomain_px=0)
    a = oracle.gauss_newton(lv, np.zeros((gw * gh, 6)), EnergyParams(), S, 3, pcg_trace=True)
    b = reference.gauss_newton(lv, np.zeros((gw * gh, 6)), EnergyParams(), S, 3, pcg_trace=True)
    assert a[5].shape == (3, 6)
    np.testing.assert_allclose(a[5], b[5], rtol=1e-12)
    assert a[5][0, 0] > a[5][0, -1] > 0.0


# ---- SPEC acceptance criteria on the restated hierarchy ---------------------------
def _epe_s(r, shift):
    return np.hypot(r.s[..., 0] - shift / 2, r.s[..., 1])[16:-16, 16:-16]


@pytest.mark.parametrize("shift,p90", [(2.0, 0.25), (8.0, 0.5), (16.0, 0.5)])
def test_spec_acceptance5_constant_disparity_recovery(oracle, shift, p90):
    """256x256 rectified pair, 5 levels, live preset: 90th-percentile EPE of the
    recovered stereo flow (half-shift convention) < 0.25 px for 2 px, < 0.5 px for 8 and 16 px.
    Global PCG (subdomain_px = 0); the reference's Schwarz mode diverges here (below)."""
    imgs = synthetic.render_pair(256, 256, s=(shift / 2, 0.0), seed=5)
    r, _ = oracle.run_scene_flow(imgs, EnergyParams(), SolveSchedule(levels=5, grid_step=8, subdomain_px=0))
    assert np.percentile(_epe_s(r, shift), 90) < p90


def test_spec_acceptance5_single_level_ablation_fails(oracle):
    """without the delta hierarchy the 16 px case must fail (median EPE > 2 px)."""
    imgs = synthetic.render_pair(256, 256, s=(8.0, 0.0), seed=5)
    r, _ = oracle.run_scene_flow(imgs, EnergyParams(), SolveSchedule(levels=1, grid_step=8, subdomain_px=0))
    assert np.median(_epe_s(r, 16.0)) > 2.0


def test_spec_acceptance6_motion_recovery(oracle):
    """moving plane, inter-frame motion 4 px (m = 2 px), 256x256. With the magnitude
    weight of the motion field at the smoothness level (m_m = 5) the median EPE of 2m is < 0.5 px.
    The live preset's m_m = 100 (energy.hpp:26) damps each level's motion update so hard that the
    default schedule stops short (EPE > 0.5 px): a property of the reference's parameters."""
    imgs = synthetic.render_pair(256, 256, m=(2.0, 0.0), seed=5)
    S = SolveSchedule(levels=5, grid_step=8, subdomain_px=0)
    r, _ = oracle.run_scene_flow(imgs, EnergyParams(m_m=5.0), S)
    assert np.median(np.hypot(2 * r.m[..., 0] - 4.0, 2 * r.m[..., 1])[16:-16, 16:-16]) < 0.5
    r, _ = oracle.run_scene_flow(imgs, EnergyParams(), S)
    assert np.median(np.hypot(2 * r.m[..., 0] - 4.0, 2 * r.m[..., 1])[16:-16, 16:-16]) > 0.5


def test_reference_schwarz_diverges_on_2x2_node_subdomains(oracle, reference):
    """The reference's schwarz_iterate (solver.cpp:414-482) is additive block-Jacobi without overlap
    or damping. With 16 px subdomains at grid step 8 (2x2 nodes, the cfg2 schedule) its sweeps
    diverge: every Gauss-Newton step raises the energy, by more than 10x over the finest level,
    while global PCG on the same input lowers it. The reference build and the port agree."""
    imgs = synthetic.render_pair(128, 128, s=(1.0, 0.0), seed=5)
    S = SolveSchedule(levels=2, grid_step=8, subdomain_px=16)
    for solver in (oracle, reference):
        _, st = solver.run_scene_flow(imgs, EnergyParams(), S)
        assert all(a > b for a, b in zip(st.energy_after[0], st.energy_before[0]))
        assert st.energy_after[0][-1] > 10 * st.energy_before[0][0]
    _, st = oracle.run_scene_flow(imgs, EnergyParams(), SolveSchedule(levels=2, grid_step=8, subdomain_px=0))
    assert st.energy_after[0][-1] < st.energy_before[0][0]


# ---- the bench schedules: the port against the reference build, in lock step and end to end -------
def test_port_lockstep_matches_reference_full_cfg1(oracle, reference):
    """Every GN iteration of the full cfg1 schedule (3 levels x 5 GN x 10 PCG), both handed the reference's
    state (tests/lockstep.py): one iteration of the port reproduces one of the reference within 1e-12 px,
    bit-exact W, and bit-exact occlusion on the same flows. (Free-running, the two part by 9e-3 px after
    15 iterations: the reference's GN amplifies one-ulp differences ~1e12; see test below.)"""
    from lockstep import lockstep
    imgs = synthetic.constant_pair(320, 240)[0]
    S = SolveSchedule(levels=3, grid_step=8, gn_per_level=[5], pcg_iters=10, subdomain_px=0, threads=8)

    def on_iter(l, it, A, B, ea, eb):
        assert np.abs(A.delta - B.delta).max() < 1e-12, (l, it)
        assert np.array_equal(A.W, B.W)
        np.testing.assert_allclose(B.nw, A.nw, rtol=1e-12)
        assert eb[1] == pytest.approx(ea[1], rel=1e-12)

    def on_level(l, A, B):
        assert np.array_equal(A.vis_prev, B.vis_prev)

    lockstep(reference, oracle, imgs, S, EnergyParams(), sync=True, on_iter=on_iter, on_level=on_level)


def test_reference_not_reproducible_to_1e3_on_full_cfg1(reference):
    """Root cause of the end-to-end gap at BASELINE configs[0]: the reference against ITSELF with a one-ulp
    change of a random half of its input pixels ends up to ~9e-3 px away (the golden envelope), while the
    same experiment on the headline cfg2 schedule stays below 1e-5 px."""
    from pathlib import Path
    g = dict(np.load(Path(__file__).parent / "golden" / "ref_headline.npz"))
    assert g["cfg1_full_draw_stats"][:, 0].max() > 1e-3  # ill-conditioned schedule
    imgs = synthetic.webcam_pair(0)[0]
    import bench
    S = bench.schedule("global")
    S.threads = 8
    r0, _ = reference.run_scene_flow(imgs, EnergyParams(), S)
    rng = np.random.default_rng(0)
    f = imgs.astype(np.float64) / 255.0
    r1, _ = reference.run_scene_flow(np.where(rng.random(f.shape) < 0.5, np.nextafter(f, 2.0), f), EnergyParams(), S)
    assert np.abs(r1.grid_total - r0.grid_total).max() < 1e-4  # well-conditioned headline schedule
    assert np.abs(r0.grid_total - g["cfg2_0_grid"]).max() == 0.0  # golden reproducible bit for bit


def test_port_matches_reference_headline_golden(oracle):
    """The oracle port at bench.py's cfg2 schedule against the reference-build golden (both CPU)."""
    from pathlib import Path
    g = dict(np.load(Path(__file__).parent / "golden" / "ref_headline.npz"))
    import bench
    S = bench.schedule("global")
    S.threads = 8
    imgs = synthetic.webcam_pair(2)[0]
    q, _ = oracle.run_scene_flow(imgs, EnergyParams(), S)
    assert np.abs(q.grid_total - g["cfg2_2_grid"]).max() < 1e-5
    assert np.array_equal(q.vis4, g["cfg2_2_vis4"])
