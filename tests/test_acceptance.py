"""SPEC.md's acceptance criteria 7-11 and 14, on the oracle (CPU) and on the device (-m gpu).

The hierarchy (occlusion, illumination, prolongation) has no reference code, so these criteria are the only
behavioural pins the reference holds for the oracle's restatement of it (oracle/hierarchy.cpp header, DESIGN.md
§2). Measured outcomes, including where the reference's own design misses a criterion, are in
profiles/r2_parity_notes.md.
"""
from __future__ import annotations

import time

import numpy as np
import pytest

import scenes
from lockstep import HierRun
from paper_1610_07159_b200 import synthetic
from paper_1610_07159_b200.hwflow import EnergyParams, LevelState, SolveSchedule, grid_dims

F_RECT = np.array([[0.0, 0.0, 0.0], [0.0, 0.0, -1.0], [0.0, 1.0, 0.0]])  # x_0^T F x_1 = y_1 - y_0


@pytest.fixture(params=["oracle", pytest.param("device", marks=pytest.mark.gpu)])
def lib(request):
    return request.getfixturevalue(request.param)


# ---- 7: convergence shape (Fig. 4) -------------------------------------------------------------
def _apply(blocks, x, gw, gh):
    """NormalSystem::apply (solver.cpp:57-72): 9-slot block SpMV, slot = (dy+1)*3 + (dx+1)."""
    X = x.reshape(gh, gw, 6)
    B = blocks.reshape(gh, gw, 9, 6, 6)
    out = np.zeros_like(X)
    for dy in (-1, 0, 1):
        for dx in (-1, 0, 1):
            s = (dy + 1) * 3 + (dx + 1)
            ys, xs = slice(max(0, -dy), gh - max(0, dy)), slice(max(0, -dx), gw - max(0, dx))
            yn, xn = slice(max(0, dy), gh + min(0, dy)), slice(max(0, dx), gw + min(0, dx))
            out[ys, xs] += np.einsum("yxij,yxj->yxi", B[ys, xs, s], X[yn, xn])
    return out.reshape(-1)


def test_acceptance7_pcg_decreases_error_every_step(lib):
    """SPEC.md:602 / Fig. 4 ("error is always decreased by the PCG iteration steps"): 5 GN x 5 PCG on the finest
    level of acceptance 5's 8 px case. The error PCG decreases monotonically is the energy-norm error, i.e. the
    quadratic model phi(x_k) = x^T A x / 2 - b^T x of each GN iteration's normal equations: it is non-increasing
    at every PCG step. The reference's logged per-step quantity, pcg_trace = ||r_k|| (solver.cpp:508-513), is not
    monotone in the reference either (CG does not minimise ||r||): its last step rises on every GN iteration of
    this case, which the test records rather than asserts away."""
    imgs = synthetic.render_pair(256, 256, s=(4.0, 0.0), seed=5)
    S = SolveSchedule(levels=5, grid_step=8, gn_per_level=[5], pcg_iters=5, subdomain_px=0, threads=8)
    P = EnergyParams()
    R = HierRun(lib, imgs, S, P)
    R.run_to(1)
    R.start_level(0)
    w, h, gw, gh = R.dims[0]
    rises = 0
    for it in range(5):
        lv = LevelState(R.pyr[0], 8, R.base + R.delta, R.delta, R.vis, R.W, R.nw, R.illum)
        W, nw = lib.refresh_weights(lv, P)  # solver.cpp:497-499, as gauss_newton does first
        lv = LevelState(R.pyr[0], 8, R.base + R.delta, R.delta, R.vis, W, nw, R.illum)
        blocks, rhs, _ = lib.build_normal_system(lv, P)
        phi = [0.0]
        for k in range(1, 6):
            x = lib.pcg_solve(gw, gh, blocks, rhs, k)
            phi.append(0.5 * x @ _apply(blocks, x, gw, gh) - rhs @ x)
        assert all(b <= a + 1e-9 * abs(a) for a, b in zip(phi, phi[1:])), (it, phi)
        _, tr = lib.pcg_solve(gw, gh, blocks, rhs, 5, trace=True)
        assert tr[1] < tr[0]  # the first step always lowers ||r|| here
        rises += int(np.any(np.diff(tr) > 0))
        R.gn(0)  # the reference's own GN iteration moves the state on
    assert rises >= 1  # pcg_trace is not monotone (reference behaviour, see docstring)


# ---- 8: Schwarz vs global ---------------------------------------------------------------------
@pytest.mark.parametrize("step", [2, 4])
def test_acceptance8_schwarz_close_to_global(lib, step):
    """64x64, one GN iteration; 5 Schwarz sweeps over 16x16 (+2) subdomains vs a global 25-iteration
    PCG: energies within 2%."""
    im = synthetic.render_pair(64, 64, s=(1.0, 0.0), m=(0.5, 0.25), seed=9, dtype=np.float64)
    Ssw = SolveSchedule(levels=1, grid_step=step, gn_per_level=[1], pcg_iters=5, patch_iters=5, subdomain_px=16,
                        boundary_px=2)
    Sgl = SolveSchedule(levels=1, grid_step=step, gn_per_level=[1], pcg_iters=25, subdomain_px=0)
    (_,), (a,) = lib.solve_batch(im[None], EnergyParams(), Ssw, outputs=("grid_total",))
    (_,), (b,) = lib.solve_batch(im[None], EnergyParams(), Sgl, outputs=("grid_total",))
    assert abs(a.final_energy() / b.final_energy() - 1.0) < 0.02


# ---- 9: occlusion maps ------------------------------------------------------------------------
def _gt_grid(w, h, step, rect, s_bg, extra):
    gw, gh = grid_dims(w, h, step)
    g = np.zeros((gh, gw, 6))
    g[..., 0] = s_bg
    ys, xs = np.meshgrid(np.arange(gh) * step, np.arange(gw) * step, indexing="ij")
    g[(xs >= rect[0]) & (xs < rect[2]) & (ys >= rect[1]) & (ys < rect[3]), 0] += extra
    return g.reshape(-1, 6)


def _rates(vis4, gt):
    v = np.stack([(vis4 >> e) & 1 for e in range(4)]).astype(bool)
    occ = ~gt
    return (occ & ~v).sum() / occ.sum(), (gt & ~v).sum() / gt.sum()


@pytest.mark.parametrize("extra", [8.0, 16.0])
def test_acceptance9_occlusion_maps_two_layer_scene(lib, extra):
    """SPEC.md:604 on compute_occlusion_maps (pins C.2/C.3 in oracle/hierarchy.cpp): the two-layer
    scene's flow (background s = 2 px, foreground square +extra, disparity gap 2*extra) on a 1 px warp grid, so
    the grid can carry the discontinuity: >= 90% of the ground-truth occluded background pixels are marked
    occluded, <= 5% of the visible ones wrongly. The ground truth is render_pair's own pull-back geometry
    (tests/scenes.py:occlusion_truth); the band lies beside the square's leading edge in one camera."""
    w, h = 256, 256
    rect = (w // 3, h // 3, 2 * w // 3, 2 * h // 3)
    vis4 = lib.compute_occlusion_maps(w, h, 1, _gt_grid(w, h, 1, rect, 2.0, extra))
    recall, fp = _rates(vis4, scenes.occlusion_truth(w, h, rect, (extra, 0.0)))
    assert recall >= 0.9 and fp <= 0.05, (recall, fp)


@pytest.mark.xfail(strict=True, reason="the reference's solver smooths the two-layer discontinuity (L2 smoothness on "
                   "the 8 px warp grid, energy.cpp:131-166), so the solved mesh never folds and the occlusion maps "
                   "stay (almost) all-visible; recall ~0 measured on the reference build (profiles/r2_parity_notes.md)")
def test_acceptance9_end_to_end_after_level2(oracle):
    w, h = 640, 480
    rect = (w // 3, h // 3, 2 * w // 3, 2 * h // 3)
    imgs = synthetic.render_pair(w, h, s=(2.0, 0.0), m=(0.5, -0.25), seed=33,
                                 occluder={"rect": rect, "extra_s": (8.0, 0.0)})
    S = SolveSchedule(levels=5, grid_step=8, pcg_iters=5, subdomain_px=0, threads=8)
    R = HierRun(oracle, imgs, S, EnergyParams())
    R.run_to(2)
    wl, hl = R.dims[2][:2]
    recall, fp = _rates(R.vis_prev, scenes.occlusion_truth(wl, hl, rect, (8.0, 0.0), level=2))
    assert recall >= 0.9 and fp <= 0.05


# ---- 10: illumination correction ---------------------------------------------------------------
def test_acceptance10_illumination_correction(lib):
    """right images brightened by +0.1; after the hierarchy, at the finest level, mean |d_0| over
    pixels visible in both images of check 0 is < 0.02 with the correction maps (vs ~0.1 without)."""
    w, h = 320, 240
    im = synthetic.render_pair(w, h, s=(2.0, 0.0), m=(0.5, -0.25), seed=21, gain_offset={"offset": [0, 0.1, 0, 0.1]})
    S = SolveSchedule(levels=4, grid_step=8, pcg_iters=5, subdomain_px=0, threads=8)
    R = HierRun(lib, im, S, EnergyParams())
    R.run_to(0)
    fl = scenes.interp_grid(R.total_prev, w, h, 8)
    a0, a1 = scenes.warped(R.pyr[0], fl, 0), scenes.warped(R.pyr[0], fl, 1)
    vis = (((R.vis >> 0) & 1) & ((R.vis >> 1) & 1)).astype(bool)  # check 0 = (1, 0) (warp_grid.hpp:85)
    corrected = np.abs((a1 + R.illum[1]) - (a0 + R.illum[0]))[vis].mean()
    raw = np.abs(a1 - a0)[vis].mean()
    assert corrected < 0.02, corrected
    assert 0.08 < raw < 0.12, raw


# ---- 11: epipolar term --------------------------------------------------------------------------
def test_acceptance11_epipolar_term(lib):
    """rectified scene, vertical-drift initialisation (coarse_s_offset = (0, 0.5)): with w_epi = 0.5 the
    median |l^T F r| at convergence is < 0.5, and with w_epi = 0 it is strictly larger (the term does work)."""
    im = synthetic.render_pair(256, 192, s=(2.0, 0.0), m=(0.5, 0.25), seed=12)
    S = SolveSchedule(levels=4, grid_step=8, pcg_iters=5, subdomain_px=0, coarse_s_offset=(0.0, 0.5))
    med = {}
    for w_epi in (0.5, 0.0):
        (r,), _ = lib.solve_batch(im[None], EnergyParams(w_epi=w_epi), S, F_RECT if w_epi > 0 else None,
                                  outputs=("grid_total",))
        med[w_epi] = float(np.median(scenes.epipolar_residuals(r.grid_total)))
    assert med[0.5] < 0.5 and med[0.0] > med[0.5], med


# ---- 14: scaling ---------------------------------------------------------------------------------
def test_acceptance14_scaling_linear_in_pixels(lib):
    """the time for 512x512 is 2.5x-6x the time for 256x256 (same schedule). On the device a batch
    of 128 pairs per call, so that both sizes fill the GPU (at 32 pairs 256x256 is still partly launch- and
    transfer-bound: ratio 2.4 measured); the second, warm call is timed."""
    n_pairs = 128 if lib.backend.startswith("cuda") else 1
    S = SolveSchedule(levels=5, grid_step=8, pcg_iters=5, subdomain_px=0, threads=1)
    ts = []
    for n in (256, 512):
        frames = np.stack([synthetic.render_pair(n, n, s=(1.0, 0.0), seed=3 + i) for i in range(n_pairs)])
        lib.solve_batch(frames, EnergyParams(), S, outputs=("grid_total",))
        t = time.perf_counter()
        lib.solve_batch(frames, EnergyParams(), S, outputs=("grid_total",))
        ts.append(time.perf_counter() - t)
    assert 2.5 <= ts[1] / ts[0] <= 6.0, ts
