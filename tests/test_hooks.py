"""The reference's test hooks at the C-ABI (hwf_assemble_jacobian, hwf_normal_dense) and what they are for.

- assemble_jacobian (include/hwflow/solver.hpp:96-111, src/solver.cpp:247-314), the derivative checker's
  input: the stacked residuals R and dR/dx as triplets. The oracle port and the device must produce the reference
  build's triplets (same rows, columns and order; values to 1e-12 / 1e-9), SPEC acceptance 1 holds (analytic
  columns = central finite differences of R), and the negative control (negate_field, SPEC.md:573's "deliberately
  corrupted sign") must make that check fail.
- NormalSystem::dense (solver.hpp:77, solver.cpp:89-98): JᵀJ as a dense matrix; "for m_s, m_m, m_d > 0
  the smallest eigenvalue of JᵀJ on small instances is > 0", and dense(J^T J) = J^T J from the triplets.
"""
from __future__ import annotations

import numpy as np
import pytest

from paper_1610_07159_b200 import synthetic
from paper_1610_07159_b200.hwflow import EnergyParams, LevelState, grid_dims


def _level(seed=3, w=24, h=18, step=4, illum=True):
    rng = np.random.default_rng(seed)
    imgs = synthetic.render_pair(w, h, s=(1.0, 0.3), m=(0.4, -0.6), seed=seed, dtype=np.float64)
    gw, gh = grid_dims(w, h, step)
    return LevelState(imgs, step, rng.normal(0, 0.5, (gw * gh, 6)), rng.normal(0, 0.2, (gw * gh, 6)),
                      rng.integers(0, 16, (h, w)).astype(np.uint8), (rng.random((h, w)) > 0.15).astype(np.uint8),
                      rng.uniform(1, 100, gw * gh), rng.normal(0, 0.02, (4, h, w)) if illum else None,
                      np.array([[0, 0, 0], [0, 0, -1], [0, 1, 0.0]]))


def _dense(J, M, D):
    R, rows, cols, vals = J
    A = np.zeros((M, D))
    np.add.at(A, (rows, cols), vals)
    return A


def _residuals_at(lib, lv, P, x):
    """R at total = lv.total + dx, delta = lv.delta + dx (both move with the unknowns, as in a GN step)."""
    dx = x.reshape(-1, 6)
    moved = LevelState(lv.images, lv.grid_step, lv.total + dx, lv.delta + dx, lv.vis4, lv.outlier, lv.node_w,
                       lv.illum, lv.fundamental)
    return lib.assemble_jacobian(moved, P)[0]


def _fd_column_errors(lib, lv, P, J, cols, h=1e-6):
    """max |analytic - central FD| / max(|analytic|, |FD|, 1e-8) over the given unknowns."""
    gw, gh = grid_dims(lv.width, lv.height, lv.grid_step)
    D = 6 * gw * gh
    A = _dense(J, J[0].size, D)
    errs = []
    for c in cols:
        e = np.zeros(D)
        e[c] = h
        fd = (_residuals_at(lib, lv, P, e) - _residuals_at(lib, lv, P, -e)) / (2 * h)
        scale = max(np.abs(A[:, c]).max(), np.abs(fd).max(), 1e-8)
        errs.append(np.abs(A[:, c] - fd).max() / scale)
    return np.array(errs)


@pytest.mark.parametrize("preset", ["live", "facial"])
def test_jacobian_port_matches_reference(oracle, reference, preset):
    lv, P = _level(), EnergyParams.preset(preset)
    for active, neg in ((7, -1), (5, 1), (7, 2)):
        a, b = oracle.assemble_jacobian(lv, P, active, neg), reference.assemble_jacobian(lv, P, active, neg)
        assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])  # same entries, same order
        np.testing.assert_allclose(a[0], b[0], rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(a[3], b[3], rtol=1e-10, atol=1e-13)


def test_jacobian_fd_and_negative_control(oracle):
    """SPEC acceptance 1 (analytic columns = central FD of R) passes; flipping one field's derivatives fails it."""
    lv, P = _level(w=16, h=16, step=2, illum=False), EnergyParams()
    gw, gh = grid_dims(16, 16, 2)
    cols = [6 * n + c for n in (gw + 1, 2 * gw + 3, 5 * gw + 4) for c in range(6)]
    good = _fd_column_errors(oracle, lv, P, oracle.assemble_jacobian(lv, P), cols)
    assert good.max() < 1e-4, good.max()
    for f in range(3):
        bad = _fd_column_errors(oracle, lv, P, oracle.assemble_jacobian(lv, P, 7, f), cols)
        hit = [e for c, e in zip(cols, bad) if (c % 6) // 2 == f]
        assert max(hit) > 0.5, (f, max(hit))  # the checker catches the corrupted chain rule


def test_normal_dense_spd_and_consistent(oracle):
    """dense(J^T J) from hwf_linearize equals J^T J from the triplets (plus the Levenberg-free regulariser pins),
    and it is SPD for m_f > 0."""
    lv, P = _level(w=16, h=12, step=4), EnergyParams()
    gw, gh = grid_dims(16, 12, 4)
    blocks, rhs, _ = oracle.build_normal_system(lv, P)
    Adense = oracle.normal_dense(gw, gh, blocks)
    J = oracle.assemble_jacobian(lv, P)
    A = _dense(J, J[0].size, 6 * gw * gh)
    np.testing.assert_allclose(Adense, A.T @ A, rtol=1e-9, atol=1e-9 * np.abs(Adense).max())
    np.testing.assert_allclose(rhs, -A.T @ J[0], rtol=1e-9, atol=1e-9 * np.abs(rhs).max())
    assert np.allclose(Adense, Adense.T)
    assert np.linalg.eigvalsh(Adense).min() > 0.0


@pytest.mark.gpu
@pytest.mark.parametrize("preset", ["live", "facial"])
def test_jacobian_device_matches_oracle(device, oracle, preset):
    lv, P = _level(), EnergyParams.preset(preset)
    for active, neg in ((7, -1), (3, 0), (7, 2)):
        a, b = device.assemble_jacobian(lv, P, active, neg), oracle.assemble_jacobian(lv, P, active, neg)
        assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
        np.testing.assert_allclose(a[0], b[0], rtol=1e-9, atol=1e-13)
        np.testing.assert_allclose(a[3], b[3], rtol=1e-9, atol=1e-13)


@pytest.mark.gpu
def test_device_negative_control_and_spd(device):
    lv, P = _level(w=16, h=16, step=2, illum=False), EnergyParams()
    gw, gh = grid_dims(16, 16, 2)
    cols = [6 * (gw + 1) + c for c in range(6)]
    assert _fd_column_errors(device, lv, P, device.assemble_jacobian(lv, P), cols).max() < 1e-4
    assert _fd_column_errors(device, lv, P, device.assemble_jacobian(lv, P, 7, 0), cols)[:2].max() > 0.5
    blocks, _, _ = device.build_normal_system(lv, P)
    assert np.linalg.eigvalsh(device.normal_dense(gw, gh, blocks)).min() > 0.0
