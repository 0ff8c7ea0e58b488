"""Geometry outputs (§8f rank 2): StereoRig::validate, triangulate_dlt, compute_scene_points,
export_mesh_obj (include/hwflow/geometry.hpp:14-59; pins G.1-G.6 in
oracle/geometry.cpp).

-m "not gpu": the oracle restatement against SPEC.md's examples and invariants.
-m gpu: the device kernels (k_triangulate, k_scene_points) against the oracle.
"""
from __future__ import annotations

import numpy as np
import pytest

from paper_1610_07159_b200.capi import InvalidArgument
from paper_1610_07159_b200.hwflow import FlowResult, StereoRig

K = np.array([[500.0, 0.0, 320.0], [0.0, 500.0, 240.0], [0.0, 0.0, 1.0]])


def _rot(ax, ay, az):
    cx, sx, cy, sy, cz, sz = np.cos(ax), np.sin(ax), np.cos(ay), np.sin(ay), np.cos(az), np.sin(az)
    Rx = np.array([[1, 0, 0], [0, cx, -sx], [0, sx, cx]])
    Ry = np.array([[cy, 0, sy], [0, 1, 0], [-sy, 0, cy]])
    Rz = np.array([[cz, -sz, 0], [sz, cz, 0], [0, 0, 1]])
    return Rz @ Ry @ Rx


def _skew(t):
    return np.array([[0, -t[2], t[1]], [t[2], 0, -t[0]], [-t[1], t[0], 0]])


def make_rig(R=None, t=(-0.12, 0.0, 0.0)) -> StereoRig:
    """P0 = K[I|0], P1 = K[R|t]; F with x_0^T F x_1 = 0 (the transpose of the usual x_1^T F' x_0)."""
    R = np.eye(3) if R is None else R
    t = np.asarray(t, np.float64)
    P0 = K @ np.hstack([np.eye(3), np.zeros((3, 1))])
    P1 = K @ np.hstack([R, t[:, None]])
    Ki = np.linalg.inv(K)
    F1 = Ki.T @ _skew(t) @ R @ Ki  # x_1^T F1 x_0 = 0
    return StereoRig(F=F1.T / np.abs(F1).max(), P0=P0, P1=P1)


def project(P, X):
    h = X @ P[:, :3].T + P[:, 3]
    return h[..., :2] / h[..., 2:3]


def _random_points(rng, n):
    return np.stack([rng.uniform(-1, 1, n), rng.uniform(-0.8, 0.8, n), rng.uniform(2.0, 8.0, n)], axis=-1)


# ---------------------------------------------------------------- oracle (CPU)
def test_triangulation_round_trip_oracle(oracle):
    """exact correspondences -> the 3D point within 1e-6, reprojection within 1e-6 px."""
    rng = np.random.default_rng(7)
    for rig in (make_rig(), make_rig(_rot(0.02, -0.05, 0.01), (-0.2, 0.01, 0.02))):
        X = _random_points(rng, 200)
        x0, x1 = project(rig.P0, X), project(rig.P1, X)
        Y, ok = oracle.triangulate_dlt(rig.P0, rig.P1, x0, x1)
        assert ok.all()
        assert np.abs(Y - X).max() < 1e-6
        assert np.abs(project(rig.P0, Y) - x0).max() < 1e-6 and np.abs(project(rig.P1, Y) - x1).max() < 1e-6


def test_parallel_rays_invalid_oracle(oracle):
    """zero disparity with a translated-parallel rig is a point at infinity -> invalid."""
    rig = make_rig()
    x = np.array([[100.0, 50.0], [320.0, 240.0], [600.5, 400.25]])
    Y, ok = oracle.triangulate_dlt(rig.P0, rig.P1, x, x)
    assert not ok.any() and np.all(Y == 0.0)


def _flow_result(w, h, s, m, d, vis=0x0F):
    r = FlowResult(width=w, height=h)
    r.s, r.m, r.d = (np.ascontiguousarray(np.broadcast_to(v, (h, w, 2)), np.float64) for v in (s, m, d))
    r.disparity = 2.0 * r.s[..., 0]
    r.vis4 = np.full((h, w), vis, np.uint8)
    return r


def test_scene_flow_zero_without_motion_oracle(oracle):
    """zero motion flow and d = 0 -> zero scene-flow vector."""
    rng = np.random.default_rng(3)
    w, h = 24, 16
    r = _flow_result(w, h, np.stack([rng.uniform(-30, -5, (h, w)), rng.uniform(-1, 1, (h, w))], -1), 0.0, 0.0)
    oracle.compute_scene_points(r, make_rig(_rot(0.0, 0.01, 0.0), (-0.15, 0.0, 0.0)))
    assert r.point_valid.all()
    assert np.all(r.scene_flow == 0.0)
    assert np.all(r.points0[..., 2] > 0)


def test_scene_points_match_motion_oracle(oracle):
    """Exact synthetic flows of a translating plane: points0/points1 are the plane at t and t+1."""
    rig = make_rig()
    w, h, Z0, dz = 32, 20, 5.0, -0.25
    f, b = K[0, 0], 0.12
    # rectified rig: x1 = x0 - f b / Z; for a fronto-parallel plane moving in depth the halfway flows are
    # s = -(f b / Z_t) / 2 along x at each t, so m and d carry the change between t = 0 and t = 1.
    sx = [-(f * b / (Z0 + k * dz)) / 2.0 for k in (0, 1)]
    s, mm, dd = 0.5 * (sx[0] + sx[1]), 0.0, 0.5 * (sx[1] - sx[0])
    # warp_position(x,f,c,t) = x + sc s + st m + sc st d; for c = 1: x + s + st d -> +-(s + st d) = sx[t]
    r = _flow_result(w, h, np.array([s, 0.0]), np.array([mm, 0.0]), np.array([dd, 0.0]))
    oracle.compute_scene_points(r, rig)
    assert r.point_valid.all()
    assert np.abs(r.points0[..., 2] - Z0).max() < 1e-9
    assert np.abs(r.points1[..., 2] - (Z0 + dz)).max() < 1e-9
    assert np.abs(r.scene_flow[..., 2] - dz).max() < 1e-9


def test_validate_rig_oracle(oracle):
    rig = make_rig(_rot(0.01, 0.02, -0.01), (-0.1, 0.005, 0.0))
    oracle.validate_rig(rig)
    oracle.validate_rig(StereoRig(F=rig.F))  # F only
    with pytest.raises(InvalidArgument, match="rank 2"):
        oracle.validate_rig(StereoRig(F=np.eye(3)))
    bad = StereoRig(F=make_rig(_rot(0.0, 0.1, 0.0)).F, P0=rig.P0, P1=rig.P1)
    with pytest.raises(InvalidArgument, match="inconsistent"):
        oracle.validate_rig(bad)
    with pytest.raises(InvalidArgument):
        oracle.compute_scene_points(_flow_result(4, 4, 0.0, 0.0, 0.0), StereoRig(F=rig.F))


def _read_obj(path):
    V, Fc = [], []
    for line in open(path):
        if line.startswith("v "):
            V.append([float(t) for t in line.split()[1:]])
        elif line.startswith("f "):
            Fc.append([int(t) for t in line.split()[1:]])
    return np.array(V).reshape(-1, 3), np.array(Fc, dtype=np.int64).reshape(-1, 3)


def test_mesh_export_oracle(oracle, tmp_path):
    """fronto-parallel plane -> planar mesh; fully occluded -> empty valid file; bounds."""
    rig = make_rig()
    w, h = 20, 14
    r = _flow_result(w, h, np.array([-6.0, 0.0]), 0.0, 0.0)
    r.vis4[3:6, 4:9] = 0x0B  # an occluded patch drops its vertices and their triangles
    oracle.compute_scene_points(r, rig)
    oracle.export_mesh_obj(r, tmp_path / "plane.obj")
    V, Fc = _read_obj(tmp_path / "plane.obj")
    assert len(V) == w * h - 15 and len(V) <= w * h
    assert 0 < len(Fc) <= 2 * (w - 1) * (h - 1)
    assert Fc.min() >= 1 and Fc.max() <= len(V)
    c = V.mean(0)
    _, _, vt = np.linalg.svd(V - c)
    dev = np.abs((V - c) @ vt[2]).max()
    assert dev < 1e-3 * np.ptp(V, axis=0).max()
    # disparity fallback: (x, y, disparity) vertices
    r2 = _flow_result(w, h, np.array([-3.0, 0.0]), 0.0, 0.0)
    oracle.export_mesh_obj(r2, tmp_path / "disp.obj")
    V2, F2 = _read_obj(tmp_path / "disp.obj")
    assert len(V2) == w * h and len(F2) == 2 * (w - 1) * (h - 1)
    assert np.all(V2[:, 2] == -6.0) and np.array_equal(V2[w + 1, :2], [1.0, 1.0])
    # fully occluded -> empty mesh, valid file
    r3 = _flow_result(w, h, 0.0, 0.0, 0.0, vis=0)
    oracle.export_mesh_obj(r3, tmp_path / "empty.obj")
    V3, F3 = _read_obj(tmp_path / "empty.obj")
    assert len(V3) == 0 and len(F3) == 0
    with pytest.raises(InvalidArgument, match="cannot open"):
        oracle.export_mesh_obj(r2, tmp_path / "missing_dir" / "x.obj")


def test_calibration_file(tmp_path):
    rig = make_rig()
    p = tmp_path / "calib.txt"
    p.write_text(" ".join(f"{v:.17g}" for v in np.concatenate([rig.F.ravel(), rig.P0.ravel(), rig.P1.ravel()])))
    r = StereoRig.load(p)
    assert np.array_equal(r.F, rig.F) and np.array_equal(r.P0, rig.P0) and np.array_equal(r.P1, rig.P1)
    p.write_text(" ".join(f"{v:.17g}" for v in rig.F.ravel()))
    assert not StereoRig.load(p).has_projections()


# ---------------------------------------------------------------- device vs oracle
@pytest.mark.gpu
def test_triangulate_device_matches_oracle(device, oracle):
    rng = np.random.default_rng(11)
    rig = make_rig(_rot(0.02, -0.03, 0.01), (-0.2, 0.01, 0.02))
    X = _random_points(rng, 4096)
    x0 = project(rig.P0, X) + rng.normal(0, 0.3, (4096, 2))  # noisy: full-rank A
    x1 = project(rig.P1, X) + rng.normal(0, 0.3, (4096, 2))
    x1[:64] = x0[:64]  # includes near-parallel rays
    Yd, okd = device.triangulate_dlt(rig.P0, rig.P1, x0, x1)
    Yo, oko = oracle.triangulate_dlt(rig.P0, rig.P1, x0, x1)
    assert np.array_equal(okd, oko)
    assert np.allclose(Yd, Yo, rtol=1e-9, atol=1e-12)
    Ye, oke = device.triangulate_dlt(rig.P0, rig.P1, project(rig.P0, X), project(rig.P1, X))
    assert oke.all() and np.abs(Ye - X).max() < 1e-6


@pytest.mark.gpu
def test_scene_points_device_matches_oracle(device, oracle, tmp_path):
    rng = np.random.default_rng(5)
    rig = make_rig(_rot(0.0, 0.02, 0.0), (-0.15, 0.0, 0.01))
    w, h = 96, 64
    r = [_flow_result(w, h, np.stack([rng.uniform(-20, -4, (h, w)), rng.uniform(-1, 1, (h, w))], -1),
                      rng.normal(0, 2, (h, w, 2)), rng.normal(0, 0.5, (h, w, 2))) for _ in range(2)]
    r[1] = _flow_result(w, h, r[0].s, r[0].m, r[0].d)
    r[0].vis4[::7] = 0x07
    r[1].vis4[::7] = 0x07
    device.compute_scene_points(r[0], rig)
    oracle.compute_scene_points(r[1], rig)
    assert np.array_equal(r[0].point_valid, r[1].point_valid)
    for k in ("points0", "points1", "scene_flow"):
        assert np.allclose(getattr(r[0], k), getattr(r[1], k), rtol=1e-9, atol=1e-9), k
    device.export_mesh_obj(r[0], tmp_path / "d.obj")
    oracle.export_mesh_obj(r[1], tmp_path / "o.obj")
    Vd, Fd = _read_obj(tmp_path / "d.obj")
    Vo, Fo = _read_obj(tmp_path / "o.obj")
    assert np.array_equal(Fd, Fo) and np.allclose(Vd, Vo, rtol=1e-9, atol=1e-9)
    device.validate_rig(rig)
    with pytest.raises(InvalidArgument):
        device.validate_rig(StereoRig(F=np.eye(3)))
