"""Ground truth and measurements for SPEC.md's acceptance criteria; test infrastructure."""
from __future__ import annotations

import numpy as np


def sample(img: np.ndarray, x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """Image::sample (image.cpp:19-46): edge-clamped bilinear at continuous positions."""
    h, w = img.shape

    def cell(v, n):
        i0 = np.clip(np.floor(v), 0, max(n - 2, 0)).astype(int)
        f = np.where(v <= 0, 0.0, np.where(v >= n - 1, 1.0, v - np.floor(v)))
        i0 = np.where(v >= n - 1, max(n - 2, 0), np.where(v <= 0, 0, i0))
        return i0, f

    ix, fx = cell(x, w)
    iy, fy = cell(y, h)
    x1, y1 = np.minimum(ix + 1, w - 1), np.minimum(iy + 1, h - 1)
    return ((1 - fx) * (1 - fy) * img[iy, ix] + fx * (1 - fy) * img[iy, x1] + (1 - fx) * fy * img[y1, ix]
            + fx * fy * img[y1, x1])


def interp_grid(grid: np.ndarray, w: int, h: int, step: int) -> np.ndarray:
    """WarpGrid::interpolate (warp_grid.cpp:41-65) of a (G, 6) grid at every pixel: (h, w, 6)."""
    gw, gh = (w - 1 + step - 1) // step + 1, (h - 1 + step - 1) // step + 1
    gw, gh = max(gw, 2), max(gh, 2)
    g = grid.reshape(gh, gw, 6)
    u, v = np.arange(w) / step, np.arange(h) / step
    a0 = np.clip(np.floor(u).astype(int), 0, gw - 2)
    b0 = np.clip(np.floor(v).astype(int), 0, gh - 2)
    fu = np.clip(u - a0, 0.0, 1.0)[None, :, None]
    fv = np.clip(v - b0, 0.0, 1.0)[:, None, None]
    B0, A0 = np.meshgrid(b0, a0, indexing="ij")
    return ((1 - fu) * (1 - fv) * g[B0, A0] + fu * (1 - fv) * g[B0, A0 + 1] + (1 - fu) * fv * g[B0 + 1, A0]
            + fu * fv * g[B0 + 1, A0 + 1])


def warped(images: np.ndarray, flow: np.ndarray, e: int) -> np.ndarray:
    """I_e(warp_position(x, f, c, t)) (warp_grid.hpp:73-77) at every halfway pixel; flow (h, w, 6)."""
    h, w = images.shape[1:]
    sc, st = (1.0 if e & 1 else -1.0), (1.0 if e >> 1 else -1.0)
    X, Y = np.meshgrid(np.arange(w, dtype=np.float64), np.arange(h, dtype=np.float64))
    wx = X + sc * flow[..., 0] + st * flow[..., 2] + sc * st * flow[..., 4]
    wy = Y + sc * flow[..., 1] + st * flow[..., 3] + sc * st * flow[..., 5]
    return sample(images[e], wx, wy)


def occlusion_truth(w: int, h: int, rect, extra_s, level: int = 0) -> np.ndarray:
    """Ground-truth visibility (4, h, w) of synthetic.render_pair's two-layer scene at pyramid level `level`
    (pixel x of level l covers full-resolution pixels 2^l x .. 2^l x + 2^l - 1; its centre is tested). A
    background halfway pixel x is hidden in image e = c + 2t iff its position there shows the foreground:
    x + warp_e(f_bg) - warp_e(f_fg) = x - sc * extra_s lies in the foreground rect (render_pair's pull-back);
    foreground pixels are front-most in every view."""
    k = 2 ** level
    X, Y = np.meshgrid(k * np.arange(w) + 0.5 * (k - 1), k * np.arange(h) + 0.5 * (k - 1))
    x0, y0, x1, y1 = rect

    def inside(px, py):
        return (px >= x0) & (px < x1) & (py >= y0) & (py < y1)

    fg = inside(X, Y)
    vis = np.empty((4, h, w), bool)
    for e in range(4):
        sc = 1.0 if e & 1 else -1.0
        vis[e] = fg | ~inside(X - sc * extra_s[0], Y - sc * extra_s[1])
    return vis


def epipolar_residuals(grid: np.ndarray) -> np.ndarray:
    """|l^T F r| at every node and t for the rectified rig F = [[0,0,0],[0,0,-1],[0,1,0]] (x_0^T F x_1 = y_1 - y_0,
    energy.cpp:168-192): x_c = warp_position(node, f, c, t), so e_t = 2 (s_y + sigma_t d_y)."""
    return np.abs(np.concatenate([2.0 * (grid[:, 1] - grid[:, 5]), 2.0 * (grid[:, 1] + grid[:, 5])]))
