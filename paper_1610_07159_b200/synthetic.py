"""Synthetic procedurally-textured stereo sequences with known flow.

The reference's generator (src/synthetic.cpp) is not
shipped; this re-creates it per SURVEY.md §8d. T(x) is seeded band-limited
value noise (octaves at lattice spacings 4/8/16/32 px, smoothstep-bilinear) plus
a little white noise, normalised to [0.1, 0.9]. Images are exact pull-back
warps of T by the ground-truth flows, I_c^t(y) = T(y - sc*s - st*m - sc*st*d),
so that I_c^t(warp_position(x, f, c, t)) = T(x) (warp_grid.hpp:73-77), then
quantised to u8 (webcam-like).
"""
from __future__ import annotations

import numpy as np


def _octave(rng: np.random.Generator, spacing: float, xs: np.ndarray, ys: np.ndarray, extent: tuple[int, int]):
    gx = int(np.ceil(extent[0] / spacing)) + 4
    gy = int(np.ceil(extent[1] / spacing)) + 4
    lat = rng.random((gy, gx))
    u = xs / spacing + 2.0
    v = ys / spacing + 2.0
    i = np.clip(np.floor(u).astype(np.int64), 0, gx - 2)
    j = np.clip(np.floor(v).astype(np.int64), 0, gy - 2)
    fu = np.clip(u - i, 0.0, 1.0)
    fv = np.clip(v - j, 0.0, 1.0)
    fu = fu * fu * (3 - 2 * fu)
    fv = fv * fv * (3 - 2 * fv)
    a = lat[j, i] * (1 - fu) + lat[j, i + 1] * fu
    b = lat[j + 1, i] * (1 - fu) + lat[j + 1, i + 1] * fu
    return a * (1 - fv) + b * fv


def _weights_1d(coord: np.ndarray, spacing: float, n: int):
    """Lattice cell and smoothstep weight along one axis (same rule as _octave)."""
    u = coord / spacing + 2.0
    i = np.clip(np.floor(u).astype(np.int64), 0, n - 2)
    f = np.clip(u - i, 0.0, 1.0)
    return i, f * f * (3 - 2 * f)


class Texture:
    """Continuous, seeded texture T(x, y) over a margin-padded domain."""

    SPACINGS = (4.0, 8.0, 16.0, 32.0)

    def __init__(self, seed: int, w: int, h: int, margin: int = 96):
        self.seed, self.margin = seed, margin
        self.extent = (w + 2 * margin, h + 2 * margin)

    def __call__(self, xs: np.ndarray, ys: np.ndarray) -> np.ndarray:
        rng = np.random.default_rng(self.seed)
        X, Y = xs + self.margin, ys + self.margin
        t = np.zeros_like(X, dtype=np.float64)
        for k, sp in enumerate(self.SPACINGS):
            t += (0.5 ** (3 - k)) * _octave(rng, sp, X, Y, self.extent)
        t /= 1.875
        return 0.1 + 0.8 * np.clip(t, 0.0, 1.0)

    def grid(self, x: np.ndarray, y: np.ndarray) -> np.ndarray:
        """T on the separable grid (y[r], x[c]); same values as __call__ on that grid,
        evaluated per octave as a 1-D blend along x for every lattice row, then along y."""
        rng = np.random.default_rng(self.seed)
        X, Y = x + self.margin, y + self.margin
        t = np.zeros((y.size, x.size))
        for k, sp in enumerate(self.SPACINGS):
            gx = int(np.ceil(self.extent[0] / sp)) + 4
            gy = int(np.ceil(self.extent[1] / sp)) + 4
            lat = rng.random((gy, gx))
            i, fu = _weights_1d(X, sp, gx)
            j, fv = _weights_1d(Y, sp, gy)
            A = lat[:, i] * (1 - fu) + lat[:, i + 1] * fu  # (gy, W)
            t += (0.5 ** (3 - k)) * (A[j] * (1 - fv)[:, None] + A[j + 1] * fv[:, None])
        t /= 1.875
        return 0.1 + 0.8 * np.clip(t, 0.0, 1.0)


def render_pair(w: int, h: int, s=(0.0, 0.0), m=(0.0, 0.0), d=(0.0, 0.0), seed: int = 1610, noise: float = 0.01,
                occluder: dict | None = None, gain_offset: dict | None = None, dtype=np.uint8,
                shift=(0.0, 0.0)) -> np.ndarray:
    """Four images (4, h, w) by image_index(c,t) = c + 2t for constant flows.

    occluder: {"rect": (x0, y0, x1, y1) in the halfway domain, "extra_s": (sx, sy)}
        foreground square with its own stereo flow s + extra_s (two-layer scene).
    gain_offset: {"offset": [o0..o3], "gain": [g0..g3]} per image (illumination change).
    """
    T = Texture(seed, w, h)
    Tf = Texture(seed + 7919, w, h) if occluder else None
    # shift: global translation of the scene (sequences: frame k of a moving texture)
    x1d, y1d = np.arange(w, dtype=np.float64) - shift[0], np.arange(h, dtype=np.float64) - shift[1]
    rng = np.random.default_rng(seed + 1)
    out = np.empty((4, h, w))
    for e in range(4):
        sc = -1.0 if (e & 1) == 0 else 1.0
        st = -1.0 if (e >> 1) == 0 else 1.0
        # constant flows: the pull-back grid is the pixel grid shifted (separable)
        img = T.grid(x1d - (sc * s[0] + st * m[0] + sc * st * d[0]), y1d - (sc * s[1] + st * m[1] + sc * st * d[1]))
        if occluder:
            x0, y0, x1, y1 = occluder["rect"]
            fs = (s[0] + occluder["extra_s"][0], s[1] + occluder["extra_s"][1])
            fx = x1d - (sc * fs[0] + st * m[0] + sc * st * d[0])
            fy = y1d - (sc * fs[1] + st * m[1] + sc * st * d[1])
            inside = ((fy >= y0) & (fy < y1))[:, None] & ((fx >= x0) & (fx < x1))[None, :]
            img = np.where(inside, Tf.grid(fx, fy), img)
        if gain_offset:
            img = img * gain_offset.get("gain", [1, 1, 1, 1])[e] + gain_offset.get("offset", [0, 0, 0, 0])[e]
        img = img + noise * rng.standard_normal(img.shape)
        out[e] = np.clip(img, 0.0, 1.0)
    if dtype == np.uint8:
        return np.round(out * 255.0).astype(np.uint8)
    return out


def webcam_truth(index: int) -> dict:
    """The known constant flow of cfg2/cfg4 pair `index` (halfway convention): s in [0, 4] px
    (disparity 2s in [0, 8]), m in [-2, 2]^2 px (inter-frame motion 2m in [-4, 4]^2), d = 0."""
    rng = np.random.default_rng(1610 + index)
    s = (float(rng.uniform(0.0, 4.0)), 0.0)
    m = (float(rng.uniform(-2.0, 2.0)), float(rng.uniform(-2.0, 2.0)))
    return {"s": s, "m": m, "d": (0.0, 0.0)}


def webcam_pair(index: int, w: int = 640, h: int = 480) -> tuple[np.ndarray, dict]:
    """cfg2/cfg4 pair `index`, seed 1610+index, flow webcam_truth(index)."""
    gt = webcam_truth(index)
    return render_pair(w, h, s=gt["s"], m=gt["m"], seed=1610 + index), gt


def flow_error(grid_total: np.ndarray, truths: list[dict]) -> dict:
    """Node error of solved finest warp grids (n, G, 6) against constant known flows: median and
    90th percentile over all nodes of |s - s_gt| and |m - m_gt| (px)."""
    g = np.asarray(grid_total).reshape(len(truths), -1, 6)
    st = np.array([t["s"] for t in truths])[:, None, :]
    mt = np.array([t["m"] for t in truths])[:, None, :]
    es = np.hypot(g[..., 0] - st[..., 0], g[..., 1] - st[..., 1])
    em = np.hypot(g[..., 2] - mt[..., 0], g[..., 3] - mt[..., 1])
    return {"s_median_px": float(np.median(es)), "s_p90_px": float(np.percentile(es, 90)),
            "m_median_px": float(np.median(em)), "m_p90_px": float(np.percentile(em, 90))}


def constant_pair(w: int = 320, h: int = 240, seed: int = 1610) -> tuple[np.ndarray, dict]:
    """cfg1: s = (1.5, 0) (disparity 3 px), m = (0.75, 0.5) (motion (1.5, 1.0)), d = 0."""
    s, m = (1.5, 0.0), (0.75, 0.5)
    return render_pair(w, h, s=s, m=m, seed=seed), {"s": s, "m": m, "d": (0.0, 0.0)}


def valgaerts_pair(index: int = 0, w: int = 1920, h: int = 1080) -> tuple[np.ndarray, dict]:
    """cfg3: two-layer occluder (foreground square with +6 px extra disparity, i.e. +3 px
    of half-disparity s) and per-camera illumination change (right camera +0.05 offset,
    t+1 gain x1.05), SURVEY.md §8d."""
    rng = np.random.default_rng(7919 + index)
    s = (float(rng.uniform(1.0, 3.0)), 0.0)
    m = (float(rng.uniform(-1.5, 1.5)), float(rng.uniform(-1.0, 1.0)))
    rect = (w // 3, h // 3, 2 * w // 3, 2 * h // 3)
    go = {"offset": [0.0, 0.05, 0.0, 0.05], "gain": [1.0, 1.0, 1.05, 1.05]}
    imgs = render_pair(w, h, s=s, m=m, seed=2000 + index, occluder={"rect": rect, "extra_s": (3.0, 0.0)},
                       gain_offset=go)
    return imgs, {"s": s, "m": m, "d": (0.0, 0.0), "rect": rect, "extra_s": (3.0, 0.0)}


def uhd_pair(index: int = 0, w: int = 3840, h: int = 2160) -> tuple[np.ndarray, dict]:
    """cfg5: one 3840x2160 pair with known constant flow."""
    rng = np.random.default_rng(4000 + index)
    s = (float(rng.uniform(1.0, 6.0)), 0.0)
    m = (float(rng.uniform(-3.0, 3.0)), float(rng.uniform(-3.0, 3.0)))
    return render_pair(w, h, s=s, m=m, seed=4000 + index), {"s": s, "m": m, "d": (0.0, 0.0)}


def sequence_pairs(n_pairs: int, w: int, h: int, s=(1.5, 0.0), v=(2.0, 1.0), seed: int = 1610) -> list[np.ndarray]:
    """A constant-velocity stereo sequence: frame t shows the texture translated by t*v (inter-frame
    motion v = 2m in the halfway convention); pair k = frames (k, k+1), i.e. render_pair with
    m = v/2 and the scene shifted by (k + 1/2) v. Noise-free so consecutive pairs share pixels."""
    m = (v[0] / 2.0, v[1] / 2.0)
    return [render_pair(w, h, s=s, m=m, seed=seed, noise=0.0, shift=((k + 0.5) * v[0], (k + 0.5) * v[1]))
            for k in range(n_pairs)]
