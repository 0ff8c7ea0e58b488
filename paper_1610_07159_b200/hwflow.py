"""Host-side mirror of the reference's hwflow:: interface over the C-ABI.

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj/include/hwflow/*.hpp and SPEC.md): EnergyParams
(energy.hpp:17-39), SolveSchedule (solver.hpp:14-35), FlowResult
(geometry.hpp:26-37), run_scene_flow, gauss_newton
(solver.hpp:152), build_pyramid (image.hpp:83), build_normal_system
(solver.hpp:91), pcg_solve (solver.hpp:117), schwarz_iterate (solver.hpp:138),
compute_occlusion_maps / compute_illumination_maps / prolongate.
SolverDivergence is raised where the reference throws it (core.hpp:19).

`Solver()` binds the product library (lib/libhwflow_cuda.so, sm_100a) and
fails loudly if it is missing or no GPU is usable — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import capi
from .capi import (DTYPE_F64, DTYPE_U8, EnergyC, EnergyParamsC, Frame4C, LevelC, ResultC, ScheduleC, StatsC,
                   SolverDivergence, dptr, u8ptr)

CUDA_LIB_PATH = Path(__file__).resolve().parent / "lib" / "libhwflow_cuda.so"

__all__ = ["EnergyParams", "SolveSchedule", "FlowResult", "GnStats", "LevelState", "Solver", "SolverDivergence",
           "image_index", "grid_dims", "level_dims", "CUDA_LIB_PATH"]


def image_index(cam: int, time: int) -> int:  # core.hpp:27
    return cam + 2 * time


def grid_dims(w: int, h: int, step: int) -> tuple[int, int]:  # warp_grid.cpp:11-14
    return max((w - 1 + step - 1) // step + 1, 2), max((h - 1 + step - 1) // step + 1, 2)


@dataclass
class EnergyParams:  # energy.hpp:17-39 (defaults = "live")
    w_reg: float = 1.0
    w_photo: float = 1.0
    w_grad: float = 2.0
    w_epi: float = 0.0
    w_smooth: float = 1.0
    w_mag: float = 1.0
    w_s: float = 5.0
    w_m: float = 5.0
    w_d: float = 0.5
    m_s: float = 5.0
    m_m: float = 100.0
    m_d: float = 1000.0
    eps_huber: float = 0.001
    eps_color: float = 0.2

    @staticmethod
    def preset(name: str) -> "EnergyParams":  # energy.cpp:9-41
        p = EnergyParams()
        if name == "live":
            return p
        if name == "facial":
            return EnergyParams(w_reg=0.5, w_photo=0.5, w_grad=5.0, w_epi=0.5, w_s=0.75, w_m=0.5, w_d=0.01,
                                m_s=0.5, m_m=10.0, m_d=100.0)
        if name == "stereo-hq":
            return EnergyParams(w_reg=5.0, w_photo=1.0, w_grad=5.0, w_epi=0.5, w_s=0.5, w_m=1.0, w_d=1.0,
                                m_s=0.1, m_m=10000.0, m_d=10000.0)
        raise ValueError(f"unknown preset: {name}")

    def validate(self) -> None:  # energy.cpp:43-50
        for k in ("w_reg", "w_photo", "w_grad", "w_epi", "w_smooth", "w_mag", "w_s", "w_m", "w_d", "m_s", "m_m",
                  "m_d"):
            if not getattr(self, k) >= 0.0:
                raise ValueError("energy weights must be >= 0")
        if not self.eps_huber > 0.0:
            raise ValueError("eps_huber must be > 0")

    def to_c(self) -> EnergyParamsC:
        return EnergyParamsC(*[float(getattr(self, n)) for n, _ in EnergyParamsC._fields_])


@dataclass
class SolveSchedule:  # solver.hpp:14-35
    levels: int = 5
    gn_per_level: list[int] = field(default_factory=list)
    pcg_iters: int = 5
    patch_iters: int = 5
    subdomain_px: int = 16
    boundary_px: int = 2
    grid_step: int = 2
    threads: int = 1
    lm_lambda: float = 0.0
    active_fields: int = 0b111
    coarse_s_offset: tuple[float, float] = (0.0, 0.0)

    def gn_for_level(self, level: int) -> int:
        if self.gn_per_level:
            return self.gn_per_level[min(level, len(self.gn_per_level) - 1)]
        return 2 if level <= 1 else 5

    def to_c(self) -> ScheduleC:
        s = ScheduleC()
        s.levels = self.levels
        s.n_gn_per_level = len(self.gn_per_level)
        for i, g in enumerate(self.gn_per_level[: capi.HWF_MAX_LEVELS]):
            s.gn_per_level[i] = g
        s.pcg_iters, s.patch_iters = self.pcg_iters, self.patch_iters
        s.subdomain_px, s.boundary_px, s.grid_step = self.subdomain_px, self.boundary_px, self.grid_step
        s.threads, s.lm_lambda, s.active_fields = self.threads, self.lm_lambda, self.active_fields
        s.coarse_s_offset[0], s.coarse_s_offset[1] = self.coarse_s_offset
        return s


@dataclass
class GnStats:  # solver.hpp:142-147, one entry per level (0 = finest)
    energy_before: list[list[float]]
    energy_after: list[list[float]]

    @staticmethod
    def from_c(st: StatsC) -> "GnStats":
        L = st.levels_used
        eb = [[st.energy_before[l][i] for i in range(st.gn_iters[l])] for l in range(L)]
        ea = [[st.energy_after[l][i] for i in range(st.gn_iters[l])] for l in range(L)]
        return GnStats(eb, ea)

    def final_energy(self) -> float:
        return self.energy_after[0][-1] if self.energy_after and self.energy_after[0] else float("nan")


@dataclass
class FlowResult:  # geometry.hpp:26-37 (3D points are out of scope)
    width: int
    height: int
    s: np.ndarray | None = None          # (h, w, 2)
    m: np.ndarray | None = None
    d: np.ndarray | None = None
    disparity: np.ndarray | None = None  # (h, w) = 2 s_x
    vis4: np.ndarray | None = None       # (h, w) bit e = visible in image e
    grid_total: np.ndarray | None = None  # (G, 6) finest accumulated warp grid


@dataclass
class LevelState:
    """What EnergyContext + PixelWeights hold at one level (energy.hpp:51-88)."""
    images: np.ndarray                    # (4, h, w) float64
    grid_step: int
    total: np.ndarray                     # (G, 6)
    delta: np.ndarray                     # (G, 6)
    vis4: np.ndarray | None = None        # (h, w) uint8, default all visible
    outlier: np.ndarray | None = None     # (h, w) uint8, default 1
    node_w: np.ndarray | None = None      # (G,), default 1
    illum: np.ndarray | None = None       # (4, h, w) or None
    fundamental: np.ndarray | None = None  # (3, 3)

    def __post_init__(self):
        self.images = np.ascontiguousarray(self.images, dtype=np.float64)
        _, h, w = self.images.shape
        gw, gh = grid_dims(w, h, self.grid_step)
        self.total = np.ascontiguousarray(self.total, dtype=np.float64).reshape(gw * gh, 6)
        self.delta = np.ascontiguousarray(self.delta, dtype=np.float64).reshape(gw * gh, 6)
        self.vis4 = np.full((h, w), 0x0F, np.uint8) if self.vis4 is None else np.ascontiguousarray(self.vis4, np.uint8)
        self.outlier = np.ones((h, w), np.uint8) if self.outlier is None else np.ascontiguousarray(self.outlier, np.uint8)
        self.node_w = np.ones(gw * gh) if self.node_w is None else np.ascontiguousarray(self.node_w, np.float64)
        if self.illum is not None:
            self.illum = np.ascontiguousarray(self.illum, dtype=np.float64)
        if self.fundamental is not None:
            self.fundamental = np.ascontiguousarray(self.fundamental, dtype=np.float64).reshape(3, 3)

    @property
    def width(self) -> int:
        return self.images.shape[2]

    @property
    def height(self) -> int:
        return self.images.shape[1]

    def to_c(self) -> LevelC:
        lv = LevelC()
        lv.width, lv.height, lv.grid_step = self.width, self.height, self.grid_step
        for e in range(4):
            lv.images[e] = dptr(self.images[e])
            lv.illum[e] = dptr(self.illum[e]) if self.illum is not None else dptr(None)
        lv.total, lv.delta = dptr(self.total), dptr(self.delta)
        lv.vis4, lv.outlier, lv.node_w = u8ptr(self.vis4), u8ptr(self.outlier), dptr(self.node_w)
        lv.fundamental = dptr(self.fundamental) if self.fundamental is not None else dptr(None)
        return lv


def level_dims(lib: capi.Library, w: int, h: int, levels: int, step: int) -> list[tuple[int, int, int, int]]:
    used = C.c_int()
    dims = (C.c_int * (4 * capi.HWF_MAX_LEVELS))()
    if lib.hwf_level_dims(w, h, levels, step, C.byref(used), dims) != capi.HWF_OK:
        raise ValueError("bad level dims")
    return [tuple(dims[4 * l: 4 * l + 4]) for l in range(used.value)]


def _frame(images: np.ndarray) -> tuple[Frame4C, np.ndarray]:
    a = np.ascontiguousarray(images)
    if a.ndim != 3 or a.shape[0] != 4:
        raise ValueError("images must be (4, h, w) indexed by image_index(c,t) = c + 2t")
    if a.dtype == np.uint8:
        dt = DTYPE_U8
    else:
        a = np.ascontiguousarray(a, dtype=np.float64)
        dt = DTYPE_F64
    f = Frame4C()
    f.width, f.height, f.dtype = a.shape[2], a.shape[1], dt
    for e in range(4):
        f.plane[e] = a[e].ctypes.data
    return f, a


class SequenceState:
    """hwf_state: the per-level delta hierarchy + accumulated grids of n pairs."""

    def __init__(self, solver: "Solver", n: int, width: int, height: int, schedule: SolveSchedule):
        self.solver, self.n, self.width, self.height = solver, n, width, height
        self.levels = level_dims(solver.lib, width, height, schedule.levels, schedule.grid_step)
        h = C.c_void_p()
        solver.ctx.check(solver.lib.hwf_state_create(solver.ctx.h, n, width, height, schedule.levels,
                                                     schedule.grid_step, C.byref(h)))
        self.h = h

    def read(self, pair: int) -> tuple[list[np.ndarray], list[np.ndarray]]:
        sizes = [6 * gw * gh for (_, _, gw, gh) in self.levels]
        d, t = np.empty(sum(sizes)), np.empty(sum(sizes))
        self.solver.ctx.check(self.solver.lib.hwf_state_read(self.solver.ctx.h, self.h, pair, dptr(d), dptr(t)))
        offs = np.cumsum([0] + sizes)
        return ([d[offs[i]:offs[i + 1]].reshape(-1, 6) for i in range(len(sizes))],
                [t[offs[i]:offs[i + 1]].reshape(-1, 6) for i in range(len(sizes))])

    def __del__(self):
        try:
            if self.h:
                self.solver.lib.hwf_state_destroy(self.h)
                self.h = None
        except Exception:
            pass


class Solver:
    """One device context (or, in tests, one CPU checker) behind the C-ABI."""

    def __init__(self, lib: capi.Library | str | Path | None = None, device: int = 0):
        if lib is None:
            if not CUDA_LIB_PATH.exists():
                raise RuntimeError(f"{CUDA_LIB_PATH} is missing: run `python -m paper_1610_07159_b200.build cuda` "
                                   "(there is no CPU fallback)")
            lib = CUDA_LIB_PATH
        self.lib = lib if isinstance(lib, capi.Library) else capi.Library(lib)
        self.ctx = capi.Context(self.lib, device)

    @property
    def backend(self) -> str:
        return self.lib.backend

    def close(self):
        self.ctx.close()

    # ---- Algorithm 1 -------------------------------------------------------
    def solve_batch(self, frames: np.ndarray, params: EnergyParams, schedule: SolveSchedule,
                    fundamental: np.ndarray | None = None, outputs=("s", "m", "d", "disparity", "vis4", "grid_total"),
                    ) -> tuple[list[FlowResult], list[GnStats]]:
        """frames: (n, 4, h, w) uint8 or float64 — n independent frame pairs, one device batch."""
        return self._solve(frames, params, schedule, fundamental, outputs, None, None)

    def _solve(self, frames, params, schedule, fundamental, outputs, prev, nxt):
        a = np.ascontiguousarray(frames)
        if a.ndim != 4 or a.shape[1] != 4:
            raise ValueError("frames must be (n, 4, h, w)")
        if a.dtype != np.uint8:
            a = np.ascontiguousarray(a, dtype=np.float64)
        n, _, h, w = a.shape
        gw, gh = grid_dims(w, h, schedule.grid_step)
        fr = (Frame4C * n)()
        for i in range(n):
            fr[i].width, fr[i].height = w, h
            fr[i].dtype = DTYPE_U8 if a.dtype == np.uint8 else DTYPE_F64
            for e in range(4):
                fr[i].plane[e] = a[i, e].ctypes.data
        res = (ResultC * n)()
        outs = []
        for i in range(n):
            o = FlowResult(w, h)
            if "s" in outputs: o.s = np.empty((h, w, 2))
            if "m" in outputs: o.m = np.empty((h, w, 2))
            if "d" in outputs: o.d = np.empty((h, w, 2))
            if "disparity" in outputs: o.disparity = np.empty((h, w))
            if "vis4" in outputs: o.vis4 = np.empty((h, w), np.uint8)
            if "grid_total" in outputs: o.grid_total = np.empty((gw * gh, 6))
            res[i].s, res[i].m, res[i].d = dptr(o.s), dptr(o.m), dptr(o.d)
            res[i].disparity, res[i].vis4, res[i].grid_total = dptr(o.disparity), u8ptr(o.vis4), dptr(o.grid_total)
            outs.append(o)
        stats = (StatsC * n)()
        F = None if fundamental is None else np.ascontiguousarray(fundamental, np.float64).reshape(9)
        pc, sc = params.to_c(), schedule.to_c()
        if prev is None and nxt is None:
            rc = self.lib.hwf_solve_batch(self.ctx.h, n, fr, C.byref(pc), C.byref(sc), dptr(F), res, stats)
        else:
            rc = self.lib.hwf_solve_batch_seq(self.ctx.h, n, fr, C.byref(pc), C.byref(sc), dptr(F),
                                              prev.h if prev is not None else None,
                                              nxt.h if nxt is not None else None, res, stats)
        self.ctx.check(rc)
        return outs, [GnStats.from_c(stats[i]) for i in range(n)]

    # ---- sequences: temporal propagation ---------------------
    def new_state(self, n_pairs: int, width: int, height: int, schedule: SolveSchedule) -> "SequenceState":
        return SequenceState(self, n_pairs, width, height, schedule)

    def solve_batch_seq(self, frames: np.ndarray, params: EnergyParams, schedule: SolveSchedule,
                        prev: "SequenceState | None", nxt: "SequenceState | None",
                        fundamental: np.ndarray | None = None,
                        outputs=("s", "m", "d", "disparity", "vis4", "grid_total")):
        """n frame pairs, each warm-started from its own previous frame in `prev` (None: first frame)."""
        return self._solve(frames, params, schedule, fundamental, outputs, prev, nxt)

    def propagate_temporal(self, width: int, height: int, step: int, prev_delta: np.ndarray,
                           prev_total: np.ndarray) -> np.ndarray:
        pd, pt = np.ascontiguousarray(prev_delta, np.float64), np.ascontiguousarray(prev_total, np.float64)
        out = np.empty_like(pd)
        self.ctx.check(self.lib.hwf_propagate_temporal(self.ctx.h, width, height, step, dptr(pd), dptr(pt), dptr(out)))
        return out

    def run_scene_flow(self, images: np.ndarray, params: EnergyParams, schedule: SolveSchedule,
                       fundamental: np.ndarray | None = None) -> tuple[FlowResult, GnStats]:
        """SPEC.md:396-404 for one frame pair; images (4, h, w) by image_index(c,t)."""
        outs, stats = self.solve_batch(np.asarray(images)[None], params, schedule, fundamental)
        return outs[0], stats[0]

    # ---- per-stage seams ---------------------------------------------------
    def build_pyramid(self, images: np.ndarray, levels: int) -> list[np.ndarray]:
        f, keep = _frame(images)
        h, w = keep.shape[1:]
        dims, total = [], 0
        for _ in range(levels):
            dims.append((h, w))
            total += 4 * h * w
            w, h = (w + 1) // 2, (h + 1) // 2
        out = np.empty(total)
        self.ctx.check(self.lib.hwf_pyramid(self.ctx.h, C.byref(f), levels, dptr(out)))
        res, off = [], 0
        for h, w in dims:
            res.append(out[off: off + 4 * h * w].reshape(4, h, w))
            off += 4 * h * w
        return res

    def energy(self, lv: LevelState, params: EnergyParams, residuals: bool = False) -> tuple[EnergyC, np.ndarray | None]:
        c, pc, e = lv.to_c(), params.to_c(), EnergyC()
        gw, gh = grid_dims(lv.width, lv.height, lv.grid_step)
        R = np.empty(2 * lv.width * lv.height + 14 * gw * gh) if residuals else None
        self.ctx.check(self.lib.hwf_eval_energy(self.ctx.h, C.byref(c), C.byref(pc), C.byref(e), dptr(R)))
        return e, R

    def refresh_weights(self, lv: LevelState, params: EnergyParams) -> tuple[np.ndarray, np.ndarray]:
        c, pc = lv.to_c(), params.to_c()
        W = np.empty((lv.height, lv.width), np.uint8)
        nw = np.empty(lv.node_w.shape)
        self.ctx.check(self.lib.hwf_refresh_weights(self.ctx.h, C.byref(c), C.byref(pc), u8ptr(W), dptr(nw)))
        return W, nw

    def build_normal_system(self, lv: LevelState, params: EnergyParams, active_fields: int = 7,
                            lm_lambda: float = 0.0):
        c, pc = lv.to_c(), params.to_c()
        G = lv.total.shape[0]
        blocks, rhs, pre = np.empty((G, 9, 6, 6)), np.empty(6 * G), np.empty((G, 3, 2, 2))
        self.ctx.check(self.lib.hwf_linearize(self.ctx.h, C.byref(c), C.byref(pc), active_fields, lm_lambda,
                                              dptr(blocks), dptr(rhs), dptr(pre)))
        return blocks, rhs, pre

    def pcg_solve(self, gw: int, gh: int, blocks: np.ndarray, rhs: np.ndarray, iters: int, trace: bool = False):
        b, r = np.ascontiguousarray(blocks, np.float64), np.ascontiguousarray(rhs, np.float64)
        x = np.empty(6 * gw * gh)
        tr = np.empty(iters + 1) if trace else None
        self.ctx.check(self.lib.hwf_pcg(self.ctx.h, gw, gh, dptr(b), dptr(r), iters, dptr(x), dptr(tr)))
        return (x, tr) if trace else x

    def schwarz_iterate(self, gw: int, gh: int, step: int, blocks: np.ndarray, rhs: np.ndarray, patch_iters: int,
                        pcg_iters: int, tile_px: int = 16, boundary_px: int = 2) -> np.ndarray:
        b, r = np.ascontiguousarray(blocks, np.float64), np.ascontiguousarray(rhs, np.float64)
        x = np.empty(6 * gw * gh)
        self.ctx.check(self.lib.hwf_schwarz(self.ctx.h, gw, gh, step, tile_px, boundary_px, dptr(b), dptr(r),
                                            patch_iters, pcg_iters, dptr(x)))
        return x

    def gauss_newton(self, lv: LevelState, base: np.ndarray, params: EnergyParams, schedule: SolveSchedule,
                     gn_iters: int):
        """solver.cpp:484-532; returns (delta, outlier, node_w, energy_before, energy_after)."""
        c, pc, sc = lv.to_c(), params.to_c(), schedule.to_c()
        base = np.ascontiguousarray(base, np.float64).reshape(-1, 6)
        delta = lv.delta.copy()
        W, nw = lv.outlier.copy(), lv.node_w.copy()
        eb, ea = np.empty(max(gn_iters, 1)), np.empty(max(gn_iters, 1))
        self.ctx.check(self.lib.hwf_gn_level(self.ctx.h, C.byref(c), dptr(base), dptr(delta), u8ptr(W), dptr(nw),
                                             C.byref(pc), C.byref(sc), gn_iters, dptr(eb), dptr(ea)))
        return delta, W, nw, eb[:gn_iters], ea[:gn_iters]

    def compute_occlusion_maps(self, w: int, h: int, step: int, total: np.ndarray) -> np.ndarray:
        t = np.ascontiguousarray(total, np.float64)
        v = np.empty((h, w), np.uint8)
        self.ctx.check(self.lib.hwf_occlusion(self.ctx.h, w, h, step, dptr(t), u8ptr(v)))
        return v

    def compute_illumination_maps(self, images: np.ndarray, step: int, total: np.ndarray, vis4: np.ndarray):
        im = np.ascontiguousarray(images, np.float64)
        _, h, w = im.shape
        arr = (capi._dp * 4)(*[dptr(im[e]) for e in range(4)])
        t, v = np.ascontiguousarray(total, np.float64), np.ascontiguousarray(vis4, np.uint8)
        hm = np.empty((2, h, w))
        self.ctx.check(self.lib.hwf_illumination(self.ctx.h, w, h, step, arr, dptr(t), u8ptr(v), dptr(hm)))
        return hm

    def prolongate(self, wc, hc, wf, hf, step, total_c, vis_c=None, hm_c=None):
        gwf, ghf = grid_dims(wf, hf, step)
        base = np.empty((gwf * ghf, 6))
        tc = np.ascontiguousarray(total_c, np.float64)
        vc = None if vis_c is None else np.ascontiguousarray(vis_c, np.uint8)
        hc_ = None if hm_c is None else np.ascontiguousarray(hm_c, np.float64)
        vf = np.empty((hf, wf), np.uint8) if vc is not None else None
        hf_ = np.empty((2, hf, wf)) if hc_ is not None else None
        self.ctx.check(self.lib.hwf_prolongate(self.ctx.h, wc, hc, wf, hf, step, dptr(tc), u8ptr(vc), dptr(hc_),
                                               dptr(base), u8ptr(vf), dptr(hf_)))
        return base, vf, hf_
