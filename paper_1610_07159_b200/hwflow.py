"""Host-side mirror of the reference's hwflow:: interface over the C-ABI.

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj/include/hwflow/*.hpp and SPEC.md): EnergyParams
(energy.hpp:17-39), SolveSchedule (solver.hpp:14-35), FlowResult
(geometry.hpp:26-37), run_scene_flow, gauss_newton
(solver.hpp:152), build_pyramid (image.hpp:83), build_normal_system
(solver.hpp:91), pcg_solve (solver.hpp:117), schwarz_iterate (solver.hpp:138),
compute_occlusion_maps / compute_illumination_maps / prolongate,
StereoRig / triangulate_dlt / compute_scene_points / export_mesh_obj (geometry.hpp:14-59).
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
from .capi import (DTYPE_F64, DTYPE_U8, EnergyC, EnergyParamsC, Frame4C, LevelC, ResultC, RigC, ScheduleC,
                   StatsC, SolverDivergence, dptr, u8ptr)

CUDA_LIB_PATH = Path(__file__).resolve().parent / "lib" / "libhwflow_cuda.so"

__all__ = ["EnergyParams", "SolveSchedule", "FlowResult", "GnStats", "LevelState", "Solver", "SolverDivergence",
           "StereoRig", "image_index", "grid_dims", "level_dims", "CUDA_LIB_PATH"]


def image_index(cam: int, time: int) -> int:  # core.hpp:27
    return cam + 2 * time


def grid_dims(w: int, h: int, step: int) -> tuple[int, int]:  # warp_grid.cpp:8-14
    if w < 1 or h < 1 or step < 1:
        raise capi.InvalidArgument(capi.HWF_EINVAL, "WarpGrid: bad dimensions or step")
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
class FlowResult:  # geometry.hpp:26-37
    width: int
    height: int
    s: np.ndarray | None = None          # (h, w, 2)
    m: np.ndarray | None = None
    d: np.ndarray | None = None
    disparity: np.ndarray | None = None  # (h, w) = 2 s_x
    vis4: np.ndarray | None = None       # (h, w) bit e = visible in image e
    grid_total: np.ndarray | None = None  # (G, 6) finest accumulated warp grid
    has_points: bool = False             # filled by Solver.compute_scene_points
    points0: np.ndarray | None = None    # (h, w, 3) triangulated at t = 0
    points1: np.ndarray | None = None    # (h, w, 3) at t = 1
    scene_flow: np.ndarray | None = None  # (h, w, 3) = points1 - points0
    point_valid: np.ndarray | None = None  # (h, w) uint8

    def pixel_count(self) -> int:
        return self.width * self.height


@dataclass
class StereoRig:  # geometry.hpp:14-23: x_0^T F x_1 = 0 (energy.cpp:176-178), optional 3x4 projections
    F: np.ndarray = field(default_factory=lambda: np.zeros((3, 3)))
    P0: np.ndarray | None = None
    P1: np.ndarray | None = None

    def has_projections(self) -> bool:
        return self.P0 is not None and self.P1 is not None

    def to_c(self) -> RigC:
        r = RigC()
        r.F[:] = np.asarray(self.F, np.float64).ravel().tolist()
        r.has_projections = int(self.has_projections())
        if self.has_projections():
            r.P0[:] = np.asarray(self.P0, np.float64).ravel().tolist()
            r.P1[:] = np.asarray(self.P1, np.float64).ravel().tolist()
        return r

    @staticmethod
    def load(path: str | Path) -> "StereoRig":
        """Calibration file: 9 numbers (row-major F), optionally followed by 12 + 12 (P0, P1)."""
        v = np.array(Path(path).read_text().split(), dtype=np.float64)
        if v.size not in (9, 33):
            raise ValueError(f"calibration file needs 9 or 33 numbers, got {v.size}")
        rig = StereoRig(F=v[:9].reshape(3, 3))
        if v.size == 33:
            rig.P0, rig.P1 = v[9:21].reshape(3, 4), v[21:33].reshape(3, 4)
        return rig


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

    def assemble_jacobian(self, lv: LevelState, params: EnergyParams, active_fields: int = 7, negate_field: int = -1):
        """assemble_jacobian (solver.hpp:106-111, solver.cpp:247-314): (R, rows, cols, vals), the stacked residuals
        (M = 2N + 14G) and dR/dx as triplets in the reference's order; negate_field flips one flow field's analytic
        derivatives (the negative-control hook)."""
        c, pc = lv.to_c(), params.to_c()
        gw, gh = grid_dims(lv.width, lv.height, lv.grid_step)
        R = np.empty(2 * lv.width * lv.height + 14 * gw * gh)
        nnz = C.c_longlong()
        self.ctx.check(self.lib.hwf_assemble_jacobian(self.ctx.h, C.byref(c), C.byref(pc), active_fields, negate_field,
                                                      dptr(None), None, None, dptr(None), 0, C.byref(nnz)))
        n = nnz.value
        rows, cols, vals = np.empty(n, np.int32), np.empty(n, np.int32), np.empty(n)
        ip = C.POINTER(C.c_int)
        self.ctx.check(self.lib.hwf_assemble_jacobian(self.ctx.h, C.byref(c), C.byref(pc), active_fields, negate_field,
                                                      dptr(R), rows.ctypes.data_as(ip), cols.ctypes.data_as(ip),
                                                      dptr(vals), n, C.byref(nnz)))
        return R, rows, cols, vals

    def normal_dense(self, gw: int, gh: int, blocks: np.ndarray) -> np.ndarray:
        """NormalSystem::dense (solver.hpp:77, solver.cpp:89-98) of a system in hwf_linearize layout."""
        b = np.ascontiguousarray(blocks, np.float64)
        D = 6 * gw * gh
        out = np.empty((D, D))
        rc = self.lib.hwf_normal_dense(gw, gh, dptr(b), dptr(out))
        if rc != capi.HWF_OK:
            raise ValueError("hwf_normal_dense: bad arguments")
        return out

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
                     gn_iters: int, pcg_trace: bool = False):
        """solver.cpp:484-532; returns (delta, outlier, node_w, energy_before, energy_after), plus the
        per-iteration PCG residual-norm traces (gn_iters, pcg_iters + 1) when pcg_trace (global-PCG mode,
        SolveSchedule::pcg_trace, solver.cpp:508-513)."""
        c, pc, sc = lv.to_c(), params.to_c(), schedule.to_c()
        base = np.ascontiguousarray(base, np.float64).reshape(-1, 6)
        delta = lv.delta.copy()
        W, nw = lv.outlier.copy(), lv.node_w.copy()
        eb, ea = np.empty(max(gn_iters, 1)), np.empty(max(gn_iters, 1))
        tr = np.zeros((max(gn_iters, 1), schedule.pcg_iters + 1)) if pcg_trace else None
        self.ctx.check(self.lib.hwf_gn_level_trace(self.ctx.h, C.byref(c), dptr(base), dptr(delta), u8ptr(W),
                                                   dptr(nw), C.byref(pc), C.byref(sc), gn_iters, dptr(eb), dptr(ea),
                                                   dptr(tr)))
        out = (delta, W, nw, eb[:gn_iters], ea[:gn_iters])
        return out + (tr[:gn_iters],) if pcg_trace else out

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

    # ---- geometry (geometry.hpp:14-59) ------------------------------------
    def validate_rig(self, rig: StereoRig) -> None:
        """StereoRig::validate: raises InvalidArgument (a ValueError) on failure."""
        rc = rig.to_c()
        self.ctx.check(self.lib.hwf_validate_rig(self.ctx.h, C.byref(rc)))

    def triangulate_dlt(self, P0: np.ndarray, P1: np.ndarray, x0: np.ndarray, x1: np.ndarray):
        """Vectorised triangulate_dlt: x0, x1 (..., 2) -> points (..., 3), valid (...)."""
        a0, a1 = np.ascontiguousarray(x0, np.float64), np.ascontiguousarray(x1, np.float64)
        shape = a0.shape[:-1]
        n = int(np.prod(shape)) if shape else 1
        X, ok = np.zeros(shape + (3,)), np.zeros(shape, np.uint8)
        p0, p1 = np.ascontiguousarray(P0, np.float64), np.ascontiguousarray(P1, np.float64)
        self.ctx.check(self.lib.hwf_triangulate(self.ctx.h, n, dptr(p0), dptr(p1), dptr(a0), dptr(a1), dptr(X),
                                                u8ptr(ok)))
        return X, ok.astype(bool)

    def triangulate_pixel(self, x, f, t: int, rig: StereoRig):
        """geometry.hpp:50-52: f = (s, m, d) Vec2s; the correspondence (warp_position(x,f,0,t), (x,f,1,t))."""
        x, (s, m, d) = np.asarray(x, np.float64), (np.asarray(v, np.float64) for v in f)
        st = 1.0 if t else -1.0
        X, ok = self.triangulate_dlt(rig.P0, rig.P1, x - s + st * m - st * d, x + s + st * m + st * d)
        return X, bool(ok)

    def compute_scene_points(self, result: FlowResult, rig: StereoRig) -> FlowResult:
        """Fills points0/points1/scene_flow/point_valid from the dense s, m, d (geometry.hpp:54)."""
        w, h = result.width, result.height
        s, m, d = (np.ascontiguousarray(v, np.float64) for v in (result.s, result.m, result.d))
        p0, p1, sf = (np.empty((h, w, 3)) for _ in range(3))
        ok = np.empty((h, w), np.uint8)
        rc = rig.to_c()
        self.ctx.check(self.lib.hwf_scene_points(self.ctx.h, w, h, dptr(s), dptr(m), dptr(d), C.byref(rc), dptr(p0),
                                                 dptr(p1), dptr(sf), u8ptr(ok)))
        result.points0, result.points1, result.scene_flow, result.point_valid = p0, p1, sf, ok
        result.has_points = True
        return result

    def export_mesh_obj(self, result: FlowResult, path: str | Path) -> None:
        """geometry.hpp:56-59: OBJ over the pixel grid (3D points when present, else (x, y, disparity))."""
        vis = np.ascontiguousarray(result.vis4, np.uint8)
        disp = None if result.disparity is None else np.ascontiguousarray(result.disparity, np.float64)
        pts = np.ascontiguousarray(result.points0, np.float64) if result.has_points else None
        ok = np.ascontiguousarray(result.point_valid, np.uint8) if result.has_points else None
        self.ctx.check(self.lib.hwf_export_mesh_obj(self.ctx.h, result.width, result.height, dptr(disp), u8ptr(vis),
                                                    dptr(pts), u8ptr(ok), str(path).encode()))

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
