"""Algorithm 1 (oracle/hierarchy.cpp run_scene_flow) re-driven through the stage seams of
one library, one Gauss-Newton iteration at a time (test infrastructure, also used by tools/hier_trace.py).

Lock-step parity: at every level and GN iteration of a full schedule, both libraries are handed the SAME
state (the checker's) and each takes one iteration (`gauss_newton`, solver.cpp:484-532, via hwf_gn_level);
their outputs are then compared. This isolates one iteration of the implementation from the reference's
own amplification of round-off over long schedules.
"""
from __future__ import annotations

import numpy as np

from paper_1610_07159_b200.hwflow import LevelState, Solver, level_dims


class HierRun:
    """One library's hierarchy state (mirrors orc::run_scene_flow's locals)."""

    def __init__(self, solver: Solver, imgs: np.ndarray, S, P, F=None):
        self.s, self.S, self.P, self.F = solver, S, P, F
        self.dims = level_dims(solver.lib, imgs.shape[2], imgs.shape[1], S.levels, S.grid_step)
        self.pyr = solver.build_pyramid(imgs, len(self.dims))
        self.total_prev = self.vis_prev = self.hm_prev = None

    @property
    def L(self) -> int:
        return len(self.dims)

    def start_level(self, l: int) -> None:
        w, h, gw, gh = self.dims[l]
        G = gw * gh
        self.base = np.zeros((G, 6))
        self.vis = np.full((h, w), 0x0F, np.uint8)
        self.illum = None
        if l == self.L - 1:  # C.6 coarsest level
            self.base[:, 0] += self.S.coarse_s_offset[0]
            self.base[:, 1] += self.S.coarse_s_offset[1]
        else:  # C.1/C.3/C.4 prolongation of grid, masks and illumination
            wc, hc = self.dims[l + 1][:2]
            self.base, self.vis, hm = self.s.prolongate(wc, hc, w, h, self.S.grid_step, self.total_prev,
                                                        self.vis_prev, self.hm_prev)
            self.illum = np.stack([hm[0], -hm[0], hm[1], -hm[1]])
        self.delta = np.zeros((G, 6))
        self.W = np.ones((h, w), np.uint8)
        self.nw = np.ones(G)

    def gn(self, l: int) -> tuple[float, float]:
        lv = LevelState(self.pyr[l], self.S.grid_step, self.base, self.delta, self.vis, self.W, self.nw,
                        self.illum, self.F)
        self.delta, self.W, self.nw, eb, ea = self.s.gauss_newton(lv, self.base, self.P, self.S, 1)
        return float(eb[0]), float(ea[0])

    def end_level(self, l: int) -> None:
        w, h = self.dims[l][:2]
        total = self.base + self.delta
        vis_new = self.s.compute_occlusion_maps(w, h, self.S.grid_step, total)
        if l > 0:
            self.hm_prev = self.s.compute_illumination_maps(self.pyr[l], self.S.grid_step, total, vis_new)
        self.total_prev, self.vis_prev = total, vis_new

    def run_to(self, l_stop: int) -> None:
        """Algorithm 1 from the coarsest level down to level l_stop inclusive (its GN iterations, then its
        occlusion and, above the finest level, illumination maps)."""
        for l in range(self.L - 1, l_stop - 1, -1):
            self.start_level(l)
            for _ in range(self.S.gn_for_level(l)):
                self.gn(l)
            self.end_level(l)

    def copy_from(self, o: "HierRun") -> None:
        for k in ("base", "delta", "W", "nw", "vis", "illum", "total_prev", "vis_prev", "hm_prev"):
            v = getattr(o, k, None)
            setattr(self, k, None if v is None else v.copy())


def lockstep(a: Solver, b: Solver, imgs, S, P, F=None, sync: bool = True, on_iter=None, on_level=None):
    """Drive both libraries through the full schedule. With sync, b is re-seeded from a's state before every
    GN iteration and before every level's occlusion/illumination, so each callback sees one step's own
    divergence. on_iter(l, it, A, B, ea, eb); on_level(l, A, B) after both ran end_level."""
    A, B = HierRun(a, imgs, S, P, F), HierRun(b, imgs, S, P, F)
    assert A.dims == B.dims
    for l in range(A.L - 1, -1, -1):
        A.start_level(l)
        B.start_level(l)
        for it in range(S.gn_for_level(l)):
            if sync:
                B.copy_from(A)
            ea, eb = A.gn(l), B.gn(l)
            if on_iter:
                on_iter(l, it, A, B, ea, eb)
        if sync:
            B.copy_from(A)
        A.end_level(l)
        B.end_level(l)
        if on_level:
            on_level(l, A, B)
    return A, B
