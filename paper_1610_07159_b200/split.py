"""Strip-split solve of one frame pair across ranks (SURVEY.md §8e, 4K mode).

The C side is include/hwflow_split.h. This file is the driver that sequences its steps and
moves data between ranks.
  - The product (libhwflow_cuda.so): one rank per GPU, `TorchComm` over NCCL.
  - The CPU tests: the oracle (host buffers) on gloo ranks, or on in-process `LocalComm`
    ranks that copy rows directly.
Collectives and data movement per frame:
  - Schwarz mode, after every sweep but the last: halo exchange of the published x rows next
    to each strip (P2P), 2 node rows per rank.
  - Global-PCG mode (the headline schedule), per PCG iteration: two all-gathers of the dot
    partials (each rank's tiles, a few hundred KB at 4K); every rank then sums the same
    partials in the same order, so the scalars agree bitwise. The z halo the next spmv needs
    rides in the second gather's buffer (each rank appends its first and last z rows), so it
    costs no collective of its own.
  - After every Gauss-Newton iteration: all-gather of the owned total/delta rows. Occlusion,
    illumination, prolongation and the next linearisation read the whole grid.
  - At the end: sum-all-reduce of the energy partials and OR of the divergence flags.
Schwarz sweeps are Jacobi across subdomains (solver.cpp:430-480), and the global PCG's dots
sum per-tile partials in a fixed order, so a split with exact halos reproduces the unsplit solve
bit for bit in both modes.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist

from .capi import DTYPE_F64, DTYPE_U8, Frame4C, ResultC, StatsC, dptr, u8ptr
from .hwflow import EnergyParams, FlowResult, GnStats, SolveSchedule, Solver, grid_dims

__all__ = ["SplitRank", "LocalComm", "TorchComm", "solve_split"]


class _DevArray:  # zero-copy view of library-owned device memory for torch
    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 2}


class SplitRank:
    """One rank's hwf_split: device buffers (CUDA library) or host buffers (oracle)."""

    def __init__(self, solver: Solver, width: int, height: int, dtype: int, params: EnergyParams,
                 schedule: SolveSchedule, fundamental: np.ndarray | None, rank: int, world: int):
        self.solver, self.lib, self.rank, self.world = solver, solver.lib, rank, world
        self.on_device = solver.backend.startswith("cuda")
        self.width, self.height, self.dtype = width, height, dtype
        self._pc, self._sc = params.to_c(), schedule.to_c()
        self._F = None if fundamental is None else np.ascontiguousarray(fundamental, np.float64).reshape(9)
        h = C.c_void_p()
        self._check(self.lib.hwf_split_create(solver.ctx.h, width, height, dtype, C.byref(self._pc),
                                              C.byref(self._sc), dptr(self._F), rank, world, C.byref(h)))
        self.h = h
        L, gn = C.c_int(), (C.c_int * 8)()
        self._check(self.lib.hwf_split_schedule(self.h, C.byref(L), gn))
        self.levels, self.gn = L.value, [gn[l] for l in range(L.value)]
        self.patch_iters = schedule.patch_iters
        self.pcg_iters = schedule.pcg_iters
        self.global_mode = schedule.subdomain_px <= 0
        self._row_elems = {}
        self.rows = []  # per level: (n0, n1, gw)
        for l in range(self.levels):
            n0, n1, gw = C.c_int(), C.c_int(), C.c_int()
            self._check(self.lib.hwf_split_rows(self.h, l, C.byref(n0), C.byref(n1), C.byref(gw)))
            self.rows.append((n0.value, n1.value, gw.value))
        self.stream = (torch.cuda.ExternalStream(self.lib.hwf_stream(solver.ctx.h)) if self.on_device else None)

    def _check(self, rc: int):
        self.solver.ctx.check(rc)

    def buffer(self, level: int, name: str) -> torch.Tensor:
        p, n = C.c_void_p(), C.c_longlong()
        self._check(self.lib.hwf_split_buffer(self.h, level, name.encode(), C.byref(p), C.byref(n)))
        flags = name == "flags"
        if self.on_device:
            return torch.as_tensor(_DevArray(p.value, n.value, "<i4" if flags else "<f8"), device="cuda")
        ct = C.c_int32 if flags else C.c_double
        return torch.from_numpy(np.ctypeslib.as_array(C.cast(p, C.POINTER(ct)), shape=(n.value,)))

    def row_elems(self, level: int, name: str = "total") -> int:
        key = (level, name)
        if key not in self._row_elems:
            e = C.c_longlong()
            self._check(self.lib.hwf_split_row_elems(self.h, level, name.encode(), C.byref(e)))
            self._row_elems[key] = e.value
        return self._row_elems[key]

    def row_slice(self, level: int, r0: int, r1: int, name: str = "total") -> slice:
        w = self.row_elems(level, name)
        return slice(w * r0, w * r1)

    # steps (include/hwflow_split.h)
    def begin(self, frame: Frame4C):
        self._check(self.lib.hwf_split_begin(self.h, C.byref(frame)))

    def upload(self, frame: Frame4C):
        self._check(self.lib.hwf_split_upload(self.h, C.byref(frame)))

    def prologue(self):
        self._check(self.lib.hwf_split_prologue(self.h))

    def level_begin(self, l: int):
        self._check(self.lib.hwf_split_level_begin(self.h, l))

    def linearize(self, l: int, it: int):
        self._check(self.lib.hwf_split_linearize(self.h, l, it))

    def sweep(self, l: int, s: int):
        self._check(self.lib.hwf_split_sweep(self.h, l, s))

    def pcg(self, l: int, phase: int, it: int = 0):
        self._check(self.lib.hwf_split_pcg(self.h, l, phase, it))

    def pcg_scalars(self, l: int, phase: int, it: int = 0):
        self._check(self.lib.hwf_split_pcg_scalars(self.h, l, phase, it))

    def energy_after(self, l: int):
        self._check(self.lib.hwf_split_energy_after(self.h, l))

    def level_end(self, l: int):
        self._check(self.lib.hwf_split_level_end(self.h, l))

    def finish(self) -> tuple[FlowResult, GnStats]:
        w, h = self.width, self.height
        gw, gh = grid_dims(w, h, self._sc.grid_step)
        o = FlowResult(w, h)
        o.s, o.m, o.d = np.empty((h, w, 2)), np.empty((h, w, 2)), np.empty((h, w, 2))
        o.disparity, o.vis4, o.grid_total = np.empty((h, w)), np.empty((h, w), np.uint8), np.empty((gw * gh, 6))
        r = ResultC(dptr(o.s), dptr(o.m), dptr(o.d), dptr(o.disparity), u8ptr(o.vis4), dptr(o.grid_total))
        st = StatsC()
        self._check(self.lib.hwf_split_finish(self.h, C.byref(r), C.byref(st)))
        return o, GnStats.from_c(st)

    def close(self):
        if self.h:
            self.lib.hwf_split_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _owner(rows: list[tuple[int, int]], q: int) -> int:
    for r, (n0, n1) in enumerate(rows):
        if n0 <= q < n1:
            return r
    raise ValueError(f"node row {q} has no owner")


class LocalComm:
    """All ranks in this process (oracle on CPU, or several splits sharing one device context):
    rows move by direct copies, in step order."""

    def _streamed(self, ranks):
        s = ranks[0].stream
        return torch.cuda.stream(s) if s is not None else _Null()

    def halo(self, ranks: list[SplitRank], level: int, name: str):
        rows = [r.rows[level][:2] for r in ranks]
        gh = max(n1 for _, n1 in rows)
        with self._streamed(ranks):
            for r, (n0, n1) in zip(ranks, rows):
                if n1 <= n0:
                    continue
                for q in (n0 - 1, n1):
                    if 0 <= q < gh:
                        src = ranks[_owner(rows, q)]
                        sl = r.row_slice(level, q, q + 1, name)
                        r.buffer(level, name)[sl].copy_(src.buffer(level, name)[sl])

    def allgather_rows(self, ranks: list[SplitRank], level: int, name: str):
        with self._streamed(ranks):
            for src in ranks:
                n0, n1, _ = src.rows[level]
                if n1 <= n0:
                    continue
                sl = src.row_slice(level, n0, n1, name)
                for dst in ranks:
                    if dst is not src:
                        dst.buffer(level, name)[sl].copy_(src.buffer(level, name)[sl])

    def allgather_rows_halo(self, ranks: list[SplitRank], level: int, name: str, halo_name: str):
        """allgather_rows(name) and halo(halo_name) as one exchange (TorchComm fuses them)."""
        self.allgather_rows(ranks, level, name)
        self.halo(ranks, level, halo_name)

    def allreduce_sum(self, ranks: list[SplitRank], name: str):
        with self._streamed(ranks):
            bufs = [r.buffer(0, name) for r in ranks]
            tot = bufs[0].clone()
            for b in bufs[1:]:
                tot += b
            for b in bufs:
                b.copy_(tot)

    def allreduce_or(self, ranks: list[SplitRank], name: str):
        with self._streamed(ranks):
            bufs = [r.buffer(0, name) for r in ranks]
            acc = bufs[0].clone()
            for b in bufs[1:]:
                acc |= b
            for b in bufs:
                b.copy_(acc)


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


class TorchComm:
    """One rank per process over torch.distributed (NCCL for device buffers, gloo for host buffers)."""

    def __init__(self, rank: SplitRank, group=None):
        self.group = group
        self.world = dist.get_world_size(group)
        me = torch.tensor([v for (n0, n1, _) in rank.rows for v in (n0, n1)], dtype=torch.int64)
        dev = "cuda" if rank.on_device else "cpu"
        gathered = torch.empty(self.world * me.numel(), dtype=torch.int64, device=dev)
        dist.all_gather_into_tensor(gathered, me.to(dev), group=group)
        self.table = gathered.view(self.world, -1, 2).cpu().tolist()  # [rank][level][n0, n1]

    def _streamed(self, ranks):
        s = ranks[0].stream
        return torch.cuda.stream(s) if s is not None else _Null()

    def halo(self, ranks: list[SplitRank], level: int, name: str):
        (me,) = ranks
        rows = [self.table[r][level] for r in range(self.world)]
        gh = max(n1 for _, n1 in rows)
        buf = me.buffer(level, name)
        ops = []
        for r, (n0, n1) in enumerate(rows):
            if n1 <= n0 or r == me.rank:
                continue
            for tag, q in ((0, n0 - 1), (1, n1)):
                if 0 <= q < gh and _owner(rows, q) == me.rank:  # r needs my row q
                    ops.append(dist.P2POp(dist.isend, buf[me.row_slice(level, q, q + 1, name)], r, self.group, tag))
        n0, n1 = rows[me.rank]
        if n1 > n0:
            for tag, q in ((0, n0 - 1), (1, n1)):
                if 0 <= q < gh:
                    ops.append(dist.P2POp(dist.irecv, buf[me.row_slice(level, q, q + 1, name)], _owner(rows, q),
                                          self.group, tag))
        if not ops:
            return
        with self._streamed(ranks):
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    def allgather_rows(self, ranks: list[SplitRank], level: int, name: str):
        (me,) = ranks
        rows = [self.table[r][level] for r in range(self.world)]
        w = me.row_elems(level, name)
        span = w * max(n1 - n0 for n0, n1 in rows)
        if span == 0:
            return
        buf = me.buffer(level, name)
        with self._streamed(ranks):
            n0, n1 = rows[me.rank]
            slab = torch.zeros(span, dtype=buf.dtype, device=buf.device)
            slab[: w * (n1 - n0)].copy_(buf[me.row_slice(level, n0, n1, name)])
            out = torch.empty(self.world * span, dtype=buf.dtype, device=buf.device)
            dist.all_gather_into_tensor(out, slab, group=self.group)
            for r, (a, b) in enumerate(rows):
                if r != me.rank and b > a:
                    buf[me.row_slice(level, a, b, name)].copy_(out[r * span: r * span + w * (b - a)])

    def allgather_rows_halo(self, ranks: list[SplitRank], level: int, name: str, halo_name: str):
        """One all-gather carries both: every rank's `name` rows, then its first and last `halo_name` rows.
        Strips are contiguous, so the halo row above a strip is its owner's last row and the one below is
        its owner's first; the P2P exchange of halo() is folded into the collective the protocol already
        makes (the PCG's partial-sum gather)."""
        (me,) = ranks
        rows = [self.table[r][level] for r in range(self.world)]
        w, wh = me.row_elems(level, name), me.row_elems(level, halo_name)
        span = w * max(n1 - n0 for n0, n1 in rows)
        if span == 0:
            return
        buf, hb = me.buffer(level, name), me.buffer(level, halo_name)
        gh = max(n1 for _, n1 in rows)
        n0, n1 = rows[me.rank]
        with self._streamed(ranks):
            slab = torch.zeros(span + 2 * wh, dtype=buf.dtype, device=buf.device)
            if n1 > n0:
                slab[: w * (n1 - n0)].copy_(buf[me.row_slice(level, n0, n1, name)])
                slab[span: span + wh].copy_(hb[me.row_slice(level, n0, n0 + 1, halo_name)])
                slab[span + wh:].copy_(hb[me.row_slice(level, n1 - 1, n1, halo_name)])
            stride = span + 2 * wh
            out = torch.empty(self.world * stride, dtype=buf.dtype, device=buf.device)
            dist.all_gather_into_tensor(out, slab, group=self.group)
            for r, (a, b) in enumerate(rows):
                if r != me.rank and b > a:
                    buf[me.row_slice(level, a, b, name)].copy_(out[r * stride: r * stride + w * (b - a)])
            if n1 > n0:
                for q in (n0 - 1, n1):
                    if 0 <= q < gh:
                        o = _owner(rows, q)
                        at = o * stride + span + (0 if q == rows[o][0] else wh)
                        hb[me.row_slice(level, q, q + 1, halo_name)].copy_(out[at: at + wh])

    def allreduce_sum(self, ranks: list[SplitRank], name: str):
        (me,) = ranks
        with self._streamed(ranks):
            dist.all_reduce(me.buffer(0, name), op=dist.ReduceOp.SUM, group=self.group)

    def allreduce_or(self, ranks: list[SplitRank], name: str):
        (me,) = ranks
        buf = me.buffer(0, name)
        with self._streamed(ranks):
            out = torch.empty(self.world * buf.numel(), dtype=buf.dtype, device=buf.device)
            dist.all_gather_into_tensor(out, buf.clone(), group=self.group)
            acc = out.view(self.world, -1)[0].clone()
            for r in range(1, self.world):
                acc |= out.view(self.world, -1)[r]
            buf.copy_(acc)


def _frame(images: np.ndarray) -> tuple[Frame4C, np.ndarray]:
    a = np.ascontiguousarray(images)
    if a.dtype != np.uint8:
        a = np.ascontiguousarray(a, dtype=np.float64)
    f = Frame4C()
    f.width, f.height = a.shape[2], a.shape[1]
    f.dtype = DTYPE_U8 if a.dtype == np.uint8 else DTYPE_F64
    for e in range(4):
        f.plane[e] = a[e].ctypes.data
    return f, a


def _pcg_split(ranks: list[SplitRank], comm, l: int):
    """pcg_solve (solver.cpp:365-380) across the strips, include/hwflow_split.h's protocol."""
    def phase(ph: int, it: int = 0, z_halo: bool = False):
        for r in ranks:
            r.pcg(l, ph, it)
        if z_halo:  # phases 0 and 2 leave z for the next spmv: its halo rides on the partials' gather
            comm.allgather_rows_halo(ranks, l, "pcg_part", "z")
        else:
            comm.allgather_rows(ranks, l, "pcg_part")
        for r in ranks:
            r.pcg_scalars(l, ph, it)

    phase(0, z_halo=True)
    for it in range(ranks[0].pcg_iters):
        phase(1, it)
        phase(2, it, z_halo=it < ranks[0].pcg_iters - 1)


def _split_body(ranks: list[SplitRank], comm):
    """Everything between the frame upload and hwf_split_finish: device enqueues and collectives only (no host
    synchronisation), so that SplitGraph can capture it into one CUDA graph."""
    r0 = ranks[0]
    for r in ranks:
        r.prologue()
    for l in reversed(range(r0.levels)):
        for r in ranks:
            r.level_begin(l)
        for it in range(r0.gn[l]):
            for r in ranks:
                r.linearize(l, it)
            if r0.global_mode:
                _pcg_split(ranks, comm, l)
            else:
                for s in range(r0.patch_iters):
                    for r in ranks:
                        r.sweep(l, s)
                    if s < r0.patch_iters - 1:
                        comm.halo(ranks, l, r0.lib.hwf_split_swept(s).decode())
            comm.allgather_rows(ranks, l, "total")
            comm.allgather_rows(ranks, l, "delta")
        for r in ranks:
            r.energy_after(l)
        for r in ranks:
            r.level_end(l)
    comm.allreduce_sum(ranks, "energy")
    comm.allreduce_or(ranks, "flags")


def solve_split(ranks: list[SplitRank], comm, images: np.ndarray) -> list[tuple[FlowResult, GnStats]]:
    """run_scene_flow of one frame pair (4, h, w), split across `ranks`
    (all of them for LocalComm, this process's one for TorchComm). Returns each local rank's
    (FlowResult, GnStats); every rank ends with the full result."""
    frame, keep = _frame(images)
    for r in ranks:
        r.upload(frame)
    _split_body(ranks, comm)
    out = [r.finish() for r in ranks]
    del keep
    return out


class SplitGraph:
    """The split solve as ONE CUDA graph per process: the steps of every local rank, the halo exchanges and the
    PCG dot-partial all-gathers (NCCL collectives under TorchComm, device copies under LocalComm) are captured
    once; a frame is then upload -> graph replay -> finish, with no host code between PCG phases.
    Device libraries only (the CPU oracle has no graphs)."""

    def __init__(self, ranks: list[SplitRank], comm, images: np.ndarray):
        if not all(r.on_device for r in ranks):
            raise ValueError("SplitGraph needs the CUDA library")
        self.ranks, self.comm = ranks, comm
        stream = ranks[0].stream
        frame, keep = _frame(images)
        for r in ranks:  # warm-up: plans, workspaces and NCCL communicators exist before capture
            r.upload(frame)
        _split_body(ranks, comm)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=stream):
            _split_body(ranks, comm)
        torch.cuda.synchronize()
        del keep

    def replay(self):
        """The captured solve on the frame last uploaded (device time only; no transfers), launched on the
        library's stream so that it is ordered after the upload and before the download."""
        with torch.cuda.stream(self.ranks[0].stream):
            self.graph.replay()

    def __call__(self, images: np.ndarray) -> list[tuple[FlowResult, GnStats]]:
        frame, keep = _frame(images)
        for r in self.ranks:
            r.upload(frame)
        self.replay()
        out = [r.finish() for r in self.ranks]
        del keep
        return out
