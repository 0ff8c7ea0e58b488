"""Per-rank device time of the 4K strip split (include/hwflow_split.h), measured on ONE GPU.

The world's ranks run in this process with LocalComm, all on one context (one stream). Every
step call of every rank is bracketed with CUDA events, so each rank's busy time is measured on the
device. The halo and all-gather copies are not counted here. The exchanged bytes are counted, and
the script prints a projected N-GPU frame time: max over ranks of busy time, plus the exchanges
at an assumed NVLink rate and per-collective latency. This is an estimate, labelled as such. With
one GPU per gpurun call, multi-GPU runs cannot be measured here.

    python tools/split_estimate.py --worlds 1 2 4 8 [--mode global|schwarz]
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_1610_07159_b200 import build, synthetic  # noqa: E402
from paper_1610_07159_b200.capi import DTYPE_U8  # noqa: E402
from paper_1610_07159_b200.hwflow import EnergyParams, SolveSchedule, Solver  # noqa: E402
from paper_1610_07159_b200.split import LocalComm, SplitGraph, SplitRank, solve_split  # noqa: E402

NVLINK_GBS = 700.0      # assumed effective NVLink 5 P2P / all-gather rate per GPU (B200 spec: 900 GB/s/dir)
LATENCY_US = 15.0       # assumed per-collective latency, host-launched collectives
GRAPH_LATENCY_US = 6.0  # assumed per-collective latency of small NCCL all-gathers inside one CUDA graph


class Timed(SplitRank):
    def __init__(self, *a, **k):
        super().__init__(*a, **k)
        self.ms = 0.0

    def _t(self, fn, *args):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(self.stream)
        fn(*args)
        e1.record(self.stream)
        self._ev.append((e0, e1))

    def upload(self, f):  # transfers are not busy time; the step timing starts with the pyramid
        self._ev = []
        super().upload(f)

    def prologue(self):
        self._t(super().prologue)

    def level_begin(self, l):
        self._t(super().level_begin, l)

    def linearize(self, l, it):
        self._t(super().linearize, l, it)

    def sweep(self, l, s):
        self._t(super().sweep, l, s)

    def pcg(self, l, phase, it=0):
        self._t(super().pcg, l, phase, it)

    def pcg_scalars(self, l, phase, it=0):
        self._t(super().pcg_scalars, l, phase, it)

    def energy_after(self, l):
        self._t(super().energy_after, l)

    def level_end(self, l):
        self._t(super().level_end, l)

    def finish(self):
        torch.cuda.synchronize()
        self.ms = sum(a.elapsed_time(b) for a, b in self._ev)
        return super().finish()


class NullComm(LocalComm):
    """No exchanges: one rank's own device work, for its busy time."""

    def halo(self, *a):
        pass

    def allgather_rows(self, *a):
        pass

    def allgather_rows_halo(self, *a):
        pass

    def allreduce_sum(self, *a):
        pass

    def allreduce_or(self, *a):
        pass


def graph_busy_ms(dev, w, h, S, imgs, world: int, reps: int) -> list[float]:
    """Per-rank device time of the rank's whole frame as one captured CUDA graph (split.py SplitGraph with the
    exchanges left out), median of `reps` replays: no host launch gaps."""
    out = []
    for r in range(world):
        rank = SplitRank(dev, w, h, DTYPE_U8, EnergyParams(), S, None, r, world)
        g = SplitGraph([rank], NullComm(), imgs)
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(rank.stream)
            g.replay()
            e1.record(rank.stream)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        out.append(sorted(ts)[len(ts) // 2])
        del g
        rank.close()
    return out


class CountingComm(LocalComm):
    def __init__(self):
        self.halo_bytes = self.gather_bytes = 0
        self.halos = self.gathers = 0

    def halo(self, ranks, level, name):
        w = ranks[0].row_elems(level, name)
        self.halo_bytes += 2 * w * 8  # one row each way per boundary, per rank (upper bound)
        self.halos += 1
        super().halo(ranks, level, name)

    def allgather_rows(self, ranks, level, name):
        w = ranks[0].row_elems(level, name)
        gh = max(r.rows[level][1] for r in ranks)
        self.gather_bytes += w * gh * 8  # every rank receives the whole buffer
        self.gathers += 1
        super().allgather_rows(ranks, level, name)

    def allgather_rows_halo(self, ranks, level, name, halo_name):
        """One collective (TorchComm folds the halo rows into the gather)."""
        h, hb = self.halos, self.halo_bytes
        super().allgather_rows_halo(ranks, level, name, halo_name)
        self.halos = h
        self.halo_bytes = hb + 2 * ranks[0].row_elems(level, halo_name) * 8 * len(ranks)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--worlds", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--mode", choices=["global", "schwarz"], default="global")
    ap.add_argument("--graph", action="store_true", help="per-rank busy time from a captured CUDA graph (SplitGraph)")
    a = ap.parse_args()
    dev = Solver(build.CUDA_LIB)
    imgs = synthetic.uhd_pair(0)[0]
    S = SolveSchedule(levels=5, grid_step=4, pcg_iters=5, patch_iters=5, subdomain_px=16 if a.mode == "schwarz" else 0)
    h, w = imgs.shape[1:]
    out = []
    for world in a.worlds:
        ranks = [Timed(dev, w, h, DTYPE_U8, EnergyParams(), S, None, r, world) for r in range(world)]
        for _ in range(a.reps):  # last rep counts
            comm = CountingComm()
            solve_split(ranks, comm, imgs)
        busy = [r.ms for r in ranks]
        if a.graph:
            busy = graph_busy_ms(dev, w, h, S, imgs, world, max(a.reps, 5))
        xfer_ms = (comm.halo_bytes + comm.gather_bytes) / (NVLINK_GBS * 1e9) * 1e3
        lat_ms = (comm.halos + comm.gathers) * (GRAPH_LATENCY_US if a.graph else LATENCY_US) / 1e3 if world > 1 else 0.0
        proj = max(busy) + (xfer_ms + lat_ms if world > 1 else 0.0)
        row = {"mode": a.mode, "graph": a.graph, "world": world, "rank_busy_ms": [round(b, 3) for b in busy], "max_busy_ms": round(max(busy), 3),
               "exchanges": comm.halos + comm.gathers, "exchange_MB": round((comm.halo_bytes + comm.gather_bytes) / 1e6, 2),
               "projected_frame_ms": round(proj, 3), "projected_hz": round(1000.0 / proj, 1)}
        out.append(row)
        print(json.dumps(row), flush=True)
        for r in ranks:
            r.close()
    return out


if __name__ == "__main__":
    main()
