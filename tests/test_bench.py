"""bench.py's JSON line contract (the driver parses it): the reference arm on CPU, our arm on the GPU."""
from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _line(args, timeout):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], cwd=ROOT, capture_output=True, text=True,
                         timeout=timeout, check=True).stdout
    return json.loads(out.strip().splitlines()[-1])


def test_reference_arm_line():
    """--impl reference: the reference's CPU path (oracle/_ref, else the port), same metric and config."""
    d = _line(["--impl", "reference", "--steps", "1", "--warmup", "3"], 600)
    assert d["impl"] == "reference" and d["metric"].startswith("frame-pairs/s") and d["value"] > 0
    assert d["higher_is_better"] is True and d["unit"] == "frame-pairs/s"
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert "global PCG" in d["config"]["workload"]


@pytest.mark.gpu
def test_bench_line_contract():
    d = _line(["--steps", "2", "--warmup", "3", "--batch", "8", "--no-extra", "--no-cpu"], 900)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks", "flow_error"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3 and d["value"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 8 * 4 * 640 * 480 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0 and d["clocks"]["sm_mhz"]
    assert d["flow_error"]["s_median_px"] < 0.2  # the headline schedule recovers the known stereo flow


def test_gpus_flag_spawns_ranks_with_disjoint_shards():
    """`bench.py --gpus 2` without a launcher re-execs itself under torch.distributed.run with 2 ranks
    (frame mode: rank r owns pairs [rB, (r+1)B), no collective); --dry runs the plumbing on gloo."""
    d = _line(["--gpus", "2", "--batch", "8", "--dry"], 300)
    assert d["dry"] is True and d["n_gpus"] == 2
    ranks = sorted(d["ranks"])
    assert [r[0] for r in ranks] == [0, 1]
    assert [(r[1], r[2]) for r in ranks] == [(0, 8), (8, 16)]  # disjoint, contiguous shards
    assert ranks[0][3] != ranks[1][3]  # two processes
    assert d["max_over_ranks"] == 2.0  # the timing max reduces over both ranks


@pytest.mark.gpu
def test_bench_two_gpus():
    """`bench.py --gpus 2` on a 2-GPU node: two NCCL ranks, one line with n_gpus 2 and the whole-job value. Skipped
    on the 1-GPU boxes this project is measured on."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip(f"needs 2 GPUs, found {torch.cuda.device_count()}")
    d = _line(["--gpus", "2", "--steps", "2", "--warmup", "3", "--batch", "8", "--no-extra", "--no-cpu"], 1200)
    assert d["n_gpus"] == 2 and d["value"] > 0 and "x2" in d["config"]["parallelism"]
    assert d["e2e"]["value"] > 0
