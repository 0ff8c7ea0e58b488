"""Per-kernel roofline table from one ncu metrics pass over a replay (north_star: "each kernel's choices are
evidenced by ncu: achieved HBM GB/s and L2/shared throughput against B200 peak").

    # on the GPU box (cold, serialised launches; never a bench number):
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,\
l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,\
smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/kr.csv \
        python tools/prof_run.py --batch 256 --mode global --warmup 0 --runs 1
    # here:
    python tools/kernel_roofline.py gpurun_out/kr.csv > profiles/r2_kernel_roofline.md   (+ .json beside it)

Per kernel (template arguments kept): launches, total time and share, and for its largest launch (the finest
level): duration, DRAM bytes, DRAM GB/s and its fraction of MEASURED_PEAKS.json's copy bandwidth, L2 GB/s,
shared-memory wavefronts, FP64-pipe and issue-slot utilisation. The profiled replay runs twice under ncu
(capture + replay), so counts are per 2 replays.
"""
import collections
import csv
import json
import re
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def main():
    src = sys.argv[1]
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    rows = list(csv.reader(open(src)))
    hdr, launches = None, collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = d["ID"]
        name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("hwf::(anonymous namespace)::", "")
        name = name.replace("void ", "").replace("unnamed>::", "")
        L = launches.setdefault(key, {"name": name})
        try:
            v = float(d["Metric Value"].replace(",", ""))
        except ValueError:
            continue
        unit = d.get("Metric Unit", "")
        m = d["Metric Name"]
        if m == "gpu__time_duration.sum":
            v *= {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}.get(unit, 1e-9)
        elif m.startswith(("dram__bytes", "lts__t_bytes")):
            v *= {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1.0)
        L[m] = v
    by = collections.defaultdict(list)
    for L in launches.values():
        if "gpu__time_duration.sum" in L:
            by[L["name"]].append(L)
    total = sum(L["gpu__time_duration.sum"] for ls in by.values() for L in ls)
    out = []
    for name, ls in sorted(by.items(), key=lambda kv: -sum(L["gpu__time_duration.sum"] for L in kv[1])):
        t = sum(L["gpu__time_duration.sum"] for L in ls)
        big = max(ls, key=lambda L: L["gpu__time_duration.sum"])
        dur = big["gpu__time_duration.sum"]
        dram = big.get("dram__bytes_read.sum", 0.0) + big.get("dram__bytes_write.sum", 0.0)
        out.append({
            "kernel": name, "launches": len(ls), "ms": 1e3 * t, "share": t / total,
            "largest_launch_us": 1e6 * dur, "dram_bytes": dram, "dram_gbs": dram / dur / 1e9,
            "dram_frac": dram / dur / 1e9 / peak, "l2_gbs": big.get("lts__t_bytes.sum", 0.0) / dur / 1e9,
            "smem_wavefronts": big.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
            "fp64_pipe_pct": big.get("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
            "issue_pct": big.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        })
    json_path = Path(sys.argv[2]) if len(sys.argv) > 2 else None
    if json_path:
        json_path.write_text(json.dumps({"source": src, "hbm_peak_gbs": peak, "total_ms": 1e3 * total,
                                         "kernels": out}, indent=1))
    print(f"Per-kernel rooflines (ncu, cold serialised launches; total {1e3 * total:.1f} ms; HBM peak {peak} GB/s "
          f"measured copy bandwidth, MEASURED_PEAKS.json). Columns for each kernel's largest (finest-level) launch.\n")
    print("| kernel | launches | ms | share | largest launch µs | DRAM GB/s | of HBM peak | L2 GB/s | FP64 pipe % | issue % |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for k in out:
        f = lambda v, fmt: (fmt % v) if v is not None else "–"
        print(f"| `{k['kernel']}` | {k['launches']} | {k['ms']:.2f} | {100 * k['share']:.1f}% | {k['largest_launch_us']:.0f} | "
              f"{k['dram_gbs']:.0f} | {100 * k['dram_frac']:.0f}% | {k['l2_gbs']:.0f} | {f(k['fp64_pipe_pct'], '%.0f')} | "
              f"{f(k['issue_pct'], '%.0f')} |")


if __name__ == "__main__":
    main()
