"""Key metrics + stall reasons from an ncu --set full report (run here, no GPU)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
want = ["Duration", "DRAM Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
        "Executed Instructions", "Memory Throughput", "Block Limit Registers", "Block Limit Shared Mem", "Grid Size", "Block Size"]
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") in want:
        print(f"  {d['Metric Name']:38s} {d['Metric Value']:>14s} {d.get('Metric Unit','')}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rr[0], rr[1], (rr[2] if len(rr) > 2 else rr[1])
m = dict(zip(hdr, vals))
u = dict(zip(hdr, units))
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
def f(k):
    try: return float(m.get(k, "nan").replace(",", ""))
    except ValueError: return float("nan")
def nbytes(k):
    return f(k) * SCALE.get(u.get(k, "byte"), 1.0)
rd, wr = nbytes('dram__bytes_read.sum'), nbytes('dram__bytes_write.sum')
print(f"  dram bytes read+write: {(rd + wr) / 1e9:.4g} GB  (read {rd / 1e9:.4g} GB, write {wr / 1e9:.4g} GB)")
stalls = {k: f(k) for k in hdr if k.startswith("smsp__average_warp_latency_issue_stalled") or k.startswith("smsp__pcsamp_warps_issue_stalled")}
tot = sum(v for k, v in stalls.items() if k.startswith("smsp__pcsamp_warps_issue_stalled") and v == v)
top = sorted(((v, k) for k, v in stalls.items() if k.startswith("smsp__pcsamp_warps_issue_stalled") and v == v), reverse=True)[:8]
for v, k in top:
    print(f"  stall {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):35s} {100 * v / tot:5.1f}%")
