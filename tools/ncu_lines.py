"""Per-source-line and per-opcode breakdown of one kernel in an ncu report (run here, no GPU).

    python tools/ncu_lines.py report.ncu-rep [--top 40] [--op IMAD]

Reads `ncu --page source --print-source cuda,sass --csv` and sums, per CUDA source line, the warp-level
instructions executed, the stall samples, and the FP64 / shared / local instructions; plus a per-opcode table.
"""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
want_op = sys.argv[sys.argv.index("--op") + 1] if "--op" in sys.argv else None
by_op = collections.Counter()  # (line, full opcode) -> instructions, for --op
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
lines = collections.defaultdict(lambda: collections.Counter())
ops = collections.Counter()
opsamp = collections.Counter()
src_text = {}
fname = None
hdr = None
cur = None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or len(row) < 8:
        continue
    if row[0].isdigit():  # a CUDA source line (its metrics are the sum of its SASS rows below)
        cur = (fname, int(row[0]))
        src_text.setdefault(cur, row[1].strip()[:90])
        continue
    if cur is None or not row[2].startswith("0x"):
        continue
    d = dict(zip(hdr[2:], row[2:]))
    sass = row[3].strip()
    try:
        ie = float(d.get("Instructions Executed", "0") or 0)
        smp = float(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        continue
    body = sass.split(None, 1)[1] if sass.startswith("@") else sass
    op = re.split(r"[ .]", body)[0]
    c = lines[cur]
    c["inst"] += ie
    c["samples"] += smp
    if op in ("DFMA", "DADD", "DMUL"):
        c["fp64"] += ie
    if op in ("LDS", "STS"):
        c["shared"] += ie
    if op in ("LDL", "STL"):
        c["local"] += ie
    ops[op] += ie
    opsamp[op] += smp
    if op == want_op:
        by_op[(cur, body.split(None, 1)[0])] += ie
tot = sum(c["inst"] for c in lines.values())
tsm = sum(c["samples"] for c in lines.values())
print(f"total warp instructions {tot:.4g}, stall samples {tsm:.4g}")
print(f"{'file:line':22s} {'inst%':>6s} {'samp%':>6s} {'fp64%':>6s} {'lds/sts':>8s} {'ldl/stl':>8s}  source  (fp64% = DFMA/DADD/DMUL share of the line's instructions)")
for key, c in sorted(lines.items(), key=lambda kv: -kv[1]["samples"])[:top]:
    print(f"{key[0][:14]}:{key[1]:<6d} {100*c['inst']/tot:6.2f} {100*c['samples']/tsm:6.2f} {100*c['fp64']/max(c['inst'],1):6.1f} "
          f"{c['shared']:8.3g} {c['local']:8.3g}  {src_text[key]}")
print("\nopcode            inst%   samp%")
for op, v in ops.most_common(30):
    print(f"{op:16s} {100*v/tot:6.2f} {100*opsamp[op]/tsm:6.2f}")
if want_op:
    print(f"\n{want_op} by source line (full opcode), share of all instructions")
    for (key, full), v in by_op.most_common(top):
        print(f"{key[0][:14]}:{key[1]:<6d} {full:22s} {100*v/tot:6.2f}  {src_text[key]}")
