"""Static SASS opcode mix of one kernel in an object/.so (no GPU): python tools/sass_mix.py file.o k_pixelILb1ELb1E"""
import collections, re, subprocess, sys
out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
pat = sys.argv[2]
cur, mix = None, collections.Counter()
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    if cur and pat in cur:
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9]+)", line)
        if m:
            mix[m.group(2)] += 1
tot = sum(mix.values())
fp64 = sum(v for k, v in mix.items() if k in ("DFMA", "DADD", "DMUL"))
print(f"{pat}: {tot} instructions, FP64 {fp64}, " + ", ".join(f"{k} {v}" for k, v in mix.most_common(14)))
