"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections, csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: [0, 0.0])
seq = []
for d in data:
    n = re.sub(r'\(.*', '', d['Kernel Name']).replace('hwf::(anonymous namespace)::', '').replace('void ', '').replace('unnamed>::', '')
    v = float(d['Metric Value']) / 1000.0  # ns -> us
    agg[n][0] += 1
    agg[n][1] += v
    seq.append(f"{n}:{v:.0f}")
tot = sum(v for _, v in agg.values())
print(f"{'kernel':30s} {'n':>4s} {'us':>9s} {'share':>6s}")
for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:30s} {n:4d} {v:9.1f} {100 * v / tot:5.1f}%")
print(f"total {tot:.1f} us over {len(data)} launches")
if len(sys.argv) > 2:
    print(" ".join(seq))
