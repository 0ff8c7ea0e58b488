"""A/B variants of the library: build here, time on the B200.

    python tools/ab.py build NAME=DEF1,DEF2 NAME2=DEF ...     # lib/variants/NAME/libhwflow_cuda.so
    python tools/ab.py run [--batch 256] [--reps 3] base NAME NAME2 ...   # on the GPU box

`run` times every variant (and `base` = the in-tree library) with tools/prof_run.py (global-PCG headline,
device-resident replays, in-graph k_pixel<LIN> events), interleaving the variants `--reps` times, and prints the
median ms per replay of each.
"""
import statistics
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    if sys.argv[1] == "build":
        from paper_1610_07159_b200 import build
        for spec in sys.argv[2:]:
            name, _, defs = spec.partition("=")
            print(build.build_cuda(defines=tuple(d for d in defs.split(",") if d), variant=name))
        return
    args = sys.argv[2:]
    batch, reps = "256", 3
    if "--batch" in args:
        i = args.index("--batch")
        batch = args[i + 1]
        del args[i:i + 2]
    if "--reps" in args:
        i = args.index("--reps")
        reps = int(args[i + 1])
        del args[i:i + 2]
    res = {n: [] for n in args}
    pix = {n: [] for n in args}
    for _ in range(reps):
        for n in args:
            lib = ROOT / "paper_1610_07159_b200" / "lib" / ("libhwflow_cuda.so" if n == "base" else f"variants/{n}/libhwflow_cuda.so")
            out = subprocess.run([sys.executable, str(ROOT / "tools" / "prof_run.py"), "--lib", str(lib), "--batch", batch,
                                  "--mode", "global", "--warmup", "3", "--runs", "10", "--profiling"],
                                 capture_output=True, text=True).stdout.strip().splitlines()
            kv = dict(x.split("=") for x in out[-1].split()) if out else {}
            res[n].append(float(kv.get("ms_per_replay", "nan")))
            pix[n].append(float(kv.get("pixel_lin_L0_ms_per_launch", "nan")))
    for n in args:
        print(f"{n:24s} ms/replay median {statistics.median(res[n]):8.3f} {res[n]}  k_pixel<LIN> L0 ms/launch "
              f"{statistics.median(pix[n]):.3f}", flush=True)


if __name__ == "__main__":
    main()
