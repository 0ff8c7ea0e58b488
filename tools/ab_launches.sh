#!/usr/bin/env bash
# Launch lists (ncu gpu__time_duration, cold, serialised) of A/B variants: tools/ab_launches.sh base tma ...
for v in "$@"; do
  lib=paper_1610_07159_b200/lib/libhwflow_cuda.so; [ "$v" != base ] && lib=paper_1610_07159_b200/lib/variants/$v/libhwflow_cuda.so
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$v.csv \
    python tools/prof_run.py --lib $lib --batch 256 --mode global --warmup 0 --runs 1 > /dev/null 2>&1
  echo "== $v"; python tools/launches.py gpurun_out/launches_$v.csv | head -14
done
