#!/usr/bin/env bash
# Rebuild in tree, then on one B200: the GPU test suite and a 128-pair timing (tools/prof_run.py).
#   tools/gpu_check.sh [pytest -k expr]
set -e
cd "$(dirname "$0")/.."
python -m paper_1610_07159_b200.build > /dev/null
K=""; [ -n "$1" ] && K="-k '$1'"
timeout 2400 /usr/local/graft/bin/gpurun --timeout 1800 -- "timeout 900 python -m pytest tests -m gpu -x -q $K > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log; python tools/prof_run.py --batch 128 --warmup 3 --runs 10 2>&1 | tail -1" 2>&1 | tail -5
