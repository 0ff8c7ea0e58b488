for v in base e6 e8; do
  lib=paper_1610_07159_b200/lib/libhwflow_cuda.so; [ $v != base ] && lib=paper_1610_07159_b200/lib/variants/$v/libhwflow_cuda.so
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --kernel-name-base demangled -k "regex:k_pixel<.bool.0, .bool.1" --log-file gpurun_out/e_$v.csv python tools/prof_run.py --lib $lib --batch 256 --mode global --warmup 0 --runs 1 > /dev/null 2>&1
  echo $v; grep -o '"[0-9.]*"$' gpurun_out/e_$v.csv | tail -2
done
python tools/ab.py run --reps 2 base e6 e8 | tail -3
