#!/bin/bash
# A/B whole-path kernel timings of library variants (config 2, 1M points)
for lib in paper_2410_01231_b200/libpgk.so "$@"; do
  echo "== $lib" >> gpurun_out/all_ab.log
  PGK_LIB_PATH=$lib python tools/prof_path.py --stage all --config 2 --n 1000000 --reps 3 --kernels 2>&1 \
    | grep -v -i warn | awk '$1+0 > 0.1 || /n=/' >> gpurun_out/all_ab.log
done
