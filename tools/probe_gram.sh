#!/bin/bash
# Gram-kernel role timing (GRAM_STATS=1 variant) and structural variants,
# phase A at config 2, 1M points (run on the GPU box).
out=${1:-gpurun_out}
true \
  python tools/prof_path.py --stage prune --config 2 --n 1000000 --reps 2 > $out/gram_stats.log 2>&1
for lib in paper_2410_01231_b200/libpgk.so paper_2410_01231_b200/variants/libpgk_g*.so; do
  echo "== $lib" >> $out/gram_ab.log
  PGK_LIB_PATH=$lib python tools/prof_path.py --stage prune --config 2 --n 1000000 --reps 3 --kernels 2>&1 \
    | grep -v -i warn | awk '$1+0 > 0.05 || /n=/' >> $out/gram_ab.log
done
