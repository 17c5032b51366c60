#!/bin/bash
# pass-1 coverage (P1_MULT variants) x pass-2 guess factor, pool stage at config 2 1M
for lib in paper_2410_01231_b200/libpgk.so paper_2410_01231_b200/variants/libpgk_p1m3.so paper_2410_01231_b200/variants/libpgk_p1m2.so; do
  for sh in 0.93 0.90 0.87; do
    echo "== $lib shrink $sh" >> gpurun_out/p1_sweep.log
    PGK_LIB_PATH=$lib PGK_SEED_SHRINK=$sh python tools/prof_path.py --stage pool --config 2 --n 1000000 --reps 3 2>&1 | grep "pool n" | tail -2 >> gpurun_out/p1_sweep.log
  done
done
