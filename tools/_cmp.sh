PGK_GRAM=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for v in default ng3; do
  if [ $v = default ]; then unset PGK_LIB_PATH; else export PGK_LIB_PATH=$PWD/paper_2410_01231_b200/variants/libpgk_$v.so; fi
  echo "== $v"; PGK_GRAM=1 timeout 200 python tools/prof_path.py --stage all --n 1000000 --reps 3 --kernels 2>&1 | grep -v Warn | grep "gram\|all n" | tail -5
done
PGK_LIB_PATH=$PWD/paper_2410_01231_b200/variants/libpgk_stats.so PGK_GRAM=1 timeout 200 python tools/prof_path.py --stage all --n 1000000 --reps 1 2>&1 | grep "gram stats"
