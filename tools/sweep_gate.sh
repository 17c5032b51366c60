for sh in 0.93 0.90 0.87; do
  echo "== shrink $sh" >> gpurun_out/gate.log
  PGK_SEED_SHRINK=$sh python tools/prof_path.py --stage pool --config 2 --n 1000000 --reps 3 2>&1 | grep "pool n" | tail -2 >> gpurun_out/gate.log
done
PGK_SEED_SHRINK=0.85 python -m pytest tests/test_gpu_tc.py -x -q > gpurun_out/g27_tc85.log 2>&1
python -m pytest tests/test_gpu_tc.py tests/test_gpu_fullscale.py -x -q -k "not float and not graph and not 4m" > gpurun_out/g27_tc.log 2>&1
