for sh in 0.93 0.94 0.95 0.92; do
  echo "== shrink $sh" >> gpurun_out/shrink.log
  PGK_SEED_SHRINK=$sh python tools/prof_path.py --stage pool --config 2 --n 1000000 --reps 3 --kernels 2>&1 | grep -v -i warn | awk '$1+0 > 0.08 || /n=/' >> gpurun_out/shrink.log
done
python tools/prof_path.py --stage reverse --config 2 --n 1000000 --reps 3 --kernels 2>&1 | grep -v -i warn > gpurun_out/reverse_kernels.log
