#!/bin/bash
# Round-end evidence on the GPU box: the bench line, the ncu launch list of the
# same command (--metrics gpu__time_duration.sum, clock-control none), and
# --set full captures of the top kernels.  Usage: bash tools/round_profile.sh TAG
tag=${1:-r02c}
o=gpurun_out
python bench.py --steps 10 --warmup 3 > $o/${tag}_bench.json 2> $o/${tag}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file $o/${tag}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-parity \
    --extra-cfg3 0 > $o/${tag}_ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:prune_gram_kernel -c 1 \
    -o $o/${tag}_gram python tools/prof_path.py --stage prune --config 2 --n 1000000 --reps 1 \
    > $o/${tag}_ncu_gram.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:tc_pool_u8_kernel -s 2 -c 1 \
    -o $o/${tag}_tcp2 python tools/prof_path.py --stage pool --config 2 --n 1000000 --reps 1 \
    > $o/${tag}_ncu_tcp2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:tc_finalize -c 1 \
    -o $o/${tag}_fin python tools/prof_path.py --stage pool --config 2 --n 1000000 --reps 1 \
    > $o/${tag}_ncu_fin.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:merge_prune_kernel -c 1 \
    -o $o/${tag}_mprune python tools/prof_path.py --stage all --config 2 --n 1000000 --reps 1 \
    > $o/${tag}_ncu_mprune.log 2>&1
