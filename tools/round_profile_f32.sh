#!/bin/bash
# Float-path evidence on the GPU box: ncu --set full captures of the tensor-core
# float pool pass 2 and the float Gram selection (phase A) on a config-3
# prefix, plus the tools' own timing lines.  Usage: bash tools/round_profile_f32.sh TAG [N]
tag=${1:-r02e}
n=${2:-300000}
o=gpurun_out
PGK_TILES_STATS=1 python tools/f32_tc_check.py --config 3 --n 1000000 --kernels --modes 0,2 --reps 1 \
    > $o/${tag}_f32_pool_cfg3.log 2>&1
PGK_GRAM_F32_STATS=1 python tools/gram_f32_check.py --config 3 --n 1000000 --reps 2 \
    > $o/${tag}_f32_gram_cfg3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:tc_pool_f32_kernel -s 1 -c 1 \
    -o $o/${tag}_tcf32_pass2 python tools/f32_tc_check.py --config 3 --n $n --reps 1 --modes 2 \
    --out /tmp/p.npz > $o/${tag}_ncu_tcf32.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:prune_gram_f32_kernel -c 1 \
    -o $o/${tag}_gramf32 python tools/gram_f32_check.py --config 3 --n $n --reps 1 \
    --out /tmp/g.npz > $o/${tag}_ncu_gramf32.log 2>&1
