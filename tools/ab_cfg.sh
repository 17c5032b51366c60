#!/bin/bash
# A/B per-kernel timing of library variants on a given config:
#   bash tools/ab_cfg.sh CONFIG N STAGE VARIANT [VARIANT ...]
cfg=$1; n=$2; stage=$3; shift 3
for lib in "$@"; do
  echo "== $lib"
  PGK_LIB_PATH=$lib python tools/prof_path.py --stage $stage --config $cfg --n $n --reps 2 --kernels 2>&1 \
    | grep -v -i warn | awk '$1+0 > 5 || /n=/'
done
