#!/bin/bash
# A/B per-kernel timing of library variants on the GPU box:
#   bash tools/ab.sh STAGE N VARIANT [VARIANT ...]   (VARIANT = path to a libpgk*.so)
stage=$1; n=$2; shift 2
for lib in "$@"; do
  echo "== $lib"
  PGK_LIB_PATH=$lib python tools/prof_path.py --stage $stage --config 2 --n $n --reps 3 --kernels 2>&1 \
    | grep -v -i warn | awk '$1+0 > 0.1 || /n=/'
done
