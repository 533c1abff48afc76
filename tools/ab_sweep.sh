#!/bin/bash
# A/B sweep on the GPU box: the in-tree library vs build/ab/libnavix_<tag>.so
# (same ABI), interleaved per library so clocks/thermal drift hit both alike.
# usage: bash tools/ab_sweep.sh OUTDIR ENVS SIZES [TAGS...]
OUT=$1; ENVS=$2; SIZES=$3; shift 3
mkdir -p $OUT
for rep in 1 2; do
  for tag in new "$@"; do
    if [ "$tag" = new ]; then LIB=""; else LIB=build/ab/libnavix_$tag.so; fi
    NAVIX_LIBRARY=$LIB timeout 600 python tools/sweep.py --envs $ENVS --sizes $SIZES --steps 256 --runs 3 \
      --out $OUT/sweep_${tag}_$rep.json > $OUT/sweep_${tag}_$rep.txt 2>&1
  done
done
