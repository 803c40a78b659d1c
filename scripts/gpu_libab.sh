#!/bin/bash
# device query bench with alternative in-tree libraries (NBVH_LIB) vs the default build
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT=gpurun_out; TAG=${1:-ab}; mkdir -p $OUT
B="python bench.py --steps 20 --warmup 3 --train 0 --lod 0 --pt 0 --cpu-seconds 0"
timeout 200 $B > $OUT/bench_${TAG}_def.json 2>> $OUT/sweep_$TAG.err
for L in $LIBS; do
  NBVH_LIB=$PWD/paper_2405_16237_b200/$L timeout 200 $B > $OUT/bench_${TAG}_$L.json 2>> $OUT/sweep_$TAG.err
done
timeout 200 $B > $OUT/bench_${TAG}_def2.json 2>> $OUT/sweep_$TAG.err
