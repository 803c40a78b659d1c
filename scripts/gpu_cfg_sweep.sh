#!/bin/bash
# query timing under traversal variants and list capacities
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT=gpurun_out; TAG=${1:-c}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
B="python bench.py --steps 20 --warmup 3 --train 0 --lod 0 --pt 0 --cpu-seconds 0"
NBVH_TRAVERSE=packet timeout 300 $B > $OUT/bench_${TAG}_packet.json 2>> $OUT/sweep_$TAG.err
for k in 8 10 12 16; do
  timeout 300 $B --list-cap $k > $OUT/bench_${TAG}_k$k.json 2>> $OUT/sweep_$TAG.err
done
