#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT=gpurun_out; TAG=${1:-ck}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
B="python bench.py --steps 20 --warmup 3 --train 0 --lod 0 --pt 0 --cpu-seconds 0"
for c in ${CHUNKS:-16 256 1024 4096}; do
  NBVH_QUERY_CHUNK=$c timeout 200 $B > $OUT/bench_${TAG}_$c.json 2>> $OUT/sweep_$TAG.err
done
