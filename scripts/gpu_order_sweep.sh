#!/bin/bash
# query timing under the three ray orders
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT=gpurun_out; TAG=${1:-o}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for o in tiles tiles_rows rows; do
  timeout 300 python bench.py --steps 10 --warmup 3 --train 0 --lod 0 --pt 0 --cpu-seconds 0 --order $o > $OUT/bench_${TAG}_$o.json 2>> $OUT/sweep_$TAG.err
done
