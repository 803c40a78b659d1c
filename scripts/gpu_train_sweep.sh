#!/bin/bash
# training-step timing under a few tuning-hook settings (NBVH_PRIV_BYTES)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT=gpurun_out; TAG=${1:-s}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for pb in default 20480 6000; do
  if [ "$pb" = default ]; then unset NBVH_PRIV_BYTES; else export NBVH_PRIV_BYTES=$pb; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --lod 0 --pt 0 --cpu-seconds 0 > $OUT/bench_${TAG}_$pb.json 2>> $OUT/sweep_$TAG.err
done
