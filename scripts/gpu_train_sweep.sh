#!/bin/bash
# training-step timing under tuning-hook settings: warp-aggregated scatter levels
# (NBVH_SCATTER_AGG) x shared-memory privatisation budget (NBVH_PRIV_BYTES)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT=gpurun_out; TAG=${1:-s}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
DEF="0:default 8:default 10:default 12:default 10:0 10:20480 16:0"
for cfg in ${SWEEP:-$DEF}; do
  agg=${cfg%%:*}; pb=${cfg##*:}
  export NBVH_SCATTER_AGG=$agg
  if [ "$pb" = default ]; then unset NBVH_PRIV_BYTES; else export NBVH_PRIV_BYTES=$pb; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --lod 0 --pt 0 --cpu-seconds 0 > $OUT/bench_${TAG}_a${agg}_p$pb.json 2>> $OUT/sweep_$TAG.err
done
unset NBVH_SCATTER_AGG NBVH_PRIV_BYTES
if [ -n "$TESTS" ]; then
  timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_train_elementwise.py -x -q > $OUT/tests_$TAG.log 2>&1
  echo "tests exit $?" >> $OUT/tests_$TAG.log
fi
