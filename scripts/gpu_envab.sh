#!/bin/bash
# device query bench under environment A/B settings (ENVS="VAR=val ..." each run), default first
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT=gpurun_out; TAG=${1:-env}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
B="python bench.py --steps 20 --warmup 3 --train 0 --lod ${LOD:-0} --pt ${PT:-0} --cpu-seconds 0"
timeout 300 $B > $OUT/bench_${TAG}_def.json 2>> $OUT/sweep_$TAG.err
i=0
for E in $ENVS; do
  i=$((i+1))
  env $(echo $E | tr ',' ' ') timeout 300 $B > $OUT/bench_${TAG}_$i.json 2>> $OUT/sweep_$TAG.err
done
if [ -n "$TESTENV" ]; then
  env $(echo $TESTENV | tr ',' ' ') timeout 900 python -m pytest tests/test_gpu_query.py -x -q --timeout=240 > $OUT/tests_$TAG.log 2>&1
  echo "tests exit $?" >> $OUT/tests_$TAG.log
fi
