#!/bin/bash
# training-step timing under environment A/B settings (ENVS="VAR=val,VAR=val ..."), default first,
# then the training parity tests (TESTS=1)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT=gpurun_out; TAG=${1:-te}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
B="python bench.py --steps 10 --warmup 3 --lod 0 --pt 0 --cpu-seconds 0"
timeout 300 $B > $OUT/bench_${TAG}_def.json 2>> $OUT/sweep_$TAG.err
i=0
for E in $ENVS; do
  i=$((i+1))
  env $(echo $E | tr ',' ' ') timeout 300 $B > $OUT/bench_${TAG}_$i.json 2>> $OUT/sweep_$TAG.err
done
if [ -n "$TESTS" ]; then
  timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_train_elementwise.py -x -q --timeout=300 > $OUT/tests_$TAG.log 2>&1
  echo "tests exit $?" >> $OUT/tests_$TAG.log
fi
