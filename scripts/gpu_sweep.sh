#!/bin/bash
# Parity tests + bench sweep over the leaf-list capacity K (no ncu).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT=gpurun_out; TAG=${1:-sweep}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $OUT/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> $OUT/pytest_gpu_$TAG.log
for K in ${CAPS:-2 4 8 16}; do
  timeout 300 python bench.py --steps 10 --warmup 3 --cpu-seconds 0 --list-cap $K > $OUT/bench_${TAG}_K$K.json 2> $OUT/bench_${TAG}_K$K.err
done
