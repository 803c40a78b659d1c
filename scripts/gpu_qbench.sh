#!/bin/bash
# query bench (device + e2e) and the query parity tests
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT=gpurun_out; TAG=${1:-qb}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
B="python bench.py --steps 20 --warmup 3 --train 0 --lod 0 --pt 0 --cpu-seconds 0"
timeout 200 $B > $OUT/bench_${TAG}.json 2>> $OUT/sweep_$TAG.err
timeout 200 $B > $OUT/bench_${TAG}_2.json 2>> $OUT/sweep_$TAG.err
timeout 900 python -m pytest tests/test_gpu_query.py -x -q > $OUT/tests_$TAG.log 2>&1
echo "tests exit $?" >> $OUT/tests_$TAG.log
