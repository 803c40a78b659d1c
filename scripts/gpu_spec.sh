#!/bin/bash
# speculative tail rows in k_query_warp: device bench, e2e and the query parity tests, on / off
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT=gpurun_out; TAG=${1:-sp}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
B="python bench.py --steps 20 --warmup 3 --train 0 --lod 1 --pt 1 --cpu-seconds 0"
timeout 300 $B > $OUT/bench_${TAG}_on.json 2>> $OUT/sweep_$TAG.err
NBVH_QUERY_SPEC=0 timeout 300 $B > $OUT/bench_${TAG}_off.json 2>> $OUT/sweep_$TAG.err
timeout 900 python -m pytest tests/test_gpu_query.py tests/test_gpu_pathtrace.py -x -q > $OUT/tests_$TAG.log 2>&1
echo "tests exit $?" >> $OUT/tests_$TAG.log
