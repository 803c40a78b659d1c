#!/bin/bash
# query bench (device + e2e + LoD + path tracing) twice and the query / path-tracing parity tests
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT=gpurun_out; TAG=${1:-qb}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
B="python bench.py --steps 20 --warmup 3 --train 0 --lod ${LOD:-1} --pt ${PT:-1} --cpu-seconds 0"
timeout 300 $B > $OUT/bench_${TAG}.json 2>> $OUT/sweep_$TAG.err
timeout 300 $B > $OUT/bench_${TAG}_2.json 2>> $OUT/sweep_$TAG.err
timeout 900 python -m pytest tests/test_gpu_query.py tests/test_gpu_pathtrace.py -x -q -v --timeout=240 > $OUT/tests_$TAG.log 2>&1
echo "tests exit $?" >> $OUT/tests_$TAG.log
