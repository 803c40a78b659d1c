#!/bin/bash
# k_query_warp variants: 16 vs 32 slots per warp (NBVH_QUERY_Q), MLP as one 32-row call or two
# 16-row calls (NBVH_QUERY_MB=1), then the query parity tests
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT=gpurun_out; TAG=${1:-q}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
B="python bench.py --steps 20 --warmup 3 --train 0 --lod 0 --pt 0 --cpu-seconds 0"
timeout 300 $B > $OUT/bench_${TAG}_q16.json 2>> $OUT/sweep_$TAG.err
NBVH_QUERY_Q=32 timeout 300 $B > $OUT/bench_${TAG}_q32.json 2>> $OUT/sweep_$TAG.err
NBVH_QUERY_Q=32 NBVH_QUERY_MB=1 timeout 300 $B > $OUT/bench_${TAG}_q32mb1.json 2>> $OUT/sweep_$TAG.err
NBVH_QUERY_Q=32 NBVH_QUERY_WARPS=14 timeout 300 $B > $OUT/bench_${TAG}_q32w14.json 2>> $OUT/sweep_$TAG.err
timeout 900 python -m pytest tests/test_gpu_query.py -x -q -s -k "deep_cut or mlp or variants or end_to_end" > $OUT/tests_$TAG.log 2>&1
echo "tests exit $?" >> $OUT/tests_$TAG.log
