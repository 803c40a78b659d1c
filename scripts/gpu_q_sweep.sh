#!/bin/bash
# k_query_warp variants: warps per CTA (NBVH_QUERY_WARPS: less shared memory, larger L1),
# shared-memory carve-out, then the query parity tests on the default
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT=gpurun_out; TAG=${1:-q}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
B="python bench.py --steps 20 --warmup 3 --train 0 --lod 0 --pt 0 --cpu-seconds 0"
timeout 300 $B > $OUT/bench_${TAG}_w16.json 2>> $OUT/sweep_$TAG.err
for w in 14 13 12; do
  NBVH_QUERY_WARPS=$w timeout 300 $B > $OUT/bench_${TAG}_w$w.json 2>> $OUT/sweep_$TAG.err
done
NBVH_QUERY_WARPS=13 NBVH_QUERY_CARVEOUT=56 timeout 300 $B > $OUT/bench_${TAG}_w13c56.json 2>> $OUT/sweep_$TAG.err
NBVH_QUERY_CARVEOUT=100 timeout 300 $B > $OUT/bench_${TAG}_w16c100.json 2>> $OUT/sweep_$TAG.err
timeout 900 python -m pytest tests/test_gpu_query.py -x -q -s -k "deep_cut or mlp or variants or end_to_end" > $OUT/tests_$TAG.log 2>&1
echo "tests exit $?" >> $OUT/tests_$TAG.log
