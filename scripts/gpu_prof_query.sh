#!/bin/bash
# ncu --set full of the query kernel(s) in a short bench run (no training / LoD / path tracing)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT=gpurun_out; TAG=${1:-q}; KRE=${2:-k_query}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
CMD="python bench.py --steps 2 --warmup 1 --cpu-seconds 0 --train 0 --lod 0 --pt 0"
timeout 600 $CMD > $OUT/prof_plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s ${SKIP:-0} -c ${COUNT:-1} \
    -o $OUT/prof_$TAG -f $CMD > $OUT/prof_$TAG.log 2>&1
echo "ncu exit $?" >> $OUT/prof_$TAG.log
