#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT=gpurun_out; TAG=${1:-dw}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_train_(dw|bias|fwd|label|select)" -s 0 -c 5 \
    -o $OUT/prof_dw_$TAG -f python bench.py --steps 2 --warmup 1 --cpu-seconds 0 --lod 0 --pt 0 > $OUT/prof_dw_$TAG.log 2>&1
echo "ncu exit $?" >> $OUT/prof_dw_$TAG.log
