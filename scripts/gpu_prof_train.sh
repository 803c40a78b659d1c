#!/bin/bash
# ncu --set full of the training kernels (one step of the bench's cfg-5 workload)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT=gpurun_out; TAG=${1:-t}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
CMD="python bench.py --steps 2 --warmup 1 --cpu-seconds 0 --lod 0 --pt 0"
timeout 600 $CMD > $OUT/prof_plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_train_(select|fwd|bwd|label|dw|bias)" -s 0 -c 6 \
    -o $OUT/prof_train_$TAG -f $CMD > $OUT/prof_train_$TAG.log 2>&1
echo "ncu exit $?" >> $OUT/prof_train_$TAG.log
