#!/bin/bash
# ncu --set full of the T7 scatter kernels: the plain one (privatised levels 0-2) and the
# warp-aggregated one (NBVH_SCATTER_AGG=6, no privatisation)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT=gpurun_out; TAG=${1:-t}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
CMD="python bench.py --steps 2 --warmup 1 --cpu-seconds 0 --lod 0 --pt 0"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_train_scatter" -s 0 -c 2 \
    -o $OUT/prof_scatter_$TAG -f $CMD > $OUT/prof_scatter_$TAG.log 2>&1
echo "ncu exit $?" >> $OUT/prof_scatter_$TAG.log
NBVH_SCATTER_AGG=6 NBVH_PRIV_BYTES=0 timeout 600 ncu --set full --clock-control none --import-source on \
    -k regex:"k_train_scatter" -s 0 -c 2 -o $OUT/prof_scatter_agg_$TAG -f $CMD > $OUT/prof_scatter_agg_$TAG.log 2>&1
echo "ncu exit $?" >> $OUT/prof_scatter_agg_$TAG.log
