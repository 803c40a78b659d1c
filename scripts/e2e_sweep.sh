#!/bin/bash
# e2e (host-buffer) rate for chunk plans (NBVH_HOST_WEIGHTS) and interleave block sizes
# (NBVH_HOST_BLOCK, rays per block)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
: > gpurun_out/e2e_sweep.log
for B in ${BLOCKS:-1024 4096 8192 16384}; do
for Wt in ${PLANS:-"1,2,3,3,2,1"}; do
  v=$(NBVH_HOST_BLOCK=$B NBVH_HOST_WEIGHTS=$Wt timeout 120 python bench.py --steps 10 --warmup 3 --cpu-seconds 0 --train 0 --lod 0 --pt 0 2>/dev/null | tail -1 | python -c 'import json,sys; print(round(json.loads(sys.stdin.read())["e2e"]["value"],1))')
  echo "block=$B weights=$Wt e2e=$v" >> gpurun_out/e2e_sweep.log
done; done
