#!/bin/bash
# e2e (host-buffer) rate for chunk plans: NBVH_HOST_WEIGHTS x NBVH_HOST_CONTIG
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
: > gpurun_out/e2e_sweep.log
for c in 0 1; do for Wt in "1,2,3,3,2,1" "1,1,1,1,1,1" "2,3,3,2" "1,2,2,2,1" "1,1,1,1,1,1,1,1"; do
  v=$(NBVH_HOST_CONTIG=$c NBVH_HOST_WEIGHTS=$Wt timeout 120 python bench.py --steps 10 --warmup 3 --cpu-seconds 0 --train 0 --lod 0 --pt 0 2>/dev/null | tail -1 | python -c 'import json,sys; print(round(json.loads(sys.stdin.read())["e2e"]["value"],1))')
  echo "contig=$c weights=$Wt e2e=$v" >> gpurun_out/e2e_sweep.log
done; done
