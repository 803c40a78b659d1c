#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for Wt in "1" "1,1,1,1" "1,2,2,1" "1,2,2,2,1" "1,2,3,3,2,1" "1,3,3,3,1" "1,2,2,2,2,2,1"; do
  echo "weights $Wt: $(NBVH_HOST_WEIGHTS=$Wt python bench.py --steps 10 --warmup 3 --cpu-seconds 0 --train 0 --lod 0 | python -c 'import json,sys; d=json.load(sys.stdin); print(d["e2e"]["value"])')"
done
