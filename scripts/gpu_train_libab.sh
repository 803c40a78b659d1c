#!/bin/bash
# training-step timing with alternative in-tree libraries (NBVH_LIB=$LIBS) vs the default
# build, interleaved (def, alt..., def), then the phase table
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT=gpurun_out; TAG=${1:-tl}; mkdir -p $OUT
B="python bench.py --steps 10 --warmup 3 --lod 0 --pt 0 --cpu-seconds 0"
timeout 300 $B > $OUT/bench_${TAG}_def.json 2>> $OUT/sweep_$TAG.err
for L in $LIBS; do
  NBVH_LIB=$PWD/paper_2405_16237_b200/$L timeout 300 $B > $OUT/bench_${TAG}_$L.json 2>> $OUT/sweep_$TAG.err
done
timeout 300 $B > $OUT/bench_${TAG}_def2.json 2>> $OUT/sweep_$TAG.err
python - "$OUT" "$TAG" <<'PY'
import glob, json, sys
for f in sorted(glob.glob(f"{sys.argv[1]}/bench_{sys.argv[2]}_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1]); t = d["train"]
        print(f, round(t["ms_per_step"], 4), {k: round(v, 4) for k, v in t["phase_ms_rank0"].items()})
    except Exception as e:
        print(f, "ERR", e)
PY
