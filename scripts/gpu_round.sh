#!/bin/bash
# One GPU session: parity tests, smoke, bench (fp16 and bf16), ncu launch list + full captures
# of the dominant kernels.  Usage (from the repo root, on the GPU box):  bash scripts/gpu_round.sh [tag]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
TAG=${1:-r2}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi > $OUT/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $OUT/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> $OUT/pytest_gpu_$TAG.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1
echo "smoke exit $?" >> $OUT/smoke_$TAG.log
timeout 600 python bench.py --steps 10 --warmup 3 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
echo "bench exit $?" >> $OUT/bench_$TAG.err
timeout 300 python bench.py --steps 10 --warmup 3 --mlp-dtype bf16 --train 0 --lod 0 --pt 0 --cpu-seconds 0 \
    > $OUT/bench_${TAG}_bf16.json 2>> $OUT/bench_$TAG.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_${TAG}_reference.json 2>> $OUT/bench_$TAG.err
if [ "${SKIP_NCU:-0}" != "1" ]; then
  CMD="python bench.py --steps 2 --warmup 1 --cpu-seconds 0 --lod 0 --pt 0"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/launches_$TAG.csv $CMD > $OUT/ncu_launches.log 2>&1
  echo "ncu launches exit $?" >> $OUT/ncu_launches.log
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_query_warp|k_traverse" -s 0 -c 2 \
      -o $OUT/prof_query_$TAG -f $CMD --train 0 > $OUT/ncu_full.log 2>&1
  echo "ncu full exit $?" >> $OUT/ncu_full.log
  timeout 900 ncu --set full --clock-control none --import-source on \
      -k regex:"k_train_(select|fwd|bwd|label|dw|bias|scatter)" -s 0 -c 8 \
      -o $OUT/prof_train_$TAG -f $CMD > $OUT/ncu_full_train.log 2>&1
  echo "ncu full train exit $?" >> $OUT/ncu_full_train.log
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_mlp_tc" -s 0 -c 1 \
      -o $OUT/prof_mlp_$TAG -f $CMD --train 0 > $OUT/ncu_full_mlp.log 2>&1
  echo "ncu full mlp exit $?" >> $OUT/ncu_full_mlp.log
fi
