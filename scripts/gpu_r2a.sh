#!/bin/bash
# round-2 first GPU session: tests, smoke, bench (tiles vs rows order)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "${KSEL:-}" > $OUT/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
echo "smoke exit $?" >> $OUT/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/bench_tiles.json 2> $OUT/bench_tiles.err
echo "bench exit $?" >> $OUT/bench_tiles.err
timeout 300 python bench.py --steps 10 --warmup 3 --order rows --train 0 --lod 0 --pt 0 --cpu-seconds 0 > $OUT/bench_rows.json 2> $OUT/bench_rows.err
echo "bench exit $?" >> $OUT/bench_rows.err
