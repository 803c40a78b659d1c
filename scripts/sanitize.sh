#!/bin/bash
# compute-sanitizer memcheck (one tool per call) over a few small GPU tests.  (The GPU pool
# refuses compute-sanitizer runs; tests/test_gpu_debug_checks.py runs the device-side bounds
# checks of the debug build instead.)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 compute-sanitizer --tool ${TOOL:-memcheck} --error-exitcode 9 --print-limit 20 \
    python -m pytest tests/test_gpu_query.py tests/test_gpu_pathtrace.py -q -p no:cacheprovider \
    -k "tiny_end_to_end or refill or lod_slots or chunked or intersect_mesh or pt_shade" \
    > gpurun_out/sanitize_${TOOL:-memcheck}.log 2>&1
echo "sanitizer exit $?" >> gpurun_out/sanitize_${TOOL:-memcheck}.log
