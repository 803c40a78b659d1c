"""The debug-checks build (device-side bounds asserts on grid cells, hash indices, work-list
records, list positions, traversal fill and gradient-scatter indices; build.py debug=True)
runs the tiny query, host path (with list refills), training steps and the tcgen05 MLP
without a failed check.  (compute-sanitizer is not available on the GPU pool.)"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_debug_checks_build_runs_clean():
    from paper_2405_16237_b200 import build as b
    lib = b.build(debug=True)
    env = dict(os.environ, NBVH_LIB=lib)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "helpers", "debug_checks_run.py")],
                         capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert out.returncode == 0, (out.stdout[-2000:], out.stderr[-4000:])
    assert "debug checks ok" in out.stdout
