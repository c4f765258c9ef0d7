"""The CTA-pair (cta_group::2) GEMM path, opt-in via SPIN_GEMM_PAIR_MIN_T (gemm_plan reads it
once per process, so the T > 256 shapes of tests/test_gpu_gemm.py run in a child process with
pairs enabled) against the same numpy fp32 reference."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_pair_gemm_shapes_match_fp32():
    env = dict(os.environ, SPIN_GEMM_PAIR_MIN_T="257")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", os.path.join(ROOT, "tests", "test_gpu_gemm.py"),
                        "-k", "partial and (645 or 1280 or 512)"], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "skipped" not in r.stdout.split("\n")[-2], r.stdout[-500:]
