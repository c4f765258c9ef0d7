"""Both GEMM paths for T > 256 against the numpy fp32 reference: the default runs CTA pairs
(cta_group::2) there (tests/test_gpu_gemm.py), so the T > 256 shapes run again in a child
process with pairs off (SPIN_GEMM_PAIR_MIN_T=0, read once per process by gemm_plan): the
single-CTA grouped stream-K path stays parity-tested."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_single_cta_path_for_large_t_matches_fp32():
    env = dict(os.environ, SPIN_GEMM_PAIR_MIN_T="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", os.path.join(ROOT, "tests", "test_gpu_gemm.py"),
                        "-k", "partial and (645 or 1280 or 512)"], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout, r.stdout[-500:]
