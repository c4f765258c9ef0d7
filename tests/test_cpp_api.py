"""Runs the C++ drop-in API tests (tests/cpp) and the drop-in proof binary
(the reference's unmodified bandit/matching/policies sources linked to the B200
SlotEngine, oracle/_ref/lbss_on_b200)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "build", "test_specsim_api")
DROPIN = os.path.join(ROOT, "oracle", "_ref", "lbss_on_b200")


def _build():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2503_15921_b200", "csrc")], check=True)
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)


def test_cpp_api_host_parts():
    _build()
    r = subprocess.run([BIN, "host"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


@pytest.mark.gpu
def test_cpp_api_on_gpu():
    _build()
    r = subprocess.run([BIN, "gpu"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


@pytest.mark.gpu
def test_reference_selector_drives_b200_engine():
    if not os.path.exists(DROPIN):
        pytest.skip("drop-in binary not built (needs /root/reference at build time: make -C oracle dropin)")
    r = subprocess.run([DROPIN, "16"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["lbss_tokens"] > 0 and out["greedy_tokens"] > 0
    assert out["lbss_time_s"] > 0 and out["greedy_time_s"] > 0
