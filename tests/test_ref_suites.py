"""Gate on the oracle build: the reference's own unit suites
(proj/tests/test_*.cpp, compiled unmodified against oracle/shim) pass on it,
with the assertion counts of SURVEY §0.5."""
import os
import subprocess

import pytest

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")
SUITES = {"test_collective": 47656, "test_model_fusion": 2464, "test_task_graph": 83,
          "test_simulate": 602, "test_cost_model": 2939, "test_analysis": 3776,
          "test_gp": 1102, "test_tuner": 146}


@pytest.mark.parametrize("suite", sorted(SUITES))
def test_reference_suite_passes(suite):
    exe = os.path.join(REF, suite)
    if not os.path.exists(exe):
        if not os.path.exists("/root/reference/proj/src/collective.cpp"):
            pytest.skip("reference build absent and /root/reference not mounted")
        subprocess.run(["make", "-s", "-C", os.path.dirname(REF), "ref"], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert f"assertions: {SUITES[suite]} | {SUITES[suite]} passed | 0 failed" in out.stdout
