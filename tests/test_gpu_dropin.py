"""The drop-in boundary exercised from the reference side: the unmodified
reference library (oracle/_ref objects) calls the engine through
integration/pccp_gpu_shim.hpp — run_gpu vs run_sequential, solve_gpu vs
solve_parallel, generic commands rejected, N-Queens 8 through enumerate_gpu."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEMO = os.path.join(ROOT, "oracle", "_ref", "dropin_demo")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(DEMO), reason="oracle/_ref/dropin_demo not built (needs /root/reference)")
def test_reference_calls_engine_through_shim():
    out = subprocess.run([DEMO], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["ok"] and r["fixpoint_equal"] and r["valid"] and r["generic_rejected"]
    assert r["cpu_objective"] == r["gpu_objective"] == 84
    assert r["q8"] == [779, 92, 298]
