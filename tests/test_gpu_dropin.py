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
    # GpuConfig{devices = {0, 0}}: two linked shards on one device match solve_parallel
    assert r["sharded_equal"] and r["sharded_optima"] == "84/84, 60/60"
    assert r["persistent"]  # one GpuEngine, lowered once, three solves
    assert r["batch_equal"] == 64  # propagate_batch_gpu == run_sequential on 64 sub-boxes


VERIFY = os.path.join(ROOT, "oracle", "_ref", "verify_gpu")


@pytest.mark.skipif(not os.path.exists(VERIFY), reason="oracle/_ref/verify_gpu not built (needs /root/reference)")
def test_reference_confluence_check_with_gpu_engine():
    """`pccp verify` (tools/pccp.cpp:97-188) over the 110 corpus instances and the
    RCPSP30 parity seeds with the device fixed points (4 launch shapes) beside
    seq, fair x 10 and par x {1, 2, 4, 8}: every run agrees cell for cell; the
    non-monotone generic mutant is rejected by the device path (ModelError)."""
    out = subprocess.run([VERIFY], capture_output=True, text=True, timeout=1200)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["ok"] and r["pass"] == r["instances"] == 116, r
    assert r["gpu_runs"] >= 3 * r["instances"]
    assert r["mutant_checked"] == r["mutant_rejected"] == 10
