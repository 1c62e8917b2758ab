"""The pccp_gpu CLI against the reference CLI's own tests (tests/test_cli.cpp):
report keys, JSON keys, exit codes (0 / 2 UNKNOWN / 1 error), JSON ingest and
verify.  Parsing and argument errors need no GPU; solving does."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2207_12116_b200", "pccp_gpu")

# test_cli.cpp:39-53
CHAIN_TOY = "4 1\n1\n0 0 2 2 3\n2 1 2 3 4\n3 1 1 4\n0 0 0\n"
UNSAT_TOY = "3 1\n0\n0 0 1 2\n4 1 1 3\n0 0 0\n"
CHAIN_JSON = """{
    "tasks": [{"duration": 0}, {"duration": 2, "usages": [1]},
              {"duration": 3, "usages": [1]}, {"duration": 0}],
    "precedences": [[0, 1], [1, 2], [1, 3], [2, 3]],
    "capacities": [1]
  }"""


def run(args, env=None, timeout=300):
    e = dict(os.environ)
    e.update(env or {})
    p = subprocess.run([CLI] + args, capture_output=True, text=True, env=e, timeout=timeout)
    return p.returncode, p.stdout, p.stderr


def write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


@pytest.fixture(scope="module", autouse=True)
def built():
    if not os.path.exists(CLI):
        pytest.skip("pccp_gpu not built (python -c 'import __graft_entry__ as g; g.build()')")


# ---- no GPU needed -------------------------------------------------------------------
def test_bad_files_and_flags_exit_one(tmp_path):
    """test_cli.cpp:100-105."""
    assert run(["solve", "/nonexistent.rcp"])[0] == 1
    trunc = write(tmp_path, "trunc.rcp", "7 1\n1\n0 0 1")
    code, _, err = run(["solve", trunc])
    assert code == 1 and "truncated" in err
    assert run(["solve", "--engine", "bogus", trunc])[0] != 0
    assert run(["solve", "--timeout", "x", trunc])[0] != 0
    assert run(["bogus"])[0] != 0
    assert run([])[0] != 0


@pytest.mark.parametrize("text,what", [
    ('{"tasks": [{"duration": 1}], "capacities": [1], "precedences": [[0]]}', "pairs"),
    ('{"tasks": [{"duration": 1}', "bad json"),
    ('{"capacities": []}', "tasks"),
    ('{"tasks": [{"duration": 1}, {"duration": 1}], "precedences": [[0, 1], [1, 0]]}', "cyclic"),
    ('{"tasks": [{"duration": -1}]}', "negative"),
    ('{"tasks": [{"duration": 1.5}]}', "integer"),
])
def test_bad_json_instances_exit_one(tmp_path, text, what):
    code, _, err = run(["solve", write(tmp_path, "bad.json", text)])
    assert code == 1 and what in err, err


def test_gen_round_trips_through_the_parser(tmp_path):
    """`gen` prints random_patterson as Patterson text; the parser must read it
    back into the same model (same slots and command count as the generator)."""
    from paper_2207_12116_b200 import Model
    code, text, _ = run(["gen", "1", "30", "4"])
    assert code == 0
    a = Model.rcpsp_patterson(text).tables()
    b = Model.rcpsp_random(1, 30, 4).tables()
    assert a.n_cmds == b.n_cmds and a.n_words == b.n_words
    assert list(a.slot_word) == list(b.slot_word) and list(a.cands) == list(b.cands)


# ---- on the B200 -----------------------------------------------------------------------
gpu = pytest.mark.gpu


@gpu
def test_solve_prints_the_documented_report(tmp_path):
    """test_cli.cpp:56-65."""
    code, out, _ = run(["solve", write(tmp_path, "chain.rcp", CHAIN_TOY)])
    assert code == 0
    assert "status: OPTIMAL" in out and "objective: 5" in out
    for k in ("nodes: ", "time_ms: ", "nodes_per_sec: "):
        assert k in out


@gpu
def test_json_output_keys(tmp_path):
    """test_cli.cpp:67-77."""
    code, out, _ = run(["solve", "--json", write(tmp_path, "chain.rcp", CHAIN_TOY)])
    assert code == 0
    j = json.loads(out)
    assert j["status"] == "OPTIMAL" and j["objective"] == 5
    assert isinstance(j["nodes"], int) and j["nodes"] >= 0
    assert isinstance(j["time_ms"], int) and isinstance(j["nodes_per_sec"], int)
    assert list(j) == sorted(j)  # nlohmann's sorted object keys


@gpu
def test_unsat_reports_objective_none(tmp_path):
    """test_cli.cpp:79-89."""
    f = write(tmp_path, "unsat.rcp", UNSAT_TOY)
    code, out, _ = run(["solve", f])
    assert code == 0 and "status: UNSAT" in out and "objective: none" in out
    assert json.loads(run(["solve", "--json", f])[1])["objective"] is None


@gpu
def test_forced_timeout_is_unknown_exit_two(tmp_path):
    """test_cli.cpp:91-98 (a corpus-sized instance whose root is no solution)."""
    _, text, _ = run(["gen", "4", "30", "4"])
    code, out, _ = run(["solve", "--timeout", "0.000001", write(tmp_path, "big.rcp", text)])
    assert code == 2 and "status: UNKNOWN" in out


@gpu
def test_reports_deterministic_apart_from_timing(tmp_path):
    """test_cli.cpp:107-118: status and objective; node counts of a parallel
    search depend on timing, so they are compared for the
    one-shard enumeration-free toy only."""
    f = write(tmp_path, "chain.rcp", CHAIN_TOY)
    a = json.loads(run(["solve", "--json", "--engine", "seq", "--seed", "3", "--workers", "1", f])[1])
    b = json.loads(run(["solve", "--json", "--engine", "seq", "--seed", "3", "--workers", "1", f])[1])
    assert (a["status"], a["objective"], a["nodes"]) == (b["status"], b["objective"], b["nodes"])


@gpu
def test_json_ingest_solves_the_same_instance(tmp_path):
    """test_cli.cpp:120-130."""
    out = run(["solve", "--json", write(tmp_path, "chain.json", CHAIN_JSON)])[1]
    assert json.loads(out)["objective"] == 5


@gpu
def test_verify_passes_on_healthy_instances(tmp_path):
    """test_cli.cpp:132-137, plus a 30-task instance (tables in shared and global memory)."""
    code, out, _ = run(["verify", write(tmp_path, "chain.rcp", CHAIN_TOY)])
    assert code == 0 and "PASS" in out
    _, text, _ = run(["gen", "1", "30", "4"])
    code, out, _ = run(["verify", write(tmp_path, "r30.rcp", text)])
    assert code == 0 and "PASS" in out and "1184 cells" in out


@gpu
def test_empty_model_verifies_and_solves_to_zero(tmp_path):
    """test_cli.cpp:139-148."""
    f = write(tmp_path, "empty.json", '{"tasks": [], "capacities": []}')
    code, out, _ = run(["verify", f])
    assert code == 0 and "PASS" in out
    code, out, _ = run(["solve", "--json", f])
    assert code == 0 and json.loads(out)["objective"] == 0


@gpu
def test_workers_env_default(tmp_path):
    """test_cli.cpp:175-179."""
    assert run(["solve", "--json", write(tmp_path, "chain.rcp", CHAIN_TOY)], env={"PCCP_WORKERS": "2"})[0] == 0


@gpu
@pytest.mark.parametrize("seed,optimum", [(1, 84), (5, 73), (11, 99)])
def test_rcpsp30_optimum_through_the_cli(tmp_path, seed, optimum):
    _, text, _ = run(["gen", str(seed), "30", "4"])
    f = write(tmp_path, f"r30s{seed}.rcp", text)
    j = json.loads(run(["solve", "--json", "--timeout", "60", f])[1])
    assert j["status"] == "OPTIMAL" and j["objective"] == optimum


@gpu
@pytest.mark.parametrize("shards", [2, 4])
def test_sharded_solve_with_linked_incumbents(tmp_path, shards):
    """--gpus N on one device (--devices 0,0,..): N contexts on N host threads,
    EPS shards i mod N, incumbents linked by pccp_gpu_link_peers.  The optimum
    and the proof must be those of one context."""
    _, text, _ = run(["gen", "2", "30", "4"])
    f = write(tmp_path, "r30s2.rcp", text)
    devs = ",".join(["0"] * shards)
    code, out, _ = run(["solve", "--json", "--stats", "--devices", devs, "--timeout", "120", f])
    j = json.loads(out)
    assert code == 0 and j["status"] == "OPTIMAL" and j["objective"] == 77 and j["gpus"] == shards


@gpu
def test_primal_phase_through_the_cli(tmp_path):
    _, text, _ = run(["gen", "1", "120", "4"])
    f = write(tmp_path, "r120.rcp", text)
    code, out, _ = run(["solve", "--json", "--stats", "--timeout", "3", "--primal-ms", "3000", f])
    j = json.loads(out)
    assert code == 0 and j["status"] == "SAT" and j["objective"] >= 237 and j["primal_nodes"] > 0
