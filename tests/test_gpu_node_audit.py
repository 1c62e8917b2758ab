"""Per-node parity of the persistent search itself ("identical
propagation fixed points per node").  The engine samples nodes of its own
search (cfg audit_nodes / audit_shift): the store as materialised (parent fixed
point + decision + objective bound) and the fixed point the search computed.
The C oracle, pinned to the reference, recomputes run_sequential
(engine.cpp:13-32) from every sampled store and must agree exactly.  Also the
reference's error behaviour for unbounded branching candidates."""
import numpy as np
import pytest

from oracle.port import Oracle
from test_gpu_parity import build

pytestmark = pytest.mark.gpu


def audited(name, n, shift, run, **cfg):
    from paper_2207_12116_b200 import Engine
    m = build(name)
    with Engine(0, audit_nodes=n, audit_shift=shift, **cfg) as e:
        e.load(m)
        out = run(e)
        pre, post, failed = e.audit()
    return m, out, pre, post, failed


def check_samples(m, pre, post, failed):
    o = Oracle(m.tables())
    assert len(pre) > 0
    for k in range(len(pre)):
        f, w, _, _ = o.run_sequential(pre[k])
        assert f == failed[k], k
        if not f:
            assert np.array_equal(w, post[k]), k


# eps_factor 1 keeps the decomposition small, so most nodes are the search's
@pytest.mark.parametrize("name,shift", [("nqueens12", 10), ("nqueens13", 12)])
def test_enumeration_nodes(name, shift):
    m, r, pre, post, failed = audited(name, 96, shift, lambda e: e.enumerate(), eps_factor=1)
    assert r["exhausted"]
    check_samples(m, pre, post, failed)


def test_csp_nodes_depth_capped():
    m, r, pre, post, failed = audited("csp1", 48, 6, lambda e: e.enumerate(depth_cap=17), eps_factor=1)
    check_samples(m, pre, post, failed)


@pytest.mark.parametrize("seed", [1, 7])
def test_rcpsp30_branch_and_bound_nodes(seed, golden):
    """Optimisation nodes carry the incumbent's bound obj <= best - 1 in `pre`."""
    m, s, pre, post, failed = audited(f"rcpsp30_s{seed}", 48, 10, lambda e: e.solve(timeout_s=60))
    assert s.status == "OPTIMAL" and s.objective == golden[f"rcpsp30_s{seed}"]["optimum"]["value"]
    check_samples(m, pre, post, failed)


def test_rcpsp120_primal_nodes():
    m, s, pre, post, failed = audited("rcpsp120_s1", 6, 12, lambda e: e.solve(timeout_s=2), primal_ms=2000)
    assert s.status == "SAT" and m.check_solution(s.best_words)
    check_samples(m, pre, post, failed)


def test_unbounded_candidate_is_a_model_error():
    """branch() throws ModelError on an unbounded candidate (solver.cpp:41-43);
    the device search reports it as PCCP_EMODEL instead of terminating."""
    from paper_2207_12116_b200 import Engine, Model
    from paper_2207_12116_b200._native import ModelError
    m = Model()
    x = m.add_cell()
    y = m.add_cell()
    m.tell(y, 0, 3)  # x stays (-inf, +inf)
    with Engine(0) as e:
        e.load(m)
        with pytest.raises(ModelError):
            e.enumerate()
