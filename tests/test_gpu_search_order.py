"""Search-order extensions (not in the reference): variable orders 1-3 (smallest
lb first, include/pccp_gpu.h `var_order`) and the primal phase (`primal_ms`).

They change the tree, so node counts differ from the reference's; what must
not differ is checked here against the reference's goldens:
  * the solution set: the number of all-solutions leaves is the same under any
    variable order (a leaf is fp(root + assignment), failure is monotone);
  * optima and UNSAT proofs (solve_dfs / solve_parallel goldens);
  * every incumbent passes check_solution (rcpsp.cpp:275-300)."""
import pytest

from conftest import load_micro_rcpsps
from test_gpu_parity import build

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("var_order", [1, 2, 3])
@pytest.mark.parametrize("n", [6, 8, 10])
def test_solution_count_invariant_under_var_order(n, var_order, golden):
    from paper_2207_12116_b200 import Engine
    g = golden[f"nqueens{n}"]["enumerate"]
    with Engine(0, var_order=var_order) as e:
        res = e.load(build(f"nqueens{n}")).enumerate()
    assert res["exhausted"]
    assert res["solutions"] == g["solutions"]


@pytest.mark.parametrize("var_order", [2, 3])
def test_depth_capped_csp_tree_shape(var_order):
    """Depth caps cut different trees, so counts differ from the golden; the
    run must still be exhausted and a full binary tree (every branching node
    has two children: nodes = 2 * leaves - 1)."""
    from paper_2207_12116_b200 import Engine
    with Engine(0, var_order=var_order) as e:
        res = e.load(build("csp_small2")).enumerate(depth_cap=10)
    assert res["exhausted"]
    leaves = res["failures"] + res["solutions"] + res["open_leaves"]
    assert res["nodes"] == 2 * leaves - 1


@pytest.mark.parametrize("seed", [1, 2, 5, 7, 9, 11])
def test_rcpsp30_optimum_with_primal_phase(seed, golden):
    from paper_2207_12116_b200 import Engine
    m = build(f"rcpsp30_s{seed}")
    with Engine(0, primal_ms=2000) as e:
        res = e.load(m).solve(timeout_s=120)
    assert res.status == "OPTIMAL"
    assert res.objective == golden[f"rcpsp30_s{seed}"]["optimum"]["value"]
    assert m.check_solution(res.best_words)
    incs = [v for v, _ in res.improvements]
    assert all(a > b for a, b in zip(incs, incs[1:]))
    assert res.primal is not None and res.primal["nodes"] > 0


@pytest.mark.parametrize("var_order", [1, 2, 3])
def test_rcpsp10_optimum_under_var_orders(var_order, golden):
    from paper_2207_12116_b200 import Engine
    with Engine(0, var_order=var_order) as e:
        for seed in range(1, 9):
            g = golden[f"rcpsp10_s{seed}"]["solve_dfs"]
            m = build(f"rcpsp10_s{seed}")
            res = e.load(m).solve()
            assert res.status == {0: "OPTIMAL", 2: "UNSAT"}[g["status"]], seed
            assert res.objective == g["objective"], seed
            if res.objective is not None:
                assert m.check_solution(res.best_words)


def test_micro_rcpsp_optimality_with_primal_phase():
    """The 200 brute-forced micro RCPSPs (acceptance_main.cpp:243-287) through
    the primal phase: same optima, UNSAT where there is no schedule."""
    from paper_2207_12116_b200 import Engine
    with Engine(0, primal_ms=500) as e:
        for t, rec in load_micro_rcpsps():
            e.load(t)
            res = e.solve()
            if rec["brute_force"] is None:
                assert res.status == "UNSAT"
            else:
                assert res.status == "OPTIMAL" and res.objective == rec["brute_force"]


def test_primal_phase_limits_and_unsat():
    from paper_2207_12116_b200 import Engine, Model
    prec = []
    for i in (1, 2, 3):
        prec += [(0, i), (i, 4)]
    m = Model.rcpsp([0, 2, 2, 2, 0], [[0], [1], [1], [1], [0]], [1], prec, 5)
    with Engine(0, primal_ms=1000) as e:
        e.load(m)
        assert e.solve(node_limit=0).status == "UNKNOWN"
        r = e.solve()
        assert r.status == "UNSAT" and r.primal["proved"]


def test_rcpsp120_primal_finds_a_valid_schedule():
    """Config 5: the reference's order finds no leaf in 300 s on 8 cores
    (SURVEY 8d); the primal phase must produce a checker-valid schedule fast."""
    from paper_2207_12116_b200 import Engine
    m = build("rcpsp120_s1")
    with Engine(0, primal_ms=3000) as e:
        res = e.load(m).solve(timeout_s=3)
    assert res.status == "SAT"
    assert m.check_solution(res.best_words)
    assert res.objective >= 237  # the root fixed point's critical-path bound
    assert res.improvements and res.improvements[0][1] < 2000.0
