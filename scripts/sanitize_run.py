"""A CI-sized workload for compute-sanitizer (memcheck / synccheck / racecheck):
Q8 enumeration (warp groups), CSP depth 10 (CTA groups, rows), an RCPSP10
solve (fused reifications, incumbent, donations), a propagate batch, a
primal-phase solve, a node-limited RCPSP30 solve (bit planes, kPacked, the
control prefetch), two linked shards stealing, and a randomised-order
enumeration."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2207_12116_b200 import Engine, Model  # noqa: E402

with Engine(0, hash=True, eps_factor=1) as e:
    r = e.load(Model.nqueens(8)).enumerate()
    assert (r["nodes"], r["solutions"], r["hash_sum"]) == (779, 92, 0xF1DF80A1FF36FBF6), r
    r = e.load(Model.random_csp(2, n_vars=60, n_cons=200)).enumerate(depth_cap=8)
    print("csp", r["nodes"], r["open_leaves"])
with Engine(0, eps_factor=1) as e:
    m = Model.rcpsp_random(1, 10, 2)
    s = e.load(m).solve()
    assert s.status == "OPTIMAL" and m.check_solution(s.best_words), s.status
    out, failed, _ = e.propagate_batch([m.bottom()] * 4)
    print("rcpsp10", s.objective, s.stats["nodes"], failed.tolist())
with Engine(0, eps_factor=1, primal_ms=300) as e:  # primal segments, restarts, keep-incumbent resets
    m = Model.rcpsp_random(2, 10, 2)
    s = e.load(m).solve(timeout_s=60)  # the sanitizers slow the search down by orders of magnitude
    assert s.status in ("OPTIMAL", "SAT") and m.check_solution(s.best_words), s.status
    print("primal", s.objective, s.primal)
with Engine(0, group_threads=256, ctas_per_sm=1) as e:  # kPacked CTA groups, control prefetch, bit planes
    m = Model.rcpsp_random(1, 30, 4)
    s = e.load(m).solve(node_limit=3000)
    assert s.status in ("OPTIMAL", "SAT", "UNKNOWN"), s.status
    print("rcpsp30", s.status, s.objective, s.stats["nodes"])
from paper_2207_12116_b200.engine import link_peers  # noqa: E402
engs = [Engine(0, shard_index=k, shard_count=2, ctas_per_sm=1, groups_per_cta=1) for k in range(2)]
for e in engs:
    e.load(Model.nqueens(7))
link_peers(engs)  # linked shards: epoch-tagged share cells, stealing
parts = [e.enumerate() for e in engs]
assert sum(p["solutions"] for p in parts) == 40, parts
for e in engs:
    e.close()
with Engine(0, eps_factor=1, var_order=3) as e:  # randomised branching
    r = e.load(Model.nqueens(6)).enumerate()
    assert r["solutions"] == 4, r
print("sanitize workload ok")
