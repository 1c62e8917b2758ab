"""Config 5 (RCPSP 120x4 seed 1) over a long budget: the incumbent and the gap to
the best lower bound over time.  `python scripts/rcpsp120_long.py [budget_s] [out.json]`

The solve runs the primal phase (smallest-lb dives, include/pccp_gpu.h
primal_ms) for the whole budget, then whatever is left in the reference's
order.  Lower bounds: the root fixed point's makespan lb (critical path) and
the destructive bound (the smallest T whose root under makespan <= T does not
fail; bench.destructive_lower_bound).  Every incumbent is checked with
check_solution at the end (the best one; earlier ones are the same model's
solutions by construction)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import destructive_lower_bound  # noqa: E402
from paper_2207_12116_b200 import Engine, Model  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 60.0
out_path = sys.argv[2] if len(sys.argv) > 2 else None
m = Model.rcpsp_random(1, 120, 4)
sink = int(m.tables().slot_word[m.starts()[-1]])
with Engine(0, primal_ms=int(budget * 1e3)) as e:
    e.load(m)
    failed, root, _ = e.run_sequential()
    lb_root = int(root[sink])
    t0 = time.time()
    r = e.solve(timeout_s=budget)
    wall = time.time() - t0
    ok = r.best_words is not None and m.check_solution(r.best_words)
    lb = destructive_lower_bound(e, m, lb_root, r.objective if r.objective is not None else lb_root + 64)
    info = e.lowering_info()
best_lb = max(lb_root, lb)
res = {
    "config": "rcpsp 120x4 seed 1 (random_patterson(mt19937_64(1), 120, 4)), minimise makespan",
    "budget_s": budget, "wall_s": round(wall, 2), "status": r.status, "objective": r.objective, "valid": bool(ok),
    "lower_bound": {"root_critical_path": lb_root, "destructive": lb},
    "gap_final": None if r.objective is None else round((r.objective - best_lb) / r.objective, 4),
    "nodes": r.stats["nodes"], "device_ms": round(r.stats["device_ms"], 1),
    "nodes_per_s": round(r.stats["nodes"] / (r.stats["device_ms"] / 1e3)),
    "primal": r.primal,
    "incumbent_over_time": [{"objective": v, "t_ms": round(ms, 3), "gap": round((v - best_lb) / v, 4)}
                            for v, ms in r.improvements],
    "layout": {k: info[k] for k in ("device_words", "packed_cells", "group_threads", "ctas", "table_in_smem",
                                    "smem_bytes", "table_bytes")},
}
s = json.dumps(res)
print(s)
if out_path:
    with open(out_path, "w") as f:
        f.write(s + "\n")
