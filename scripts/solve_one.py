"""One RCPSP solve for profiling: `python scripts/solve_one.py tasks seed [timeout_s] [node_limit] [reps]`
(a warm-up solve first, then `reps` solves; ncu -s 1 skips the warm-up's k_search)."""
import sys

from paper_2207_12116_b200 import Engine, Model

n, seed = int(sys.argv[1]), int(sys.argv[2])
timeout = float(sys.argv[3]) if len(sys.argv) > 3 else 60.0
limit = int(sys.argv[4]) if len(sys.argv) > 4 and int(sys.argv[4]) > 0 else None
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 1
m = Model.rcpsp_random(seed, n, 4)
with Engine(0, verbose=True) as e:
    e.load(m)
    e.solve(timeout_s=timeout, node_limit=limit)
    for _ in range(reps):
        r = e.solve(timeout_s=timeout, node_limit=limit)
        print(r.status, r.objective, r.stats["nodes"], r.stats["device_ms"], r.stats["rounds"])
