"""RCPSP30 parity seeds with a short primal phase: `python scripts/r30_primal.py primal_ms`
(PCCP_PRIMAL_STALL_MS sets the stall window).  Median device time to proof of 3 solves."""
import json
import statistics
import sys

from paper_2207_12116_b200 import Engine, Model

pm = int(sys.argv[1]) if len(sys.argv) > 1 else 0
want = {1: 84, 2: 77, 5: 73, 7: 60, 9: 61, 11: 99}
out, tot = {}, 0.0
for seed, opt in want.items():
    m = Model.rcpsp_random(seed, 30, 4)
    with Engine(0, primal_ms=pm) as e:
        e.load(m)
        ts, ns, first = [], [], []
        for _ in range(int(__import__("os").environ.get("REPS", "3"))):
            r = e.solve(timeout_s=60)
            assert r.status == "OPTIMAL" and r.objective == opt, (seed, r.status, r.objective)
            ts.append(r.stats["device_ms"])
            ns.append(r.stats["nodes"])
            first.append(min(ms for v, ms in r.improvements if v == opt))
    out[seed] = (round(statistics.median(ts), 3), int(statistics.median(ns)), round(statistics.median(first), 3))
    tot += statistics.median(ts)
print(json.dumps({"primal_ms": pm, "total_ms": round(tot, 3), "seeds": out}))
