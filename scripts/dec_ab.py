"""EPS target A/B: `PCCP_DEC_TARGET=k python scripts/dec_ab.py` -> device ms of Q8, Q14, CSP d22 (median of 5)."""
import json
import statistics

from paper_2207_12116_b200 import Engine, Model

out = {}
for name, m, depth in (("q8", Model.nqueens(8), -1), ("q14", Model.nqueens(14), -1), ("csp", Model.random_csp(1), 22)):
    with Engine(0) as e:
        e.load(m)
        for _ in range(2):
            e.enumerate(depth_cap=depth)
        ts, ds = [], []
        for _ in range(5):
            r = e.enumerate(depth_cap=depth)
            ts.append(r["device_ms"])
            ds.append(r["decompose_ms"])
        out[name] = (round(statistics.median(ts), 4), round(statistics.median(ds), 4), r["subproblems"])
print(json.dumps(out))
