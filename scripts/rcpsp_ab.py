"""A/B timing of the RCPSP configs for one engine configuration:
`python scripts/rcpsp_ab.py [group_threads] [ctas_per_sm]` (env knobs such as
PCCP_NO_PACK=1 select the layout).  RCPSP30 parity seeds: device time to proof
(median of 3); RCPSP120 seed 1: reference-order nodes/s over 3 s."""
import json
import statistics
import sys

from paper_2207_12116_b200 import Engine, Model

gt = int(sys.argv[1]) if len(sys.argv) > 1 else 0
cps = int(sys.argv[2]) if len(sys.argv) > 2 else 0
want = {1: 84, 2: 77, 5: 73, 7: 60, 9: 61, 11: 99}
out = {"group_threads": gt, "ctas_per_sm": cps}
tot = 0.0
for seed, opt in want.items():
    m = Model.rcpsp_random(seed, 30, 4)
    with Engine(0, group_threads=gt, ctas_per_sm=cps) as e:
        e.load(m)
        info = e.lowering_info()
        ts, nodes = [], []
        for _ in range(3):
            r = e.solve(timeout_s=60)
            assert r.status == "OPTIMAL" and r.objective == opt, (seed, r.status, r.objective)
            assert m.check_solution(r.best_words)
            ts.append(r.stats["device_ms"])
            nodes.append(r.stats["nodes"])
    med = statistics.median(ts)
    tot += med
    out[f"s{seed}"] = {"ms": round(med, 3), "nodes": int(statistics.median(nodes)),
                       "Mnodes_s": round(statistics.median(nodes) / med / 1e3, 2)}
out["r30_total_ms"] = round(tot, 3)
out["r30_layout"] = {k: info[k] for k in ("device_words", "packed_cells", "group_threads", "groups_per_cta", "ctas",
                                          "smem_bytes", "table_in_smem", "table_bytes")}
m = Model.rcpsp_random(1, 120, 4)
with Engine(0, group_threads=gt, ctas_per_sm=cps) as e:
    e.load(m)
    info = e.lowering_info()
    r = e.solve(timeout_s=3.0)
    out["r120_ref_order"] = {"nodes": r.stats["nodes"], "device_ms": round(r.stats["device_ms"], 1),
                             "nodes_per_s": round(r.stats["nodes"] / (r.stats["device_ms"] / 1e3))}
    out["r120_layout"] = {k: info[k] for k in ("device_words", "packed_cells", "group_threads", "groups_per_cta",
                                               "ctas", "smem_bytes", "table_in_smem", "table_bytes")}
print(json.dumps(out))
