"""A one-device proxy for cross-GPU work stealing: N linked shards of one
search run concurrently on one B200, each with a slice of the SMs (ctas_per_sm
= 1; two 512-thread CTAs fit per SM), from N host threads, like `pccp_gpu
solve --gpus N`.  For each workload, with and without stealing
(PCCP_NO_STEAL), every shard's device time, nodes and stolen subproblems, and
the job's time (the slowest shard); with stealing alone and with the
cross-GPU donation of pending branches as well.  `python scripts/steal_proxy.py [N] [out.json]`."""
import json
import os
import sys
import threading

from paper_2207_12116_b200 import Engine, Model
from paper_2207_12116_b200.distributed import combine_enum, combine_solve
from paper_2207_12116_b200.engine import link_peers

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
out_path = sys.argv[2] if len(sys.argv) > 2 else None
WORK = [("rcpsp30-s7", lambda: Model.rcpsp_random(7, 30, 4), "solve", 60),
        ("rcpsp30-s3", lambda: Model.rcpsp_random(3, 30, 4), "solve", 30),
        ("rcpsp30-s6", lambda: Model.rcpsp_random(6, 30, 4), "solve", 30),
        ("csp-d22", lambda: Model.random_csp(1), "enum", 22)]


def run(name, make, kind, arg, steal):
    """steal: 0 static split, 1 stealing only, 2 stealing and cross-GPU donation."""
    for k in ("PCCP_NO_STEAL", "PCCP_NO_REMOTE_DONATE"):
        os.environ.pop(k, None)
    if steal == 0:
        os.environ["PCCP_NO_STEAL"] = "1"
    elif steal == 1:
        os.environ["PCCP_NO_REMOTE_DONATE"] = "1"
    m = make()
    engs = [Engine(0, shard_index=k, shard_count=n, ctas_per_sm=1, mix_order=-1) for k in range(n)]
    for e in engs:
        e.load(m)
    link_peers(engs)
    res = [None] * n

    def work(k):
        e = engs[k]
        if kind == "solve":
            r = e.solve(timeout_s=arg)
            res[k] = {"status": r.status, "objective": r.objective, "device_ms": r.stats["device_ms"],
                      "nodes": r.stats["nodes"], "stolen": r.stats["stolen"],
                      "exhausted": r.status in ("OPTIMAL", "UNSAT"), "proved": r.primal_proved,
                      "solutions": r.stats["solutions"], "has_store": r.best_words is not None,
                      "remote_in": r.stats["remote_in"], "remote_out": r.stats["remote_out"]}
        else:
            r = e.enumerate(depth_cap=arg)
            res[k] = dict(r)

    # warm-up, one after the other: a first search allocates its buffers, and an
    # allocation synchronises the whole device (it would serialise the shards)
    for k in range(n):
        work(k)
    for e in engs:
        e.reset_shared()
    th = [threading.Thread(target=work, args=(k,)) for k in range(n)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in engs:
        e.close()
    shards = [{"device_ms": round(r["device_ms"], 3), "nodes": int(r["nodes"]), "stolen": int(r["stolen"]),
               "remote_in": int(r.get("remote_in", 0)), "remote_out": int(r.get("remote_out", 0))} for r in res]
    job = {"job_ms": max(s["device_ms"] for s in shards), "shards": shards}
    if kind == "solve":
        c = combine_solve(res)
        job.update(status=c["status"], objective=c["objective"])
    else:
        c = combine_enum(res)
        job.update(nodes=c["nodes"], hash_ok=None)
    return job


report = {"n_shards": n, "note": "one B200, shards concurrent on SM slices (ctas_per_sm 1), reference order"}
for name, make, kind, arg in WORK:
    report[name] = {"static": run(name, make, kind, arg, 0), "stealing": run(name, make, kind, arg, 1),
                    "stealing+donation": run(name, make, kind, arg, 2)}
    print(name, json.dumps(report[name]), flush=True)
for k in ("PCCP_NO_STEAL", "PCCP_NO_REMOTE_DONATE"):
    os.environ.pop(k, None)
if out_path:
    with open(out_path, "w") as f:
        json.dump(report, f, indent=1)
