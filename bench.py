#!/usr/bin/env python
"""Headline benchmark: search nodes/s of the B200 propagate-and-search engine.

Workload (BASELINE.json configs[1]): N-Queens 14, all-solutions enumeration —
the whole 8,567,767-node tree (pairwise != decomposition, 1,106 guarded
commands over 28 words).  One step = one full enumeration through the C ABI
(EPS decomposition on the device + persistent DFS); the device time of the
step comes from CUDA events on the engine's own stream.

    python bench.py                                  # 1 GPU, 5 timed steps, 3 warm-up
    torchrun --nproc-per-node N bench.py --gpus N    # EPS frontier sharded i mod N, no data-path collective
    python bench.py --impl reference                 # the reference CPU path on this host's cores

The `cpu_baseline` object (rank 0, N=1) times the reference itself
(oracle/_ref: the reference library compiled from its sources, driven by the
harness DFS enumerator over its public API) on a bounded sample of the same
workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "q14": dict(workload="nqueens14-all-solutions", n=14, depth=-1,
                expect=dict(nodes=8567767, solutions=365596, failures=3918288, hash_sum=0xDB0839842A068562)),
    "q12": dict(workload="nqueens12-all-solutions", n=12, depth=-1, expect=dict(nodes=278923, solutions=14200)),
    "csp": dict(workload="random-linear-csp-seed1-depth22", csp=1, depth=22,
                expect=dict(nodes=108611, failures=23228, open_leaves=31078, hash_sum=0x6C8868DADE5564A8)),
}


def build_model(w):
    from paper_2207_12116_b200 import Model
    if "n" in w:
        return Model.nqueens(w["n"])
    return Model.random_csp(w["csp"])


def ref_model(w):
    from oracle.refh import RefModel
    if "n" in w:
        return RefModel.nqueens(w["n"])
    return RefModel.csp(w["csp"])


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


# ---- clocks (B200_PROFILING.md recipe) --------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, devices):
        self.devices = devices
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", ",".join(str(d) for d in self.devices), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        rows = []
        with open(self.path) as f:
            for line in f:
                p = [x.strip() for x in line.split(",")]
                if len(p) >= 9:
                    rows.append(p)
        os.unlink(self.path)
        if not rows:
            return None

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[1]) for r in rows if num(r[1]) is not None]
        smax = [num(r[2]) for r in rows if num(r[2]) is not None]
        power = [num(r[3]) for r in rows if num(r[3]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        # under load: samples drawing more than idle power
        loaded = [s for s, pw in zip(sm, power) if pw is not None and pw > 0.25 * max(power)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(rows), "power_w_max": max(power) if power else None}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def smem_peak_gbs(sm_mhz):
    """Shared-memory bandwidth: 148 SMs x 128 B/clk at the given SM clock."""
    return 148 * 128 * sm_mhz * 1e6 / 1e9


def roofline(st, info, sm_mhz, world=1):
    """Roofline of the persistent search kernel (k_search) from one search's
    stats, on the LOWERED records' byte model (pccp_lowering_info): a round
    reads store_bytes_per_round of the store (shared memory) and
    table_bytes_per_round of the tables (shared memory when table_in_smem,
    else L2).  achieved = search rounds x bytes per round / k_search time.

    Also reported, not used for `frac`: the per-reference-command model of
    SURVEY 8(d) (alg_bytes_per_eval x evals), which counts a word once per
    reference command reading it — a fused record reads it once for several
    commands, so that ratio can pass 1 (`per_command_model_ratio`)."""
    ks = st["kernel_ms"] / 1e3
    if ks <= 0:
        return None
    rounds = st["search_evals"] / max(info["n_cmds"], 1)
    tis = bool(info["table_in_smem"])
    bpr = info["store_bytes_per_round"] + (info["table_bytes_per_round"] if tis else 0.0)
    achieved = rounds * bpr / ks / 1e9 / world
    peak = smem_peak_gbs(sm_mhz)
    d = {"bound": "smem", "kernel": "k_search", "achieved": achieved, "peak": peak, "unit": "GB/s",
         "frac": achieved / peak, "bytes_per_round": bpr, "store_bytes_per_round": info["store_bytes_per_round"],
         "table_bytes_per_round": info["table_bytes_per_round"], "table_in_smem": tis,
         "search_rounds": rounds, "kernel_ms": st["kernel_ms"],
         "evals_per_s": st["search_evals"] / ks / world,
         "per_command_model_ratio": st["search_evals"] * info["alg_bytes_per_eval"] / ks / 1e9 / world / peak,
         "peak_source": f"148 SMs x 128 B/clk x {sm_mhz:.0f} MHz"}
    if not tis:
        d["l2_table_gbs"] = rounds * info["table_bytes_per_round"] / ks / 1e9 / world
    return d


def ncu_kernel(workload):
    """The committed ncu --set full summary of k_search for a workload (profiles/)."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            return json.load(f)[workload]["k_search"]
    except Exception:
        return None


# ---- CPU reference -----------------------------------------------------------------
def cpu_reference(w, budget_s, threads):
    """The reference path on host cores: refh_enumerate over oracle/_ref."""
    from oracle import refh
    if refh.available():
        m = ref_model(w)
        r = m.enumerate(depth_cap=w["depth"], threads=threads, budget_s=budget_s)
        secs = r["elapsed_ms"] / 1e3
        return dict(value=r["nodes"] / secs, nodes=r["nodes"], seconds=secs, cores=threads, kind="reference",
                    sample=f"{budget_s:g} s of the {w['workload']} DFS (reference run_sequential/branch/materialize "
                           f"from oracle/_ref, harness enumerator oracle/ref_harness.cpp) over a BFS frontier of "
                           f"{8 * threads} subtrees on {threads} threads")
    # fallback: the plain-C restatement, one thread, bounded by nodes
    from oracle.port import Oracle
    m = build_model(w)
    o = Oracle(m.tables())
    t = time.perf_counter()
    r = o.enumerate(m.bottom(), w["depth"], node_budget=200000)
    secs = time.perf_counter() - t
    return dict(value=r["nodes"] / secs, nodes=r["nodes"], seconds=secs, cores=1, kind="port",
                sample=f"first {r['nodes']} nodes of the {w['workload']} DFS on the C oracle port (1 thread)")


TTO_SEEDS = (1, 2, 5, 7, 9, 11)  # SURVEY 8(d) config 4 parity seeds
TTO_OPTIMA = {1: 84, 2: 77, 5: 73, 7: 60, 9: 61, 11: 99}


def time_to_optimum(local, rank, world, dist):
    """Config 4 (RCPSP 30x4): optimum, time to the first optimal incumbent and
    time to the proof on the GPU(s) (at N = 1 the median of three solves, all
    three listed).  With N > 1 the incumbent is shared
    through CUDA IPC + system-scope atomicMin (paper_2207_12116_b200/distributed.py)."""
    from paper_2207_12116_b200 import Engine, Model
    from paper_2207_12116_b200.distributed import attach_incumbents, run_solve
    eng = Engine(local, shard_index=rank, shard_count=world)
    ref = Engine(local, mix_order=-1) if world == 1 else None  # the reference's order alone, for comparison
    attached = False
    out = {}
    for seed in TTO_SEEDS:
        m = Model.rcpsp_random(seed, 30, 4)
        eng.load(m)
        if world > 1 and not attached:
            attach_incumbents(eng)
            attached = True
        if world > 1:
            dist.barrier()
            res = run_solve(eng, timeout_s=120, check=m.check_solution)
            status, obj, ok = res["status"], res["objective"], res.get("checked")
            local_r = res["local"]
        else:
            # three solves: the search order (and so the node count) depends on
            # incumbent timing; the median run by time to proof is reported
            runs = [eng.solve(timeout_s=120) for _ in range(3)]
            assert len({(x.status, x.objective) for x in runs}) == 1, [(x.status, x.objective) for x in runs]
            runs.sort(key=lambda x: x.stats["device_ms"])
            r = runs[1]
            status, obj = r.status, r.objective
            ok = all(x.best_words is not None and m.check_solution(x.best_words) for x in runs)
            local_r = r
        t_first = min((ms for v, ms in local_r.improvements if v == obj), default=float("inf"))
        t_proof = local_r.stats["device_ms"]
        if world > 1:
            t_first = min(x for x in _gather_obj(dist, t_first))
            t_proof = max(_gather_obj(dist, t_proof))
        st = local_r.stats
        sm_mhz = load_peaks().get("sm_max_mhz", 1965.0)
        out[str(seed)] = {"status": status, "objective": obj, "valid": bool(ok),
                          "matches_reference": obj == TTO_OPTIMA[seed], "t_first_optimal_ms": t_first,
                          "t_proof_ms": t_proof, "t_wall_ms": local_r.stats["elapsed_ms"],
                          "nodes": local_r.stats["nodes"],
                          "tree_nodes": local_r.stats["nodes"] - local_r.stats["rematerialised"],
                          "roofline": roofline(st, eng.lowering_info(), sm_mhz)}
        if world == 1:
            out[str(seed)]["t_proof_ms_runs"] = [x.stats["device_ms"] for x in runs]
        if ref is not None:
            rr = ref.load(m).solve(timeout_s=120)
            out[str(seed)]["reference_order"] = {
                "status": rr.status, "objective": rr.objective, "t_proof_ms": rr.stats["device_ms"],
                "t_first_optimal_ms": min((ms for v, ms in rr.improvements if v == rr.objective), default=None),
                "nodes": rr.stats["nodes"]}
    eng.close()
    if ref is not None:
        ref.close()
    return {"config": "rcpsp 30 tasks x 4 resources, random_patterson(mt19937_64(seed)), minimise makespan",
            "note": "node counts differ from the CPU only through search order and incumbent timing; the "
                    "default search mixes branching orders (every 48th group branches by smallest lb, LST "
                    "ties: cfg mix_order), 'reference_order' is the same solve in branch()'s order alone",
            "gpu": out}


STRETCH_SEEDS = (3, 4, 6, 8, 10, 12)  # unproven by the reference at 60 s (1 core) / 120 s (8 cores)
STRETCH_CPU_BEST = {3: 62, 4: 74, 6: 71, 8: 73, 10: 91, 12: 112}  # best reference incumbents (W=1 60 s, W=8 120 s)


def _solve_on_ranks(eng, m, world, dist, timeout_s):
    from paper_2207_12116_b200.distributed import run_solve
    if world > 1:
        dist.barrier()
        res = run_solve(eng, timeout_s=timeout_s, check=m.check_solution)
        return res["status"], res["objective"], res.get("checked"), res["local"]
    r = eng.solve(timeout_s=timeout_s)
    ok = r.best_words is not None and m.check_solution(r.best_words)
    return r.status, r.objective, ok, r


def stretch_and_large(local, rank, world, dist, timeout_s, large_timeout_s):
    """Configs 4 (stretch seeds) and 5 (RCPSP 120x4) with the primal phase
    (smallest-lb dives, LST tie-break, stall restarts; include/pccp_gpu.h
    primal_ms) ahead of the reference-order exact search."""
    from paper_2207_12116_b200 import Engine, Model
    from paper_2207_12116_b200.distributed import attach_incumbents
    eng = Engine(local, shard_index=rank, shard_count=world, primal_ms=int(timeout_s * 1e3))
    if world > 1:
        attach_incumbents(eng)
    out = {}
    for seed in STRETCH_SEEDS:
        m = Model.rcpsp_random(seed, 30, 4)
        eng.load(m)
        status, obj, ok, r = _solve_on_ranks(eng, m, world, dist, timeout_s)
        t_best = min((ms for v, ms in r.improvements if v == obj), default=None)
        out[str(seed)] = {"status": status, "objective": obj, "valid": bool(ok), "t_best_ms": t_best,
                          "t_end_ms": r.stats["device_ms"], "nodes": r.stats["nodes"],
                          "cpu_reference_best": STRETCH_CPU_BEST[seed]}
    eng.close()
    stretch = {"config": "rcpsp 30x4 stretch seeds (unproven by the reference CPU solver)",
               "timeout_s": timeout_s, "gpu": out}

    large = rcpsp120(local, rank, world, dist, large_timeout_s)
    return stretch, large


def destructive_lower_bound(eng, m, lo, hi):
    """The smallest makespan T in [lo, hi) whose root fixed point under
    `makespan <= T` does not fail: every T below it is refuted by propagation
    alone, so it is a lower bound on the optimum (the classic destructive
    bound).  All candidate T go through one pccp_gpu_propagate_batch."""
    import numpy as np
    if hi <= lo:
        return lo
    t = m.tables()
    ub_word = int(t.slot_word[m.starts()[-1]]) + 1
    ts = np.arange(lo, hi, dtype=np.int64)
    stores = np.repeat(m.bottom()[None, :], len(ts), axis=0)
    stores[:, ub_word] = np.minimum(stores[:, ub_word], ts)
    _, failed, _ = eng.propagate_batch(stores)
    ok = np.nonzero(~failed)[0]
    return int(ts[ok[0]]) if ok.size else int(hi)


def rcpsp120(local, rank, world, dist, budget_s):
    """Config 5: RCPSP 120x4 seed 1.  (1) The reference's branching order alone
    (branch(), solver.cpp:19-47; no incumbent is found in that order) for a few
    seconds: nodes/s and the k_search roofline.  (2) The solve with the primal
    phase for `budget_s`: the incumbent over time (every improvement) and the
    gap to the best lower bound (root critical path; destructive bound)."""
    from paper_2207_12116_b200 import Engine, Model
    from paper_2207_12116_b200.distributed import attach_incumbents
    m = Model.rcpsp_random(1, 120, 4)
    sm = load_peaks().get("sm_max_mhz", 1965.0)
    # the reference's order alone: no mixed orders (cfg mix_order -1)
    with Engine(local, shard_index=rank, shard_count=world, mix_order=-1) as e0:  # unlinked: nothing to share
        e0.load(m)
        r0 = e0.solve(timeout_s=3.0)
        ref_order = {"status": r0.status, "nodes": r0.stats["nodes"], "device_ms": r0.stats["device_ms"],
                     "nodes_per_s": r0.stats["nodes"] / (r0.stats["device_ms"] / 1e3),
                     "rounds": "filtered (kPackedF, the default for this model)"}
        if world > 1:
            ref_order["nodes_per_s_all_ranks"] = sum(_gather_obj(dist, ref_order["nodes_per_s"]))
    # the same search in eventless rounds (every record every round): the
    # roofline's byte model describes this loop; filtered rounds do less work
    # per node, not the same work faster
    os.environ["PCCP_PACKED_FILTER"] = "0"
    try:
        with Engine(local, shard_index=rank, shard_count=world, mix_order=-1) as e1:
            e1.load(m)
            r1 = e1.solve(timeout_s=3.0)
            ref_order["eventless"] = {"nodes": r1.stats["nodes"], "device_ms": r1.stats["device_ms"],
                                      "nodes_per_s": r1.stats["nodes"] / (r1.stats["device_ms"] / 1e3),
                                      "roofline": roofline(r1.stats, e1.lowering_info(), sm)}
    finally:
        del os.environ["PCCP_PACKED_FILTER"]
    eng = Engine(local, shard_index=rank, shard_count=world, primal_ms=int(budget_s * 1e3))
    eng.load(m)
    if world > 1:
        attach_incumbents(eng)
    failed, root, _ = eng.run_sequential()
    sink = int(m.tables().slot_word[m.starts()[-1]])
    status, obj, ok, r = _solve_on_ranks(eng, m, world, dist, budget_s)
    first = r.improvements[0] if r.improvements else (None, None)
    t_best = min((ms for v, ms in r.improvements if v == obj), default=None)
    if world > 1:
        t_best = min(x for x in _gather_obj(dist, t_best if t_best is not None else float("inf")))
    lb_root = int(root[sink])
    lb = destructive_lower_bound(eng, m, lb_root, obj if obj is not None else lb_root + 64)
    eng.close()
    return {"config": "rcpsp 120x4 seed 1 (random_patterson(mt19937_64(1), 120, 4)), minimise makespan",
            "timeout_s": budget_s, "status": status, "objective": obj, "valid": bool(ok),
            "lower_bound": {"root_critical_path": lb_root, "destructive": lb},
            "gap": None if obj is None else (obj - lb) / obj,
            "first": {"objective": first[0], "t_ms": first[1]}, "t_best_ms": t_best,
            "incumbent_over_time": [[v, ms] for v, ms in r.improvements],
            "nodes": r.stats["nodes"], "nodes_per_s": r.stats["nodes"] / (r.stats["device_ms"] / 1e3),
            "primal": r.primal, "reference_order": ref_order,
            "note": "the reference's branching order reaches no leaf (SURVEY 8d); the primal phase's incumbents "
                    "are ordinary solutions of the same model, checked by check_solution"}


def cpu_large(threads, budget_s):
    """The reference solve_parallel on RCPSP 120x4 seed 1 for a bounded budget."""
    from oracle import refh
    if not refh.available():
        return None
    r = refh.RefModel.rcpsp(1, 120, 4).solve_parallel(workers=threads, timeout_s=budget_s)
    return {"status": ["OPTIMAL", "SAT", "UNSAT", "UNKNOWN"][r["status"]], "objective": r["objective"],
            "t_ms": r["elapsed_ms"], "nodes": r["nodes"], "nodes_per_s": r["nodes"] / max(r["elapsed_ms"], 1) * 1e3,
            "workers": threads}


def enumeration_configs(local, rank, world, dist, cpu, threads):
    """Configs 1 and 3 beside the headline: N-Queens 8 and the random linear CSP
    (seed 1, depth cap 22), full trees, counts and hash-sums checked against the
    reference's; the reference itself on the host for comparison."""
    from paper_2207_12116_b200 import Engine
    from paper_2207_12116_b200.distributed import combine_enum, _gather
    cases = [("nqueens8-all-solutions", dict(n=8, depth=-1),
              dict(nodes=779, failures=298, solutions=92, hash_sum=0xF1DF80A1FF36FBF6)),
             ("random-linear-csp-seed1-depth22", WORKLOADS["csp"], WORKLOADS["csp"]["expect"])]
    out = {}
    for name, w, exp in cases:
        m = build_model(w)
        with Engine(local, shard_index=rank, shard_count=world) as eng:
            eng.load(m)
            info = eng.lowering_info()
            for _ in range(3):
                r = eng.enumerate(depth_cap=w["depth"])
            runs = []
            for _ in range(5):
                runs.append(eng.enumerate(depth_cap=w["depth"]))
        with Engine(local, shard_index=rank, shard_count=world, hash=True) as heng:
            hr = heng.load(m).enumerate(depth_cap=w["depth"])
        if world > 1:
            hr = combine_enum(_gather(hr))
            ms = [max(_gather(r["device_ms"])) for r in runs]
            nodes = combine_enum(_gather(runs[-1]))["nodes"]
        else:
            ms = [r["device_ms"] for r in runs]
            nodes = runs[-1]["nodes"]
        d = {"nodes": nodes, "device_ms": statistics.median(ms), "nodes_per_s": nodes / (statistics.median(ms) / 1e3),
             "parity": all(int(hr[k]) == v for k, v in exp.items())}
        if world == 1:
            r = runs[-1]
            d["decompose_ms"] = r["decompose_ms"]
            d["roofline"] = roofline(r, info, load_peaks().get("sm_max_mhz", 1965.0))
        if cpu:
            c = cpu_reference(dict(w, workload=name), 3.0, threads)
            d["cpu_reference"] = {"nodes_per_s": c["value"], "threads": c["cores"], "kind": c["kind"],
                                  "sample": f"{c['seconds']:.2f} s"}
        out[name] = d
    return out


def _gather_obj(dist, v):
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, v)
    return out


def host_cpu():
    """nproc, the lscpu model and clocks of this host."""
    info = {"threads": os.cpu_count() or 1}
    try:
        txt = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in txt.splitlines():
            k, _, v = line.partition(":")
            k, v = k.strip(), v.strip()
            if k == "Model name":
                info["model"] = v
            elif k in ("CPU max MHz", "CPU MHz", "Socket(s)", "Core(s) per socket", "Thread(s) per core"):
                info[k.lower().replace("(s)", "s").replace(" ", "_")] = v
    except Exception:
        pass
    return info


def cpu_time_to_optimum(threads, timeout_s=90.0):
    """The reference solve_parallel (oracle/_ref: the reference library compiled
    from its sources) on all six parity seeds, with W = 1 and W = host threads
    (solver.cpp:229-283, EngineConfig Seq, eps_factor 8 — the call of
    `pccp solve`, tools/pccp.cpp:61-62), timed in this run.  The six W = 1
    solves run at the same time, one host thread each (ctypes releases the
    GIL; each is single-threaded), the W = nproc solves one after the other."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import refh
    if not refh.available():
        return None

    def one(seed, workers):
        r = refh.RefModel.rcpsp(seed, 30, 4).solve_parallel(workers=workers, timeout_s=timeout_s)
        return {"status": ["OPTIMAL", "SAT", "UNSAT", "UNKNOWN"][r["status"]], "objective": r["objective"],
                "t_proof_ms": r["elapsed_ms"] if r["status"] == 0 else None, "t_ms": r["elapsed_ms"],
                "nodes": r["nodes"], "workers": workers}
    concurrent = min(len(TTO_SEEDS), max(1, threads // 2))
    with ThreadPoolExecutor(concurrent) as ex:
        w1 = list(ex.map(lambda sd: one(sd, 1), TTO_SEEDS))
    wn = [one(sd, threads) for sd in TTO_SEEDS]
    return {"timeout_s": timeout_s, "w1_concurrent_solves": concurrent, "host": host_cpu(),
            "seeds": {str(sd): {"w1": a, "wN": b} for sd, a, b in zip(TTO_SEEDS, w1, wn)}}


def run_reference_arm(a, w):
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    try:
        from oracle import refh
        if not refh.available():
            raise FileNotFoundError("oracle/_ref/libpccp_ref.so is not built")
    except Exception as e:  # the C port is still the reference's algorithm, say so
        print(json.dumps({"impl": "reference", "unavailable": f"reference library missing ({e})"}))
        return 0
    for _ in range(a.warmup):
        cpu_reference(w, min(2.0, a.ref_budget), threads)
    nodes, secs = 0, 0.0
    last = None
    for _ in range(a.steps):
        last = cpu_reference(w, a.ref_budget, threads)
        nodes += last["nodes"]
        secs += last["seconds"]
    value = nodes / secs
    line = {
        "impl": "reference", "metric": "search nodes/sec", "value": value, "unit": "nodes/s",
        "n_gpus": 0, "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * secs / a.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": w["workload"], "parallelism": f"cpu-threads{threads}"},
        "cpu_baseline": {"value": value, "unit": "nodes/s", "cores": threads, "kind": last["kind"],
                         "sample": last["sample"]},
        "e2e": {"value": value, "unit": "nodes/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ---- our arm -------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="q14", choices=sorted(WORKLOADS))
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--ref-budget", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-tto", action="store_true", help="skip the RCPSP time-to-optimum sections")
    ap.add_argument("--stretch-timeout", type=float, default=10.0)
    ap.add_argument("--large-timeout", type=float, default=20.0)
    ap.add_argument("--cpu-tto-timeout", type=float, default=60.0,
                    help="budget of each reference solve_parallel in the time-to-optimum comparison")
    a = ap.parse_args()
    w = WORKLOADS[a.config]
    if a.impl == "reference":
        return run_reference_arm(a, w)

    import torch
    import torch.distributed as dist

    from paper_2207_12116_b200 import Engine

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    if world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world}")
    # PCCP_BENCH_SHARE_DEVICE=1 (tests only): every rank on cuda:0 over gloo, to
    # exercise the N>1 path (sharding, IPC incumbents, max-over-ranks) on a 1-GPU box
    shared = os.environ.get("PCCP_BENCH_SHARE_DEVICE") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def allreduce(vals, op):
        if world == 1:
            return vals
        t = torch.tensor(vals, dtype=torch.float64, device="cpu" if shared else f"cuda:{local}")
        dist.all_reduce(t, op=op)
        return t.tolist()

    model = build_model(w)
    tables = model.tables()
    eng = Engine(local, shard_index=rank, shard_count=world)
    if world > 1:  # linked shards: the share cells (work stealing) and the incumbent, over IPC
        from paper_2207_12116_b200.distributed import attach_incumbents
        attach_incumbents(eng)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=f"cuda:{local}")

    def step():
        flush.zero_()  # L2 flush between steps (outside the step's own events)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.load(tables)
        r = eng.enumerate(depth_cap=w["depth"])
        return r, time.perf_counter() - t0

    for _ in range(max(a.warmup, 0)):
        step()
    eng.load(tables)
    info = eng.lowering_info()

    sampler = ClockSampler([local]) if rank == 0 else None
    barrier()
    if sampler:
        sampler.start()
        time.sleep(0.3)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    per_step = []
    t_region = time.perf_counter()
    for _ in range(a.steps):
        per_step.append(step())
    barrier()
    ev1.record()
    torch.cuda.synchronize()
    region_ms = ev0.elapsed_time(ev1)
    region_wall = time.perf_counter() - t_region
    clocks = sampler.stop() if sampler else None

    nodes = [float(r["nodes"]) for r, _ in per_step]
    dev_ms = [r["device_ms"] for r, _ in per_step]
    e2e_s = [s for _, s in per_step]
    kern_ms = [r["kernel_ms"] for r, _ in per_step]
    sevals = [float(r["search_evals"]) for r, _ in per_step]
    launches = sum(r["launches"] for r, _ in per_step)
    # whole job: nodes summed over ranks, time = max over ranks, per step
    nodes_all = allreduce(nodes, dist.ReduceOp.SUM if world > 1 else None)
    dev_max = allreduce(dev_ms, dist.ReduceOp.MAX if world > 1 else None)
    e2e_max = allreduce(e2e_s, dist.ReduceOp.MAX if world > 1 else None)
    kern_max = allreduce(kern_ms, dist.ReduceOp.MAX if world > 1 else None)
    sevals_all = allreduce(sevals, dist.ReduceOp.SUM if world > 1 else None)
    launches_all = allreduce([float(launches)], dist.ReduceOp.SUM if world > 1 else None)[0]
    r0 = per_step[-1][0]
    h2d = tables.nbytes() + r0["h2d_bytes"]
    d2h = r0["d2h_bytes"]

    # parity on the full workload (every step) and one hashed verification run
    exp = w["expect"]
    counts = {k: int(allreduce([float(r0[k])], dist.ReduceOp.SUM if world > 1 else None)[0])
              for k in ("nodes", "failures", "solutions", "open_leaves")}
    parity = {k: counts[k] == exp[k] for k in counts if k in exp}
    if "hash_sum" in exp:
        heng = Engine(local, shard_index=rank, shard_count=world, hash=True)
        if world > 1:
            attach_incumbents(heng)
        hr = heng.load(tables).enumerate(depth_cap=w["depth"])
        hs = int(hr["hash_sum"])
        if world > 1:
            hl = [None] * world
            dist.all_gather_object(hl, hs)
            hs = sum(hl) % 2**64
        parity["hash_sum"] = hs == exp["hash_sum"]
        heng.close()

    tto = None if a.no_tto else time_to_optimum(local, rank, world, dist)
    others = None if a.no_tto else enumeration_configs(local, rank, world, dist,
                                                       world == 1 and not a.no_cpu_baseline, os.cpu_count() or 1)
    stretch, large = (None, None) if a.no_tto else stretch_and_large(local, rank, world, dist, a.stretch_timeout,
                                                                     a.large_timeout)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    total_nodes = sum(nodes_all)
    total_dev_s = sum(dev_max) / 1e3
    value = total_nodes / total_dev_s
    e2e_value = total_nodes / sum(e2e_max)
    peaks = load_peaks()
    sm_mhz = (clocks or {}).get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
    # roofline of k_search over the timed steps (lowered-record byte model)
    rl_steps = [roofline({"kernel_ms": km, "search_evals": se, "n_cmds": info["n_cmds"]}, info, sm_mhz, world)
                for se, km in zip(sevals_all, kern_max)]
    rl = dict(rl_steps[-1])
    for k in ("achieved", "frac", "evals_per_s", "per_command_model_ratio", "kernel_ms", "search_rounds"):
        rl[k] = statistics.mean(x[k] for x in rl_steps)
    nk = ncu_kernel(w["workload"])
    ncu = None
    if nk:  # the committed capture of this build, on its own (cold-cache, serialised) launch time
        t = nk["duration_ms"] / 1e3
        clk = nk.get("sm_clock_mhz", sm_mhz)
        ncu = {"source": nk["source"], "duration_ms": nk["duration_ms"], "sm_clock_mhz": clk,
               "smem_wavefront_frac": nk["smem_wavefronts"] * 128 / t / 1e9 / smem_peak_gbs(clk),
               "issue_frac": nk["warp_instructions"] / t / (148 * 4 * clk * 1e6),
               "issue_active_pct": nk.get("issue_active_pct"),
               "bank_conflict_share": nk.get("smem_bank_conflicts", 0) / max(nk.get("smem_wavefronts", 1), 1),
               "l2_bytes_per_launch": nk.get("l2_bytes_per_launch"),
               "note": "measured by ncu on the same command line and build, not in this run: wavefronts include "
                       "bank conflicts and partial-warp accesses, so the physical fraction exceeds the byte model's"}
    rl["traffic"] = nk["dram_bytes_per_launch"] if nk else None
    rl["traffic_source"] = nk["source"] if nk else None
    rl["hbm_peak_gbs"] = peaks.get("hbm_gbs")
    rl["ncu"] = ncu
    line = {
        "metric": "search nodes/sec", "value": value, "unit": "nodes/s", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": 1e3 * total_dev_s / a.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": w["workload"], "commands": tables.n_cmds, "words": tables.n_words,
                   "parallelism": f"eps-shard{world}", "l2": "flushed between steps (256 MiB write)",
                   "group_threads": info["group_threads"], "groups_per_cta": info["groups_per_cta"],
                   "ctas": info["ctas"], "table_in_smem": bool(info["table_in_smem"])},
        "e2e": {"value": e2e_value, "unit": "nodes/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "note": "pccp_gpu_load (table upload; the context keeps the lowering of an identical model)  + pccp_gpu_enumerate from host buffers, host clock"},
        "gpu_launches": int(launches_all),
        "roofline": rl,
        "parity": {"exact": all(parity.values()), **parity},
        "region_ms": region_ms, "region_wall_s": region_wall,
        "kernel_ms_per_step": statistics.mean(kern_max),
    }
    if clocks:
        line["clocks"] = clocks
    if world == 1 and not a.no_cpu_baseline:
        cb = cpu_reference(w, a.cpu_budget, os.cpu_count() or 1)
        line["cpu_baseline"] = {"value": cb["value"], "unit": "nodes/s", "cores": cb["cores"], "kind": cb["kind"],
                                "sample": cb["sample"]}
    if tto is not None:
        if world == 1 and not a.no_cpu_baseline:
            tto["cpu_reference"] = cpu_time_to_optimum(os.cpu_count() or 1, a.cpu_tto_timeout)
        line["time_to_optimum"] = tto
    if others is not None:
        line["other_configs"] = others
    if stretch is not None:
        line["stretch"] = stretch
        if world == 1 and not a.no_cpu_baseline:
            large["cpu_reference"] = cpu_large(os.cpu_count() or 1, min(a.large_timeout, 30.0))
        line["rcpsp120"] = large
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
