"""Multi-GPU driver: one process per GPU, the EPS frontier sharded i mod N.

Enumeration (configs 1-3) has no data-path exchange: every rank computes the
same deterministic frontier, drains its own shard (and, with peers attached,
steals positions of the peers' shards nobody has reached), and the counters
are combined once at the end (sums; the hash-sum mod 2^64).  Minimisation
(configs 4-5) shares one int32: each rank exports the IPC handle of its
control cells, attaches every peer's, and improving solutions are pushed with
system-scope atomicMin over NVLink from inside the search kernel.

Collectives here go through torch.distributed (NCCL on the GPU box, gloo in
the CPU tests); they run once per call, never per node.
"""
from __future__ import annotations

from typing import Callable

import numpy as np

U64 = 2**64


def shard_indices(n_frontier: int, index: int, count: int) -> range:
    """Frontier positions owned by shard `index` (the k_search work queue maps
    its k-th pop to index + k*count)."""
    if not 0 <= index < max(count, 1):
        raise ValueError("shard index out of range")
    return range(index, n_frontier, max(count, 1))


SUM_KEYS = ("nodes", "failures", "solutions", "open_leaves", "rounds", "evals", "search_evals", "launches",
            "h2d_bytes", "d2h_bytes")


def combine_enum(results: list[dict]) -> dict:
    """Whole-job enumeration result from per-rank results (rank 0 first)."""
    out = {k: sum(int(r.get(k, 0)) for r in results) for k in SUM_KEYS}
    out["hash_sum"] = sum(int(r.get("hash_sum", 0)) for r in results) % U64
    out["exhausted"] = all(bool(r.get("exhausted", True)) for r in results)
    out["subproblems"] = int(results[0].get("subproblems", 0)) if results else 0
    out["max_depth"] = max((int(r.get("max_depth", 0)) for r in results), default=0)
    for k in ("device_ms", "kernel_ms", "decompose_ms", "elapsed_ms"):
        out[k] = max((float(r.get(k, 0.0)) for r in results), default=0.0)  # ranks run concurrently
    return out


def combine_solve(results: list[dict]) -> dict:
    """finish() (solver.cpp:148-162) over the union of the shards: a proof needs
    every shard exhausted — the shards partition one bound-free EPS frontier
    (engine.cu run_search) — or one rank's primal dive exhausted the WHOLE tree
    (`proved`); the objective is the minimum over ranks."""
    exhausted = all(r["exhausted"] for r in results) or any(r.get("proved", False) for r in results)
    objs = [r["objective"] for r in results if r["objective"] is not None]
    obj = min(objs) if objs else None
    if obj is not None:
        status = "OPTIMAL" if exhausted else "SAT"
    else:
        status = "UNSAT" if exhausted else "UNKNOWN"
    owner = None
    for i, r in enumerate(results):
        if r["objective"] == obj and r.get("has_store"):
            owner = i
            break
    return {"status": status, "objective": obj, "owner": owner, "exhausted": exhausted,
            "nodes": sum(int(r["nodes"]) for r in results), "solutions": sum(int(r["solutions"]) for r in results)}


def _gather(obj, group=None):
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, obj, group=group)
    return out


def run_enumerate(engine, depth_cap: int = -1, root=None, group=None) -> dict:
    """Enumerate this rank's shard (engine built with shard_index=rank,
    shard_count=world) and return the combined whole-job result on every rank."""
    local = engine.enumerate(root=root, depth_cap=depth_cap)
    return combine_enum(_gather(local, group))


def attach_incumbents(engine, group=None) -> None:
    """Exchange the IPC handles of every rank's control cells (incumbent, done
    flag, share cell) in rank order and attach every peer: minimisation shares
    the incumbent, and any sharded search steals untouched frontier positions
    from the peers' shares (engine.cu run_search)."""
    import torch.distributed as dist
    handles = _gather(engine.incumbent_handle(), group)
    engine.attach_peers(handles, dist.get_rank(group))


def run_solve(engine, timeout_s: float = 0.0, root=None, group=None,
              check: Callable[[np.ndarray], bool] | None = None) -> dict:
    """Branch and bound over this rank's shard with the shared incumbent; returns
    the combined result (and the best store, gathered from its owner) on every rank."""
    import torch.distributed as dist
    # every rank resets its cross-rank cells before any rank starts: a peer's
    # push must not be wiped by a late reset (include/pccp_gpu.h)
    engine.reset_shared()
    dist.barrier(group)
    r = engine.solve(root=root, timeout_s=timeout_s)
    local = {"objective": r.objective, "exhausted": r.status in ("OPTIMAL", "UNSAT"),
             "proved": bool(getattr(r, "primal_proved", False)),
             "nodes": r.stats["nodes"], "solutions": r.stats["solutions"], "has_store": r.best_words is not None}
    res = combine_solve(_gather(local, group))
    stores = _gather(r.best_words.tolist() if r.best_words is not None else None, group)
    best = stores[res["owner"]] if res["owner"] is not None else None
    res["best_words"] = None if best is None else np.asarray(best, np.int32)
    if check is not None and res["best_words"] is not None:
        res["checked"] = bool(check(res["best_words"]))
    res["local"] = r  # this rank's SolveResult (improvement log, device timings)
    return res
