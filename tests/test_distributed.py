"""Multi-rank host logic on CPU: world_size 2 over gloo (the GPU box runs the
same code over NCCL).  The device search is replaced by a fake engine with a
known per-shard answer; the frontier partition itself is checked against a
CPU restatement of the EPS sharding."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2207_12116_b200.distributed import (combine_enum, combine_solve, run_enumerate, run_solve,
                                               shard_indices)


class FakeEnumEngine:
    def __init__(self, rank):
        self.rank = rank

    def enumerate(self, root=None, depth_cap=-1):
        # shard k holds 100+k nodes, hashes near 2^64 so the sum wraps
        return {"nodes": 100 + self.rank, "failures": 10, "solutions": 3 + self.rank, "open_leaves": 0,
                "hash_sum": 2**64 - 5 + self.rank, "exhausted": True, "rounds": 7, "evals": 70,
                "device_ms": 1.0 + self.rank, "subproblems": 64}


class FakeSolveEngine:
    def __init__(self, rank, objective, exhausted, proved=False):
        self.rank, self.objective, self.exhausted, self.proved = rank, objective, exhausted, proved
        self.resets = 0

    def reset_shared(self):
        self.resets += 1

    def solve(self, root=None, timeout_s=0.0):
        import numpy as np

        class R:
            pass
        r = R()
        r.objective = self.objective
        r.status = ("OPTIMAL" if self.objective is not None else "UNSAT") if self.exhausted else (
            "SAT" if self.objective is not None else "UNKNOWN")
        r.stats = {"nodes": 1000, "solutions": 1 if self.objective is not None else 0}
        r.best_words = None if self.objective is None else np.full(4, self.objective, np.int32)
        r.primal_proved = self.proved
        return r


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        e = run_enumerate(FakeEnumEngine(rank))
        s1 = run_solve(FakeSolveEngine(rank, [57, 55][rank], True))
        s2 = run_solve(FakeSolveEngine(rank, [None, 61][rank], [True, False][rank]))
        s3 = run_solve(FakeSolveEngine(rank, None, True))
        # rank 1's primal dive exhausted the whole tree; rank 0 was told to stop (unfinished)
        f4 = FakeSolveEngine(rank, [70, 64][rank], False, proved=rank == 1)
        s4 = run_solve(f4)
        q.put((rank, e, s1["status"], s1["objective"], int(s1["best_words"][0]), s2["status"], s2["objective"],
               s3["status"], s4["status"], s4["objective"], f4.resets))
    finally:
        dist.destroy_process_group()


def test_two_rank_combination_over_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, e, st1, ob1, bw, st2, ob2, st3, st4, ob4, resets in out:
        assert e["nodes"] == 201 and e["solutions"] == 7 and e["failures"] == 20
        assert e["hash_sum"] == (2 * 2**64 - 9) % 2**64
        assert e["exhausted"] and e["device_ms"] == 2.0
        assert (st1, ob1, bw) == ("OPTIMAL", 55, 55)   # min over ranks, store from the owner
        assert (st2, ob2) == ("SAT", 61)               # one shard unfinished: no proof
        assert st3 == "UNSAT"
        assert (st4, ob4, resets) == ("OPTIMAL", 64, 1)  # a whole-tree primal proof is the job's proof


def test_shards_partition_the_frontier():
    for n in (0, 1, 7, 64, 1000):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                seen.extend(shard_indices(n, r, world))
            assert sorted(seen) == list(range(n))
    with pytest.raises(ValueError):
        shard_indices(10, 2, 2)


def test_combine_rules():
    assert combine_solve([{"objective": None, "exhausted": False, "nodes": 1, "solutions": 0}])["status"] == "UNKNOWN"
    two = [{"objective": 9, "exhausted": True, "nodes": 1, "solutions": 1},
           {"objective": 8, "exhausted": False, "nodes": 1, "solutions": 1}]
    assert combine_solve(two)["status"] == "SAT"
    two[0]["proved"] = True
    assert combine_solve(two)["status"] == "OPTIMAL" and combine_solve(two)["objective"] == 8
    r = combine_enum([{"nodes": 5, "hash_sum": 2**64 - 1, "exhausted": True},
                      {"nodes": 6, "hash_sum": 2, "exhausted": False}])
    assert r["nodes"] == 11 and r["hash_sum"] == 1 and not r["exhausted"]
