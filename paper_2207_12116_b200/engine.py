"""Engine: the device search entry points (include/pccp_gpu.h) from Python.

Each method mirrors a reference entry point:
    propagate_batch / run_sequential  ->  run_sequential   (engine.cpp:13-32)
    replay                            ->  materialize      (solver.cpp:91-102)
    enumerate                         ->  dfs order of solver.cpp:122-146, all solutions
    solve                             ->  solve_parallel   (solver.cpp:229-283)
There is no CPU fallback: without a B200 and the built library, Engine() raises.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .model import INT32_MAX, Model, Tables


def _vp(a):
    return a.ctypes.data_as(C.c_void_p)


def _stats(s: N.PccpStats) -> dict:
    return {k: getattr(s, k) for k, _ in N.PccpStats._fields_}


@dataclass
class SolveResult:
    status: str
    objective: int | None
    stats: dict
    best_words: np.ndarray | None
    improvements: list = field(default_factory=list)  # (objective, ms since search start)
    best_on_peer: bool = False
    primal: dict | None = None  # {nodes, device_ms, proved} when a primal phase ran (cfg primal_ms)
    primal_proved: bool = False  # a primal dive exhausted the whole tree: a proof for every shard


def device_count() -> int:
    n = C.c_int32(0)
    N.lib().pccp_gpu_device_count(C.byref(n))
    return n.value


class Engine:
    """One device context (one GPU).  Not re-entrant."""

    def __init__(self, device: int = 0, *, group_threads: int = 0, groups_per_cta: int = 0, ctas_per_sm: int = 0,
                 eps_factor: int = 0, shard_index: int = 0, shard_count: int = 1, hash: bool = False,
                 value_order: int = -1, var_order: int = 0, primal_ms: int = 0, audit_nodes: int = 0,
                 audit_shift: int = 0, record_frontier: bool = False, verbose: bool = False, mix_order: int = 0):
        L = N.lib()
        self.cfg = N.PccpGpuCfg(device, group_threads, groups_per_cta, ctas_per_sm, eps_factor, shard_index,
                                shard_count, int(hash), int(verbose), value_order, var_order, primal_ms, audit_nodes,
                                audit_shift, int(record_frontier), mix_order)
        h = C.c_void_p()
        N.check(L.pccp_gpu_open(C.byref(self.cfg), C.byref(h)))
        self._h = h
        self.tables: Tables | None = None

    def close(self):
        if getattr(self, "_h", None) and N._lib is not None:
            N._lib.pccp_gpu_close(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ---- model
    def load(self, model) -> "Engine":
        """Lower and upload a model (Model, Tables, or any object with table attributes)."""
        t = Tables.coerce(model)
        s, keep = t.as_struct()
        N.check(N.lib().pccp_gpu_load(self._h, C.byref(s)))
        del keep
        self.tables = t
        return self

    def lowering_info(self) -> dict:
        i = N.PccpLoweringInfo()
        N.check(N.lib().pccp_gpu_lowering_info(self._h, C.byref(i)))
        return {k: getattr(i, k) for k, _ in N.PccpLoweringInfo._fields_}

    def _root(self, root):
        return self.tables.bottom() if root is None else np.ascontiguousarray(root, np.int32)

    # ---- K1
    def propagate_batch(self, stores):
        """Fixed points of independent stores: (out, failed[bool], rounds)."""
        a = np.ascontiguousarray(stores, np.int32).reshape(-1, self.tables.n_words)
        n = a.shape[0]
        out = np.empty_like(a)
        st = np.zeros(n, np.uint8)
        rd = np.zeros(n, np.uint32)
        N.check(N.lib().pccp_gpu_propagate_batch(self._h, _vp(a), n, _vp(out), _vp(st), _vp(rd)))
        return out, st.astype(bool), rd

    def run_sequential(self, words=None):
        """(failed, fixpoint words, rounds) for one store (bottom by default)."""
        out, st, rd = self.propagate_batch(self._root(words)[None, :])
        return bool(st[0]), out[0], int(rd[0])

    def replay(self, paths, best=None, root=None):
        """materialize() of each decision path [(var, upper, mid), ...] -> (words, failed)."""
        off = np.zeros(len(paths) + 1, np.uint32)
        flat = []
        for i, p in enumerate(paths):
            flat.extend(p)
            off[i + 1] = len(flat)
        dec = (N.PccpDecision * max(len(flat), 1))(*[N.PccpDecision(int(v), int(u), int(m)) for v, u, m in flat])
        b = np.full(len(paths), INT32_MAX, np.int32) if best is None else np.ascontiguousarray(best, np.int32)
        r = self._root(root)
        out = np.zeros((len(paths), self.tables.n_words), np.int32)
        st = np.zeros(len(paths), np.uint8)
        N.check(N.lib().pccp_gpu_replay(self._h, _vp(r), len(paths), _vp(off), C.cast(dec, C.c_void_p), _vp(b),
                                        _vp(out), _vp(st)))
        return out, st.astype(bool)

    # ---- search
    def enumerate(self, root=None, depth_cap: int = -1, timeout_s: float = 0.0, node_limit: int | None = None):
        lim = N.PccpLimits(timeout_s, 2**64 - 1 if node_limit is None else node_limit)
        res = N.PccpEnumResult()
        N.check(N.lib().pccp_gpu_enumerate(self._h, _vp(self._root(root)), depth_cap, C.byref(lim), C.byref(res)))
        d = _stats(res.stats)
        d["exhausted"] = bool(res.exhausted)
        return d

    def solve(self, root=None, timeout_s: float = 0.0, node_limit: int | None = None) -> SolveResult:
        lim = N.PccpLimits(timeout_s, 2**64 - 1 if node_limit is None else node_limit)
        res = N.PccpSolveResult()
        best = np.zeros(max(self.tables.n_words, 1), np.int32)
        N.check(N.lib().pccp_gpu_solve(self._h, _vp(self._root(root)), C.byref(lim), C.byref(res), _vp(best)))
        imp = [(res.improvements[k], res.improvement_ms[k]) for k in range(res.n_improvements)]
        has = res.has_objective
        primal = None
        if self.cfg.primal_ms > 0:
            primal = {"nodes": res.primal_nodes, "device_ms": res.primal_device_ms, "proved": bool(res.primal_proved),
                      "restarts": res.primal_restarts}
        return SolveResult(N.STATUS_NAMES[res.status], res.objective if has else None, _stats(res.stats),
                           best[: self.tables.n_words] if has == 1 else None, imp, best_on_peer=has == 2,
                           primal=primal, primal_proved=bool(res.primal_proved))

    def audit(self):
        """(pre, post, failed) of the nodes the last search sampled (cfg audit_nodes)."""
        k, nw = max(self.cfg.audit_nodes, 1), self.tables.n_words
        pre = np.zeros((k, nw), np.int32)
        post = np.zeros((k, nw), np.int32)
        fl = np.zeros(k, np.uint8)
        n = C.c_uint32(0)
        N.check(N.lib().pccp_gpu_audit(self._h, _vp(pre), _vp(post), _vp(fl), C.byref(n)))
        return pre[: n.value], post[: n.value], fl[: n.value].astype(bool)

    # ---- multi-GPU incumbent sharing
    def incumbent_handle(self) -> bytes:
        buf = (C.c_uint8 * 64)()
        N.check(N.lib().pccp_gpu_incumbent_handle(self._h, buf))
        return bytes(buf)

    def attach_peers(self, handles: list, self_index: int) -> None:
        raw = b"".join(h.ljust(64, b"\0")[:64] for h in handles)
        buf = (C.c_uint8 * max(len(raw), 1)).from_buffer_copy(raw or b"\0")
        N.check(N.lib().pccp_gpu_attach_peers(self._h, buf, len(handles), self_index))

    def reset_shared(self) -> None:
        """Reset the cross-rank cells (incumbent, best lock, done flag); with peers
        attached a solve never does it itself (include/pccp_gpu.h)."""
        N.check(N.lib().pccp_gpu_reset_shared(self._h))

    def offer_incumbent(self, value: int) -> None:
        """atomicMin a known objective value into the incumbent cell."""
        N.check(N.lib().pccp_gpu_offer_incumbent(self._h, int(value)))

    def frontier(self):
        """(all, share): store hashes of the last search's shared EPS frontier and of
        this shard's positions (cfg record_frontier)."""
        na, ns = C.c_uint32(0), C.c_uint32(0)
        N.check(N.lib().pccp_gpu_frontier(self._h, None, C.byref(na), None, C.byref(ns), 0))
        a = np.zeros(max(na.value, 1), np.uint64)
        b = np.zeros(max(ns.value, 1), np.uint64)
        N.check(N.lib().pccp_gpu_frontier(self._h, _vp(a), C.byref(na), _vp(b), C.byref(ns), max(a.size, b.size)))
        return a[: na.value], b[: ns.value]


def link_peers(engines: list) -> None:
    """pccp_gpu_link_peers: contexts of one process share the incumbent (and the
    done flag) through peer memory; contexts on one device are linked directly."""
    arr = (C.c_void_p * len(engines))(*[e._h.value for e in engines])
    N.check(N.lib().pccp_gpu_link_peers(arr, len(engines)))
