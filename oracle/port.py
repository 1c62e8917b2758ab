"""ctypes view of oracle/liboracle.so, the plain-C restatement — TEST INFRASTRUCTURE ONLY.

Operates on flat tables (any object with slot_kind, slot_word, n_words,
cmd_off, cmd_code, cands, obj_slot numpy attributes — e.g. oracle.refh.Tables
or the product's model views).  Only tests/, __graft_entry__.smoke and
bench.py's cpu_baseline use it, always as the checker.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
INT32_MAX = 2**31 - 1

_lib = None


class PccpModel(C.Structure):
    """struct pccp_model of include/pccp_gpu.h."""

    _fields_ = [
        ("n_slots", C.c_uint32),
        ("slot_kind", C.c_void_p),
        ("slot_word", C.c_void_p),
        ("n_words", C.c_uint32),
        ("n_cmds", C.c_uint32),
        ("cmd_off", C.c_void_p),
        ("cmd_code", C.c_void_p),
        ("n_cands", C.c_uint32),
        ("cands", C.c_void_p),
        ("obj_slot", C.c_int32),
    ]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C oracle port`")
        L = C.CDLL(LIB_PATH)
        P = C.POINTER
        vp, u64 = C.c_void_p, C.c_uint64
        L.orc_run_sequential.argtypes = [P(PccpModel), vp, P(u64), P(u64)]
        L.orc_run_sequential.restype = C.c_int
        L.orc_is_failed.argtypes = [P(PccpModel), vp]
        L.orc_branch.argtypes = [P(PccpModel), vp, P(C.c_int32), P(C.c_int32)]
        L.orc_replay.argtypes = [P(PccpModel), vp, C.c_int, vp, C.c_int32, vp]
        L.orc_store_hash.argtypes = [C.c_uint32, vp]
        L.orc_store_hash.restype = C.c_uint64
        L.orc_enumerate.argtypes = [P(PccpModel), vp, C.c_int, u64, vp]
        L.orc_solve_dfs.argtypes = [P(PccpModel), vp, u64, vp, vp, vp]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


class Oracle:
    """The C restatement bound to one model's flat tables."""

    def __init__(self, t):
        self._keep = [np.ascontiguousarray(t.slot_kind, np.uint8), np.ascontiguousarray(t.slot_word, np.uint32),
                      np.ascontiguousarray(t.cmd_off, np.uint32), np.ascontiguousarray(t.cmd_code, np.int32),
                      np.ascontiguousarray(t.cands, np.int32)]
        k, w, off, code, cands = self._keep
        self.n_words = int(t.n_words)
        self.m = PccpModel(len(k), _p(k), _p(w), self.n_words, len(off) - 1, _p(off), _p(code), len(cands),
                           _p(cands), int(t.obj_slot))
        self.obj_slot = int(t.obj_slot)

    def bottom(self):
        """Store::reset (store.cpp:29-39): every cell at bottom."""
        words = np.zeros(self.n_words, np.int32)
        k, w = self._keep[0], self._keep[1]
        bot = {0: -(2**31), 1: 2**31 - 1, 2: 0, 3: 1}
        for kind, first in zip(k, w):
            if kind == 4:
                words[first] = -(2**31)
                words[first + 1] = 2**31 - 1
            else:
                words[first] = bot[int(kind)]
        return words

    def run_sequential(self, words):
        w = np.array(words, np.int32, copy=True)
        it, ap = C.c_uint64(), C.c_uint64()
        r = lib().orc_run_sequential(C.byref(self.m), _p(w), C.byref(it), C.byref(ap))
        if r < 0:
            raise RuntimeError("ModelError: scalar tell without a scalar expression")
        return bool(r), w, it.value, ap.value

    def is_failed(self, words):
        w = np.ascontiguousarray(words, np.int32)
        return bool(lib().orc_is_failed(C.byref(self.m), _p(w)))

    def branch(self, words):
        w = np.ascontiguousarray(words, np.int32)
        v, m = C.c_int32(), C.c_int32()
        r = lib().orc_branch(C.byref(self.m), _p(w), C.byref(v), C.byref(m))
        if r < 0:
            raise RuntimeError("ModelError: branch on an unbounded variable")
        return None if r == 0 else (v.value, m.value)

    def replay(self, root, decisions, best=INT32_MAX):
        dec = np.ascontiguousarray(np.asarray(decisions, np.int32).reshape(-1, 3))
        rt = np.ascontiguousarray(root, np.int32)
        out = np.zeros(self.n_words, np.int32)
        r = lib().orc_replay(C.byref(self.m), _p(rt), len(dec), _p(dec), best, _p(out))
        return bool(r), out

    def enumerate(self, root, depth_cap=-1, node_budget=0):
        out = np.zeros(7, np.uint64)
        rt = np.ascontiguousarray(root, np.int32)
        r = lib().orc_enumerate(C.byref(self.m), _p(rt), depth_cap, node_budget, _p(out))
        if r < 0:
            raise RuntimeError("ModelError during enumeration")
        keys = ["nodes", "failures", "solutions", "open_leaves", "hash_sum", "sweeps", "exhausted"]
        return {k: int(v) for k, v in zip(keys, out)}

    def solve_dfs(self, root, node_limit=2**64 - 1):
        if self.obj_slot < 0:
            raise ValueError("model has no objective")
        out = np.zeros(3, np.int32)
        st = np.zeros(2, np.uint64)
        best = np.zeros(self.n_words, np.int32)
        rt = np.ascontiguousarray(root, np.int32)
        r = lib().orc_solve_dfs(C.byref(self.m), _p(rt), node_limit, _p(out), _p(st), _p(best))
        if r < 0:
            raise RuntimeError("ModelError during search")
        return dict(status=int(out[0]), objective=int(out[2]) if out[1] else None, nodes=int(st[0]),
                    solutions=int(st[1]), best_words=best if out[1] else None)


def store_hash(words) -> int:
    w = np.ascontiguousarray(words, np.int32)
    return int(lib().orc_store_hash(len(w), _p(w)))
