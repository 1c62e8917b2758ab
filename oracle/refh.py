"""ctypes view of oracle/_ref/libpccp_ref.so — TEST INFRASTRUCTURE ONLY.

The library is the unmodified reference (/root/reference/proj/src) plus the
harness in oracle/ref_harness.cpp, built by `make -C oracle ref`.  Only
tests/, bench.py (cpu_baseline and --impl reference) and the golden generator
use this module; the product never imports anything under oracle/.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libpccp_ref.so")

_lib = None

INT32_MAX = 2**31 - 1
INT32_MIN = -(2**31)


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C oracle ref` where /root/reference exists")
        L = C.CDLL(LIB_PATH)
        vp, u32, i32, u64, dbl = C.c_void_p, C.c_uint32, C.c_int32, C.c_uint64, C.c_double
        P = C.POINTER
        sig = {
            "refh_last_error": (C.c_char_p, []),
            "refh_free": (None, [vp]),
            "refh_model_nqueens": (vp, [C.c_int]),
            "refh_model_csp": (vp, [u64, C.c_int, C.c_int, C.c_int, C.c_int]),
            "refh_model_rcpsp": (vp, [u64, C.c_int, C.c_int]),
            "refh_model_corpus": (vp, [C.c_int]),
            "refh_model_patterson": (vp, [C.c_char_p]),
            "refh_rng_new": (vp, [u64]),
            "refh_rng_free": (None, [vp]),
            "refh_model_micro_csp": (vp, [vp]),
            "refh_model_micro_rcpsp": (vp, [vp]),
            "refh_brute_force_makespan": (i32, [vp]),
            "refh_n_slots": (u32, [vp]),
            "refh_n_words": (u32, [vp]),
            "refh_n_cmds": (u32, [vp]),
            "refh_code_len": (u32, [vp]),
            "refh_n_cands": (u32, [vp]),
            "refh_obj_slot": (i32, [vp]),
            "refh_tables": (None, [vp, vp, vp, vp, vp, vp]),
            "refh_root": (None, [vp, vp]),
            "refh_run_sequential": (C.c_int, [vp, vp, vp, P(u64), P(u64)]),
            "refh_run_parallel": (C.c_int, [vp, vp, vp, C.c_uint, P(u64)]),
            "refh_replay": (C.c_int, [vp, vp, C.c_int, vp, i32, vp, P(u64)]),
            "refh_branch": (C.c_int, [vp, vp, P(i32), P(i32)]),
            "refh_enumerate": (C.c_int, [vp, C.c_int, C.c_int, dbl, u64, vp, P(dbl)]),
            "refh_solve_parallel": (C.c_int, [vp, C.c_uint, dbl, u64, C.c_uint, vp, vp, P(dbl), vp]),
            "refh_solve_dfs": (C.c_int, [vp, dbl, u64, vp, vp, P(dbl), vp]),
            "refh_check_solution": (C.c_int, [vp, vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


@dataclass
class Tables:
    """Flat command tables of include/pccp_gpu.h (numpy views)."""

    slot_kind: np.ndarray
    slot_word: np.ndarray
    n_words: int
    cmd_off: np.ndarray
    cmd_code: np.ndarray
    cands: np.ndarray
    obj_slot: int

    @property
    def n_cmds(self) -> int:
        return len(self.cmd_off) - 1


class RefModel:
    """A model built by the reference's own API (owned handle)."""

    def __init__(self, handle):
        if not handle:
            raise RuntimeError("reference harness: " + lib().refh_last_error().decode())
        self.h = handle
        L = lib()
        ns, nw, nc, cl, nk = (L.refh_n_slots(handle), L.refh_n_words(handle), L.refh_n_cmds(handle),
                              L.refh_code_len(handle), L.refh_n_cands(handle))
        kind = np.zeros(ns, np.uint8)
        word = np.zeros(ns, np.uint32)
        off = np.zeros(nc + 1, np.uint32)
        code = np.zeros(max(cl, 1), np.int32)
        cands = np.zeros(max(nk, 1), np.int32)
        L.refh_tables(handle, _ptr(kind), _ptr(word), _ptr(off), _ptr(code), _ptr(cands))
        self.tables = Tables(kind, word, int(nw), off, code[:cl], cands[:nk], int(L.refh_obj_slot(handle)))

    def __del__(self):
        try:
            if self.h and _lib is not None:
                _lib.refh_free(self.h)
        except Exception:
            pass

    # ---- builders
    @classmethod
    def nqueens(cls, n: int) -> "RefModel":
        return cls(lib().refh_model_nqueens(n))

    @classmethod
    def csp(cls, seed: int, n_vars=200, n_cons=1000, dom_hi=100, variant=0) -> "RefModel":
        return cls(lib().refh_model_csp(seed, n_vars, n_cons, dom_hi, variant))

    @classmethod
    def rcpsp(cls, seed: int, n_real: int, resources: int) -> "RefModel":
        return cls(lib().refh_model_rcpsp(seed, n_real, resources))

    @classmethod
    def corpus(cls, idx: int) -> "RefModel":
        return cls(lib().refh_model_corpus(idx))

    @classmethod
    def patterson(cls, text: str) -> "RefModel":
        return cls(lib().refh_model_patterson(text.encode()))

    @property
    def n_words(self) -> int:
        return self.tables.n_words

    def root(self) -> np.ndarray:
        w = np.zeros(self.n_words, np.int32)
        lib().refh_root(self.h, _ptr(w))
        return w

    def run_sequential(self, words=None):
        """(failed, out_words, iterations, applications) — engine.cpp:13-32."""
        out = np.zeros(self.n_words, np.int32)
        it, ap = C.c_uint64(), C.c_uint64()
        inp = None if words is None else np.ascontiguousarray(words, np.int32)
        r = lib().refh_run_sequential(self.h, None if inp is None else _ptr(inp), _ptr(out), C.byref(it), C.byref(ap))
        if r < 0:
            raise RuntimeError(lib().refh_last_error().decode())
        return bool(r), out, it.value, ap.value

    def run_parallel(self, words=None, workers=4):
        out = np.zeros(self.n_words, np.int32)
        it = C.c_uint64()
        inp = None if words is None else np.ascontiguousarray(words, np.int32)
        r = lib().refh_run_parallel(self.h, None if inp is None else _ptr(inp), _ptr(out), workers, C.byref(it))
        if r < 0:
            raise RuntimeError(lib().refh_last_error().decode())
        return bool(r), out, it.value

    def replay(self, decisions, best=INT32_MAX, root=None):
        """materialize (solver.cpp:91-102): decisions = [(var, upper, mid), ...]."""
        dec = np.asarray(decisions, np.int32).reshape(-1, 3)
        rt = self.root() if root is None else np.ascontiguousarray(root, np.int32)
        out = np.zeros(self.n_words, np.int32)
        it = C.c_uint64()
        r = lib().refh_replay(self.h, _ptr(rt), len(dec), _ptr(np.ascontiguousarray(dec)), best, _ptr(out), C.byref(it))
        if r < 0:
            raise RuntimeError(lib().refh_last_error().decode())
        return bool(r), out

    def branch(self, words):
        v, m = C.c_int32(), C.c_int32()
        w = np.ascontiguousarray(words, np.int32)
        r = lib().refh_branch(self.h, _ptr(w), C.byref(v), C.byref(m))
        if r < 0:
            raise RuntimeError(lib().refh_last_error().decode())
        return None if r == 0 else (v.value, m.value)

    def enumerate(self, depth_cap=-1, threads=1, budget_s=0.0, node_budget=0):
        out = np.zeros(7, np.uint64)
        ms = C.c_double()
        r = lib().refh_enumerate(self.h, depth_cap, threads, budget_s, node_budget, _ptr(out), C.byref(ms))
        if r < 0:
            raise RuntimeError(lib().refh_last_error().decode())
        keys = ["nodes", "failures", "solutions", "open_leaves", "hash_sum", "sweeps", "exhausted"]
        d = {k: int(v) for k, v in zip(keys, out)}
        d["elapsed_ms"] = ms.value
        return d

    def solve_parallel(self, workers=1, timeout_s=0.0, node_limit=2**64 - 1, eps_factor=8):
        out = np.zeros(3, np.int32)
        st = np.zeros(2, np.uint64)
        ms = C.c_double()
        best = np.zeros(self.n_words, np.int32)
        r = lib().refh_solve_parallel(self.h, workers, timeout_s, node_limit, eps_factor, _ptr(out), _ptr(st),
                                      C.byref(ms), _ptr(best))
        if r < 0:
            raise RuntimeError(lib().refh_last_error().decode())
        return dict(status=int(out[0]), objective=int(out[2]) if out[1] else None, nodes=int(st[0]),
                    solutions=int(st[1]), elapsed_ms=ms.value, best_words=best if out[1] else None)

    def solve_dfs(self, timeout_s=0.0, node_limit=2**64 - 1):
        out = np.zeros(3, np.int32)
        st = np.zeros(2, np.uint64)
        ms = C.c_double()
        best = np.zeros(self.n_words, np.int32)
        r = lib().refh_solve_dfs(self.h, timeout_s, node_limit, _ptr(out), _ptr(st), C.byref(ms), _ptr(best))
        if r < 0:
            raise RuntimeError(lib().refh_last_error().decode())
        return dict(status=int(out[0]), objective=int(out[2]) if out[1] else None, nodes=int(st[0]),
                    solutions=int(st[1]), elapsed_ms=ms.value, best_words=best if out[1] else None)

    def check_solution(self, words) -> bool:
        w = np.ascontiguousarray(words, np.int32)
        r = lib().refh_check_solution(self.h, _ptr(w))
        if r < 0:
            raise RuntimeError("not an RCPSP model")
        return bool(r)

    def brute_force_makespan(self):
        v = lib().refh_brute_force_makespan(self.h)
        return None if v == INT32_MIN else v


class RefRng:
    """std::mt19937_64 shared across reference generator calls."""

    def __init__(self, seed: int):
        self.h = lib().refh_rng_new(seed)

    def __del__(self):
        try:
            if self.h and _lib is not None:
                _lib.refh_rng_free(self.h)
        except Exception:
            pass

    def micro_csp(self) -> RefModel:
        return RefModel(lib().refh_model_micro_csp(self.h))

    def micro_rcpsp(self) -> RefModel:
        return RefModel(lib().refh_model_micro_rcpsp(self.h))
