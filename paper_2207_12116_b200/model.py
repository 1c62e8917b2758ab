"""Model construction: a thin Python face over the native host builder.

Mirrors the reference's model API (store.hpp SchemaBuilder, propagation.hpp
constraint constructors, compile / compile_reified, rcpsp.hpp build_model /
check_solution) on top of include/pccp_host.h.  The output is the flat command
tables (`Tables`) that `Engine.load` consumes; tables serialised from the
reference library itself load the same way.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np

from . import _native as N

INT32_MAX = 2**31 - 1
INT32_MIN = -(2**31)


class Kind:
    """pccp::Kind (lattice.hpp:16)."""

    ZInc, ZDec, BInc, BDec, Interval = N.ZINC, N.ZDEC, N.BINC, N.BDEC, N.INTERVAL


@dataclass
class Tables:
    """Flat command tables of include/pccp_gpu.h (owned numpy arrays)."""

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

    @property
    def n_slots(self) -> int:
        return len(self.slot_kind)

    def bottom(self) -> np.ndarray:
        """Store::reset (store.cpp:29-39)."""
        w = np.zeros(self.n_words, np.int32)
        bot = {N.ZINC: INT32_MIN, N.ZDEC: INT32_MAX, N.BINC: 0, N.BDEC: 1}
        for k, first in zip(self.slot_kind, self.slot_word):
            if k == N.INTERVAL:
                w[first] = INT32_MIN
                w[first + 1] = INT32_MAX
            else:
                w[first] = bot[int(k)]
        return w

    def nbytes(self) -> int:
        return sum(a.nbytes for a in (self.slot_kind, self.slot_word, self.cmd_off, self.cmd_code, self.cands))

    def as_struct(self):
        """(PccpModel, keepalive) borrowing these arrays."""
        keep = [np.ascontiguousarray(self.slot_kind, np.uint8), np.ascontiguousarray(self.slot_word, np.uint32),
                np.ascontiguousarray(self.cmd_off, np.uint32), np.ascontiguousarray(self.cmd_code, np.int32),
                np.ascontiguousarray(self.cands, np.int32)]
        p = [a.ctypes.data_as(C.c_void_p) for a in keep]
        s = N.PccpModel(len(keep[0]), p[0], p[1], int(self.n_words), len(keep[2]) - 1, p[2], p[3], len(keep[4]),
                        p[4], int(self.obj_slot))
        return s, keep

    @staticmethod
    def coerce(t) -> "Tables":
        if isinstance(t, Tables):
            return t
        if isinstance(t, Model):
            return t.tables()
        return Tables(np.asarray(t.slot_kind, np.uint8), np.asarray(t.slot_word, np.uint32), int(t.n_words),
                      np.asarray(t.cmd_off, np.uint32), np.asarray(t.cmd_code, np.int32),
                      np.asarray(t.cands, np.int32), int(t.obj_slot))


# ---- constraint expressions (propagation.hpp:17-66), prefix-encoded ---------------
@dataclass(frozen=True)
class Operand:
    var: int = -1
    value: int = 0
    is_const: bool = False

    @staticmethod
    def v(slot: int) -> "Operand":
        return Operand(slot, 0, False)

    @staticmethod
    def c(k: int) -> "Operand":
        return Operand(-1, k, True)


def _op(o) -> Operand:
    return o if isinstance(o, Operand) else Operand.v(int(o))


@dataclass(frozen=True)
class Constraint:
    code: tuple

    def encode(self) -> np.ndarray:
        return np.asarray(self.code, np.int32)


def linear_leq(terms: Iterable[tuple[int, int]], c: int) -> Constraint:
    """sum coef*x <= c, coef >= 0 (linear_leq, propagation.cpp:8-13)."""
    terms = list(terms)
    out = [0, len(terms)]
    for coef, slot in terms:
        if coef < 0:
            raise N.ModelError(N.EMODEL, "linear_leq: coefficients must be nonnegative")
        out += [int(coef), int(slot)]
    return Constraint(tuple(out + [int(c)]))


def leq_offset(x, offset: int, y) -> Constraint:
    """x + offset <= y."""
    x, y = _op(x), _op(y)
    return Constraint((1, int(x.is_const), x.value if x.is_const else x.var, int(offset), int(y.is_const),
                       y.value if y.is_const else y.var))


def leq(x, y) -> Constraint:
    return leq_offset(x, 0, y)


def lt(x, y) -> Constraint:
    return leq_offset(x, 1, y)


def precedes(x, d: int, y) -> Constraint:
    return leq_offset(x, d, y)


def and_c(a: Constraint, b: Constraint) -> Constraint:
    return Constraint((2,) + a.code + b.code)


def iff_c(a: Constraint, b: Constraint) -> Constraint:
    return Constraint((3,) + a.code + b.code)


def not_c(a: Constraint) -> Constraint:
    return Constraint((4,) + a.code)


class Model:
    """A schema plus its guarded commands (SchemaBuilder + compiled propagators)."""

    def __init__(self, handle=None, *, is_rcpsp=False):
        L = N.lib()
        self._h = handle if handle is not None else L.pccp_host_new()
        if not self._h:
            raise N.ModelError(N.EMODEL, L.pccp_host_last_error().decode())
        self.is_rcpsp = is_rcpsp
        self._tables = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and N._lib is not None:
            N._lib.pccp_host_free(h)
            self._h = None

    @staticmethod
    def _wrap(h, is_rcpsp=False) -> "Model":
        if not h:
            raise N.ModelError(N.EMODEL, N.lib().pccp_host_last_error().decode())
        return Model(h, is_rcpsp=is_rcpsp)

    # ---- benchmark configurations
    @staticmethod
    def nqueens(n: int) -> "Model":
        return Model._wrap(N.lib().pccp_host_nqueens(n))

    @staticmethod
    def random_csp(seed: int, n_vars: int = 200, n_cons: int = 1000, dom_hi: int = 100) -> "Model":
        return Model._wrap(N.lib().pccp_host_random_csp(seed, n_vars, n_cons, dom_hi))

    @staticmethod
    def rcpsp_random(seed: int, n_real: int, resources: int) -> "Model":
        return Model._wrap(N.lib().pccp_host_rcpsp_random(seed, n_real, resources), True)

    @staticmethod
    def rcpsp_patterson(text: str) -> "Model":
        return Model._wrap(N.lib().pccp_host_rcpsp_patterson(text.encode()), True)

    @staticmethod
    def rcpsp(durations: Sequence[int], usages: Sequence[Sequence[int]], capacities: Sequence[int],
              precedences: Sequence[tuple[int, int]], horizon: int | None = None) -> "Model":
        d = np.asarray(durations, np.int32)
        n, r = len(d), len(capacities)
        u = np.asarray(usages, np.int32).reshape(n, r) if n and r else np.zeros((n, r), np.int32)
        cap = np.asarray(capacities, np.int32)
        pr = np.asarray(precedences, np.int32).reshape(-1, 2)
        h = int(d.sum()) if horizon is None else int(horizon)
        vp = lambda a: np.ascontiguousarray(a).ctypes.data_as(C.c_void_p)
        u, pr = np.ascontiguousarray(u), np.ascontiguousarray(pr)
        return Model._wrap(N.lib().pccp_host_rcpsp(n, vp(d), r, vp(u), vp(cap), len(pr), vp(pr), h), True)

    # ---- generic construction
    def _err(self, code):
        if code != N.OK:
            raise N.ModelError(code, N.lib().pccp_host_last_error().decode())

    def add_cell(self, kind: int = Kind.Interval) -> int:
        s = N.lib().pccp_host_add_cell(self._h, kind)
        if s < 0:
            self._err(N.EMODEL)
        self._tables = None
        return s

    def tell(self, slot: int, lo: int, hi: int) -> None:
        """Unguarded constant interval tell (tell_const + gnf)."""
        self._err(N.lib().pccp_host_tell(self._h, slot, lo, hi))
        self._tables = None

    def post(self, c: Constraint) -> None:
        """Compile and append a constraint's propagator (compile, propagation.cpp:408-413)."""
        e = c.encode()
        self._err(N.lib().pccp_host_post(self._h, e.ctypes.data_as(C.c_void_p), len(e)))
        self._tables = None

    def post_reified(self, b: int, c: Constraint) -> None:
        """b <-> c on a 0/1 interval b (compile_reified, propagation.cpp:415-431)."""
        e = c.encode()
        self._err(N.lib().pccp_host_post_reified(self._h, b, e.ctypes.data_as(C.c_void_p), len(e)))
        self._tables = None

    def set_objective(self, slot: int) -> None:
        self._err(N.lib().pccp_host_set_objective(self._h, slot))
        self._tables = None

    def set_candidates(self, slots: Sequence[int]) -> None:
        a = np.ascontiguousarray(slots, np.int32)
        self._err(N.lib().pccp_host_set_candidates(self._h, a.ctypes.data_as(C.c_void_p), len(a)))
        self._tables = None

    def tables(self) -> Tables:
        if self._tables is None:
            v = N.PccpModel()
            self._err(N.lib().pccp_host_view(self._h, C.byref(v)))

            def arr(ptr, ctype, n, dt):
                if n == 0:
                    return np.zeros(0, dt)
                return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ctype)), (n,)).astype(dt, copy=True)

            off = arr(v.cmd_off, C.c_uint32, v.n_cmds + 1, np.uint32)
            self._tables = Tables(arr(v.slot_kind, C.c_uint8, v.n_slots, np.uint8),
                                  arr(v.slot_word, C.c_uint32, v.n_slots, np.uint32), int(v.n_words), off,
                                  arr(v.cmd_code, C.c_int32, int(off[-1]), np.int32),
                                  arr(v.cands, C.c_int32, v.n_cands, np.int32), int(v.obj_slot))
        return self._tables

    @property
    def n_words(self) -> int:
        return self.tables().n_words

    def bottom(self) -> np.ndarray:
        return self.tables().bottom()

    # ---- RCPSP helpers (rcpsp.hpp:57-68)
    def starts(self) -> np.ndarray:
        n = N.lib().pccp_host_rcpsp_tasks(self._h)
        if n < 0:
            raise N.ModelError(N.EMODEL, "not an RCPSP model")
        s = np.zeros(n, np.int32)
        N.lib().pccp_host_rcpsp_starts(self._h, s.ctypes.data_as(C.c_void_p))
        return s

    def check_solution(self, words) -> bool:
        """check_solution on the start lower bounds of a solved store."""
        w = np.ascontiguousarray(words, np.int32)
        r = N.lib().pccp_host_rcpsp_check(self._h, w.ctypes.data_as(C.c_void_p))
        if r < 0:
            raise N.ModelError(N.EMODEL, N.lib().pccp_host_last_error().decode() or "not an RCPSP model")
        return bool(r)
