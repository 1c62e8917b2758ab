"""The C ABI library loads on a CPU-only host and exports every entry point
declared in include/*.h; entry points that need a device fail loudly (no CPU
fallback); the host-only lowering classifies the benchmark models."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2207_12116_b200 import Model, _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pccp_[a-z0-9_]+)\s*\(", src)))


@pytest.mark.parametrize("header", ["pccp_gpu.h", "pccp_host.h"])
def test_every_declared_symbol_is_exported(header):
    lib = C.CDLL(N.LIB_PATH)
    names = declared(header)
    assert len(names) >= 10
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a():
    data = open(N.LIB_PATH, "rb").read()
    assert b"sm_100a" in data


def test_device_entry_points_fail_loudly_without_gpu():
    from paper_2207_12116_b200 import Engine, EngineError, device_count
    if device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(EngineError):
        Engine(0)


def lower(m):
    L = N.lib()
    L.pccp_lower_only.argtypes = [C.POINTER(N.PccpModel), C.POINTER(N.PccpLoweringInfo), C.c_void_p]
    s, keep = m.tables().as_struct()
    info = N.PccpLoweringInfo()
    sc = np.zeros(6, np.uint32)
    N.check(L.pccp_lower_only(C.byref(s), C.byref(info), sc.ctypes.data_as(C.c_void_p)))
    return info, sc


def test_lowering_shapes():
    info, sc = lower(Model.nqueens(14))
    # every not(and(leq_offset, leq_offset)) fuses: 91 pairs x 3 offsets, nothing left over
    assert info.n_folded == 28 and sc[3] == 273 and sc[0] == 0 and info.n_generic == 0 and info.n_rows == 0
    assert sc[4] == (1 if os.environ.get("PCCP_FILTERED") else 0)  # filtered rounds are opt-in
    info, sc = lower(Model.random_csp(1))
    assert info.n_rows == 690 and info.n_generic == 0
    info, sc = lower(Model.rcpsp_random(1, 30, 4))
    # 930 overlap reifications fuse (11 commands each); precedences are unit records
    assert info.n_rows == 128 and info.n_generic == 0 and sc[5] == 930 and sc[1] == 0 and sc[0] == 80
    assert abs(lower(Model.nqueens(8))[0].alg_bytes_per_eval - 15.8139) < 1e-3  # Q8 15.8 B


def test_lowering_rejects_malformed_tables():
    t = Model.nqueens(4).tables()
    bad = type(t)(t.slot_kind, t.slot_word, t.n_words, t.cmd_off, t.cmd_code.copy(), t.cands, t.obj_slot)
    bad.cmd_code[3] = 99  # target word no longer matches the schema
    with pytest.raises(N.ModelError):
        lower(Model.__new__(Model)) if False else None
        L = N.lib()
        s, keep = bad.as_struct()
        N.check(L.pccp_lower_only(C.byref(s), C.byref(N.PccpLoweringInfo()), None))


def fast_mask(m, stores):
    L = N.lib()
    L.pccp_lower_fast_paths.argtypes = [C.POINTER(N.PccpModel), C.c_void_p, C.c_uint32, C.c_void_p]
    s, keep = m.tables().as_struct()
    a = np.ascontiguousarray(stores, np.int32).reshape(-1, m.tables().n_words)
    out = np.zeros(1, np.uint32)
    N.check(L.pccp_lower_fast_paths(C.byref(s), a.ctypes.data_as(C.c_void_p), a.shape[0],
                                    out.ctypes.data_as(C.c_void_p)))
    return int(out[0])


def test_value_range_analysis_decisions():
    """lower.cpp fast_paths: the benchmark models take the 32-bit paths from their
    bottom stores; unbounded or huge inputs, and domains whose sums could pass
    2^30, fall back to the widened int64 arithmetic (command.cpp:11-27)."""
    NE, ROWS, REIF, UNIT = 1, 2, 4, 8
    q = Model.nqueens(14)
    assert fast_mask(q, q.bottom()) == NE
    r = Model.rcpsp_random(1, 30, 4)
    assert fast_mask(r, r.bottom()) == ROWS | REIF | UNIT
    c = Model.random_csp(1)
    assert fast_mask(c, c.bottom()) == ROWS | UNIT
    # a store whose words sit near the sentinels: everything widened
    b = q.bottom().copy()
    b[:] = 2**30
    assert fast_mask(q, b) == 0
    # domains large enough that a row sum could pass 2^30: rows widened, units not
    big = Model.random_csp(1, dom_hi=10**8)
    assert fast_mask(big, big.bottom()) & ROWS == 0
