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


def layout(m, stores):
    """pccp_lower_layout: (device words, device stores, stores converted back)."""
    t = m.tables()
    s, keep = t.as_struct()
    a = np.ascontiguousarray(stores, np.int32).reshape(-1, t.n_words)
    dw = C.c_uint32(0)
    N.check(N.lib().pccp_lower_layout(C.byref(s), None, 0, None, None, C.byref(dw)))
    dev = np.zeros((a.shape[0], dw.value), np.int32)
    back = np.zeros_like(a)
    N.check(N.lib().pccp_lower_layout(C.byref(s), a.ctypes.data_as(C.c_void_p), a.shape[0],
                                      dev.ctypes.data_as(C.c_void_p), back.ctypes.data_as(C.c_void_p), C.byref(dw)))
    return dw.value, dev, back


def test_bit_plane_layout():
    """lower_packed: RCPSP's n^2 overlap booleans (rcpsp.cpp:197-213) become bit
    cells (RCPSP30: 2,240 words -> 258, RCPSP120: 30,500 -> 1,666); N-Queens
    and the CSP have none.  Reference -> device -> reference is the identity on
    every store whose 0/1 cells hold (0,0), (0,1), (1,1) or the empty (1,0),
    and a cell outside [0, 1] after its folded constants stays empty."""
    from oracle.port import Oracle
    assert lower(Model.nqueens(14))[0].packed_cells == 0
    assert lower(Model.random_csp(1))[0].packed_cells == 0
    info = lower(Model.rcpsp_random(1, 120, 4))[0]
    assert (info.packed_cells, info.device_words) == (122 * 122, 1666)  # + one zero pair after the planes
    r = Model.rcpsp_random(1, 30, 4)
    info = lower(r)[0]
    assert (info.packed_cells, info.device_words) == (32 * 32, 258)
    t = r.tables()
    failed, root, _, _ = Oracle(t).run_sequential(r.bottom())
    assert not failed
    rng = np.random.default_rng(7)
    n = 32  # tasks incl. dummies
    bw = np.array([t.slot_word[n + k] for k in range(n * n)])  # overlap cells follow the starts
    stores = np.repeat(root[None, :], 64, axis=0)
    for s in stores[1:]:
        v = rng.integers(0, 4, bw.size)  # (0,1), (1,1), (0,0), (1,0) = empty
        s[bw] = np.where(v == 1, 1, np.where(v == 3, 1, 0))
        s[bw + 1] = np.where(v == 2, 0, np.where(v == 3, 0, 1))
    # the folded constants of each cell: the bottom store converted and back
    _, _, fb = layout(r, r.bottom()[None, :])
    flb, fub = fb[0, bw], fb[0, bw + 1]
    assert set(np.unique(flb)) <= {0, 1} and set(np.unique(fub)) <= {0, 1}
    want = stores.copy()
    lb, ub = np.maximum(stores[:, bw], flb), np.minimum(stores[:, bw + 1], fub)
    empty = lb > ub
    want[:, bw], want[:, bw + 1] = np.where(empty, 1, lb), np.where(empty, 0, ub)
    dw, dev, back = layout(r, stores)
    assert dw == 258
    assert np.array_equal(back, want)
    assert np.array_equal(layout(r, root[None, :])[2][0], root)
    assert np.array_equal(dev[:, :64], stores[:, :64])  # the starts keep their words
    # outside [0, 1]: lb 2 / ub -1 are empty after the folds, and stay empty
    s = root.copy()
    s[bw[5]] = 2
    s[bw[9] + 1] = -1
    _, _, back = layout(r, s[None, :])
    assert back[0, bw[5]] > back[0, bw[5] + 1] and back[0, bw[9]] > back[0, bw[9] + 1]
