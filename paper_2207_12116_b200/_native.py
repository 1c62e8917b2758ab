"""ctypes binding of libpccp_b200.so (include/pccp_gpu.h, include/pccp_host.h).

The library is built in-tree by `make -C paper_2207_12116_b200/csrc` (or
`__graft_entry__.build()`).  There is no fallback: if it is missing, importing
the engine raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PCCP_LIB") or os.path.join(HERE, "libpccp_b200.so")  # PCCP_LIB: build variants

OK, EMODEL, ECUDA, ELIMIT, EARG = 0, 1, 2, 3, 4
ZINC, ZDEC, BINC, BDEC, INTERVAL = 0, 1, 2, 3, 4
OPTIMAL, SAT, UNSAT, UNKNOWN = 0, 1, 2, 3
STATUS_NAMES = {OPTIMAL: "OPTIMAL", SAT: "SAT", UNSAT: "UNSAT", UNKNOWN: "UNKNOWN"}


class PccpModel(C.Structure):
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


class PccpDecision(C.Structure):
    _fields_ = [("var", C.c_int32), ("upper", C.c_int32), ("mid", C.c_int32)]


class PccpGpuCfg(C.Structure):
    _fields_ = [
        ("device", C.c_int32),
        ("group_threads", C.c_int32),
        ("groups_per_cta", C.c_int32),
        ("ctas_per_sm", C.c_int32),
        ("eps_factor", C.c_int32),
        ("shard_index", C.c_int32),
        ("shard_count", C.c_int32),
        ("hash", C.c_int32),
        ("verbose", C.c_int32),
        ("value_order", C.c_int32),
        ("var_order", C.c_int32),
        ("primal_ms", C.c_int32),
        ("audit_nodes", C.c_int32),
        ("audit_shift", C.c_int32),
        ("record_frontier", C.c_int32),
        ("mix_order", C.c_int32),
    ]


class PccpLimits(C.Structure):
    _fields_ = [("timeout_s", C.c_double), ("node_limit", C.c_uint64)]


class PccpStats(C.Structure):
    _fields_ = [
        ("nodes", C.c_uint64),
        ("failures", C.c_uint64),
        ("solutions", C.c_uint64),
        ("open_leaves", C.c_uint64),
        ("hash_sum", C.c_uint64),
        ("rounds", C.c_uint64),
        ("evals", C.c_uint64),
        ("subproblems", C.c_uint64),
        ("max_depth", C.c_uint64),
        ("elapsed_ms", C.c_double),
        ("kernel_ms", C.c_double),
        ("decompose_ms", C.c_double),
        ("launches", C.c_uint64),
        ("search_evals", C.c_uint64),
        ("h2d_bytes", C.c_uint64),
        ("d2h_bytes", C.c_uint64),
        ("device_ms", C.c_double),
        ("bfs_levels", C.c_uint64),
        ("donations", C.c_uint64),
        ("rematerialised", C.c_uint64),
        ("stolen", C.c_uint64),
        ("remote_in", C.c_uint64),
        ("remote_out", C.c_uint64),
    ]


class PccpEnumResult(C.Structure):
    _fields_ = [("stats", PccpStats), ("exhausted", C.c_int32)]


class PccpSolveResult(C.Structure):
    _fields_ = [
        ("stats", PccpStats),
        ("status", C.c_int32),
        ("has_objective", C.c_int32),
        ("objective", C.c_int32),
        ("n_improvements", C.c_int32),
        ("improvements", C.c_int32 * 64),
        ("improvement_ms", C.c_double * 64),
        ("phases", C.c_int32),
        ("primal_proved", C.c_int32),
        ("primal_nodes", C.c_uint64),
        ("primal_device_ms", C.c_double),
        ("primal_restarts", C.c_int32),
    ]


class PccpLoweringInfo(C.Structure):
    _fields_ = [
        ("n_words", C.c_uint32),
        ("n_cmds", C.c_uint32),
        ("n_folded", C.c_uint32),
        ("n_small", C.c_uint32),
        ("n_rows", C.c_uint32),
        ("n_row_terms", C.c_uint32),
        ("n_generic", C.c_uint32),
        ("table_bytes", C.c_uint32),
        ("store_bytes", C.c_uint32),
        ("group_threads", C.c_uint32),
        ("groups_per_cta", C.c_uint32),
        ("ctas", C.c_uint32),
        ("smem_bytes", C.c_uint32),
        ("table_in_smem", C.c_uint32),
        ("stack_in_smem", C.c_uint32),
        ("stack_depth", C.c_uint32),
        ("alg_bytes_per_eval", C.c_double),
        ("store_bytes_per_round", C.c_double),
        ("table_bytes_per_round", C.c_double),
        ("packed_cells", C.c_uint32),
        ("device_words", C.c_uint32),
    ]


_lib = None


def lib():
    """Load the native engine; raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `make -C {os.path.join(HERE, 'csrc')}`")
    L = C.CDLL(LIB_PATH)
    vp, i32, u32, u64, P = C.c_void_p, C.c_int32, C.c_uint32, C.c_uint64, C.POINTER
    sigs = {
        # engine
        "pccp_gpu_last_error": (C.c_char_p, []),
        "pccp_gpu_version": (C.c_char_p, []),
        "pccp_gpu_device_count": (C.c_int, [P(i32)]),
        "pccp_gpu_open": (C.c_int, [P(PccpGpuCfg), P(vp)]),
        "pccp_gpu_close": (None, [vp]),
        "pccp_gpu_load": (C.c_int, [vp, P(PccpModel)]),
        "pccp_gpu_lowering_info": (C.c_int, [vp, P(PccpLoweringInfo)]),
        "pccp_gpu_propagate_batch": (C.c_int, [vp, vp, u32, vp, vp, vp]),
        "pccp_gpu_replay": (C.c_int, [vp, vp, u32, vp, vp, vp, vp, vp]),
        "pccp_gpu_enumerate": (C.c_int, [vp, vp, i32, P(PccpLimits), P(PccpEnumResult)]),
        "pccp_gpu_solve": (C.c_int, [vp, vp, P(PccpLimits), P(PccpSolveResult), vp]),
        "pccp_gpu_incumbent_handle": (C.c_int, [vp, vp]),
        "pccp_gpu_attach_peers": (C.c_int, [vp, vp, i32, i32]),
        "pccp_gpu_audit": (C.c_int, [vp, vp, vp, vp, vp]),
        "pccp_gpu_link_peers": (C.c_int, [vp, i32]),
        "pccp_gpu_reset_shared": (C.c_int, [vp]),
        "pccp_gpu_offer_incumbent": (C.c_int, [vp, i32]),
        "pccp_gpu_frontier": (C.c_int, [vp, vp, P(u32), vp, P(u32), u32]),
        "pccp_lower_layout": (C.c_int, [P(PccpModel), vp, u32, vp, vp, P(u32)]),
        # host model builder
        "pccp_host_last_error": (C.c_char_p, []),
        "pccp_host_new": (vp, []),
        "pccp_host_free": (None, [vp]),
        "pccp_host_nqueens": (vp, [i32]),
        "pccp_host_random_csp": (vp, [u64, i32, i32, i32]),
        "pccp_host_rcpsp_random": (vp, [u64, i32, i32]),
        "pccp_host_rcpsp_patterson": (vp, [C.c_char_p]),
        "pccp_host_rcpsp": (vp, [i32, vp, i32, vp, vp, i32, vp, i32]),
        "pccp_host_add_cell": (i32, [vp, i32]),
        "pccp_host_tell": (C.c_int, [vp, i32, i32, i32]),
        "pccp_host_post": (C.c_int, [vp, vp, i32]),
        "pccp_host_post_reified": (C.c_int, [vp, i32, vp, i32]),
        "pccp_host_set_objective": (C.c_int, [vp, i32]),
        "pccp_host_set_candidates": (C.c_int, [vp, vp, i32]),
        "pccp_host_view": (C.c_int, [vp, P(PccpModel)]),
        "pccp_host_bottom": (C.c_int, [vp, vp]),
        "pccp_host_rcpsp_tasks": (i32, [vp]),
        "pccp_host_rcpsp_starts": (C.c_int, [vp, vp]),
        "pccp_host_rcpsp_check": (C.c_int, [vp, vp]),
    }
    for name, (res, args) in sigs.items():
        if os.environ.get("PCCP_LIB") and not hasattr(L, name):
            continue  # an older build variant (A/B timing) may lack newer entry points
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


class EngineError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{ {1: 'ModelError', 2: 'CudaError', 3: 'LimitError', 4: 'ArgError'}.get(code, code)}] {msg}")
        self.code = code


class ModelError(EngineError):
    pass


def check(code: int):
    if code != OK:
        msg = lib().pccp_gpu_last_error().decode()
        raise (ModelError if code == EMODEL else EngineError)(code, msg)
