"""paper_2207_12116_b200 — B200-native propagate-and-search engine (PCCP / Turbo, arXiv 2207.12116).

    from paper_2207_12116_b200 import Model, Engine
    m = Model.nqueens(14)
    with Engine() as eng:
        print(eng.load(m).enumerate())

The compute path is libpccp_b200.so (sm_100a kernels behind include/pccp_gpu.h);
this package is its host-side face.
"""
from ._native import ECUDA, EMODEL, EngineError, ModelError  # noqa: F401
from .engine import Engine, SolveResult, device_count  # noqa: F401
from .model import (INT32_MAX, INT32_MIN, Constraint, Kind, Model, Operand, Tables, and_c, iff_c, leq,  # noqa: F401
                    leq_offset, linear_leq, lt, not_c, precedes)

__all__ = ["Engine", "Model", "Tables", "Kind", "Operand", "Constraint", "linear_leq", "leq", "lt", "leq_offset",
           "precedes", "and_c", "iff_c", "not_c", "device_count", "SolveResult", "EngineError", "ModelError"]
