"""A/B timing of an enumeration (k_search device time) for the package on
sys.path: `python scripts/time_q14.py [reps] [q14|csp]`; run with different
PCCP_LIB (or PYTHONPATH) to compare builds on one box."""
import statistics
import sys

import paper_2207_12116_b200 as pkg
from paper_2207_12116_b200 import Engine, Model

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
which = sys.argv[2] if len(sys.argv) > 2 else "q14"
m, depth, nodes = {"q14": (Model.nqueens(14), -1, 8567767), "csp": (Model.random_csp(1), 22, 108611)}[which]
with Engine(0) as e:
    e.load(m)
    for _ in range(3):
        e.enumerate(depth_cap=depth)
    ks, dv = [], []
    for _ in range(reps):
        r = e.enumerate(depth_cap=depth)
        ks.append(r["kernel_ms"])
        dv.append(r["device_ms"])
    assert r["nodes"] == nodes
print(f"{which} {pkg.__file__}: kernel_ms median {statistics.median(ks):.3f} min {min(ks):.3f}; device_ms median {statistics.median(dv):.3f}")
