"""A/B timing of the Q14 enumeration (k_search device time) for the package on
sys.path: `python scripts/time_q14.py [reps]`; run twice with different
PYTHONPATH to compare builds on one box."""
import statistics
import sys

import paper_2207_12116_b200 as pkg
from paper_2207_12116_b200 import Engine, Model

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
m = Model.nqueens(14)
with Engine(0) as e:
    e.load(m)
    for _ in range(3):
        e.enumerate()
    ks, dv = [], []
    for _ in range(reps):
        r = e.enumerate()
        ks.append(r["kernel_ms"])
        dv.append(r["device_ms"])
    assert r["nodes"] == 8567767
print(f"{pkg.__file__}: kernel_ms median {statistics.median(ks):.3f} min {min(ks):.3f}; device_ms median {statistics.median(dv):.3f}")
