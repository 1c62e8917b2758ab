"""One enumeration for profiling: `python scripts/enum_one.py q14|q8|csp [reps]` (three
warm-up runs first; ncu -s 3 skips their k_search launches)."""
import sys

from paper_2207_12116_b200 import Engine, Model

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
m, depth = {"q14": (Model.nqueens(14), -1), "q8": (Model.nqueens(8), -1),
            "csp": (Model.random_csp(1), 22)}[name]
with Engine(0, verbose=True) as e:
    e.load(m)
    for _ in range(3 + reps):
        r = e.enumerate(depth_cap=depth)
    print(name, r["nodes"], r["solutions"], r["kernel_ms"], r["device_ms"])
