"""Repeat RCPSP30 solves: python scripts/_seed_rep.py SEEDS REPS [TIMEOUT_S] (variance checks, ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_12116_b200 import Engine, Model  # noqa: E402

eng = Engine(0)
timeout = float(sys.argv[3]) if len(sys.argv) > 3 else 20.0
for s in [int(x) for x in sys.argv[1].split(",")]:
    m = Model.rcpsp_random(s, 30, 4)
    eng.load(m)
    for i in range(int(sys.argv[2])):
        r = eng.solve(timeout_s=timeout)
        st = r.stats
        tb = r.improvements[-1][1] if r.improvements else None
        print(s, r.status, r.objective, st['nodes'], st['rounds'], f"k={st['kernel_ms']:.1f} dec={st['decompose_ms']:.1f} "
              f"don={st['donations']} tbest={tb}", flush=True)
