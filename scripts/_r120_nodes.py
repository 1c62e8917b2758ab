"""RCPSP120 seed 1, reference branching order, bounded by a node limit (ncu
captures: a timeout would cut the replay passes short)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_12116_b200 import Engine, Model  # noqa: E402

eng = Engine(0)
m = Model.rcpsp_random(1, 120, 4)
eng.load(m)
r = eng.solve(node_limit=int(sys.argv[1]) if len(sys.argv) > 1 else 1000000)
st = r.stats
print(r.status, st["nodes"], st["rounds"], f"k={st['kernel_ms']:.1f}ms dec={st['decompose_ms']:.1f}ms",
      f"nodes/s={st['nodes'] / (st['device_ms'] / 1e3):.3e}")
