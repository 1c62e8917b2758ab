import json, sys
from paper_2207_12116_b200 import Engine, Model
m = Model.rcpsp_random(1, 120, 4)
with Engine(0) as e:
    e.load(m)
    for _ in range(3):
        r = e.solve(timeout_s=3.0)
        print("r120 ref order Mnodes/s %.2f" % (r.stats["nodes"] / r.stats["device_ms"] / 1e3), r.stats["rounds"] / r.stats["nodes"])
