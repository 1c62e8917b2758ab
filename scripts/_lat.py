import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2207_12116_b200 import Engine, Model
for name, m, gt in [("csp", Model.random_csp(1), 0), ("csp1024", Model.random_csp(1), 1024), ("q14", Model.nqueens(14), 0), ("r30", Model.rcpsp_random(1, 30, 4), 0)]:
    with Engine(0, group_threads=gt) as e:
        e.load(m)
        f, root, r = e.run_sequential()
        # a child of the root: branch like the search would, then time single-store propagation
        stores = np.stack([root] * 1)
        for _ in range(5): e.propagate_batch(stores)
        t = time.perf_counter(); n = 50
        for _ in range(n): out, st, rd = e.propagate_batch(stores)
        dt1 = (time.perf_counter() - t) / n
        big = np.stack([root] * 4096)
        e.propagate_batch(big)
        t = time.perf_counter(); out, st, rd = e.propagate_batch(big); dt2 = time.perf_counter() - t
        print(f"{name}: single-store call {dt1*1e6:.1f} us (rounds {rd[0]}), 4096 stores {dt2*1e3:.2f} ms = {dt2/4096*1e6:.2f} us/store")
