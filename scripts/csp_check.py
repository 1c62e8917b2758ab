"""Repeatability check of the CSP depth-22 enumeration under lowering variants."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_12116_b200 import Engine, Model  # noqa: E402

want = (108611, 23228, 31078, 0x6C8868DADE5564A8)
depth = int(sys.argv[1]) if len(sys.argv) > 1 else 22
gt = int(sys.argv[2]) if len(sys.argv) > 2 else 0
m = Model.random_csp(1)
with Engine(0, hash=True, group_threads=gt) as e:
    e.load(m)
    for rep in range(4):
        r = e.enumerate(depth_cap=depth)
        got = (r["nodes"], r["failures"], r["open_leaves"], r["hash_sum"])
        print(os.environ.get("PCCP_NO_UNIT"), os.environ.get("PCCP_NO_ROWS"), gt, got, got == want, flush=True)
