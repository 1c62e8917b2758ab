"""Split bench.py's end-to-end step (pccp_gpu_load + pccp_gpu_enumerate from
host buffers) into its parts on the host clock: lowering + upload, the
enumerate call, and the device time the call reports."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2207_12116_b200 import Engine, Model  # noqa: E402

q = Model.nqueens(int(sys.argv[1]) if len(sys.argv) > 1 else 14)
t = q.tables()
eng = Engine(0)
smi = None
if len(sys.argv) > 2 and sys.argv[2] == "smi":  # the bench's clock sampler running beside the steps
    import subprocess
    smi = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,"
                            "clocks_event_reasons.active", "--format=csv,noheader,nounits", "-lms", "100"],
                           stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    time.sleep(0.3)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda:0")
rows = []
for i in range(40):
    flush.zero_()
    torch.cuda.synchronize()
    ta = time.perf_counter()
    st, keep = t.as_struct()
    t0 = time.perf_counter()
    eng.load(t)
    t1 = time.perf_counter()
    r = eng.enumerate()
    t2 = time.perf_counter()
    rows.append({"as_struct_ms": (t0 - ta) * 1e3, "load_ms": (t1 - t0) * 1e3, "enum_ms": (t2 - t1) * 1e3, "device_ms": r["device_ms"],
                 "elapsed_ms": r["elapsed_ms"], "kernel_ms": r["kernel_ms"], "decompose_ms": r["decompose_ms"]})
for i in range(3):  # without re-loading
    t1 = time.perf_counter()
    r = eng.enumerate()
    t2 = time.perf_counter()
    rows.append({"noload_enum_ms": (t2 - t1) * 1e3, "device_ms": r["device_ms"], "elapsed_ms": r["elapsed_ms"]})
if smi:
    smi.terminate()
for r in rows:
    print(json.dumps({k: round(v, 3) for k, v in r.items()}))
