"""Summarise ncu reports into profiles/: per-kernel key metrics (JSON) plus the
full details page (text), and a launch-list share table.

    python scripts/ncu_summary.py --rep gpurun_out/q14_search_full2.ncu-rep --workload nqueens14-all-solutions \
        --tag r01_q14 [--launches gpurun_out/launches_q14_r1d.csv]
"""
import argparse
import collections
import csv
import io
import json
import os
import shutil
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "smsp__inst_executed.sum": "warp_instructions",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum": "smem_atomic_wavefronts",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "lts__t_bytes.sum": "l2_bytes",
    "lts__t_sectors.sum": "l2_sectors",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3,
         "Ghz": 1e3, "Mhz": 1.0}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--workload", required=True)
    ap.add_argument("--tag", required=True)
    ap.add_argument("--launches")
    a = ap.parse_args()
    hdr, units, rows = raw(a.rep)
    summ_path = os.path.join(PROF, "ncu_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    for r in rows:
        name = r[hdr.index("Kernel Name")].split("(")[0].split("<")[0].split("::")[-1].replace("void ", "").strip()
        d = {"source": f"ncu --set full --clock-control none ({os.path.basename(a.rep)}); "
                       f"details in profiles/{a.tag}_{name}_details.txt"}
        for k, short in METRICS.items():
            if k in hdr:
                i = hdr.index(k)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if short == "duration":
                    d["duration_ms"] = v * SCALE.get(u, 1.0)
                elif short == "sm_clock":
                    d["sm_clock_mhz"] = v * SCALE.get(u, 1.0)
                elif short.startswith("dram") or short == "l2_bytes":
                    d[short + "_bytes"] = v * SCALE.get(u, 1.0)
                else:
                    d[short] = v
        d["dram_bytes_per_launch"] = d.get("dram_read_bytes", 0) + d.get("dram_write_bytes", 0)
        if "l2_sectors" in d:
            d["l2_bytes_per_launch"] = d["l2_sectors"] * 32
        t = d.get("duration_ms", 0) / 1e3
        if t > 0:  # achieved bandwidths of the launch (cold-cache, serialised replay)
            d["achieved_gbs"] = {"smem": d.get("smem_wavefronts", 0) * 128 / t / 1e9,
                                 "l2": d.get("l2_bytes_per_launch", 0) / t / 1e9,
                                 "dram": d["dram_bytes_per_launch"] / t / 1e9}
        summ.setdefault(a.workload, {})[name] = d
        det = subprocess.run(["ncu", "-i", a.rep, "--page", "details"], capture_output=True, text=True).stdout
        with open(os.path.join(PROF, f"{a.tag}_{name}_details.txt"), "w") as f:
            f.write(det)
        print(a.workload, name, json.dumps(d))
    json.dump(summ, open(summ_path, "w"), indent=1, sort_keys=True)
    if a.launches:
        agg = collections.defaultdict(lambda: [0, 0.0])
        lh = None
        for r in csv.reader(open(a.launches)):
            if r and r[0] == "ID":
                lh = r
                continue
            if lh and len(r) == len(lh):
                k = r[lh.index("Kernel Name")].split("(")[0]
                agg[k][0] += 1
                agg[k][1] += float(r[lh.index("Metric Value")])
        tot = sum(v[1] for v in agg.values())
        with open(os.path.join(PROF, f"{a.tag}_launches_summary.txt"), "w") as f:
            f.write(f"ncu --metrics gpu__time_duration.sum --clock-control none ({os.path.basename(a.launches)})\n"
                    "cold-cache, serialised launches: compare shares, not absolutes\n\n")
            for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
                f.write(f"{k:70s} {n:5d} launches {t / 1e6:10.3f} ms {100 * t / tot:6.2f}%\n")
        shutil.copyfile(a.launches, os.path.join(PROF, f"{a.tag}_launches.csv"))


if __name__ == "__main__":
    main()
