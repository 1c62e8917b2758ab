"""Per-source-line stall samples and instructions of one ncu report (the
`--page source --print-source cuda,sass` view): `python scripts/ncu_lines.py rep [top]`."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
f = None
agg = {}
h = None
for r in rows:
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        h = r
        continue
    if not h or len(r) < 8 or not r[0]:
        continue
    si, ii = 4, 7
    try:
        s, n = int(r[si] or 0), int(r[ii] or 0)
    except ValueError:
        continue
    agg[(f, int(r[0]))] = (s, n, r[1].strip()[:100])
ts = sum(v[0] for v in agg.values()) or 1
tn = sum(v[1] for v in agg.values()) or 1
print(f"samples {ts} instructions {tn}")
for (f, ln), (s, n, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * s / ts:5.1f}% smp {100 * n / tn:5.1f}% ins  {f}:{ln}  {src}")
