"""Per-line instruction counts (warp-instructions per instance) from an ncu report.
Usage: python tools/ncu_phases.py report.ncu-rep N_INSTANCES [min_per_instance]"""
import csv
import subprocess
import sys

rep, n = sys.argv[1], int(sys.argv[2])
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 8
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = cur = None
agg, fname = {}, ""
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ie = hdr.index("Instructions Executed")
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0] != "":
        cur = (fname, int(r[0]), r[1].strip()[:90])
        agg.setdefault(cur, 0)
        continue
    if r[2] == "...":
        continue
    try:
        agg[cur] += int(r[ie] or 0)
    except ValueError:
        pass
tot = sum(agg.values())
print(f"total {tot / n:.0f} warp-instructions per instance")
for (f, l, s), v in sorted(agg.items(), key=lambda x: (x[0][0], x[0][1])):
    if v / n >= thr:
        print(f"{f}:{l:4d} {v / n:7.1f}  {s}")
