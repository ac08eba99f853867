"""Summarise an ncu source page (cuda,sass) CSV: per CUDA source line, instructions
executed and warp-stall samples. Usage: python tools/ncu_lines.py report.ncu-rep [topN]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
cur = None
agg = {}
fname = ""
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ie = hdr.index("Instructions Executed")
        ss = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0] != "":
        cur = (fname, int(r[0]), r[1].strip()[:90])
        agg.setdefault(cur, [0, 0])
        continue
    if cur is None or r[2] == "...":
        continue
    try:
        agg[cur][0] += int(r[ie] or 0)
        agg[cur][1] += int(r[ss] or 0)
    except ValueError:
        pass
tot_i = sum(v[0] for v in agg.values()) or 1
tot_s = sum(v[1] for v in agg.values()) or 1
print(f"total warp-instructions {tot_i:,}  stall samples {tot_s:,}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{100*v[0]/tot_i:5.1f}% inst {100*v[1]/tot_s:5.1f}% stall  {k[0]}:{k[1]}  {k[2]}")
