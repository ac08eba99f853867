"""Instruction / stall share per code region of admit_kernel (regions = marker comments
in pf_admit.cuh). Usage: python tools/ncu_regions.py report.ncu-rep N_INSTANCES"""
import csv
import os
import subprocess
import sys

rep, N = sys.argv[1], int(sys.argv[2])
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
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
        ss = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0] != "":
        cur = (fname, int(r[0]))
        agg.setdefault(cur, [0, 0])
        continue
    if r[2] == "...":
        continue
    try:
        agg[cur][0] += int(r[ie] or 0)
        agg[cur][1] += int(r[ss] or 0)
    except ValueError:
        pass
src = open(os.path.join(ROOT, "paper_2507_10150_b200/csrc/pf_admit.cuh")).read().split("\n")
keys = ["// ---- instance scalars", "// ---- a3:", "// ---- a4:", "auto finish", "// running requests e",
        "// queued requests j", "if (T.any(my_bad", "// ---- a5/a6:", "auto evaluate", "// walk: exact T",
        "Eval ev;", "// ---- refinement", "// Many candidate bins", "// ---- a7:", "// p_max(",
        "// rebuild binQ"]
marks = {}
for i, l in enumerate(src, 1):
    for key in keys:
        if key in l and key not in marks:
            marks[key] = i
order = sorted(marks.items(), key=lambda x: x[1])


def region(l):
    name = "helpers (Team, lookups)"
    for k, v in order:
        if l >= v:
            name = k
    return name


byr = {}
for (f, l), v in agg.items():
    key = region(l) if f == "pf_admit.cuh" else "other:" + f
    x = byr.setdefault(key, [0, 0])
    x[0] += v[0]
    x[1] += v[1]
tot = sum(v[0] for v in byr.values()) or 1
tots = sum(v[1] for v in byr.values()) or 1
print(f"{'region':32s} {'warp-inst/inst':>14s} {'inst %':>7s} {'stall %':>8s}")
for k, v in sorted(byr.items(), key=lambda x: -x[1][0]):
    print(f"{k:32s} {v[0] / N:14.0f} {100 * v[0] / tot:6.1f}% {100 * v[1] / tots:7.1f}%")
