"""Opcode histogram (warp-instructions per instance) of one kernel from an ncu source page
exported with `--page source --csv --print-source sass`.
usage: python tools/sass_hist.py sass.csv N_INSTANCES [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
h = rows[1]
ia, isrc, iex = h.index("Address"), h.index("Source"), h.index("Instructions Executed")
ist = h.index("Warp Stall Sampling (All Samples)")
ops = collections.Counter()
stall = collections.Counter()
tot = 0
seq = []
for r in rows[2:]:
    if len(r) <= iex:
        continue
    src = r[isrc].strip()
    ex = int(r[iex] or 0)
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    base = op.split(".")[0]
    ops[base] += ex
    stall[base] += int(r[ist] or 0)
    tot += ex
    seq.append((r[ia], src, ex, int(r[ist] or 0)))
print(f"total {tot / n:.1f} warp-inst per instance")
for op, c in ops.most_common(top):
    print(f"{op:12s} {c / n:8.1f}  stall-samples {stall[op]}")
