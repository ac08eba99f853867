"""Per-basic-block instruction counts of a kernel from an ncu source page (sass):
python tools/ncu_blocks.py report.ncu-rep N_INSTANCES [min_share]
A block starts at a branch target or after a branch; prints blocks by instructions executed."""
import csv
import re
import subprocess
import sys

rep, N = sys.argv[1], int(sys.argv[2])
mins = float(sys.argv[3]) if len(sys.argv) > 3 else 0.005
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ia, isrc, ie = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
iss = hdr.index("Warp Stall Sampling (All Samples)")
ins = [(int(r[ia], 16), r[isrc].strip(), int(r[ie] or 0), int(r[iss] or 0)) for r in rows[2:] if len(r) > ie]
base = ins[0][0]
targets = set()
for a, s, _, _ in ins:
    m = re.search(r"BRA.*?(0x[0-9a-f]+)", s)
    if m:
        targets.add(int(m.group(1), 16) + (base if int(m.group(1), 16) < base else 0))
blocks, cur = [], None
for idx, (a, s, e, st) in enumerate(ins):
    if cur is None or a in targets or a - base in targets:
        cur = [a - base, a - base, 0, 0, 0, s]
        blocks.append(cur)
    cur[1] = a - base
    cur[2] += e
    cur[3] += 1
    cur[4] += st
    if "BRA" in s or "EXIT" in s or "RET" in s:
        cur = None
tot = sum(b[2] for b in blocks)
tst = sum(b[4] for b in blocks) or 1
print(f"total {tot / N:.0f} warp-inst/instance")
for b in sorted(blocks, key=lambda b: -b[2]):
    if b[2] / tot < mins:
        break
    execs = b[2] / max(b[3], 1) / N
    print(f"{b[0]:#06x}-{b[1]:#06x} n={b[3]:4d} {100 * b[2] / tot:5.1f}% inst  {100 * b[4] / tst:5.1f}% stall  "
          f"{b[2] / N:7.1f}/inst  x{execs:5.2f}/inst  {b[5][:40]}")
