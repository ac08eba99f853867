"""Top SASS instructions of admit_kernel by sampled stalls (total and long-scoreboard),
with the CUDA source line they belong to.
Usage: python tools/ncu_stalls.py report.ncu-rep [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, fname, cur, recs = None, "", None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path" or r[0] == "File Name":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0] != "":
        cur = f"{fname}:{r[0]}"
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        tot = float(d["Warp Stall Sampling (All Samples)"] or 0)
        lsb = float(d["stall_long_sb"] or 0)
    except (KeyError, ValueError):
        continue
    recs.append((tot, lsb, cur, d["Address"], r[3][:60]))
T = sum(x[0] for x in recs) or 1
L = sum(x[1] for x in recs) or 1
print(f"samples {T:.0f}, long_sb {L:.0f} ({100 * L / T:.1f}%)")
for tot, lsb, cur, addr, s in sorted(recs, reverse=True)[:top]:
    print(f"{100 * tot / T:5.1f}% lsb {100 * lsb / T:5.1f}%  {cur:24s} {addr:>6s} {s}")
