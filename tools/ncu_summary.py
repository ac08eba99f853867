"""Write a compact text summary of an ncu --set full report (for profiles/).
Usage: python tools/ncu_summary.py report.ncu-rep N_INSTANCES ALG_BYTES > out.txt"""
import csv
import subprocess
import sys

rep, n, alg = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
keys = ("Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "No Eligible", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "L1/TEX Hit Rate", "L2 Hit Rate", "Warp Cycles Per Issued Instruction")
rows = list(csv.reader(det.splitlines()))
print(f"report: {rep}")
if rows:
    h = rows[0]
    kn = h.index("Kernel Name") if "Kernel Name" in h else None
    if kn is not None and len(rows) > 1:
        print("kernel:", rows[1][kn])
    mn, mu, mv = h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    seen = set()
    for r in rows[1:]:
        if len(r) > mv and r[mn] in keys and r[mn] not in seen:
            seen.add(r[mn])
            print(f"  {r[mn]:40s} {r[mv]:>14s} {r[mu]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
h, u, v = rr[0], rr[1], rr[2]
def get(name):
    return float(v[h.index(name)].replace(",", "")) if name in h else None
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
def getb(name):
    return get(name) * SCALE.get(u[h.index(name)], 1) if name in h else 0.0
traffic = getb("dram__bytes_read.sum") + getb("dram__bytes_write.sum")
print(f"  dram bytes read+write (per launch)       {traffic:,.0f}")
print(f"  algorithmic bytes (per launch)           {alg:,}")
inst = get("smsp__inst_executed.sum")
if inst:
    print(f"  warp-instructions / instance             {inst / n:,.0f}")
stalls = []
for i, name in enumerate(h):
    if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("not_issued"):
        try:
            stalls.append((float(v[i].replace(",", "")), name.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
tot = sum(s for s, _ in stalls) or 1
print("  top stall reasons (pc sampling): " + ", ".join(f"{nm} {100 * s / tot:.0f}%" for s, nm in sorted(stalls)[::-1][:5]))
