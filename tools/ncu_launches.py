"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of bench.py:
launches per kernel, mean/min/max duration, and each kernel's share of the step.
Usage: python tools/ncu_launches.py launches.csv "command that produced it" > summary.txt"""
import collections
import csv
import sys

OURS = ("admit_kernel", "admit_group_kernel", "update_hist_kernel", "update_sorted_kernel", "group_tables_kernel",
        "init_ring_kernel", "hist_rows_kernel", "sort_rows_kernel", "baseline_kernel", "sim_",
        "gram_kernel", "adjacent_kernel", "cosine_kernel")
path, cmd = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
hdr = rows[0]
ik, im, iu, iv = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
t = collections.OrderedDict()
units = set()
for r in rows[1:]:
    if len(r) <= iv or r[im] != "gpu__time_duration.sum" or not any(n in r[ik] for n in OURS):
        continue
    v = float(r[iv].replace(",", ""))
    u = r[iu]
    units.add(u)
    v = v / 1000.0 if u == "ns" else (v * 1000.0 if u == "ms" else v)  # -> us
    t.setdefault(r[ik], []).append(v)
print(f"ncu launch list of: {cmd}")
print(f"(gpu__time_duration.sum, --clock-control none, units {sorted(units)}; cold-cache and serialised:")
print(" compare SHARES, not absolutes; only this library's kernels are listed)\n")
for k, v in t.items():
    print(f"{len(v):4d} launches  mean {sum(v) / len(v):9.1f} us  min {min(v):9.1f}  max {max(v):9.1f}  {k[:110]}")
mean = {k: sum(v) / len(v) for k, v in t.items()}
step = {"admit": sum(m for k, m in mean.items() if "admit" in k),
        "update_history": sum(m for k, m in mean.items() if "update_" in k),
        "group_tables": sum(m for k, m in mean.items() if "group_tables" in k)}
tot = sum(step.values())
print("\nper-step share (mean launch times): " + "  ".join(f"{k} {100 * v / tot:.1f}%" for k, v in step.items())
      + f"  (step sum {tot:.0f} us)")
