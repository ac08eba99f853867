"""Record the per-launch DRAM traffic and instruction count of the admit kernel from
ncu --set full captures into profiles/admit_traffic.json (read by bench.py's roofline).
Usage: python tools/ncu_traffic.py CFG=REPORT.ncu-rep [CFG=REPORT ...] --tag r02"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "admit_traffic.json")
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def metrics(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    h, u, v = rr[0], rr[1], rr[2]

    def get(name, scaled=False):
        x = float(v[h.index(name)].replace(",", ""))
        return x * SCALE.get(u[h.index(name)], 1) if scaled else x
    return {"bytes": int(get("dram__bytes_read.sum", True) + get("dram__bytes_write.sum", True)),
            "warp_instructions": int(get("smsp__inst_executed.sum")),
            "kernel": v[h.index("Kernel Name")] if "Kernel Name" in h else "admit_kernel"}


def main():
    tag = "r02"
    args = [a for a in sys.argv[1:]]
    if "--tag" in args:
        tag = args[args.index("--tag") + 1]
        args = [a for a in args if a not in ("--tag", tag)]
    d = json.load(open(OUT)) if os.path.exists(OUT) else {}
    d = {k: v for k, v in d.items() if isinstance(v, dict)}
    for a in args:
        cfg, rep = a.split("=", 1)
        m = metrics(rep)
        m["source"] = (f"profiles/{tag}/ncu_admit_{cfg}.txt: ncu --set full of one admit launch "
                       f"(dram__bytes_read.sum + dram__bytes_write.sum; smsp__inst_executed.sum)")
        d[cfg] = m
    json.dump(d, open(OUT, "w"), indent=1)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main()
