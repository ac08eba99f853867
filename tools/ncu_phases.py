"""Warp-instructions per instance by PHASE of admit_kernel, from an ncu --set full report
captured with --import-source on (the DESIGN.md §6.3 budget table).

Every SASS instruction is attributed to the source line ncu shows it under. Lines of the
kernel body in pf_admit.cuh map to a phase by the body's section markers; instructions of
inlined helpers (pf_common.cuh hash / scans, the Team primitives, CUDA intrinsics headers)
inherit the phase of the nearest preceding body instruction in address order (the compiler
lays the inlined code out at its call site).

Usage: python tools/ncu_phases.py report.ncu-rep N_INSTANCES [--src pf_admit.cuh | --group]"""
import csv
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_2507_10150_b200", "csrc", "pf_admit.cuh")
MARKERS = [  # (regex of the first line of a section, phase)
    (r"^admit_kernel\(AdmitParams p\)", "prologue (scalars, validation, tables, key)"),
    (r"// ---- a4: predictions", "a4 predict (loads, hash, lookups, binning)"),
    (r"if \(T\.any\(my_bad != 0\)\)", "prologue (scalars, validation, tables, key)"),
    (r"auto evaluate = ", "a5/a6 evaluation (bins, scans, bounds)"),
    (r"// ---- refinement of the wide bins", "a5/a6 refinement (list walks)"),
    (r"// ---- a7: Alg.1 lines 7-14", "a7 cutting plane (p_max scan, binQ rebuild)"),
]


# admit_group_kernel (pf_admit_group.cuh): --group
GROUP_SRC = os.path.join(ROOT, "paper_2507_10150_b200", "csrc", "pf_admit_group.cuh")
GROUP_MARKERS = [
    (r"^__device__ __forceinline__ void group_one\(", "prologue (scalars, validation, prefetch, key)"),
    (r"// ---- a4 \(Alg.1 l.3-9\)", "a4 predict (loads, hash, lookups, binning)"),
    (r"if \(__any_sync\(0xffffffffu, \(mx_lp > lpmax\)", "prologue (scalars, validation, prefetch, key)"),
    (r"auto evaluate = ", "a5/a6 evaluation (bins, scans, bounds)"),
    (r"// ---- refinement of the wide bins", "a5/a6 refinement (list walks)"),
    (r"// ---- a7: Alg.1 lines 7-14", "a7 cutting plane (p_max scan, binQ rebuild)"),
    (r"^// Cost-weighted partition", "kernel loop (partition, segments, instance counter)"),
]


def sections(src=SRC):
    lines = open(src).read().splitlines()
    out = []
    for i, l in enumerate(lines, 1):
        for rx, ph in (GROUP_MARKERS if src == GROUP_SRC else MARKERS):
            if re.search(rx, l):
                out.append((i, ph))
    end = next(i for i, l in enumerate(lines, 1) if l.startswith("}  // namespace pf"))
    return sorted(out), end


def phase_of(line, secs, end):
    ph = None
    for start, name in secs:
        if line >= start:
            ph = name
    return ph if (ph and line < end) else None


def main():
    rep, n = sys.argv[1], int(sys.argv[2])
    # --src FILE: the pf_admit.cuh the report was built from (e.g. an older commit's)
    src = GROUP_SRC if "--group" in sys.argv else (
        sys.argv[sys.argv.index("--src") + 1] if "--src" in sys.argv else SRC)
    secs, end = sections(src)
    base = os.path.basename(src)
    first = secs[0][0]
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, fname, cur, ins = None, "", None, []
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
            cur = (fname, int(r[0]))
            continue
        try:
            addr, cnt = int(r[2], 16), int(r[ie] or 0)
        except ValueError:
            continue
        ins.append((addr, cur, cnt))
    ins.sort()
    agg, last = {}, "prologue (scalars, validation, tables, key)"
    for addr, (f, line), cnt in ins:
        ph = phase_of(line, secs, end) if (f == base and line >= first) else None
        if ph is None:
            ph = last
        else:
            last = ph
        agg[ph] = agg.get(ph, 0) + cnt
    tot = sum(agg.values())
    print(f"{'phase':48s} warp-inst/instance   share")
    for ph, v in sorted(agg.items(), key=lambda kv: -kv[1]):
        print(f"{ph:48s} {v / n:10.0f}   {100 * v / tot:5.1f} %")
    print(f"{'total':48s} {tot / n:10.0f}")


if __name__ == "__main__":
    main()
