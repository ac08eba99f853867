"""Print the key counters of one ncu --set full capture (raw page CSV from `ncu -i X --page raw --csv`).
usage: python tools/ncu_keys.py raw.csv [n_instances]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h, u = rows[hi], rows[hi + 1]
KEYS = [
    ("Kernel Name", None), ("gpu__time_duration.sum", None),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", None),
    ("sm__inst_issued.avg.pct_of_peak_sustained_active", None),
    ("smsp__inst_executed.sum", "per_inst"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", None),
    ("l1tex__data_pipe_lsu_wavefronts.sum", "per_inst"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "per_inst"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum", "per_inst"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "per_inst"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum", "per_inst"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "per_inst"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum", "per_inst"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "per_inst"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "per_inst"),
    ("l1tex__t_requests_pipe_lsu_mem_local_op_ld.sum", "per_inst"),
    ("l1tex__t_requests_pipe_lsu_mem_local_op_st.sum", "per_inst"),
    ("l1tex__lsuin_requests.avg.pct_of_peak_sustained_elapsed", None),
    ("dram__bytes_read.sum", None),
    ("launch__registers_per_thread", None), ("launch__occupancy_limit_registers", None),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", None),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", None),
]
for r in rows[hi + 2:]:
    if not r or len(r) < len(h):
        continue
    d = dict(zip(h, r))
    for k, mode in KEYS:
        if k not in d:
            continue
        v = d[k]
        extra = ""
        if mode == "per_inst":
            try:
                extra = f"   ({float(v.replace(',', '')) / n:.1f} per instance)"
            except ValueError:
                pass
        print(f"{k:70s} {v} {u[h.index(k)]}{extra}")
    stalls = sorted(((float(d[k].replace(',', '') or 0), k) for k in h
                     if k.startswith("smsp__average_warp_latency_issue_stalled_") and k.endswith(".ratio")
                     and d[k]), reverse=True)[:8]
    if not stalls:
        stalls = sorted(((float(d[k].replace(',', '') or 0), k) for k in h
                         if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")
                         and d[k]), reverse=True)[:8]
    for v, k in stalls:
        print(f"  stall {k:70s} {v:.3f}")
    print("-" * 40)
