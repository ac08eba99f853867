"""Profiling driver: build a full-size config on the GPU and run T ticks of
update_history + admit (ncu target: -k regex:admit_kernel)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import workload as W  # noqa: E402
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--ticks", type=int, default=3)
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--mode", type=int, default=0)
a = ap.parse_args()
cfg = W.CONFIGS[a.config]
if a.n:
    cfg = W.scaled(cfg, a.n)
bd = W.make_batch(cfg, device="cuda")
s = bench.scheduler_for(cfg, bd, 0, 1, a.mode, 500, 0x5EED)
n = bd.n
adm = torch.empty(n, dtype=torch.int32, device="cuda")
pk = torch.empty_like(adm)
pkr = torch.empty_like(adm)
for t in range(a.ticks):
    co, cl = W.make_completions(cfg, t, bd.row_ids)
    s.update_history(co, cl)
    if cfg.q[1] == 0:
        s.estimate_peak(bd.run_off, bd.input_len, bd.generated, bd.max_new, t, peak_out=pk)
    else:
        s.admit(bd.run_off, bd.input_len, bd.generated, bd.q_off, bd.q_input_len, bd.max_new, bd.capacity, t,
                admitted_out=adm, peak_out=pk, peak_running_out=pkr)
torch.cuda.synchronize()
print("bytes", bench.algorithmic_bytes(cfg, bd), "device_error", s.device_error())
