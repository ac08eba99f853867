"""Per-rank compute of cfg 5 at P ranks, measured on ONE GPU (the multi-GPU scaling proxy of
DESIGN.md §7): rank 0's shard (2^20 / P instances, owned history shards s ≡ 0 mod P) runs
bench.py's pipelined step — update_history + group tables on a side stream overlapping the
admit — with the exchange replaced by the caller-side commit of the local partial sums (the
NCCL all-reduce of the 1.3 MB buffer is emulated by a device copy of the exact all-reduced
histogram, kept by a one-member-per-group reference context fed every shard's completions).
Prints per P: admit ms,
step ms, and the strong-scaling efficiency t(1) / (P · t(P)) the compute alone allows.

  python tools/shard_probe.py [--steps 50]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import workload as W  # noqa: E402
from workload.gen import owned_shards  # noqa: E402
from paper_2507_10150_b200 import Scheduler  # noqa: E402


PRIO = int(os.environ.get("PROBE_SIDE_PRIORITY", "-1"))  # bench.py's choice; 0 = default priority


def run(P, steps):
    cfg = W.CONFIGS[5]
    M = cfg.members_per_group
    bd = W.make_batch(cfg, rank=0, nranks=P, shards=owned_shards(cfg, 0, P), device="cuda")
    s = Scheduler(n_instances=bd.n, window=cfg.window, max_len=cfg.max_len, max_input_len=cfg.max_input_len,
                  max_entries=cfg.max_entries, n_groups=cfg.n_groups, group_off=bd.group_off,
                  members_per_group=M, member_base=0, mode=0, reserved_bp=500, seed=0x5EED, rank=0,
                  nranks=P, init_history=bd.hist_rows)
    # the all-reduced group histograms H_g: a reference context holding every shard row
    full = W.make_batch(W.scaled(cfg, cfg.n_groups), device="cuda")
    ref = Scheduler(n_instances=full.n, window=cfg.window, max_len=cfg.max_len, max_input_len=cfg.max_input_len,
                    max_entries=cfg.max_entries, n_groups=cfg.n_groups, group_off=full.group_off,
                    members_per_group=1, member_base=0, mode=0, reserved_bp=500, seed=0x5EED,
                    init_history=full.hist_rows)
    xb, xr = s.exchange_buffer(), ref.exchange_buffer()
    xb.copy_(xr)
    s.commit_history()
    pool = [W.make_completions(cfg, t, bd.row_ids) for t in range(16)]
    rpool = [W.make_completions(cfg, t, full.row_ids) for t in range(16)]
    n = bd.n
    adm = torch.empty(n, dtype=torch.int32, device="cuda")
    pk = torch.empty_like(adm)
    main = torch.cuda.current_stream()
    side = torch.cuda.Stream(priority=PRIO)  # -1: high priority (its CTAs dispatch ahead of admit's)
    ready, done = {}, {}

    def tables(t):
        with torch.cuda.stream(side):
            if t - 2 in done:
                side.wait_event(done.pop(t - 2))
            co, cl = pool[t % 16]
            s.update_history(co, cl)
            if P > 1:
                ref.update_history(*rpool[t % 16])
                xb.copy_(xr)  # stands in for ncclAllReduce(sum) of the partial histograms
                s.commit_history()
            e = torch.cuda.Event()
            e.record(side)
            ready[t] = e

    def admit(t, ev=None):
        main.wait_event(ready.pop(t))
        if ev:
            ev[0].record(main)
        s.admit(bd.run_off, bd.input_len, bd.generated, bd.q_off, bd.q_input_len, bd.max_new, bd.capacity, t,
                admitted_out=adm, peak_out=pk)
        if ev:
            ev[1].record(main)
        e = torch.cuda.Event()
        e.record(main)
        done[t] = e

    tables(0)
    for t in range(5):
        admit(t)
        tables(t + 1)
    torch.cuda.synchronize()
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    import time
    e0.record(main)
    h0 = time.perf_counter()
    for j in range(steps):
        admit(5 + j, kev[j])
        tables(6 + j)
    host_ms = (time.perf_counter() - h0) * 1e3 / steps
    main.wait_event(ready[5 + steps])
    e1.record(main)
    torch.cuda.synchronize()
    step = e0.elapsed_time(e1) / steps
    adm_ms = sum(a.elapsed_time(b) for a, b in kev) / steps
    s.close()
    ref.close()
    return n, bd.slots(), adm_ms, step, host_ms


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=50)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    base = None
    for P in (1, 2, 4, 8):
        n, slots, adm_ms, step, host_ms = run(P, a.steps)
        base = base or step
        print(json.dumps({"P": P, "instances_per_rank": n, "slots_per_rank": slots, "admit_ms": round(adm_ms, 4),
                          "step_ms": round(step, 4), "host_enqueue_ms_per_step": round(host_ms, 4),
                          "compute_strong_scaling_eff": round(base / (P * step), 3)}),
              flush=True)


if __name__ == "__main__":
    main()
