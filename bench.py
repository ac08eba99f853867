#!/usr/bin/env python
"""bench.py — Past-Future scheduler hot path on B200 (arXiv 2507.10150).

One STEP = one scheduler tick over the whole batch of instances, i.e. every §8(a)
row of SURVEY.md: update_history (record the tick's completions, Eq.(eq:5)) →
[shared mode, N>1: NCCL all-reduce of the group histograms] → group CDF tables →
admit (predict l̂ for every running/queued request, sort, scan, M*, FIFO prefix
search; Alg.1 + Eq.(eq:1)-(eq:3)).

Default workload (N=1): BASELINE.json configs[4] ("cfg5"): 2^20 instances, ragged
k ~ U[128,384] running / q ~ U[32,96] queued, mixed length classes, shared-history
groups (G=64, W=10,000 = 8 shards x 1,250), sampling mode, R=1, reserved 5 %.
Inputs (2.45 GB) are larger than the 126 MB L2, so no L2 flush is needed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C]

Prints ONE JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workload as W  # noqa: E402
from workload.gen import owned_shards  # noqa: E402

METRIC = "peak-memory estimates/s (request-slots/s) and % HBM peak at 1/2/4/8 B200"
UNIT = "request-slots/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-i", str(self.gpu), "-lms", "50"], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ helpers
def algorithmic_bytes(cfg: W.WorkloadConfig, b: W.Batch) -> int:
    """B_inst = 8k + 4q + H + S + O per instance (int32):
    l_p,l_t per running request; l_p per queued request; H = 4·min(w, Lmax+1) history
    bytes (0 in shared mode: group tables are read once per CTA from L2); S = 16 B
    scalars (run_off, q_off, max_new, capacity); O = 12 B outputs (admitted, peak,
    peak_running)."""
    k = int(b.run_off[-1])
    q = int(b.q_off[-1])
    n = b.n
    H = 0 if cfg.shared else 4 * min(cfg.window, cfg.max_len + 1)
    S = 16 if cfg.q[1] > 0 else 8
    O = 12 if cfg.q[1] > 0 else 4
    return 8 * k + 4 * q + n * (H + S + O)


def scheduler_for(cfg, bd, rank, nranks, mode, bp, seed):
    from paper_2507_10150_b200 import Scheduler
    kw = {}
    if cfg.shared:
        M = cfg.members_per_group
        kw = dict(n_groups=cfg.n_groups, group_off=bd.group_off, members_per_group=M,
                  member_base=rank * M // nranks)
    else:
        kw = dict(instance_base=int(bd.inst_ids[0]))
    return Scheduler(n_instances=bd.n, window=cfg.window, max_len=cfg.max_len,
                     max_input_len=cfg.max_input_len, max_entries=cfg.max_entries, mode=mode,
                     repetitions=1, reserved_bp=bp, seed=seed, rank=rank, nranks=nranks,
                     init_history=bd.hist_rows, **kw)


def cpu_oracle_rate(cfg, budget_s: float, n_threads: int, seed: int, bp: int, mode: int):
    """Time the oracle (as it stands) on a bounded, evenly spaced sample of the workload."""
    import oracle as O
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from harness import make_oracle, oracle_admit

    def run(m):
        ids = torch.linspace(0, cfg.n_instances - 1, m).round().long().unique()
        sub = W.make_batch(cfg, ids)
        orc = make_oracle(sub)
        t0 = time.perf_counter()
        oracle_admit(orc, sub, mode=mode, bp=bp, seed=seed, R=1, tick=0, estimate=cfg.q[1] == 0)
        dt = time.perf_counter() - t0
        return sub.slots(), sub.n, dt

    m = max(16, n_threads * 2)
    slots, n, dt = run(m)
    if dt < budget_s / 4:
        m = int(min(cfg.n_instances, max(m, m * budget_s / max(dt, 1e-3))))
        slots, n, dt = run(m)
    return slots / dt, n / dt, n, slots, dt


# ------------------------------------------------------------------ reference arm (oracle)
def run_reference(args, rank, world):
    if rank != 0:
        return
    cfg = W.CONFIGS[args.config]
    nt = os.cpu_count() or 1
    # calibrate a per-step sample so the whole --steps/--warmup run takes ~budget seconds
    budget = float(os.environ.get("PF_REF_BUDGET_S", "150"))
    per_step = max(0.05, budget / max(1, args.steps + args.warmup))
    rate_slots, rate_dec, n_cal, _, _ = cpu_oracle_rate(cfg, min(per_step * 4, 20.0), nt, args.seed, args.bp,
                                                        args.mode)
    import oracle as O  # noqa: F401
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from harness import make_oracle, oracle_admit
    m = max(8, int(rate_dec * per_step))
    ids = torch.linspace(0, cfg.n_instances - 1, min(m, cfg.n_instances)).round().long().unique()
    sub = W.make_batch(cfg, ids)
    times = []
    for s in range(args.warmup + args.steps):
        orc = make_oracle(sub)
        t0 = time.perf_counter()
        oracle_admit(orc, sub, mode=args.mode, bp=args.bp, seed=args.seed, R=1, tick=s,
                     estimate=cfg.q[1] == 0)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
    t = sum(times) / len(times)
    value = sub.slots() / t
    sample = (f"{sub.n} evenly spaced instances of {cfg.n_instances} ({sub.slots()} request-slots) per step, "
              f"oracle admit (Alg.1 literal, tick-stepped M*), {nt} threads")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": cfg.describe(), "decisions_per_s": sub.n / t},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": nt, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--mode", type=int, default=0, help="0 sample (C-8 hash), 1 quantile")
    ap.add_argument("--bp", type=int, default=500, help="reserved ratio, basis points (paper: 3/5/10 %%)")
    ap.add_argument("--seed", type=int, default=0x5EED)
    ap.add_argument("--tick-pool", type=int, default=16, help="distinct completion sets cycled over steps")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    assert args.warmup >= 3, "W >= 3 warm-up steps"

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.impl == "reference":
        run_reference(args, rank, world)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return

    torch.cuda.set_device(local)
    cfg = W.CONFIGS[args.config]
    shards = owned_shards(cfg, rank, world) if cfg.shared else None
    bd = W.make_batch(cfg, rank=rank, nranks=world, device="cuda", shards=shards)
    torch.cuda.synchronize()
    sched = scheduler_for(cfg, bd, rank, world, args.mode, args.bp, args.seed)
    pool = [W.make_completions(cfg, t, bd.row_ids) for t in range(args.tick_pool)]
    n = bd.n
    dev = "cuda"
    adm = torch.empty(n, dtype=torch.int32, device=dev)
    pk = torch.empty(n, dtype=torch.int32, device=dev)
    pkr = torch.empty(n, dtype=torch.int32, device=dev)
    estimate = cfg.q[1] == 0
    xbuf = sched.exchange_buffer() if (cfg.shared and world > 1) else None
    if xbuf is not None:  # pf_create left the group tables for the all-reduce
        import torch.distributed as dist
        dist.all_reduce(xbuf)
        sched.commit_history()
    stream = torch.cuda.current_stream()

    def step(t, ev=None):
        co, cl = pool[t % len(pool)]
        sched.update_history(co, cl)
        if xbuf is not None:
            import torch.distributed as dist
            dist.all_reduce(xbuf)
            sched.commit_history()
        if ev is not None:
            ev[0].record(stream)
        if estimate:
            sched.estimate_peak(bd.run_off, bd.input_len, bd.generated, bd.max_new, t, peak_out=pk)
        else:
            sched.admit(bd.run_off, bd.input_len, bd.generated, bd.q_off, bd.q_input_len, bd.max_new,
                        bd.capacity, t, admitted_out=adm, peak_out=pk, peak_running_out=pkr)
        if ev is not None:
            ev[1].record(stream)

    # Shared mode (cfg 5): tick t+1's update_history / NCCL all-reduce / group tables run
    # on a side stream while tick t's admit runs (the library double-buffers the group
    # tables, include/pfsched.h pf_commit_history); tables(t+2) wait for admit(t).
    pipelined = bool(cfg.shared)
    side = torch.cuda.Stream() if pipelined else None
    tab_ready, admit_done = {}, {}

    def tables(t):
        with torch.cuda.stream(side):
            if t - 2 in admit_done:
                side.wait_event(admit_done.pop(t - 2))
            co, cl = pool[t % len(pool)]
            sched.update_history(co, cl)
            if xbuf is not None:
                import torch.distributed as dist
                dist.all_reduce(xbuf)
                sched.commit_history()
            e = torch.cuda.Event()
            e.record(side)
            tab_ready[t] = e

    def admit_only(t, ev=None):
        stream.wait_event(tab_ready.pop(t))
        if ev is not None:
            ev[0].record(stream)
        sched.admit(bd.run_off, bd.input_len, bd.generated, bd.q_off, bd.q_input_len, bd.max_new,
                    bd.capacity, t, admitted_out=adm, peak_out=pk, peak_running_out=pkr)
        if ev is not None:
            ev[1].record(stream)
        e = torch.cuda.Event()
        e.record(stream)
        admit_done[t] = e

    def run_steps(t0, n, kev=None):
        # admit(t) is enqueued before tables(t+1): the host-side table flip happens at the
        # tables call, so admit(t) reads the half built for tick t
        if not pipelined:
            for j in range(n):
                step(t0 + j, kev[j] if kev else None)
            return
        if t0 not in tab_ready:
            tables(t0)
        for j in range(n):
            admit_only(t0 + j, kev[j] if kev else None)
            tables(t0 + j + 1)
        stream.wait_event(tab_ready[t0 + n])  # the timed region holds n table builds too

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    run_steps(0, args.warmup)
    barrier()
    K = args.steps
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.15)
    e0.record(stream)
    run_steps(args.warmup, K, kev)
    e1.record(stream)
    barrier()
    clk = clocks.stop()
    step_ms = e0.elapsed_time(e1) / K
    kern_ms = sum(a.elapsed_time(b) for a, b in kev) / K
    code, idx = sched.device_error()
    assert code == 0, f"device error {code} at {idx}"

    # max over ranks; whole-job units
    slots_local = bd.slots()
    t_step = torch.tensor([step_ms, kern_ms], dtype=torch.float64, device=dev)
    tot = torch.tensor([slots_local, n], dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t_step, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot)
    step_ms, kern_ms = float(t_step[0]), float(t_step[1])
    slots, decisions = float(tot[0]), float(tot[1])
    value = slots / (step_ms * 1e-3)

    # roofline of the dominant kernel (admit), algorithmic bytes of THIS rank's launch
    peak_gbs, peak_src = peaks()
    abytes = algorithmic_bytes(cfg, bd)
    achieved = abytes / (kern_ms * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "admit_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(f"cfg{args.config}")
        except Exception:
            traffic = None

    # e2e through the public API with HOST buffers (pinned), copies inside the timed region
    host = {k: getattr(bd, k).cpu().pin_memory() for k in
            ("run_off", "input_len", "generated", "q_off", "q_input_len", "max_new", "capacity")}
    hpool = [(co.cpu().pin_memory(), cl.cpu().pin_memory()) for co, cl in pool]
    dbuf = {k: torch.empty_like(v, device=dev) for k, v in host.items()}
    dco = [(torch.empty_like(a, device=dev), torch.empty_like(b, device=dev)) for a, b in hpool]
    h_adm = torch.empty(n, dtype=torch.int32).pin_memory()
    h_pk = torch.empty(n, dtype=torch.int32).pin_memory()
    h2d = sum(v.numel() * 4 for v in host.values())
    h2d_c = sum(a.numel() * 4 + b.numel() * 4 for a, b in hpool) / len(hpool)
    d2h = (0 if estimate else n * 4) + n * 4

    # Pipelined e2e: step t+1's inputs are copied (copy stream, second device buffer set)
    # while step t computes; every step still copies its inputs in and its results out.
    dsets = [dbuf, {k: torch.empty_like(v, device=dev) for k, v in host.items()}]
    dcos = [dco, [(torch.empty_like(a, device=dev), torch.empty_like(b, device=dev)) for a, b in hpool]]
    cs = torch.cuda.Stream()
    copied, used = {}, {}

    def copy_in(t, j):  # inputs of step t (tick j) into buffer set t % 2
        with torch.cuda.stream(cs):
            if t - 2 in used:
                cs.wait_event(used.pop(t - 2))
            for k, v in host.items():
                dsets[t % 2][k].copy_(v, non_blocking=True)
            a, b = hpool[j % len(hpool)]
            da, db = dcos[t % 2][j % len(hpool)]
            da.copy_(a, non_blocking=True)
            db.copy_(b, non_blocking=True)
            e = torch.cuda.Event()
            e.record(cs)
            copied[t] = e

    def e2e_compute(t, j):
        stream.wait_event(copied.pop(t))
        d = dsets[t % 2]
        da, db = dcos[t % 2][j % len(hpool)]
        sched.update_history(da, db)
        if xbuf is not None:
            import torch.distributed as dist
            dist.all_reduce(xbuf)
            sched.commit_history()
        if estimate:
            sched.estimate_peak(d["run_off"], d["input_len"], d["generated"], d["max_new"], j, peak_out=pk)
        else:
            sched.admit(d["run_off"], d["input_len"], d["generated"], d["q_off"], d["q_input_len"],
                        d["max_new"], d["capacity"], j, admitted_out=adm, peak_out=pk)
            h_adm.copy_(adm, non_blocking=True)
        h_pk.copy_(pk, non_blocking=True)
        e = torch.cuda.Event()
        e.record(stream)
        used[t] = e

    def e2e_run(E, j0):
        start = torch.cuda.Event()
        start.record(stream)
        cs.wait_event(start)  # the first copy starts inside the timed region
        copy_in(0, j0)
        for t in range(E):
            if t + 1 < E:
                copy_in(t + 1, j0 + t + 1)
            e2e_compute(t, j0 + t)
        copied.clear()
        used.clear()

    e2e_run(1, 999)
    barrier()
    E = max(1, args.e2e_steps)
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record(stream)
    e2e_run(E, 1000)
    a1.record(stream)
    barrier()
    e2e_ms = torch.tensor([a0.elapsed_time(a1) / E], dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_value = slots / (float(e2e_ms[0]) * 1e-3)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        nt = os.cpu_count() or 1
        rs, rd, ns, ss, dt = cpu_oracle_rate(cfg, args.cpu_budget, nt, args.seed, args.bp, args.mode)
        cpu = {"value": rs, "unit": UNIT, "cores": nt, "kind": "oracle",
               "sample": f"{ns} evenly spaced instances ({ss} request-slots) of {cfg.name}, one admit "
                         f"tick, oracle as it stands (Alg.1 literal, tick-stepped M*) on {nt} threads, "
                         f"{dt:.1f} s", "decisions_per_s": rd}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "int32", "data": "synthetic",
            "config": {"workload": cfg.describe(), "instances": int(decisions), "request_slots": int(slots),
                       "decisions_per_s": decisions / (step_ms * 1e-3), "mode": "sample" if args.mode == 0
                       else "quantile", "reserved_bp": args.bp, "parallelism": f"instances sharded x{world}",
                       "l2": "inputs 2.45 GB > 126 MB L2 (no flush needed)" if args.config == 5 else
                       "see DESIGN.md", "admit_kernel_ms": kern_ms,
                       "step": "update_history + group tables + admit" + (" + NCCL allreduce" if xbuf is not None else "")
                       + (" (tick t+1's history/tables on a side stream, overlapping tick t's admit)" if pipelined else "")},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak_gbs, "unit": "GB/s",
                         "frac": achieved / peak_gbs, "traffic": traffic, "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": abytes, "kernel": "admit_kernel",
                         "frac_of_8TBs_spec": achieved / 8000.0},
            "e2e": {"value": e2e_value, "unit": UNIT, "pipelined": "step t+1's H2D overlaps step t",
                    "h2d_bytes_per_step": int(h2d + h2d_c),
                    "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": 3 * K,
            "clocks": clk,
        }
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
