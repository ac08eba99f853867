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


def scheduler_for(cfg, bd, rank, nranks, mode, bp, seed, nccl_id=None):
    from paper_2507_10150_b200 import Scheduler
    kw = {}
    if cfg.shared:
        M = cfg.members_per_group
        kw = dict(n_groups=cfg.n_groups, group_off=bd.group_off, members_per_group=M,
                  member_base=rank * M // nranks, nccl_id=nccl_id)
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


def cpu_fast_rate(cfg, budget_s: float, n_threads: int, seed: int, bp: int, mode: int):
    """Context next to cpu_baseline: the optimized multithreaded CPU implementation
    (baselines/cpu_fast.cpp: O(1) lookups, sort-form M*, binary search over the prefix)
    on a bounded, evenly spaced sample of the workload."""
    import baselines
    baselines.lib()  # build outside the timed region

    def run(m):
        ids = torch.linspace(0, cfg.n_instances - 1, m).round().long().unique()
        sub = W.make_batch(cfg, ids)
        rows = baselines.dist_rows_of(sub)
        t0 = time.perf_counter()
        baselines.admit(sub, rows, mode=mode, bp=bp, seed=seed, tick=0, threads=n_threads)
        return sub.slots(), sub.n, time.perf_counter() - t0

    m = max(64, n_threads * 16)
    slots, n, dt = run(m)
    if dt < budget_s / 4:
        m = int(min(cfg.n_instances, max(m, m * budget_s / max(dt, 1e-3))))
        slots, n, dt = run(m)
    return slots / dt, n, slots, dt


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
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": cfg.describe(), "decisions_per_s": sub.n / t},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": nt, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ launcher
def relaunch_under_torchrun(args):
    """`bench.py --gpus N` without a torchrun environment: re-exec this script as N
    ranks (one process per GPU) under torch.distributed.run on 127.0.0.1."""
    import socket
    n_dev = torch.cuda.device_count()
    if n_dev and args.gpus > n_dev and not SINGLE_DEVICE:
        sys.exit(f"bench.py: --gpus {args.gpus} but only {n_dev} CUDA device(s) are visible")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    if "NCCL_DEBUG" not in env:                   # INIT lines show every rank joining, on
        env["NCCL_DEBUG"] = "INFO"                # stderr: stdout carries only the JSON line
        env["NCCL_DEBUG_SUBSYS"] = "INIT"
        env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    sys.stdout.flush()
    os.execvpe(cmd[0], cmd, env)


def dry_launch(args):
    """The launcher path without a GPU (CPU test): every rank joins a gloo group and the
    ranks are counted with an all-reduce."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    n = torch.ones(1)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        dist.all_reduce(n)
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"dry_launch": True, "n_gpus": world, "ranks_counted": int(n.item())}), flush=True)


# Test hook for one-GPU boxes (tests/test_gpu_bench_multirank.py): every rank on cuda:0,
# a gloo process group, and the shared-history exchange done by the caller (exchange
# buffer -> torch all-reduce -> pf_commit_history) instead of the library's NCCL
# communicator (NCCL refuses two ranks on one device). Everything else is the N-rank path.
SINGLE_DEVICE = os.environ.get("PFBENCH_SINGLE_DEVICE") == "1"


def dist_setup(args):
    """(rank, world, local): WORLD_SIZE from torchrun; NCCL process group with device_id."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = 0 if SINGLE_DEVICE else int(os.environ.get("LOCAL_RANK", "0"))
    if SINGLE_DEVICE and world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("gloo")
        return rank, world, local
    if world != args.gpus:
        print(f"bench.py: WORLD_SIZE={world} overrides --gpus {args.gpus}", file=sys.stderr)
    if world > 1:
        import torch.distributed as dist
        if "NCCL_DEBUG" not in os.environ:
            os.environ["NCCL_DEBUG"] = "INFO"
            os.environ["NCCL_DEBUG_SUBSYS"] = "INIT"
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def bench_config(args, world):
    """The workload this run times: strong scaling = BASELINE's config split over the ranks;
    --weak = the config's instance count PER GPU (world × n instances in total)."""
    cfg = W.CONFIGS[args.config]
    if args.weak and world > 1:
        cfg = W.scaled(cfg, cfg.n_instances * world)
    return cfg


def share_nccl_id(rank, world):
    """Rank 0 creates the ncclUniqueId of the library-owned communicator (pf_nccl_unique_id)
    and broadcasts its 128 bytes over the torch process group."""
    import torch.distributed as dist
    from paper_2507_10150_b200 import nccl_unique_id
    buf = torch.zeros(128, dtype=torch.uint8, device="cuda")
    if rank == 0:
        buf.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(buf, 0)
    return bytes(buf.cpu().tolist())


def output_check(cfg, bd, adm, pk, pkr, estimate, bp):
    """Properties of the timed step's outputs that hold at any size (no oracle in the timed
    path): Alg.1's outputs are in range, M* >= current usage (tick 0 of Eq.(eq:3)), and the
    admitted peak respects the capacity rule while M* is monotone in p."""
    n = bd.n
    k = (bd.run_off[1:] - bd.run_off[:-1]).long()
    own = torch.repeat_interleave(torch.arange(n, device=bd.run_off.device), k)
    cur = torch.zeros(n, dtype=torch.int64, device=own.device).index_add_(
        0, own, (bd.input_len + bd.generated).long())
    peak_r = (pk if estimate else pkr).long()
    bad = int((peak_r < cur).sum())
    if not estimate:
        q = (bd.q_off[1:] - bd.q_off[:-1]).long()
        a, p, pr = adm.long(), pk.long(), pkr.long()
        cmax = ((10000 - bp) * bd.capacity.long()) // 10000
        bad += int(((a < 0) | (a > q)).sum())
        bad += int(((a > 0) & (p > cmax)).sum())          # admitted set fits
        bad += int((p < pr).sum())                        # M* monotone in admitted requests
        bad += int(((a == 0) & (p != pr)).sum())          # p* = 0 reports M*(R)
        pstar0 = int((a == 0).sum()); pall = int((a == q).sum())
        return {"violations": bad, "p_star_0": pstar0, "p_star_q": pall, "interior": n - pstar0 - pall}
    return {"violations": bad}


# ------------------------------------------------------------------ our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--weak", action="store_true", help="N>1: the config's instances per GPU (weak scaling)")
    ap.add_argument("--mode", type=int, default=0, help="0 sample (C-8 hash), 1 quantile")
    ap.add_argument("--bp", type=int, default=500, help="reserved ratio, basis points (paper: 3/5/10 %%)")
    ap.add_argument("--seed", type=int, default=0x5EED)
    ap.add_argument("--tick-pool", type=int, default=16, help="distinct completion sets cycled over steps")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dry-launch", action="store_true",
                    help="test hook: start the ranks (gloo), count them, print one line, no GPU work")
    args = ap.parse_args()
    assert args.warmup >= 3, "W >= 3 warm-up steps"
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args)
    if args.dry_launch:
        return dry_launch(args)

    rank, world, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, rank, world)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    if args.config == 1:
        return run_latency(args, rank, world, local)

    torch.cuda.set_device(local)
    cfg = bench_config(args, world)
    shards = owned_shards(cfg, rank, world) if cfg.shared else None
    bd = W.make_batch(cfg, rank=rank, nranks=world, device="cuda", shards=shards)
    torch.cuda.synchronize()
    nccl_id = share_nccl_id(rank, world) if (cfg.shared and world > 1 and not SINGLE_DEVICE) else None
    # cfg2's inputs (43 MB) and per-instance histograms (34 MB) fit the 126 MB L2: rotate
    # ROT independent (context, input set) pairs so no step finds the previous one's data
    rot = 9 if args.config == 2 else 1
    sets = [bd] + [bd.clone() for _ in range(rot - 1)]
    scheds = [scheduler_for(cfg, b_, rank, world, args.mode, args.bp, args.seed, nccl_id) for b_ in sets]
    sched = scheds[0]
    caller_exchange = bool(cfg.shared and world > 1 and nccl_id is None)  # (SINGLE_DEVICE test hook)

    def exchange(sc):
        if caller_exchange:
            import torch.distributed as dist
            dist.all_reduce(sc.exchange_buffer())
            sc.commit_history()

    exchange(sched)  # pf_create left the group tables for the caller's all-reduce
    pool = [W.make_completions(cfg, t, bd.row_ids) for t in range(args.tick_pool)]
    n = bd.n
    dev = "cuda"
    adm = torch.empty(n, dtype=torch.int32, device=dev)
    pk = torch.empty(n, dtype=torch.int32, device=dev)
    pkr = torch.empty(n, dtype=torch.int32, device=dev)
    estimate = cfg.q[1] == 0
    stream = torch.cuda.current_stream()

    def admit_call(sc, b_, t):
        if estimate:
            sc.estimate_peak(b_.run_off, b_.input_len, b_.generated, b_.max_new, t, peak_out=pk)
        else:
            sc.admit(b_.run_off, b_.input_len, b_.generated, b_.q_off, b_.q_input_len, b_.max_new,
                     b_.capacity, t, admitted_out=adm, peak_out=pk, peak_running_out=pkr)

    def step(t, ev=None):
        sc, b_ = scheds[t % rot], sets[t % rot]
        co, cl = pool[t % len(pool)]
        sc.update_history(co, cl)
        if ev is not None:
            ev[0].record(stream)
        admit_call(sc, b_, t)
        if ev is not None:
            ev[1].record(stream)

    # Shared mode (cfg 5): tick t+1's update_history (+ the library's NCCL all-reduce at
    # N > 1) / group tables run on a side stream while tick t's admit runs (the library
    # double-buffers the group tables, include/pfsched.h pf_commit_history); tables(t+2)
    # wait for admit(t).
    pipelined = bool(cfg.shared)
    # high priority: the side stream's few small CTAs dispatch as soon as admit CTAs retire,
    # instead of after all of admit's pending CTAs (tools/shard_probe.py: at P = 8 the
    # step − admit gap falls from 35 to 3 µs)
    side = torch.cuda.Stream(priority=-1) if pipelined else None
    tab_ready, admit_done = {}, {}

    def tables(t):
        with torch.cuda.stream(side):
            if t - 2 in admit_done:
                side.wait_event(admit_done.pop(t - 2))
            co, cl = pool[t % len(pool)]
            sched.update_history(co, cl)
            exchange(sched)
            e = torch.cuda.Event()
            e.record(side)
            tab_ready[t] = e

    def admit_only(t, ev=None):
        stream.wait_event(tab_ready.pop(t))
        if ev is not None:
            ev[0].record(stream)
        admit_call(sched, bd, t)
        if ev is not None:
            ev[1].record(stream)
        e = torch.cuda.Event()
        e.record(stream)
        admit_done[t] = e

    def run_steps(t0, n_, kev=None):
        # admit(t) is enqueued before tables(t+1): the host-side table flip happens at the
        # tables call, so admit(t) reads the half built for tick t
        if not pipelined:
            for j in range(n_):
                step(t0 + j, kev[j] if kev else None)
            return
        if t0 not in tab_ready:
            tables(t0)
        for j in range(n_):
            admit_only(t0 + j, kev[j] if kev else None)
            tables(t0 + j + 1)
        stream.wait_event(tab_ready[t0 + n_])  # the timed region holds n table builds too

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
    for sc in scheds:
        code, idx = sc.device_error()
        assert code == 0, f"device error {code} at {idx}"
    check = output_check(cfg, sets[(args.warmup + K - 1) % rot], adm, pk, pkr, estimate, args.bp)
    assert check["violations"] == 0, f"output check failed: {check}"

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
    traffic, traffic_src, inst = measured_traffic(args.config, world, args.weak)
    issue = None
    if inst and clk.get("sm_mhz"):
        # issue roofline next to the HBM one: the kernel's measured warp-instructions (ncu) per
        # launch ÷ its live launch time vs 4 warp-instructions per SM-cycle × SMs × SM clock
        sms = torch.cuda.get_device_properties(local).multi_processor_count
        peak_wi = 4 * sms * clk["sm_mhz"] * 1e6
        ach_wi = inst / (kern_ms * 1e-3)
        issue = {"achieved": ach_wi / 1e12, "peak": peak_wi / 1e12, "unit": "Twarp-instr/s",
                 "frac": ach_wi / peak_wi, "warp_instructions_per_launch": inst,
                 "per_instance": inst / n, "source": traffic_src}

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
            for k_, v in host.items():
                dsets[t % 2][k_].copy_(v, non_blocking=True)
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
        exchange(sched)
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

    cpu = cpu_fast = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        nt = os.cpu_count() or 1
        rs, rd, ns, ss, dt = cpu_oracle_rate(cfg, args.cpu_budget, nt, args.seed, args.bp, args.mode)
        cpu = {"value": rs, "unit": UNIT, "cores": nt, "kind": "oracle",
               "sample": f"{ns} evenly spaced instances ({ss} request-slots) of {cfg.name}, one admit "
                         f"tick, oracle as it stands (Alg.1 literal, tick-stepped M*) on {nt} threads, "
                         f"{dt:.1f} s", "decisions_per_s": rd}
        if cfg.q[1] > 0:
            try:
                fs, fn, fsl, fdt = cpu_fast_rate(cfg, 3.0, nt, args.seed, args.bp, args.mode)
                cpu_fast = {"value": fs, "unit": UNIT, "cores": nt,
                            "kind": "optimized CPU implementation (baselines/cpu_fast.cpp: O(1) lookups, "
                                    "sort-form M*, binary search over the prefix; not the oracle)",
                            "sample": f"{fn} evenly spaced instances ({fsl} request-slots), one admit tick, "
                                      f"{nt} threads, {fdt:.2f} s"}
            except Exception as ex:  # context only: never fail the bench line on it
                cpu_fast = {"unavailable": str(ex)[:200]}

    if rank == 0:
        if args.config == 2:
            l2 = (f"{rot} independent (context, input set) pairs rotated step by step: "
                  f"{rot} x {(abytes / 1e6):.0f} MB > 3 x 126 MB L2")
        else:
            l2 = f"inputs {abytes / 1e9:.2f} GB per rank > 126 MB L2 (no flush needed)"
        scaling = "weak" if (args.weak and world > 1) else "strong"
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": step_ms, "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
            "dtype": "int32", "data": "synthetic",
            "config": {"workload": cfg.describe(), "instances": int(decisions), "request_slots": int(slots),
                       "decisions_per_s": decisions / (step_ms * 1e-3), "mode": "sample" if args.mode == 0
                       else "quantile", "reserved_bp": args.bp,
                       "parallelism": f"instances sharded x{world}" + (
                           ", shared-history all-reduce by the library's NCCL communicator" if nccl_id else ""),
                       "l2": l2, "admit_kernel_ms": kern_ms,
                       "step": "update_history" + (" (+ NCCL all-reduce)" if nccl_id else "")
                       + (" + group tables" if cfg.shared else "") + " + " + ("estimate_peak" if estimate else "admit")
                       + (" (tick t+1's history/tables on a side stream, overlapping tick t's admit)" if pipelined else ""),
                       "output_check": check},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak_gbs, "unit": "GB/s",
                         "frac": achieved / peak_gbs, "traffic": traffic, "traffic_source": traffic_src,
                         "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": abytes,
                         "kernel": "admit_group_kernel" if (cfg.shared and os.environ.get("PFSCHED_GROUP_KERNEL", "1") != "0")
                         else "admit_kernel",
                         "frac_of_8TBs_spec": achieved / 8000.0, "issue": issue},
            "e2e": {"value": e2e_value, "unit": UNIT, "pipelined": "step t+1's H2D overlaps step t",
                    "h2d_bytes_per_step": int(h2d + h2d_c),
                    "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": (3 if cfg.shared else 2) * K,
            "clocks": clk,
        }
        if cpu:
            line["cpu_baseline"] = cpu
        if cpu_fast:
            line["cpu_fast"] = cpu_fast
    # release the library contexts (and their NCCL communicators) and the process group
    # before the JSON line, so nothing follows it on stdout
    for sc in scheds:
        sc.close()
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


def measured_traffic(config, world, weak):
    """ncu dram__bytes_read.sum + dram__bytes_write.sum per admit launch, from the ncu
    --set full capture of this config at N = 1 (profiles/admit_traffic.json), else None."""
    if world > 1 and not weak:
        return None, "not captured for a 1/N shard", None
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "admit_traffic.json")))
        e = d.get(f"cfg{config}")
        if isinstance(e, dict):
            return e.get("bytes"), e.get("source"), e.get("warp_instructions")
    except Exception:
        pass
    return None, "no ncu capture for this config", None


def run_latency(args, rank, world, local):
    """cfg1 (one hand-checkable instance, 8 running + 4 queued): latency per call, not a
    bandwidth number. Times update_history + admit through the C-ABI per call (host wall
    clock around a synchronised call, and device time by CUDA events)."""
    torch.cuda.set_device(local)
    b = W.config1_fixture()
    bd = b.to("cuda")
    cfg = b.cfg
    from paper_2507_10150_b200 import Scheduler
    sched = Scheduler(n_instances=1, window=cfg.window, max_len=cfg.max_len, max_input_len=cfg.max_input_len,
                      max_entries=cfg.max_entries, mode=args.mode, reserved_bp=args.bp, seed=args.seed,
                      init_history=bd.hist_rows.contiguous())
    co = torch.tensor([0, 1], dtype=torch.int32, device="cuda")
    cl = torch.tensor([1024], dtype=torch.int32, device="cuda")
    adm = torch.empty(1, dtype=torch.int32, device="cuda")
    pk = torch.empty_like(adm)
    stream = torch.cuda.current_stream()

    def call(t):
        sched.update_history(co, cl)
        sched.admit(bd.run_off, bd.input_len, bd.generated, bd.q_off, bd.q_input_len, bd.max_new,
                    bd.capacity, t, admitted_out=adm, peak_out=pk)

    for t in range(args.warmup):
        call(t)
    torch.cuda.synchronize()
    K = args.steps
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.15)
    e0.record(stream)
    for t in range(K):
        call(args.warmup + t)
    e1.record(stream)
    torch.cuda.synchronize()
    dev_ms = e0.elapsed_time(e1) / K
    walls = []
    for t in range(min(K, 200)):
        w0 = time.perf_counter()
        call(t)
        torch.cuda.synchronize()
        walls.append(time.perf_counter() - w0)
    clk = clocks.stop()
    sync_us = statistics.median(walls) * 1e6
    slots = b.slots()
    line = {"metric": METRIC, "value": slots / (dev_ms * 1e-3), "unit": UNIT, "n_gpus": 1, "steps": K,
            "warmup": args.warmup, "ms_per_step": dev_ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "int32", "data": "synthetic (SURVEY P-5 hand-checkable instance)",
            "config": {"workload": cfg.describe(), "latency_us_per_call_device": dev_ms * 1e3,
                       "latency_us_per_call_synchronous": sync_us, "admitted": int(adm.item()),
                       "peak": int(pk.item()), "l2": "latency-bound (4 KB): not a bandwidth number"},
            "roofline": None, "gpu_launches": 2 * K, "clocks": clk}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
