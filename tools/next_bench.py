"""Device timings of the §8(f) NEXT rows on one B200 (CUDA events on the launching
stream, after warm-up): the comparison policies and the override path on the cfg-5
batch, the continuous-batching simulator, the window-similarity analysis on a
BurstGPT-sized trace and cross-instance forwarding. Bytes are algorithmic (what each
call must read and write), peaks from MEASURED_PEAKS.json.

Usage: python tools/next_bench.py [--out profiles/r01/next_rows.txt]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2507_10150_b200 as P  # noqa: E402
import workload as W  # noqa: E402
import workload.sim as S  # noqa: E402
from workload.gen import CHAT, D1, D2, D3  # noqa: E402


def timed(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps / 1e3  # seconds


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    peak_gbs, src = bench.peaks()
    lines = [f"# NEXT-row device timings, one B200; HBM peak {peak_gbs} GB/s ({src})"]

    def emit(s):
        print(s, flush=True)
        lines.append(s)

    # ---- NEXT-1 on the cfg-5 batch (2^20 instances, 335.8 M request slots)
    cfg = W.CONFIGS[5]
    bd = W.make_batch(cfg, device="cuda")
    sch = bench.scheduler_for(cfg, bd, 0, 1, 0, 500, 0x5EED)
    n, nr, nq = bd.n, int(bd.run_off[-1]), int(bd.q_off[-1])
    adm = torch.empty(n, dtype=torch.int32, device="cuda")
    used = torch.empty_like(adm)
    for name, pol in (("aggressive 99%", P.PF_POLICY_AGGRESSIVE), ("conservative 100%", P.PF_POLICY_CONSERVATIVE)):
        t = timed(lambda: sch.admit_baseline(pol, 9900 if pol == P.PF_POLICY_AGGRESSIVE else 10000, bd.run_off,
                                             bd.input_len, bd.generated, bd.q_off, bd.q_input_len, bd.max_new,
                                             bd.capacity, admitted_out=adm, used_out=used))
        B = 8 * nr + 4 * nq + 4 * (n + 1) * 2 + 8 * n + 8 * n
        emit(f"NEXT-1 baseline {name:18s} cfg5: {t * 1e3:7.3f} ms  {(nr + nq) / t:.3g} slots/s  "
             f"{B / t / 1e9:7.0f} GB/s = {B / t / 1e9 / peak_gbs:.1%} of HBM")
    lhr = (bd.generated + 1).contiguous()
    lhq = torch.ones(nq, dtype=torch.int32, device="cuda") * 64
    pk = torch.empty_like(adm)
    t = timed(lambda: sch.admit_override(bd.run_off, bd.input_len, bd.generated, lhr, bd.q_off, bd.q_input_len,
                                         lhq, bd.capacity, admitted_out=adm, peak_out=pk))
    B = 12 * nr + 8 * nq + 4 * (n + 1) * 2 + 4 * n + 8 * n
    emit(f"NEXT-1 override (A12)               cfg5: {t * 1e3:7.3f} ms  {(nr + nq) / t:.3g} slots/s  "
         f"{B / t / 1e9:7.0f} GB/s = {B / t / 1e9 / peak_gbs:.1%} of HBM")
    del sch, bd
    torch.cuda.empty_cache()

    # ---- NEXT-2 simulator: 256 D1 instances x 200 requests, paper scale
    w = S.make_sim_workload(D1, 256, 200, div=1, slots=16, window=1000)
    d = {k: (v.cuda() if torch.is_tensor(v) else v) for k, v in w.items()}
    for pol, bp, name in ((P.PF_SIM_PAST_FUTURE, 500, "past-future 5%"), (P.PF_SIM_AGGRESSIVE, 9500, "aggressive 95%")):
        sim = P.Simulator(req_off=d["req_off"], req_input=d["req_input"], req_output=d["req_output"],
                          max_new=d["max_new"], capacity=d["capacity"], policy=pol, param_bp=bp, window=1000,
                          max_len=w["max_len"], max_input_len=w["max_input_len"], max_entries=256,
                          init_history=d["init_history"], seed=1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        it = sim.run(chunk=1024)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        m = sim.metrics()[0].sum(0).tolist()
        emit(f"NEXT-2 simulator {name:15s} 256 x 200 D1 requests: {it} iterations in {dt:.2f} s = "
             f"{it / dt:.0f} iterations/s, {m[0] / dt:.3g} instance-iterations/s (CUDA-graph replays, 6 kernels/iter)")
        sim.close()

    # ---- NEXT-3 analysis on a BurstGPT-sized trace
    x = S.make_length_stream([CHAT, D1, D2, D3, CHAT, D3, D1], 200000).cuda()
    N, wlen = x.numel(), 1000
    Bw = N // wlen
    t = timed(lambda: P.window_similarity(x, wlen, 5120), reps=5, warm=1)
    emit(f"NEXT-3 window_similarity 1.4 M lengths, {Bw} windows of {wlen}: {t * 1e3:7.2f} ms  "
         f"{Bw * N / t:.3g} histogram lookups/s (includes the synchronous input check)")
    t = timed(lambda: P.adjacent_similarity(x, 1000, 250, 5120), reps=5, warm=1)
    emit(f"NEXT-3 adjacent_similarity h=1000 r=250: {t * 1e3:7.2f} ms")

    # ---- NEXT-4 forwarding: cfg-4 shaped instances in clusters of 8
    cfg4 = W.scaled(W.CONFIGS[4], 4096)
    b4 = W.make_batch(cfg4, device="cuda")
    s4 = bench.scheduler_for(cfg4, b4, 0, 1, 0, 500, 7)
    Sz = 8
    cq_off = b4.q_off[::Sz][:4096 // Sz + 1].contiguous()
    qn = int(cq_off[-1])
    t = timed(lambda: s4.forward(Sz, b4.run_off, b4.input_len, b4.generated, b4.max_new, b4.capacity, cq_off,
                                 b4.q_input_len[:qn].contiguous(), 1), reps=5, warm=1)
    d4, f4, _ = s4.forward(Sz, b4.run_off, b4.input_len, b4.generated, b4.max_new, b4.capacity, cq_off,
                           b4.q_input_len[:qn].contiguous(), 1)
    emit(f"NEXT-4 forward 4096 cfg4 instances (1024 running each) in clusters of {Sz}, {qn} queued: "
         f"{t * 1e3:7.2f} ms, {int(f4.sum())} forwarded ({int(f4.sum()) / t:.3g} forwarded/s)")
    if a.out:
        with open(a.out, "w") as f:
            f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
