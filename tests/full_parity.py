"""Full-coverage parity at BASELINE.json's full sizes.

Test infrastructure (a script under tests/, not collected by pytest: it needs minutes of
CPU oracle time). For each config it runs the CUDA path through the C-ABI on the WHOLE
batch, in the bench.py launch configuration, for T ticks (update_history -> admit), and
compares EVERY instance's outputs — p*, M*(admitted), M*(R), l̂ of every running and
every queued request — bit for bit with the oracle (oracle/pf_oracle.cpp: literal Alg.1,
tick-stepped M*, Eq.(eq:1)-(eq:3) PAPER.md:263-284), in instance
chunks so host memory stays bounded. cfg5 is additionally run as P = 8 ranks (eight
contexts on the one device, owned shards s mod 8, the caller-summed exchange buffer):
every rank's outputs must equal the P = 1 run (C-18 P-invariance).

  python tests/full_parity.py [--configs 2 3 4 5] [--ticks 2] [--out FILE]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

import oracle as O  # noqa: E402
import workload as W  # noqa: E402
from harness import make_oracle, make_scheduler, np32, oracle_admit  # noqa: E402
from workload.gen import owned_shards  # noqa: E402

MODE, BP, SEED, R = 0, 500, 0x5EED, 1  # bench.py's configuration (sampling mode, R = 1, 5 %);
# --mode / --bp / --R override them (e.g. quantile mode, adaptive repetitions R = 0)


def gpu_ticks(cfg, bd, ticks):
    """Yield (tick, outputs) for ticks 1..T on the whole batch (host numpy)."""
    s = make_scheduler(bd, mode=MODE, bp=BP, seed=SEED, R=R)
    n = bd.n
    est = cfg.q[1] == 0
    for t in range(1, ticks + 1):
        co, cl = W.make_completions(cfg, t, bd.row_ids)
        s.update_history(co, cl)
        pr = torch.full((max(int(bd.run_off[-1]), 1),), -7, dtype=torch.int32, device="cuda")
        if est:
            pk = s.estimate_peak(bd.run_off, bd.input_len, bd.generated, bd.max_new, t, pred_out=pr)
            out = {"peak": pk}
        else:
            pq = torch.full((max(int(bd.q_off[-1]), 1),), -7, dtype=torch.int32, device="cuda")
            pkr = torch.full((n,), -7, dtype=torch.int32, device="cuda")
            adm, pk = s.admit(bd.run_off, bd.input_len, bd.generated, bd.q_off, bd.q_input_len, bd.max_new,
                              bd.capacity, t, peak_running_out=pkr, pred_run_out=pr, pred_q_out=pq)
            out = {"admitted": adm, "peak": pk, "peak_running": pkr, "pred_q": pq[:int(bd.q_off[-1])]}
        out["pred_run"] = pr[:int(bd.run_off[-1])]
        torch.cuda.synchronize()
        yield t, {k: np32(v) for k, v in out.items()}
    assert s.device_error() == (0, 0)
    s.close()


def compare_chunked(cfg, t, g, chunk, ro, qo):
    """Oracle on every instance (chunks of `chunk`), tick t; returns mismatch counts."""
    est = cfg.q[1] == 0
    bad = {k: 0 for k in g}
    for c0 in range(0, cfg.n_instances, chunk):
        ids = torch.arange(c0, min(cfg.n_instances, c0 + chunk), dtype=torch.int64)
        sub = W.make_batch(cfg, ids)
        orc = make_oracle(sub)
        for tt in range(1, t + 1):
            co, cl = W.make_completions(cfg, tt, sub.row_ids)
            assert orc.update_history(np32(co), np32(cl))[0] == 0
        o = oracle_admit(orc, sub, mode=MODE, bp=BP, seed=SEED, R=R, tick=t, estimate=est)
        i0, i1 = c0, c0 + sub.n
        for k in g:
            if k == "pred_run":
                gv = g[k][ro[i0]:ro[i1]]
            elif k == "pred_q":
                gv = g[k][qo[i0]:qo[i1]]
            else:
                gv = g[k][i0:i1]
            bad[k] += int(np.count_nonzero(gv != np.asarray(o[k])))
        del orc
    return bad


def shared_p8(cfg, ticks, ref):
    """cfg5 as P = 8 ranks on one device; each rank's outputs vs the P = 1 outputs."""
    from paper_2507_10150_b200 import Scheduler
    P, M = 8, cfg.members_per_group
    ranks = []
    for r in range(P):
        bd = W.make_batch(cfg, rank=r, nranks=P, shards=owned_shards(cfg, r, P), device="cuda")
        s = Scheduler(n_instances=bd.n, window=cfg.window, max_len=cfg.max_len, max_input_len=cfg.max_input_len,
                      max_entries=cfg.max_entries, n_groups=cfg.n_groups, group_off=bd.group_off,
                      members_per_group=M, member_base=r * M // P, mode=MODE, reserved_bp=BP, seed=SEED, repetitions=R,
                      rank=r, nranks=P, init_history=bd.hist_rows)
        ranks.append((bd, s))

    def exchange():
        bufs = [s.exchange_buffer() for _, s in ranks]
        tot = torch.stack(bufs).sum(0, dtype=torch.int32)
        for b, (_, s) in zip(bufs, ranks):
            b.copy_(tot)
            s.commit_history()

    exchange()
    bad = 0
    for t in range(1, ticks + 1):
        for bd, s in ranks:
            co, cl = W.make_completions(cfg, t, bd.row_ids)
            s.update_history(co, cl)
        exchange()
        for bd, s in ranks:
            adm, pk = s.admit(bd.run_off, bd.input_len, bd.generated, bd.q_off, bd.q_input_len, bd.max_new,
                              bd.capacity, t)
            ids = bd.inst_ids.cpu().numpy()
            bad += int(np.count_nonzero(np32(adm) != ref[t]["admitted"][ids]))
            bad += int(np.count_nonzero(np32(pk) != ref[t]["peak"][ids]))
    for _, s in ranks:
        assert s.device_error() == (0, 0)
        s.close()
    return bad


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[2, 3, 4, 5])
    ap.add_argument("--ticks", type=int, default=2)
    ap.add_argument("--chunk", type=int, default=1 << 14)
    ap.add_argument("--scale", type=int, default=0, help="smoke run: this many instances per config")
    ap.add_argument("--mode", type=int, default=0, help="0 sampling (C-8), 1 quantile (u = 2^31)")
    ap.add_argument("--bp", type=int, default=500)
    ap.add_argument("--R", type=int, default=1, help="repetitions (0 = adaptive max(1, ceil(64/k)))")
    ap.add_argument("--no-p8", action="store_true")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "full_parity.json"))
    a = ap.parse_args()
    global MODE, BP, R
    MODE, BP, R = a.mode, a.bp, a.R
    O.build_oracle()
    torch.cuda.set_device(0)
    results = []
    for c in a.configs:
        cfg = W.CONFIGS[c] if not a.scale else W.scaled(W.CONFIGS[c], a.scale)
        t0 = time.time()
        bd = W.make_batch(cfg, device="cuda")
        ro, qo = np32(bd.run_off), np32(bd.q_off)
        ref = {}
        for t, g in gpu_ticks(cfg, bd, a.ticks):
            if cfg.shared:
                ref[t] = {"admitted": g["admitted"], "peak": g["peak"]}
            bad = compare_chunked(cfg, t, g, a.chunk, ro, qo)
            rec = {"config": cfg.name, "tick": t, "instances": cfg.n_instances,
                   "running_requests": int(ro[-1]), "queued_requests": int(qo[-1]),
                   "outputs_compared": sorted(g), "mismatches": bad, "seconds": round(time.time() - t0, 1)}
            print(json.dumps(rec), flush=True)
            results.append(rec)
        if cfg.shared and not a.no_p8:
            del bd
            torch.cuda.empty_cache()
            bad8 = shared_p8(cfg, a.ticks, ref)
            rec = {"config": cfg.name, "check": "P=8 ranks (8 contexts, summed exchange) == P=1, every instance, "
                   f"ticks 1..{a.ticks}", "mismatches": bad8}
            print(json.dumps(rec), flush=True)
            results.append(rec)
    total = sum(sum(r["mismatches"].values()) if isinstance(r["mismatches"], dict) else r["mismatches"]
                for r in results)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump({"mode": MODE, "reserved_bp": BP, "seed": SEED, "R": R, "ticks": a.ticks,
                   "total_mismatches": total, "cores": os.cpu_count(), "results": results}, f, indent=1)
    print(json.dumps({"total_mismatches": total}))
    sys.exit(1 if total else 0)


if __name__ == "__main__":
    main()
