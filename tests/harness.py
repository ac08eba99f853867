"""Test helpers: drive the CUDA path (through the C-ABI binding) and the oracle on the
same seeded workload buffers, tick by tick. Test infrastructure only."""
from __future__ import annotations

import numpy as np
import torch

import oracle as O
import workload as W


def np32(t):
    return t.detach().cpu().numpy().astype(np.int32)


def make_oracle(batch: W.Batch) -> O.Oracle:
    cfg = batch.cfg
    rows = np32(batch.hist_rows)
    return O.Oracle(rows.shape[0], cfg.row_window, cfg.max_len, cfg.shards if cfg.shared else 1, rows)


def make_scheduler(batch_dev: W.Batch, *, mode=0, bp=500, seed=7, R=1, quantile_u=0x80000000,
                   rank=0, nranks=1, init=True):
    from paper_2507_10150_b200 import Scheduler
    cfg = batch_dev.cfg
    kw = {}
    if cfg.shared:
        M = cfg.members_per_group
        kw = dict(n_groups=cfg.n_groups, group_off=batch_dev.group_off, members_per_group=M,
                  member_base=int(batch_dev.inst_ids[0].item()) % M if batch_dev.n else 0)
    else:
        kw = dict(instance_base=int(batch_dev.inst_ids[0].item()) if batch_dev.n else 0)
    return Scheduler(n_instances=batch_dev.n, window=cfg.window, max_len=cfg.max_len,
                     max_input_len=cfg.max_input_len, max_entries=cfg.max_entries, mode=mode,
                     quantile_u=quantile_u, repetitions=R, reserved_bp=bp, seed=seed, rank=rank,
                     nranks=nranks, init_history=batch_dev.hist_rows.contiguous() if init else None,
                     **kw)


def oracle_admit(orc: O.Oracle, b: W.Batch, *, mode, bp, seed, R, tick, quantile_u=0x80000000,
                 estimate=False):
    cfg = b.cfg
    kw = dict(dist_of=np32(b.dist_of), inst_id=b.inst_ids.cpu().numpy(), run_off=np32(b.run_off),
              input_len=np32(b.input_len), generated=np32(b.generated), max_new=np32(b.max_new),
              mode=mode, quantile_u=quantile_u, repetitions=R, reserved_bp=bp, seed=seed, tick=tick,
              max_input_len=cfg.max_input_len, max_entries=cfg.max_entries, want_pred=True)
    if not estimate:
        kw.update(q_off=np32(b.q_off), q_input_len=np32(b.q_input_len), capacity=np32(b.capacity))
    return orc.admit(**kw)


def gpu_admit(sched, bd: W.Batch, tick):
    n = bd.n
    dev = bd.run_off.device
    pk_run = torch.full((n,), -7, dtype=torch.int32, device=dev)
    pr = torch.full((max(int(bd.run_off[-1]), 1),), -7, dtype=torch.int32, device=dev)
    pq = torch.full((max(int(bd.q_off[-1]), 1),), -7, dtype=torch.int32, device=dev)
    adm, pk = sched.admit(bd.run_off, bd.input_len, bd.generated, bd.q_off, bd.q_input_len, bd.max_new,
                          bd.capacity, tick, peak_running_out=pk_run, pred_run_out=pr, pred_q_out=pq)
    torch.cuda.synchronize()
    return {"admitted": np32(adm), "peak": np32(pk), "peak_running": np32(pk_run),
            "pred_run": np32(pr)[:int(bd.run_off[-1])], "pred_q": np32(pq)[:int(bd.q_off[-1])]}


def gpu_estimate(sched, bd: W.Batch, tick):
    pr = torch.full((max(int(bd.run_off[-1]), 1),), -7, dtype=torch.int32, device=bd.run_off.device)
    pk = sched.estimate_peak(bd.run_off, bd.input_len, bd.generated, bd.max_new, tick, pred_out=pr)
    torch.cuda.synchronize()
    return {"peak": np32(pk), "pred_run": np32(pr)[:int(bd.run_off[-1])]}


def assert_same(gpu: dict, orc: dict, keys, ctx=""):
    for k in keys:
        g, o = np.asarray(gpu[k]), np.asarray(orc[k])
        assert g.shape == o.shape, f"{ctx} {k}: shape {g.shape} vs {o.shape}"
        bad = np.nonzero(g != o)[0]
        assert bad.size == 0, (f"{ctx} {k}: {bad.size} mismatches, first at {bad[:5]}: "
                               f"gpu {g[bad[:5]]} oracle {o[bad[:5]]}")
