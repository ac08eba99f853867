"""Shared-history mode across ranks.

Group g's window is the union of 8 fixed shard rings; shard s is owned by rank
s mod P; after each update the ranks sum their owned-shard group histograms
(all-reduce). Results must not depend on P.

* CPU (gloo, world_size 2): the host-side sharding + all-reduce logic with the
  oracle — the reduced histogram equals the P=1 window's histogram, and every
  rank's admission results equal the P=1 oracle's for its instances.
* GPU (one device, two contexts as two ranks): the C-ABI shared-mode protocol
  pf_update_history -> (sum of exchange buffers) -> pf_commit_history -> pf_admit
  reproduces the single-rank oracle bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import workload as W
from workload.gen import local_instance_ids, owned_shards

CFG = W.scaled(W.CONFIGS[5], 64 * 8)  # 64 groups x 8 members (divisible by P = 8)
TICKS = 2


def _np(t):
    return t.detach().cpu().numpy().astype(np.int32)


def _p1_reference():
    """P = 1: the oracle with all 8 shard rows per group, after TICKS updates."""
    b = W.make_batch(CFG)
    orc = O.Oracle(b.hist_rows.shape[0], CFG.row_window, CFG.max_len, CFG.shards, _np(b.hist_rows))
    for t in range(1, TICKS + 1):
        co, cl = W.make_completions(CFG, t, b.row_ids)
        assert orc.update_history(_np(co), _np(cl))[0] == 0
    hist = np.zeros((CFG.n_groups, CFG.max_len + 1), np.int64)
    for g in range(CFG.n_groups):
        for s in range(CFG.shards):
            np.add.at(hist[g], orc.row(g * CFG.shards + s), 1)
    return b, orc, hist


def _admit(orc, b, tick):
    return orc.admit(dist_of=_np(b.dist_of), inst_id=b.inst_ids.numpy(), run_off=_np(b.run_off),
                     input_len=_np(b.input_len), generated=_np(b.generated), max_new=_np(b.max_new),
                     q_off=_np(b.q_off), q_input_len=_np(b.q_input_len), capacity=_np(b.capacity),
                     mode=0, reserved_bp=500, seed=11, tick=tick, max_input_len=CFG.max_input_len,
                     max_entries=CFG.max_entries)


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shards = owned_shards(CFG, rank, world)
    b = W.make_batch(CFG, rank=rank, nranks=world, shards=shards)
    # local oracle over the owned shard rows only (rows_per_dist = shards owned)
    orc_local = O.Oracle(b.hist_rows.shape[0], CFG.row_window, CFG.max_len, len(shards), _np(b.hist_rows))
    for t in range(1, TICKS + 1):
        co, cl = W.make_completions(CFG, t, b.row_ids)
        assert orc_local.update_history(_np(co), _np(cl))[0] == 0
    part = torch.zeros((CFG.n_groups, CFG.max_len + 1), dtype=torch.int64)
    for g in range(CFG.n_groups):
        for x in range(len(shards)):
            part[g] += torch.bincount(torch.from_numpy(orc_local.row(g * len(shards) + x)).long(),
                                      minlength=CFG.max_len + 1)
    dist.all_reduce(part)  # H_g = Σ_ranks Σ_owned shards
    # the group window as one row expanded from H_g (order is irrelevant to P(l))
    rows = [np.repeat(np.arange(CFG.max_len + 1), part[g].numpy()).astype(np.int32)
            for g in range(CFG.n_groups)]
    orc = O.Oracle(CFG.n_groups, CFG.window, CFG.max_len, 1, np.stack(rows))
    o = _admit(orc, b, TICKS)
    out[rank] = (part.numpy(), b.inst_ids.numpy(), o["admitted"], o["peak"], o["peak_running"])
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_gloo_two_ranks_match_single_rank():
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    b, orc, hist = _p1_reference()
    ref = _admit(orc, b, TICKS)
    ids = b.inst_ids.numpy()
    seen = []
    for rank in range(2):
        part, inst, adm, peak, prun = out[rank]
        assert np.array_equal(part, hist), "all-reduced histogram != single-rank window"
        pos = np.searchsorted(ids, inst)
        assert np.array_equal(ids[pos], inst)
        assert np.array_equal(adm, ref["admitted"][pos])
        assert np.array_equal(peak, ref["peak"][pos])
        assert np.array_equal(prun, ref["peak_running"][pos])
        seen.append(inst)
    assert np.array_equal(np.sort(np.concatenate(seen)), ids)


@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 4, 8])
def test_gpu_shared_mode_ranks_on_one_device(P):
    from paper_2507_10150_b200 import Scheduler
    b, orc, _ = _p1_reference()
    ref = _admit(orc, b, TICKS)
    ids = b.inst_ids.numpy()
    scheds, batches = [], []
    M = CFG.members_per_group
    for rank in range(P):
        shards = owned_shards(CFG, rank, P)
        bd = W.make_batch(CFG, rank=rank, nranks=P, shards=shards, device="cuda")
        s = Scheduler(n_instances=bd.n, window=CFG.window, max_len=CFG.max_len,
                      max_input_len=CFG.max_input_len, max_entries=CFG.max_entries, n_groups=CFG.n_groups,
                      group_off=bd.group_off, members_per_group=M, member_base=rank * M // P, mode=0,
                      reserved_bp=500, seed=11, rank=rank, nranks=P, init_history=bd.hist_rows)
        scheds.append(s)
        batches.append(bd)

    def exchange():
        bufs = [s.exchange_buffer() for s in scheds]
        total = torch.stack(bufs).sum(0, dtype=torch.int32)
        for buf, s in zip(bufs, scheds):
            buf.copy_(total)
            s.commit_history()

    exchange()  # tables after pf_create
    for t in range(1, TICKS + 1):
        for s, bd in zip(scheds, batches):
            co, cl = W.make_completions(CFG, t, bd.row_ids)
            s.update_history(co, cl)
        exchange()
    for s, bd in zip(scheds, batches):
        adm, pk = s.admit(bd.run_off, bd.input_len, bd.generated, bd.q_off, bd.q_input_len, bd.max_new,
                          bd.capacity, TICKS)
        torch.cuda.synchronize()
        pos = np.searchsorted(ids, bd.inst_ids.cpu().numpy())
        assert np.array_equal(_np(adm), ref["admitted"][pos])
        assert np.array_equal(_np(pk), ref["peak"][pos])
        assert s.device_error() == (0, 0)


def _pipelined_worker(rank, world, port, out):
    """One rank of the bench.py schedule on cuda:0: admit(t) on the main stream while
    update(t+1) -> all-reduce(exchange buffer) -> commit runs on a side stream."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2507_10150_b200 import Scheduler
    torch.cuda.set_device(0)
    M = CFG.members_per_group
    shards = owned_shards(CFG, rank, world)
    bd = W.make_batch(CFG, rank=rank, nranks=world, shards=shards, device="cuda")
    s = Scheduler(n_instances=bd.n, window=CFG.window, max_len=CFG.max_len,
                  max_input_len=CFG.max_input_len, max_entries=CFG.max_entries, n_groups=CFG.n_groups,
                  group_off=bd.group_off, members_per_group=M, member_base=rank * M // world, mode=0,
                  reserved_bp=500, seed=11, rank=rank, nranks=world, init_history=bd.hist_rows)
    xbuf = s.exchange_buffer()
    dist.all_reduce(xbuf)
    s.commit_history()
    main, side = torch.cuda.current_stream(), torch.cuda.Stream()
    ready, done, res = {}, {}, []
    slow = torch.empty(1 << 24, dtype=torch.int32, device="cuda")

    def tables(t):
        with torch.cuda.stream(side):
            if t - 2 in done:
                side.wait_event(done.pop(t - 2))
            co, cl = W.make_completions(CFG, t, bd.row_ids)
            s.update_history(co.cuda(), cl.cuda())
            dist.all_reduce(xbuf)
            s.commit_history()
            e = torch.cuda.Event()
            e.record(side)
            ready[t] = e

    tables(1)
    for t in range(1, PIPE_TICKS + 1):
        main.wait_event(ready.pop(t))
        slow.add_(1)
        adm = torch.full((bd.n,), -7, dtype=torch.int32, device="cuda")
        pk = torch.full_like(adm, -7)
        s.admit(bd.run_off, bd.input_len, bd.generated, bd.q_off, bd.q_input_len, bd.max_new,
                bd.capacity, t, admitted_out=adm, peak_out=pk)
        res.append((adm, pk))
        e = torch.cuda.Event()
        e.record(main)
        done[t] = e
        if t < PIPE_TICKS:
            tables(t + 1)
    torch.cuda.synchronize()
    out[rank] = (bd.inst_ids.cpu().numpy(), [(_np(a), _np(p)) for a, p in res], s.device_error())
    dist.destroy_process_group()


PIPE_TICKS = 4


@pytest.mark.gpu
def test_gpu_two_processes_pipelined_exchange():
    """bench.py's N > 1 schedule (side-stream exchange overlapping admit, double-buffered
    group tables) with a real all-reduce between two processes (gloo, one device):
    every tick equals the single-rank oracle."""
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_pipelined_worker, args=(2, port, out), nprocs=2, join=True)
    b = W.make_batch(CFG)
    orc = O.Oracle(b.hist_rows.shape[0], CFG.row_window, CFG.max_len, CFG.shards, _np(b.hist_rows))
    ids = b.inst_ids.numpy()
    refs = []
    for t in range(1, PIPE_TICKS + 1):
        co, cl = W.make_completions(CFG, t, b.row_ids)
        assert orc.update_history(_np(co), _np(cl))[0] == 0
        refs.append(_admit(orc, b, t))
    for rank in range(2):
        inst, res, err = out[rank]
        assert err == (0, 0)
        pos = np.searchsorted(ids, inst)
        for t, (adm, pk) in enumerate(res):
            assert np.array_equal(adm, refs[t]["admitted"][pos]), f"rank {rank} tick {t + 1}"
            assert np.array_equal(pk, refs[t]["peak"][pos]), f"rank {rank} tick {t + 1}"
