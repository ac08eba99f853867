"""GPU: tick t+1's history update / group-table rebuild on a second stream, overlapping
tick t's admit (double-buffered group tables, include/pfsched.h pf_commit_history; the
schedule bench.py times) gives exactly the per-tick results of the serial schedule, and
both equal the oracle."""
import numpy as np
import pytest
import torch

import workload as W
from harness import assert_same, make_oracle, make_scheduler, np32, oracle_admit

pytestmark = pytest.mark.gpu
KEYS = ("admitted", "peak", "peak_running")


def _outs(n):
    return [torch.full((n,), -7, dtype=torch.int32, device="cuda") for _ in range(3)]


def test_pipelined_ticks_equal_serial_and_oracle():
    cfg = W.scaled(W.CONFIGS[5], 256)
    b = W.make_batch(cfg)
    bd = b.to("cuda")
    T = 6
    pool = [W.make_completions(cfg, t, b.row_ids) for t in range(T + 1)]
    pool_d = [(co.cuda(), cl.cuda()) for co, cl in pool]

    def admit(s, t, outs):
        adm, pk, pkr = outs
        s.admit(bd.run_off, bd.input_len, bd.generated, bd.q_off, bd.q_input_len, bd.max_new,
                bd.capacity, t, admitted_out=adm, peak_out=pk, peak_running_out=pkr)

    def update(s, t):
        co, cl = pool_d[t]
        s.update_history(co, cl)  # nranks == 1: rebuilds (and flips) the group tables

    # serial schedule
    s1 = make_scheduler(bd, mode=0, bp=500)
    serial = []
    for t in range(1, T + 1):
        update(s1, t)
        o = _outs(bd.n)
        admit(s1, t, o)
        serial.append(o)
    torch.cuda.synchronize()

    # pipelined schedule: admit(t) on the main stream, update/tables(t+1) on a side stream
    s2 = make_scheduler(bd, mode=0, bp=500)
    main, side = torch.cuda.current_stream(), torch.cuda.Stream()
    ready, done, piped = {}, {}, []
    slow = torch.empty(1 << 24, dtype=torch.int32, device="cuda")

    def tables(t):
        with torch.cuda.stream(side):
            if t - 2 in done:
                side.wait_event(done.pop(t - 2))
            update(s2, t)
            e = torch.cuda.Event()
            e.record(side)
            ready[t] = e

    tables(1)
    for t in range(1, T + 1):
        main.wait_event(ready.pop(t))
        slow.add_(1)  # keep the main stream busy so the side stream really runs ahead
        o = _outs(bd.n)
        admit(s2, t, o)
        piped.append(o)
        e = torch.cuda.Event()
        e.record(main)
        done[t] = e
        if t < T:
            tables(t + 1)
    torch.cuda.synchronize()
    for t in range(T):
        for a, c in zip(serial[t], piped[t]):
            assert torch.equal(a, c), f"tick {t + 1}"

    orc = make_oracle(b)
    for t in range(1, T + 1):
        co, cl = pool[t]
        st, _ = orc.update_history(np32(co), np32(cl))
        assert st == 0
        o = oracle_admit(orc, b, mode=0, bp=500, seed=7, R=1, tick=t)
        g = {"admitted": np32(piped[t - 1][0]), "peak": np32(piped[t - 1][1]),
             "peak_running": np32(piped[t - 1][2])}
        assert_same(g, o, KEYS, f"tick {t}")
    assert s2.device_error() == (0, 0)
