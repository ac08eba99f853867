"""GPU parity of cross-instance forwarding (pf_forward, NEXT-4) with the oracle
(oracle/pf_forward_oracle.cpp): destinations, forwarded counts and peaks bit for bit."""
import numpy as np
import pytest
import torch

import oracle as O
import workload as W
from harness import make_scheduler, np32

pytestmark = pytest.mark.gpu


def _run(cfg_id, n, S, mode, bp, tick=2, seed=13):
    cfg = W.scaled(W.CONFIGS[cfg_id], n)
    b = W.make_batch(cfg)
    bd = b.to("cuda")
    qo = np32(b.q_off)
    C = b.n // S
    cq_off = qo[::S][:C + 1].copy()
    sch = make_scheduler(bd, mode=mode, bp=bp, seed=seed, R=1)
    if tick:  # histories moved on by one update
        co, cl = W.make_completions(cfg, tick, b.row_ids)
        sch.update_history(co.cuda(), cl.cuda())
        hist = np32(sch.export_history())
    else:
        hist = np32(b.hist_rows)
    d, f, pk = sch.forward(S, bd.run_off, bd.input_len, bd.generated, bd.max_new, bd.capacity,
                           torch.from_numpy(cq_off).cuda(), bd.q_input_len[:int(cq_off[-1])].contiguous(), tick)
    od, of, opk = O.forward(cluster_size=S, windows=hist, run_off=np32(b.run_off), input_len=np32(b.input_len),
                            generated=np32(b.generated), max_new=np32(b.max_new), capacity=np32(b.capacity),
                            cq_off=cq_off, cq_input_len=np32(b.q_input_len)[:int(cq_off[-1])], mode=mode,
                            reserved_bp=bp, seed=seed, tick=tick, instance_base=int(b.inst_ids[0]),
                            max_entries=cfg.max_entries)
    assert np.array_equal(f.cpu().numpy(), of)
    assert np.array_equal(pk.cpu().numpy(), opk)
    assert np.array_equal(d.cpu().numpy(), od)
    assert sch.device_error() == (0, 0)
    return of


@pytest.mark.parametrize("cfg_id,n,S,mode,bp", [(4, 16, 1, 0, 500), (4, 16, 4, 0, 500), (4, 24, 8, 1, 300),
                                                (4, 32, 16, 0, 1000)])
def test_forward_parity(cfg_id, n, S, mode, bp):
    of = _run(cfg_id, n, S, mode, bp)
    assert of.sum() > 0


def test_forward_default_history_and_tick0():
    _run(4, 8, 2, 0, 500, tick=0)
