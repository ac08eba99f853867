"""GPU parity for (1) the theoretical-optimum override (A12, PAPER.md:341/:395:
admission with the true output lengths), checked against the oracle's literal
Alg.1 (orc_admit_one, tick-stepped M*), and (2) bin pile-ups that exercise every
exact-refinement path of the sort-free M* evaluation (candidate bins with more
members than a warp, many candidate bins at once)."""
import numpy as np
import pytest
import torch

import oracle as O
import workload as W
from harness import assert_same, gpu_admit, gpu_estimate, make_oracle, make_scheduler, np32, oracle_admit

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("c,n", [(5, 128), (4, 12), (2, 24)])
def test_override_matches_literal_algorithm1(c, n):
    cfg = W.scaled(W.CONFIGS[c], n)
    b = W.make_batch(cfg)
    rng = np.random.default_rng(c)
    lt = np32(b.generated)
    lhat_run = (lt + rng.integers(1, cfg.max_len + 1, size=lt.size)).clip(max=cfg.max_len)
    lhat_run = np.maximum(lhat_run, lt + 1).astype(np.int32)  # l_t < l̂ ≤ Lmax
    nq = int(b.q_off[-1])
    lhat_q = rng.integers(1, cfg.max_len + 1, size=max(nq, 1)).astype(np.int32)[:nq]
    bd = b.to("cuda")
    s = make_scheduler(bd, mode=0, bp=300)
    pr = torch.empty(bd.n, dtype=torch.int32, device="cuda")
    adm, pk = s.admit_override(bd.run_off, bd.input_len, bd.generated, torch.from_numpy(lhat_run).cuda(),
                               bd.q_off, bd.q_input_len, torch.from_numpy(lhat_q).cuda(), bd.capacity,
                               peak_running_out=pr)
    torch.cuda.synchronize()
    ro, qo = np32(b.run_off), np32(b.q_off)
    lp, qlp, cap = np32(b.input_len), np32(b.q_input_len), np32(b.capacity)
    for i in range(b.n):
        rs, qs = slice(ro[i], ro[i + 1]), slice(qo[i], qo[i + 1])
        a_r = lp[rs] + lt[rs]
        r_r = lhat_run[rs] - lt[rs]
        p, pk_o, pr_o = O.admit_one(a_r, r_r, qlp[qs], lhat_q[qs], int(cap[i]), 300)
        assert (int(adm[i]), int(pk[i]), int(pr[i])) == (p, pk_o, pr_o), f"instance {i}"
    assert s.device_error() == (0, 0)


def test_override_rejects_prediction_not_above_generated():
    cfg = W.scaled(W.CONFIGS[4], 4)
    b = W.make_batch(cfg)
    lt = np32(b.generated)
    lhat = (lt + 1).astype(np.int32)
    lhat[int(b.run_off[2])] = lt[int(b.run_off[2])]  # l̂ = l_t in instance 2
    bd = b.to("cuda")
    s = make_scheduler(bd)
    lq = torch.full((int(b.q_off[-1]),), 100, dtype=torch.int32, device="cuda")
    adm, pk = s.admit_override(bd.run_off, bd.input_len, bd.generated, torch.from_numpy(lhat).cuda(),
                               bd.q_off, bd.q_input_len, lq, bd.capacity)
    torch.cuda.synchronize()
    assert int(adm[2]) == -1 and int(pk[2]) == -1 and int(adm[0]) >= 0
    assert s.device_error() == (7, 2)


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("c,n,lo,hi", [(5, 64, 3000, 3127), (4, 8, 2100, 2160), (3, 8, 4000, 4095),
                                         (2, 16, 1500, 1563)])
def test_bin_pileups_refine_exactly(mode, c, n, lo, hi):
    """History confined to a narrow range: l̂ concentrates in one or two wide bins, so
    candidate bins hold far more members than a warp and many bins qualify."""
    cfg = W.scaled(W.CONFIGS[c], n)
    b = W.make_batch(cfg)
    rng = np.random.default_rng(7)
    b.hist_rows = torch.from_numpy(rng.integers(lo, hi + 1, size=tuple(b.hist_rows.shape)).astype(np.int32))
    b.generated = torch.from_numpy(rng.integers(0, 40, size=b.generated.numel()).astype(np.int32))
    cur = torch.zeros(b.n, dtype=torch.int64).index_add_(
        0, torch.repeat_interleave(torch.arange(b.n), torch.diff(b.run_off.long())),
        (b.input_len + b.generated).long())
    b.capacity = (cur * 13 // 10).to(torch.int32)
    bd = b.to("cuda")
    orc = make_oracle(b)
    sch = make_scheduler(bd, mode=mode, bp=0)
    estimate = cfg.q[1] == 0
    g = gpu_estimate(sch, bd, 5) if estimate else gpu_admit(sch, bd, 5)
    o = oracle_admit(orc, b, mode=mode, bp=0, seed=7, R=1, tick=5, estimate=estimate)
    keys = ("peak", "pred_run") if estimate else ("admitted", "peak", "peak_running", "pred_run", "pred_q")
    assert_same(g, o, keys, f"cfg{c} pileup")


@pytest.mark.parametrize("c", [3, 5])
def test_whole_instance_in_one_bin(c):
    """Constant history and constant l_t: every request of an instance has the same r, so
    one bin holds all of them (512 for cfg 3: the 10-bit count field of the packed bin
    words is full at N = 512; cfg 5: up to 480 in a 9-bit field)."""
    cfg = W.scaled(W.CONFIGS[c], 8)
    b = W.make_batch(cfg)
    b.hist_rows = torch.full(tuple(b.hist_rows.shape), 4000, dtype=torch.int32)
    b.generated = torch.full((b.generated.numel(),), 10, dtype=torch.int32)
    cur = torch.zeros(b.n, dtype=torch.int64).index_add_(
        0, torch.repeat_interleave(torch.arange(b.n), torch.diff(b.run_off.long())),
        (b.input_len + b.generated).long())
    b.capacity = (cur * 3 // 2).to(torch.int32)
    bd = b.to("cuda")
    orc = make_oracle(b)
    estimate = cfg.q[1] == 0
    for mode in (0, 1):
        sch = make_scheduler(bd, mode=mode, bp=0)
        g = gpu_estimate(sch, bd, 3) if estimate else gpu_admit(sch, bd, 3)
        o = oracle_admit(orc, b, mode=mode, bp=0, seed=7, R=1, tick=3, estimate=estimate)
        keys = ("peak", "pred_run") if estimate else ("admitted", "peak", "peak_running", "pred_run", "pred_q")
        assert_same(g, o, keys, f"cfg{c} one bin")
        assert sch.device_error() == (0, 0)
