"""GPU parity: the CUDA path (through the C-ABI) vs the oracle, element by element,
bit-exact (all quantities are integer token counts / indices)."""
import json
import os

import numpy as np
import pytest
import torch

import oracle as O
import workload as W
from harness import (assert_same, gpu_admit, gpu_estimate, make_oracle, make_scheduler, np32,
                     oracle_admit)

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
ALL = ("admitted", "peak", "peak_running", "pred_run", "pred_q")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_config1_hand_example_and_p6_table():
    g = _gold("config1_p5.json")
    b = W.config1_fixture().to("cuda")
    for bp in (0, 300, 2000):
        s = make_scheduler(b, mode=1, bp=bp)
        out = gpu_admit(s, b, 0)
        assert list(out["pred_run"]) == g["expect_pred_running"]
        assert list(out["pred_q"]) == g["expect_pred_queue"]
        assert int(out["peak_running"][0]) == g["expect_peak_running"]
        assert int(out["admitted"][0]) == g["expect_admitted"][str(bp)]
        assert int(out["peak"][0]) == g["expect_peak_admitted"][str(bp)]
    s = make_scheduler(b, mode=0, bp=0, seed=0x2507101500000001)
    for t in g["sampling_mode_P6"]["ticks"]:
        out = gpu_admit(s, b, t["tick"])
        assert list(out["pred_run"]) == t["pred_running"]
        assert list(out["pred_q"]) == t["pred_queue"]
        assert int(out["peak_running"][0]) == t["peak_running"]
        assert int(out["admitted"][0]) == t["admitted"]
        assert int(out["peak"][0]) == t["peak_admitted"]


CASES = [
    # (config, instances, mode, bp, R)
    (2, 40, 0, 500, 1), (2, 24, 1, 0, 1),
    (3, 40, 0, 300, 1), (3, 16, 1, 0, 2),
    (4, 24, 0, 500, 1), (4, 12, 1, 1000, 3),
    (5, 128, 0, 500, 1), (5, 64, 1, 300, 2),
    (5, 64, 0, 500, 0), (2, 16, 0, 0, 0),  # R = 0: adaptive repetitions max(1, ceil(64/k))
]


@pytest.mark.parametrize("c,n,mode,bp,R", CASES)
def test_multi_tick_parity(c, n, mode, bp, R):
    cfg = W.scaled(W.CONFIGS[c], n)
    b = W.make_batch(cfg)
    bd = b.to("cuda")
    orc = make_oracle(b)
    s = make_scheduler(bd, mode=mode, bp=bp, seed=11 + c, R=R)
    for tick in range(3):
        if tick:
            co, cl = W.make_completions(cfg, tick, b.row_ids)
            st, _ = orc.update_history(np32(co), np32(cl))
            assert st == 0
            s.update_history(co.cuda(), cl.cuda())
        o = oracle_admit(orc, b, mode=mode, bp=bp, seed=11 + c, R=R, tick=tick, estimate=cfg.q[1] == 0)
        if cfg.q[1] == 0:
            g = gpu_estimate(s, bd, tick)
            assert_same(g, o, ("peak", "pred_run"), f"cfg{c} tick{tick}")
        else:
            g = gpu_admit(s, bd, tick)
            assert_same(g, o, ALL, f"cfg{c} tick{tick}")
            e = gpu_estimate(s, bd, tick)
            assert np.array_equal(e["peak"], g["peak_running"])
    hist = np32(s.export_history())
    for r in range(hist.shape[0]):
        assert np.array_equal(hist[r], orc.row(r)), f"history row {r}"
    assert s.device_error() == (0, 0)


def test_history_update_many_completions_and_errors():
    cfg = W.scaled(W.CONFIGS[4], 6)
    b = W.make_batch(cfg)
    bd = b.to("cuda")
    orc = make_oracle(b)
    s = make_scheduler(bd, mode=1)
    rng = np.random.default_rng(0)
    counts = np.array([0, 1, 5, 1200, 2500, 3])  # more completions than the window (w = 1000)
    comp = rng.integers(1, cfg.max_len + 1, size=counts.sum()).astype(np.int32)
    comp[-2] = cfg.max_len + 1  # invalid in the last row -> row unchanged
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    st, badrow = orc.update_history(off, comp)
    assert st == O.ORC_E_COMPLETION and badrow == 5
    s.update_history(torch.from_numpy(off).cuda(), torch.from_numpy(comp).cuda())
    assert s.device_error() == (1, 5)
    hist = np32(s.export_history())
    for r in range(6):
        assert np.array_equal(hist[r], orc.row(r)), r
    o = oracle_admit(orc, b, mode=1, bp=500, seed=7, R=1, tick=0)
    assert_same(gpu_admit(s, bd, 0), o, ALL)


def test_data_errors_give_minus_one():
    cfg = W.scaled(W.CONFIGS[2], 8)
    b = W.make_batch(cfg)
    b.generated[int(b.run_off[2]) + 3] = int(b.max_new[2])          # l_t >= max_new
    b.input_len[int(b.run_off[5])] = cfg.max_input_len + 1           # l_p too large
    b.capacity[6] = -5
    bd = b.to("cuda")
    orc = make_oracle(b)
    s = make_scheduler(bd, mode=0)
    g = gpu_admit(s, bd, 0)
    o = oracle_admit(orc, b, mode=0, bp=500, seed=7, R=1, tick=0)
    assert_same(g, o, ALL)
    assert g["admitted"][2] == g["admitted"][5] == g["admitted"][6] == -1
    code, idx = s.device_error()
    assert code in (4, 5, 6) and idx in (2, 5, 6)


def test_edge_cases_empty_and_ragged():
    # empty instances, running-only, queue-only, one entry, and maximum entries
    cfg = W.scaled(W.CONFIGS[4], 8)
    b = W.make_batch(cfg)
    k = np.array([0, 0, 1, 1024, 0, 7, 1024, 3])
    q = np.array([0, 5, 0, 256, 1, 0, 0, 256])
    rng = np.random.default_rng(1)
    lt = np.concatenate([rng.integers(0, 4096, size=x) for x in k]).astype(np.int32)
    lp = rng.integers(0, 4097, size=k.sum()).astype(np.int32)
    qlp = rng.integers(0, 4097, size=q.sum()).astype(np.int32)
    b.run_off = torch.from_numpy(np.concatenate([[0], np.cumsum(k)]).astype(np.int32))
    b.q_off = torch.from_numpy(np.concatenate([[0], np.cumsum(q)]).astype(np.int32))
    b.input_len, b.generated, b.q_input_len = map(torch.from_numpy, (lp, lt, qlp))
    b.capacity = torch.tensor([0, 10**6, 5, 4 * 10**6, 2, 10**5, 10**7, 2 * 10**6], dtype=torch.int32)
    bd = b.to("cuda")
    orc = make_oracle(b)
    for mode in (0, 1):
        s = make_scheduler(bd, mode=mode, bp=0)
        g = gpu_admit(s, bd, 3)
        o = oracle_admit(orc, b, mode=mode, bp=0, seed=7, R=1, tick=3)
        assert_same(g, o, ALL, f"mode{mode}")
        assert g["peak"][0] == 0 and g["admitted"][0] == 0


def test_ties_and_constant_history():
    # A constant window makes every prediction identical: many equal r (C-11 ties).
    cfg = W.scaled(W.CONFIGS[4], 10)
    b = W.make_batch(cfg)
    b.hist_rows[:] = 3000
    b.generated.clamp_(max=2999)
    bd = b.to("cuda")
    orc = make_oracle(b)
    for mode in (0, 1):
        s = make_scheduler(bd, mode=mode, bp=300)
        assert_same(gpu_admit(s, bd, 1), oracle_admit(orc, b, mode=mode, bp=300, seed=7, R=1, tick=1),
                    ALL, f"mode{mode}")


def test_default_init_history_is_max_len():
    cfg = W.scaled(W.CONFIGS[2], 4)
    b = W.make_batch(cfg)
    bd = b.to("cuda")
    s = make_scheduler(bd, init=False)
    assert bool((s.export_history() == cfg.max_len).all())
    b.hist_rows[:] = cfg.max_len
    orc = make_oracle(b)
    assert_same(gpu_admit(s, bd, 0), oracle_admit(orc, b, mode=0, bp=500, seed=7, R=1, tick=0), ALL)


@pytest.mark.parametrize("c", [2, 3, 4, 5])
def test_full_size_sampled_parity(c):
    """BASELINE.json full sizes, bench launch configuration; 48 sampled instances
    (plus first/last) compared one by one with the oracle."""
    cfg = W.CONFIGS[c]
    bd = W.make_batch(cfg, device="cuda")
    s = make_scheduler(bd, mode=0, bp=500, seed=3)
    tick = 1
    co, cl = W.make_completions(cfg, tick, bd.row_ids)
    s.update_history(co, cl)
    est = cfg.q[1] == 0
    g = gpu_estimate(s, bd, tick) if est else gpu_admit(s, bd, tick)
    rng = np.random.default_rng(c)
    pick = np.unique(np.concatenate([[0, cfg.n_instances - 1], rng.choice(cfg.n_instances, 48, replace=False)]))
    sub = W.make_batch(cfg, torch.from_numpy(pick))
    # oracle history for the sample: replay tick-1 completions on its rows
    orc = make_oracle(sub)
    co_s, cl_s = W.make_completions(cfg, tick, sub.row_ids)
    assert orc.update_history(np32(co_s), np32(cl_s))[0] == 0
    o = oracle_admit(orc, sub, mode=0, bp=500, seed=3, R=1, tick=tick, estimate=est)
    keys = ("peak",) if est else ("admitted", "peak", "peak_running")
    assert_same({k: g[k][pick] for k in keys}, o, keys, f"cfg{c} sampled")
    # predictions of the sampled instances
    ro = np32(bd.run_off)
    gp = np.concatenate([g["pred_run"][ro[i]:ro[i + 1]] for i in pick])
    assert np.array_equal(gp, o["pred_run"])
    assert s.device_error() == (0, 0)


@pytest.mark.parametrize("c", [3, 4, 5, 2])
def test_empty_conditional_support(c):
    # C-5: l_t at or above every history value -> l̂ = max_new. Every third running request
    # is moved to l_t = max_new - 1 (the kernel's sentinel past the end of the window).
    cfg = W.scaled(W.CONFIGS[c], 24)
    b = W.make_batch(cfg)
    for i in range(b.n):
        r0, r1 = int(b.run_off[i]), int(b.run_off[i + 1])
        b.generated[r0:r1:3] = int(b.max_new[i]) - 1
    bd = b.to("cuda")
    orc = make_oracle(b)
    for mode in (0, 1):
        s = make_scheduler(bd, mode=mode, bp=300)
        o = oracle_admit(orc, b, mode=mode, bp=300, seed=7, R=1, tick=1, estimate=cfg.q[1] == 0)
        if cfg.q[1] == 0:
            g = gpu_estimate(s, bd, 1)
            assert_same(g, o, ("peak", "pred_run"), f"cfg{c}")
        else:
            g = gpu_admit(s, bd, 1)
            assert_same(g, o, ALL, f"cfg{c}")
        pr = g["pred_run"]
        for i in range(b.n):
            r0 = int(b.run_off[i])
            if int(b.run_off[i + 1]) > r0:
                assert pr[r0] == int(b.max_new[i])
        assert s.device_error() == (0, 0)


@pytest.mark.parametrize("u", [0, 1, 0x7FFFFFFF, 0xFFFFFFFF])
@pytest.mark.parametrize("c", [2, 3, 5])
def test_quantile_extremes(c, u):
    # C-3: u = 0 is the smallest history value above l_t (upper_bound), u = 2^32 − 1 the
    # largest; both ends of ⌊u·n_gt / 2^32⌋ exercised for every layout (hist / sorted / group)
    cfg = W.scaled(W.CONFIGS[c], 24)
    b = W.make_batch(cfg)
    bd = b.to("cuda")
    orc = make_oracle(b)
    s = make_scheduler(bd, mode=1, bp=300, quantile_u=u)
    o = oracle_admit(orc, b, mode=1, bp=300, seed=7, R=1, tick=0, quantile_u=u, estimate=cfg.q[1] == 0)
    if cfg.q[1] == 0:
        assert_same(gpu_estimate(s, bd, 0), o, ("peak", "pred_run"), f"cfg{c} u={u:#x}")
    else:
        assert_same(gpu_admit(s, bd, 0), o, ALL, f"cfg{c} u={u:#x}")
    assert s.device_error() == (0, 0)
