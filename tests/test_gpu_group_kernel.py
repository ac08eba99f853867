"""GPU parity for the shared-mode admit_group_kernel (pf_admit_group.cuh):
the persistent CTA-per-SM kernel with the group tables staged in shared memory, its
group-segment walk and the cost-weighted CTA ranges (per-group cycles of the previous
launch); and the unpacked shared-mode contexts that keep admit_kernel. Every case is
compared element by element with the oracle (Alg.1; Eq.(eq:1)-(eq:3),
PAPER.md:263-284) over several ticks, so later launches run on measured partitions."""
import os

import numpy as np
import pytest
import torch

import workload as W
from harness import assert_same, gpu_admit, gpu_estimate, make_oracle, make_scheduler, np32, oracle_admit
from workload.gen import MIXED, WorkloadConfig

pytestmark = pytest.mark.gpu
ALL = ("admitted", "peak", "peak_running", "pred_run", "pred_q")


def _irregular_ids(cfg, counts, member_base=2):
    """Local instances of group g are members member_base .. member_base + counts[g] − 1
    (the shared-mode id rule of include/pfsched.h); counts may be 0 (empty groups)."""
    M = cfg.members_per_group
    return torch.cat([g * M + member_base + torch.arange(c, dtype=torch.int64)
                      for g, c in enumerate(counts)])


def _ticks(cfg, b, bd, s, orc, ticks, mode=0, bp=500, seed=7, R=1, ctx=""):
    for tick in range(ticks):
        if tick:
            co, cl = W.make_completions(cfg, tick, b.row_ids)
            st, _ = orc.update_history(np32(co), np32(cl))
            assert st == 0
            s.update_history(co.cuda(), cl.cuda())
        o = oracle_admit(orc, b, mode=mode, bp=bp, seed=seed, R=R, tick=tick)
        g = gpu_admit(s, bd, tick)
        assert_same(g, o, ALL, f"{ctx} tick{tick}")
        e = gpu_estimate(s, bd, tick)
        assert np.array_equal(e["peak"], g["peak_running"]), f"{ctx} tick{tick} estimate"
    assert s.device_error() == (0, 0)


@pytest.mark.parametrize("mode", [0, 1])
def test_irregular_and_empty_groups(mode):
    """Group segments of very different sizes, empty groups between them, and CTA ranges
    that start and end inside groups (grid = min(SMs, n))."""
    cfg = W.scaled(W.CONFIGS[5], 64 * 40)  # M = 40 members per group
    rng = np.random.default_rng(5)
    counts = rng.integers(0, 38, size=cfg.n_groups)
    counts[[0, 3, 4, 17, 63]] = 0
    counts[[9, 30]] = 38
    b = W.make_batch(cfg, inst_ids=_irregular_ids(cfg, counts))
    assert (np.diff(np32(b.group_off)) == counts).all()
    bd = b.to("cuda")
    orc = make_oracle(b)
    s = make_scheduler(bd, mode=mode)
    _ticks(cfg, b, bd, s, orc, 4, mode=mode, ctx=f"mode{mode}")


def test_group_kernel_equals_admit_kernel():
    """The same inputs through admit_group_kernel and through admit_kernel
    (PFSCHED_GROUP_KERNEL=0 at context creation): identical outputs, both = oracle."""
    cfg = W.scaled(W.CONFIGS[5], 4096)
    b = W.make_batch(cfg)
    bd = b.to("cuda")
    orc = make_oracle(b)
    old = os.environ.get("PFSCHED_GROUP_KERNEL")
    try:
        os.environ["PFSCHED_GROUP_KERNEL"] = "0"
        s0 = make_scheduler(bd, mode=0, seed=3)
    finally:
        if old is None:
            os.environ.pop("PFSCHED_GROUP_KERNEL", None)
        else:
            os.environ["PFSCHED_GROUP_KERNEL"] = old
    s1 = make_scheduler(bd, mode=0, seed=3)
    for tick in range(3):
        if tick:
            co, cl = W.make_completions(cfg, tick, b.row_ids)
            orc.update_history(np32(co), np32(cl))
            s0.update_history(co.cuda(), cl.cuda())
            s1.update_history(co.cuda(), cl.cuda())
        g0, g1 = gpu_admit(s0, bd, tick), gpu_admit(s1, bd, tick)
        for key in ALL:
            assert np.array_equal(g0[key], g1[key]), f"tick{tick} {key}"
        assert_same(g1, oracle_admit(orc, b, mode=0, bp=500, seed=3, R=1, tick=tick), ALL, f"tick{tick}")


def test_many_groups_uniform_partition():
    """G = 300 > 256: no per-group cost buffers, CTA ranges by instance count; groups of 3
    members, so every CTA walks several group segments (one table staging each)."""
    cfg = WorkloadConfig("g300", 300 * 3, (20, 120), (5, 40), 8 * 100, 5120, MIXED, n_groups=300,
                         seed=0x2507101500000300)
    b = W.make_batch(cfg)
    bd = b.to("cuda")
    orc = make_oracle(b)
    s = make_scheduler(bd, mode=0, bp=200)
    _ticks(cfg, b, bd, s, orc, 3, bp=200, ctx="G300")


def test_unpacked_shared_mode_uses_admit_kernel():
    """Lmax ≥ 8192: records and bin words cannot be packed, so a shared-mode context keeps
    admit_kernel (L1-cached tables); a 64,000-entry group window (S_g 128 KB) on the way."""
    cfg = WorkloadConfig("bigtab", 2 * 6, (10, 60), (2, 20), 8 * 8000, 30000, MIXED, n_groups=2,
                         seed=0x2507101500000301)
    b = W.make_batch(cfg)
    bd = b.to("cuda")
    orc = make_oracle(b)
    s = make_scheduler(bd, mode=0, bp=0)
    _ticks(cfg, b, bd, s, orc, 2, bp=0, ctx="bigtab")


def test_data_errors_shared_mode():
    """Data-dependent violations inside the group kernel: that instance's outputs are −1,
    the sticky error word names one of them, every other instance is exact."""
    cfg = W.scaled(W.CONFIGS[5], 64 * 4)
    b = W.make_batch(cfg)
    b.generated[int(b.run_off[7]) + 3] = int(b.max_new[7])           # l_t >= max_new
    b.input_len[int(b.run_off[100])] = cfg.max_input_len + 1          # l_p too large
    b.q_input_len[int(b.q_off[150])] = -4                             # queued l_p < 0
    b.capacity[200] = -5
    bd = b.to("cuda")
    orc = make_oracle(b)
    s = make_scheduler(bd, mode=0)
    g = gpu_admit(s, bd, 0)
    assert_same(g, oracle_admit(orc, b, mode=0, bp=500, seed=7, R=1, tick=0), ALL)
    for i in (7, 100, 150, 200):
        assert g["admitted"][i] == -1 and g["peak"][i] == -1, i
    code, idx = s.device_error()
    assert code in (4, 5, 6) and idx in (7, 100, 150, 200)


def test_cost_partition_over_many_launches():
    """Twelve launches on one context: the rotating cost buffers are read, zeroed and
    refilled every launch; every launch stays exact (the partition never changes results)."""
    cfg = W.scaled(W.CONFIGS[5], 64 * 64)
    b = W.make_batch(cfg)
    bd = b.to("cuda")
    orc = make_oracle(b)
    s = make_scheduler(bd, mode=0)
    o = oracle_admit(orc, b, mode=0, bp=500, seed=7, R=1, tick=5)
    for rep in range(12):
        assert_same(gpu_admit(s, bd, 5), o, ALL, f"launch{rep}")
