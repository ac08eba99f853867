"""GPU parity for every admit-kernel variant the public ABI can select, and for the
context / communicator plumbing.

Variants (include/pfsched.h, pfsched.cu kVariants): team width TW = 1/2/4/8 warps by
max_entries (≤512 / ≤1024 / ≤2048 / ≤4096), three history layouts (per-instance sorted
window w ≤ Lmax+1, per-instance histogram w > Lmax+1, shared groups) and packed or
unpacked bin words (unpacked: Lmax ≥ 8192, or k+q ≥ 1024). Every case is compared with
the oracle element by element over two ticks (history update included)."""
import dataclasses

import numpy as np
import pytest
import torch

import workload as W
from harness import assert_same, gpu_admit, make_oracle, make_scheduler, np32, oracle_admit
from workload.gen import CHAT, D1, D3, MIXED, WorkloadConfig

pytestmark = pytest.mark.gpu
ALL = ("admitted", "peak", "peak_running", "pred_run", "pred_q")


def _cfg(name, n, k, q, window, max_len, cls, n_groups=0, seed=0x2507101500000100):
    return WorkloadConfig(name, n, k, q, window, max_len, cls, n_groups=n_groups, seed=seed)


VARIANTS = [
    # TW = 2 (513..1024 requests): sorted / histogram / group layouts, unpacked bins
    ("tw2_sorted", _cfg("tw2s", 6, (520, 700), (100, 300), 1000, 4096, D1)),
    ("tw2_hist", _cfg("tw2h", 6, (520, 700), (100, 300), 5000, 4096, D3)),
    ("tw2_group", _cfg("tw2g", 8, (520, 700), (100, 300), 8 * 250, 5120, MIXED, n_groups=4)),
    # TW = 8 (2049..4096 requests)
    ("tw8_sorted", _cfg("tw8s", 3, (2500, 3500), (100, 500), 1000, 4096, D1)),
    ("tw8_group", _cfg("tw8g", 4, (2500, 3500), (100, 500), 8 * 250, 5120, MIXED, n_groups=4)),
    # TW = 1 unpacked (Lmax >= 8192: records cannot pack r in 13 bits)
    ("tw1_unpacked_sorted", _cfg("tw1us", 16, (100, 300), (20, 100), 1000, 10000, D1)),
    ("tw1_unpacked_hist", _cfg("tw1uh", 16, (100, 300), (20, 100), 12000, 10000, CHAT)),
    ("tw1_unpacked_group", _cfg("tw1ug", 8, (100, 300), (20, 100), 8 * 250, 9000, MIXED, n_groups=4)),
    # TW = 1, histogram layout with a large Lmax: 4 teams of 4·(Lmax+1) B tables do not fit
    # 227 KB, so the context packs fewer teams per CTA
    ("tw1_hist_big_lmax", _cfg("tw1hb", 8, (60, 120), (10, 40), 30000, 20000, CHAT)),
]


@pytest.mark.parametrize("name,cfg", VARIANTS, ids=[v[0] for v in VARIANTS])
@pytest.mark.parametrize("mode", [0, 1])
def test_variant_parity(name, cfg, mode):
    b = W.make_batch(cfg)
    bd = b.to("cuda")
    orc = make_oracle(b)
    s = make_scheduler(bd, mode=mode, bp=300, seed=5)
    for tick in range(2):
        if tick:
            co, cl = W.make_completions(cfg, tick, b.row_ids)
            assert orc.update_history(np32(co), np32(cl))[0] == 0
            s.update_history(co.cuda(), cl.cuda())
        o = oracle_admit(orc, b, mode=mode, bp=300, seed=5, R=1, tick=tick)
        assert_same(gpu_admit(s, bd, tick), o, ALL, f"{name} tick{tick}")
    assert s.device_error() == (0, 0)
    s.close()


def test_two_live_contexts_of_different_sizes():
    """The kernel attributes are process-wide: creating a smaller context of the same
    variant after a larger one must not break the larger one's launches."""
    big = W.scaled(W.CONFIGS[5], 128)                                    # max_entries 480
    small = dataclasses.replace(big, k=(20, 40), q=(4, 8), name="small")  # max_entries 48
    bb, bs = W.make_batch(big), W.make_batch(small)
    db, ds = bb.to("cuda"), bs.to("cuda")
    sb = make_scheduler(db, mode=0, bp=500, seed=9)
    ss = make_scheduler(ds, mode=0, bp=500, seed=9)   # same kernel variant, smaller footprint
    for b, d, s in ((bb, db, sb), (bs, ds, ss), (bb, db, sb)):
        o = oracle_admit(make_oracle(b), b, mode=0, bp=500, seed=9, R=1, tick=0)
        assert_same(gpu_admit(s, d, 0), o, ALL, b.cfg.name)
    sb.close()
    ss.close()


def test_library_owned_nccl_communicator_one_rank():
    """§8(b): a context that owns its NCCL communicator (nccl_unique_id; forced with one
    rank on the single GPU) all-reduces inside pf_update_history; results equal the
    oracle, and pf_commit_history is refused (the library already did it)."""
    from paper_2507_10150_b200 import PFError, nccl_unique_id
    cfg = W.scaled(W.CONFIGS[5], 64 * 4)
    b = W.make_batch(cfg)
    bd = b.to("cuda")
    orc = make_oracle(b)
    from paper_2507_10150_b200 import Scheduler
    M = cfg.members_per_group
    s = Scheduler(n_instances=bd.n, window=cfg.window, max_len=cfg.max_len, max_input_len=cfg.max_input_len,
                  max_entries=cfg.max_entries, n_groups=cfg.n_groups, group_off=bd.group_off,
                  members_per_group=M, member_base=0, mode=0, reserved_bp=500, seed=13, rank=0, nranks=1,
                  init_history=bd.hist_rows, nccl_id=nccl_unique_id())
    for tick in range(3):
        if tick:
            co, cl = W.make_completions(cfg, tick, b.row_ids)
            assert orc.update_history(np32(co), np32(cl))[0] == 0
            s.update_history(co.cuda(), cl.cuda())
        o = oracle_admit(orc, b, mode=0, bp=500, seed=13, R=1, tick=tick)
        assert_same(gpu_admit(s, bd, tick), o, ALL, f"nccl tick{tick}")
    with pytest.raises(PFError):
        s.commit_history()
    assert s.device_error() == (0, 0)
    s.close()


def test_admit_before_first_commit_is_refused():
    """nranks > 1 without a library communicator: the group tables exist only after the
    caller's all-reduce + pf_commit_history; earlier admits return PF_ESTATE."""
    from paper_2507_10150_b200 import PFError, Scheduler
    cfg = W.scaled(W.CONFIGS[5], 64 * 2)
    bd = W.make_batch(cfg, rank=0, nranks=2, shards=[0, 2, 4, 6], device="cuda")
    s = Scheduler(n_instances=bd.n, window=cfg.window, max_len=cfg.max_len, max_input_len=cfg.max_input_len,
                  max_entries=cfg.max_entries, n_groups=cfg.n_groups, group_off=bd.group_off,
                  members_per_group=cfg.members_per_group, member_base=0, mode=0, reserved_bp=500, seed=1,
                  rank=0, nranks=2, init_history=bd.hist_rows)
    with pytest.raises(PFError, match="status -3"):
        s.admit(bd.run_off, bd.input_len, bd.generated, bd.q_off, bd.q_input_len, bd.max_new, bd.capacity, 0)
    with pytest.raises(PFError, match="status -3"):
        s.estimate_peak(bd.run_off, bd.input_len, bd.generated, bd.max_new, 0)
    s.commit_history()  # (one rank's partial sums: enough to lift the state check)
    s.admit(bd.run_off, bd.input_len, bd.generated, bd.q_off, bd.q_input_len, bd.max_new, bd.capacity, 0)
    torch.cuda.synchronize()
    s.close()
