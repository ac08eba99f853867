"""The synthetic generator: deterministic, addressable per instance, and shaped like
the paper's workloads (PAPER.md:307 Distribution-1/2/3 ranges, :403 max_new 2048)."""
import torch

import workload as W
from workload.gen import local_instance_ids, owned_shards


def test_deterministic_and_subset_addressable():
    cfg = W.scaled(W.CONFIGS[4], 12)
    a = W.make_batch(cfg)
    b = W.make_batch(cfg)
    for f in ("input_len", "generated", "q_input_len", "capacity", "hist_rows"):
        assert torch.equal(getattr(a, f), getattr(b, f))
    sub = W.make_batch(cfg, torch.tensor([3, 7]))
    k = int(a.run_off[1])
    assert torch.equal(sub.input_len[:k], a.input_len[3 * k:4 * k])
    assert torch.equal(sub.hist_rows[1], a.hist_rows[7])
    assert torch.equal(sub.capacity, a.capacity[[3, 7]])


def test_ranges_match_paper_distributions():
    for c, lp_rng, L_rng in ((4, (32, 4096), (2048, 4096)), (3, (2048, 4096), (32, 4096))):
        b = W.make_batch(W.scaled(W.CONFIGS[c], 16))
        assert lp_rng[0] <= int(b.input_len.min()) and int(b.input_len.max()) <= lp_rng[1]
        assert L_rng[0] <= int(b.hist_rows.min()) and int(b.hist_rows.max()) <= L_rng[1]
        assert int(b.generated.min()) >= 0 and int(b.generated.max()) < int(b.max_new.max())
    b = W.make_batch(W.scaled(W.CONFIGS[2], 8))
    assert int(b.hist_rows.max()) <= 2048 and int(b.hist_rows.min()) >= 1
    assert int(b.input_len.min()) >= 4 and int(b.input_len.max()) <= 2047


def test_config5_ragged_and_group_major():
    cfg = W.scaled(W.CONFIGS[5], 128)
    b = W.make_batch(cfg)
    k = torch.diff(b.run_off)
    q = torch.diff(b.q_off)
    assert int(k.min()) >= 128 and int(k.max()) <= 384 and int(q.min()) >= 32 and int(q.max()) <= 96
    assert torch.equal(b.dist_of.long(), b.inst_ids // cfg.members_per_group)
    assert b.hist_rows.shape == (64 * 8, cfg.row_window)
    # class = group mod 4: group 0 chat (max_new 2048), group 1 D1 (4096), group 2 D2 (5120)
    assert int(b.max_new[0]) == 2048 and int(b.max_new[2]) == 4096 and int(b.max_new[4]) == 5120


def test_rank_sharding_partitions_instances_and_shards():
    cfg = W.scaled(W.CONFIGS[5], 64 * 8)
    allids = local_instance_ids(cfg, 0, 1)
    for P in (2, 4, 8):
        ids = torch.cat([local_instance_ids(cfg, r, P) for r in range(P)])
        assert torch.equal(ids.sort().values, allids.sort().values)
        sh = sorted(s for r in range(P) for s in owned_shards(cfg, r, P))
        assert sh == list(range(8))


def test_completions_deterministic():
    cfg = W.scaled(W.CONFIGS[4], 10)
    rows = torch.arange(10)
    o1, l1 = W.make_completions(cfg, 3, rows)
    o2, l2 = W.make_completions(cfg, 3, rows)
    assert torch.equal(o1, o2) and torch.equal(l1, l2)
    if l1.numel():
        assert int(l1.min()) >= 2048 and int(l1.max()) <= 4096
