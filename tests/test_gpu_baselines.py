"""GPU parity of the paper's comparison policies (aggressive watermark, conservative
overcommit) against the oracle, per instance."""
import numpy as np
import pytest

import oracle as O
import workload as W
from harness import make_scheduler, np32

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("c,n", [(5, 128), (4, 16), (2, 32)])
@pytest.mark.parametrize("policy,ratios", [(1, (9000, 9500, 9900)), (2, (10000, 15000))])
def test_baseline_policies_match_oracle(c, n, policy, ratios):
    from paper_2507_10150_b200 import PF_POLICY_AGGRESSIVE
    cfg = W.scaled(W.CONFIGS[c], n)
    b = W.make_batch(cfg)
    bd = b.to("cuda")
    s = make_scheduler(bd)
    ro, qo = np32(b.run_off), np32(b.q_off)
    lp, lt, ql, mx, cap = map(np32, (b.input_len, b.generated, b.q_input_len, b.max_new, b.capacity))
    for ratio in ratios:
        adm, used = s.admit_baseline(policy, ratio, bd.run_off, bd.input_len, bd.generated, bd.q_off,
                                     bd.q_input_len, bd.max_new, bd.capacity)
        adm, used = np32(adm), np32(used)
        for i in range(b.n):
            rs, qs = slice(ro[i], ro[i + 1]), slice(qo[i], qo[i + 1])
            if policy == PF_POLICY_AGGRESSIVE:
                ref = O.admit_aggressive(lp[rs], lt[rs], ql[qs], int(cap[i]), ratio)
            else:
                ref = O.admit_conservative(lp[rs], ql[qs], int(mx[i]), int(cap[i]), ratio)
            assert (int(adm[i]), int(used[i])) == ref, (i, ratio)
    assert s.device_error() == (0, 0)
