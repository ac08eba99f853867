"""The optimized CPU comparator (baselines/cpu_fast.cpp: sort-form M*, binary search over
the prefix) equals the oracle (literal Alg.1, tick-stepped M*) on every instance — a third
implementation of the same definitions, on CPU."""
import numpy as np
import pytest

import baselines
import workload as W
from harness import make_oracle, np32, oracle_admit


@pytest.mark.parametrize("c,n,mode,bp", [(2, 24, 0, 500), (3, 32, 1, 0), (4, 8, 0, 300), (5, 128, 0, 500),
                                         (5, 64, 1, 1000)])
def test_cpu_fast_equals_oracle(c, n, mode, bp):
    cfg = W.scaled(W.CONFIGS[c], n)
    b = W.make_batch(cfg)
    if cfg.q[1] == 0:  # estimate-only config: give every instance an empty queue and a capacity
        pytest.skip("estimate-only config has no queue (covered by the admit configs)")
    o = oracle_admit(make_oracle(b), b, mode=mode, bp=bp, seed=9, R=1, tick=3)
    adm, pk, pkr = baselines.admit(b, baselines.dist_rows_of(b), mode=mode, bp=bp, seed=9, tick=3)
    assert np.array_equal(adm, o["admitted"])
    assert np.array_equal(pk, o["peak"])
    assert np.array_equal(pkr, o["peak_running"])
