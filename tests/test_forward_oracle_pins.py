"""Pins for the forwarding oracle (oracle/pf_forward_oracle.cpp, NEXT-4, PAPER.md:459;
readings F-1..F-4 in DESIGN.md §13): a hand-computed cluster, the one-instance
cluster that must equal Alg.1 admission, and invariants."""
import numpy as np
import pytest

import oracle as O
import workload as W
from harness import make_oracle, np32, oracle_admit


def test_hand_cluster():
    """Quantile mode, every window = {10}: every prediction is 10.
    A: running (l_p 50, l_t 2) -> (a 52, r 8), M* 60, M = 100; B: (20, 5) -> (25, 5), M* 30, M = 60.
    j1 (l_p 10 -> (10, 10)): A 52+8+10+8 = 78 (headroom 22), B 30+15 = 45 (15) -> A.
    j2 (10):  A 96 (4), B 45 (15) -> B.   j3 (30): A 134 > 100, B 80 > 60 -> stop; j4 -> -1."""
    d, f, pk = O.forward(cluster_size=2, windows=np.full((2, 4), 10), run_off=[0, 1, 2],
                         input_len=[50, 20], generated=[2, 5], max_new=[16, 16], capacity=[100, 60],
                         cq_off=[0, 4], cq_input_len=[10, 10, 30, 1], mode=1)
    assert list(d) == [0, 1, -1, -1] and list(f) == [2] and list(pk) == [78, 45]


def test_single_instance_cluster_is_alg1():
    cfg = W.scaled(W.CONFIGS[4], 12)
    b = W.make_batch(cfg)
    orc = make_oracle(b)
    for mode, bp in ((0, 500), (1, 300)):
        o = oracle_admit(orc, b, mode=mode, bp=bp, seed=5, R=1, tick=3)
        d, f, pk = O.forward(cluster_size=1, windows=np32(b.hist_rows), run_off=np32(b.run_off),
                             input_len=np32(b.input_len), generated=np32(b.generated),
                             max_new=np32(b.max_new), capacity=np32(b.capacity), cq_off=np32(b.q_off),
                             cq_input_len=np32(b.q_input_len), mode=mode, reserved_bp=bp, seed=5,
                             tick=3, instance_base=int(b.inst_ids[0]))
        assert np.array_equal(f, o["admitted"])
        assert np.array_equal(pk, o["peak"])
        qo = np32(b.q_off)
        for i in range(b.n):
            seg = d[qo[i]:qo[i + 1]]
            assert np.all(seg[:f[i]] == 0) and np.all(seg[f[i]:] == -1)


@pytest.mark.parametrize("S", [2, 4, 8])
def test_cluster_invariants(S):
    cfg = W.scaled(W.CONFIGS[4], 16)
    b = W.make_batch(cfg)
    C = b.n // S
    qo = np32(b.q_off)
    # the cluster queue of cluster c = the queues of its instances, concatenated
    cq_off = qo[::S][:C + 1]
    cap = np32(b.capacity)
    d, f, pk = O.forward(cluster_size=S, windows=np32(b.hist_rows), run_off=np32(b.run_off),
                         input_len=np32(b.input_len), generated=np32(b.generated), max_new=np32(b.max_new),
                         capacity=cap, cq_off=cq_off, cq_input_len=np32(b.q_input_len), seed=9,
                         reserved_bp=500, tick=1, instance_base=int(b.inst_ids[0]),
                         max_entries=cfg.max_entries)
    for c in range(C):
        seg = d[cq_off[c]:cq_off[c + 1]]
        assert np.all(seg[:f[c]] >= 0) and np.all(seg[:f[c]] < S) and np.all(seg[f[c]:] == -1)
    # every instance that received a request fits its bound after forwarding
    got = np.zeros(b.n, bool)
    for c in range(C):
        for s in d[cq_off[c]:cq_off[c] + f[c]]:
            got[c * S + s] = True
    assert np.all(pk[got].astype(np.int64) * 10000 <= (10000 - 500) * cap[got].astype(np.int64))
    assert f.sum() > 0
