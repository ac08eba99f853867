"""Pins for the simulator oracle (oracle/pf_sim_oracle.cpp, NEXT-2; readings S-1..S-9 in
DESIGN.md §11): hand-stepped traces, policy equivalences that hold by construction,
end-to-end invariants, and Table 1's ordinal structure."""
import numpy as np
import pytest

import oracle as O
import workload.sim as S
from workload.gen import CHAT, D1, D2, D3

M = {name: c for c, name in enumerate(O.SIM_METRICS)}


def run(req_input, req_output, *, cap, max_new, policy, bp=0, window=4, E=8, iters=1000, **kw):
    m, g, e = O.sim_run(req_off=[0, len(req_input)], req_input=req_input, req_output=req_output,
                        max_new=[max_new], capacity=[cap], policy=policy, param_bp=bp, window=window,
                        max_len=max_new, max_entries=E, iterations=iters, **kw)
    return dict(zip(O.SIM_METRICS, m[0].tolist())), g, e


def test_single_request_walkthrough():
    # l_p = 4, L = 3, M = 100. t0: admit, decode -> 5 tokens; t1 -> 6; t2 -> 7; t3: finish.
    # consumed 5 + 6 + 7 = 18; future M* (true): 4+3, 5+2, 6+1 = 7 each -> 21.
    m, g, e = run([4], [3], cap=100, max_new=10, policy=O.SIM_OPTIMUM)
    assert m == dict(iterations=3, decode_steps=3, evictions=0, finished=1, consumed_sum=18,
                     future_sum=21, samples=3, future_max=7, forced=0, admissions=1)
    assert list(g) == [3] and list(e) == [0]


def test_fig_peak_scenario():
    """PAPER.md:286 narrative (fig:peak), as a run: M = 21; A (l_p 7, L 3), B (3, 5),
    C (4, 3). Hand-stepped (S-2..S-8):
    aggressive (watermark 100 %): t0 admits A, B, C (7+3+4 = 14 ≤ 21); occupancy 17, 20,
      then t2 needs 20 + 3 = 23 > 21 -> evict C (LIFO), re-queued with 2 tokens; t3 A
      finishes, C re-admitted (6 + 6 ≤ 21); t4 C finishes; t5 B finishes.
      consumed 17+20+16+14+8 = 75; future 23+23+23+14+8 = 91.
    theoretical optimum: t0 admits A, B (M* = 16; with C 23 > 21), t1 still rejects C
      (M* = 22 > 21: "M_{t+2} = 22"), t2 admits C at M* = 21 ≤ 21 ("at t+1"); no eviction.
      consumed 12+14+21+13+15 = 75; future 16+16+21+15+15 = 83."""
    m, g, e = run([7, 3, 4], [3, 5, 3], cap=21, max_new=5, policy=O.SIM_AGGRESSIVE, bp=10000)
    assert m == dict(iterations=5, decode_steps=5, evictions=1, finished=3, consumed_sum=75,
                     future_sum=91, samples=5, future_max=23, forced=0, admissions=4)
    assert list(g) == [3, 5, 3] and list(e) == [0, 0, 1]
    m, g, e = run([7, 3, 4], [3, 5, 3], cap=21, max_new=5, policy=O.SIM_OPTIMUM)
    assert m == dict(iterations=5, decode_steps=5, evictions=0, finished=3, consumed_sum=75,
                     future_sum=83, samples=5, future_max=21, forced=0, admissions=3)
    # conservative (no overcommit): Σ(l_p + max_new) = 12 + 8 = 20 ≤ 21 admits A, B only;
    # C (9) waits until A finishes (t3), so the run takes one iteration more.
    m, _, _ = run([7, 3, 4], [3, 5, 3], cap=21, max_new=5, policy=O.SIM_CONSERVATIVE, bp=10000)
    assert m["evictions"] == 0 and m["iterations"] == 6 and m["finished"] == 3


def test_past_future_with_exact_history_equals_optimum():
    """Every request's true length is v and the window holds only v: the conditional
    quantile is v for every l_t < v (C-3, C-4), so Alg.1 sees the true lengths and the
    past-future run must equal the theoretical-optimum run metric for metric."""
    rng = np.random.default_rng(3)
    v, n = 40, 60
    lp = rng.integers(0, 50, size=n)
    L = np.full(n, v)
    for mode in (0, 1):
        a = run(lp, L, cap=600, max_new=64, policy=O.SIM_PAST_FUTURE, window=16, E=32,
                init_history=np.full(16, v), mode=mode, seed=9)
        b = run(lp, L, cap=600, max_new=64, policy=O.SIM_OPTIMUM, window=16, E=32)
        assert a[0] == b[0]
        assert a[0]["evictions"] == 0


def _wl(cls, n_inst=3, n_req=40, div=32, slots=6):
    return S.make_sim_workload(cls, n_inst, n_req, div=div, slots=slots, window=64)


def _sim(w, policy, bp, E=48, **kw):
    return O.sim_run(req_off=w["req_off"].numpy(), req_input=w["req_input"].numpy(),
                     req_output=w["req_output"].numpy(), max_new=w["max_new"].numpy(),
                     capacity=w["capacity"].numpy(), policy=policy, param_bp=bp, window=64,
                     max_len=w["max_len"], init_history=w["init_history"].numpy(), max_entries=E,
                     iterations=10**6, seed=11, **kw)


@pytest.mark.parametrize("cls", [CHAT, D1, D2, D3])
@pytest.mark.parametrize("policy,bp", [(O.SIM_PAST_FUTURE, 300), (O.SIM_PAST_FUTURE, 1000),
                                       (O.SIM_OPTIMUM, 0), (O.SIM_AGGRESSIVE, 9900),
                                       (O.SIM_CONSERVATIVE, 10000), (O.SIM_CONSERVATIVE, 15000)])
def test_run_invariants(cls, policy, bp):
    w = _wl(cls)
    m, g, e = _sim(w, policy, bp)
    n_req = np.diff(w["req_off"].numpy())
    # every run terminates with every request complete (token-count correctness)
    assert np.array_equal(g, w["req_output"].numpy())
    assert np.array_equal(m[:, M["finished"]], n_req)
    # each eviction is followed by exactly one re-admission
    ev = np.add.reduceat(e, w["req_off"].numpy()[:-1])
    assert np.array_equal(m[:, M["evictions"]], ev)
    assert np.array_equal(m[:, M["admissions"]], n_req + ev)
    assert np.array_equal(m[:, M["samples"]], m[:, M["iterations"]])
    cap = w["capacity"].numpy().astype(np.int64)
    # consumed memory never exceeds M after the overflow step (mean ≤ M)
    assert np.all(m[:, M["consumed_sum"]] <= cap * m[:, M["samples"]])
    if policy == O.SIM_OPTIMUM:  # Table 1 "Theoretical optimum ... 0 %" evicted
        assert m[:, M["evictions"]].sum() == 0
        assert np.all(m[:, M["future_max"]] * 10000 <= (10000 - bp) * cap)
    if policy == O.SIM_CONSERVATIVE and bp == 10000:  # true length ≤ max_new: never overflows
        assert m[:, M["evictions"]].sum() == 0


def test_table1_ordinal_structure():
    """PAPER.md:339-372 on Distribution-1 (decode-heavy), at reduced scale: the
    theoretical optimum and no-overcommit conservative never evict; conservative needs
    the most decoding steps; aggressive at 99 % evicts most; past-future evicts less as
    the reserved ratio grows."""
    w = _wl(D1, n_inst=4, n_req=60, div=16, slots=8)
    res = {}
    for name, pol, bp in [("opt", O.SIM_OPTIMUM, 0), ("pf3", O.SIM_PAST_FUTURE, 300),
                          ("pf10", O.SIM_PAST_FUTURE, 1000), ("ag99", O.SIM_AGGRESSIVE, 9900),
                          ("ag90", O.SIM_AGGRESSIVE, 9000), ("cons", O.SIM_CONSERVATIVE, 10000)]:
        res[name] = _sim(w, pol, bp, E=64)[0].sum(0)
    ev = {k: v[M["evictions"]] for k, v in res.items()}
    steps = {k: v[M["decode_steps"]] for k, v in res.items()}
    assert ev["opt"] == 0 and ev["cons"] == 0
    assert ev["ag99"] > ev["ag90"] and ev["ag99"] > ev["pf3"] >= ev["pf10"]
    assert steps["cons"] == max(steps.values())
    assert steps["ag99"] <= steps["opt"] < steps["cons"]
