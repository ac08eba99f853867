"""GPU parity of the batched simulator (pf_sim_*, NEXT-2) with the simulator oracle
(oracle/pf_sim_oracle.cpp): metrics, generated tokens and eviction counts per request,
bit-exact, at the end of every run and at intermediate iteration counts."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2507_10150_b200 as P
import workload.sim as S
from workload.gen import CHAT, D1, D2, D3

pytestmark = pytest.mark.gpu

E = 48


def _wl(cls, n_inst, n_req, div, slots, window=64):
    return S.make_sim_workload(cls, n_inst, n_req, div=div, slots=slots, window=window)


def _gpu(w, policy, bp, *, init=True, window=64, mode=0, R=1, seed=11):
    d = {k: (v.cuda() if torch.is_tensor(v) else v) for k, v in w.items()}
    return P.Simulator(req_off=d["req_off"], req_input=d["req_input"], req_output=d["req_output"],
                       max_new=d["max_new"], capacity=d["capacity"], policy=policy, param_bp=bp,
                       window=window, max_len=w["max_len"], max_input_len=w["max_input_len"],
                       max_entries=E, init_history=d["init_history"] if init else None, mode=mode,
                       repetitions=R, seed=seed)


def _orc(w, policy, bp, iters, *, init=True, window=64, mode=0, R=1, seed=11):
    return O.sim_run(req_off=w["req_off"].numpy(), req_input=w["req_input"].numpy(),
                     req_output=w["req_output"].numpy(), max_new=w["max_new"].numpy(),
                     capacity=w["capacity"].numpy(), policy=policy, param_bp=bp, window=window,
                     max_len=w["max_len"], init_history=w["init_history"].numpy() if init else None,
                     max_entries=E, iterations=iters, mode=mode, repetitions=R, seed=seed)


def _same(sim, orc, what):
    m, g, e = (t.cpu().numpy() for t in sim.metrics())
    om, og, oe = orc
    for c, name in enumerate(P.SIM_METRICS):
        assert np.array_equal(m[:, c], om[:, c]), f"{what}: metric {name}: {m[:, c]} vs {om[:, c]}"
    assert np.array_equal(g, og), f"{what}: generated"
    assert np.array_equal(e, oe), f"{what}: evictions"


CASES = [
    # cls, policy, bp, mode, R
    (D1, P.PF_SIM_PAST_FUTURE, 300, 0, 1), (D2, P.PF_SIM_PAST_FUTURE, 1000, 0, 1),
    (D3, P.PF_SIM_PAST_FUTURE, 500, 1, 1), (CHAT, P.PF_SIM_PAST_FUTURE, 300, 0, 0),
    (D1, P.PF_SIM_OPTIMUM, 0, 0, 1), (D2, P.PF_SIM_OPTIMUM, 300, 0, 1),
    (D1, P.PF_SIM_AGGRESSIVE, 9900, 0, 1), (D3, P.PF_SIM_AGGRESSIVE, 9000, 0, 1),
    (D1, P.PF_SIM_CONSERVATIVE, 10000, 0, 1), (D2, P.PF_SIM_CONSERVATIVE, 15000, 0, 1),
]


@pytest.mark.parametrize("cls,policy,bp,mode,R", CASES)
def test_sim_parity_full_and_partial(cls, policy, bp, mode, R):
    w = _wl(cls, n_inst=5, n_req=40, div=32, slots=6)
    for iters in (1, 7, 40):  # mid-run states
        sim = _gpu(w, policy, bp, mode=mode, R=R)
        sim.step(iters)
        _same(sim, _orc(w, policy, bp, iters, mode=mode, R=R), f"{iters} iterations")
        sim.close()
    sim = _gpu(w, policy, bp, mode=mode, R=R)
    sim.run(chunk=64)
    assert sim.n_done() == 5
    orc = _orc(w, policy, bp, 10**6, mode=mode, R=R)
    _same(sim, orc, "complete run")
    assert orc[0][:, 3].sum() == 200  # every request finished
    assert sim.device_error() == (0, 0)


def test_sim_default_window_and_ragged_instances():
    """C-2 initial window (w copies of Lmax) and instances with different request
    counts, including an empty one (done at once)."""
    w = _wl(D1, n_inst=4, n_req=30, div=32, slots=6)
    keep = np.r_[np.arange(0, 5), np.arange(30, 60), np.arange(60, 60), np.arange(90, 117)]
    counts = np.array([5, 30, 0, 27])
    w2 = dict(w)
    w2["req_off"] = torch.from_numpy(np.r_[0, np.cumsum(counts)].astype(np.int32))
    w2["req_input"] = w["req_input"][keep].contiguous()
    w2["req_output"] = w["req_output"][keep].contiguous()
    for policy, bp in ((P.PF_SIM_PAST_FUTURE, 300), (P.PF_SIM_AGGRESSIVE, 9500)):
        sim = _gpu(w2, policy, bp, init=False)
        sim.run(chunk=32)
        _same(sim, _orc(w2, policy, bp, 10**6, init=False), f"policy {policy}")


def test_sim_table1_structure_at_scale():
    """Distribution-1 at the paper's scale (div = 1, ~16 concurrent requests, w = 1000):
    GPU runs only (the oracle would take minutes); the ordinal facts of Table 1 hold."""
    w = S.make_sim_workload(D1, 8, 120, div=1, slots=16, window=1000)
    res = {}
    for name, pol, bp in [("opt", P.PF_SIM_OPTIMUM, 0), ("pf3", P.PF_SIM_PAST_FUTURE, 300),
                          ("pf10", P.PF_SIM_PAST_FUTURE, 1000), ("ag99", P.PF_SIM_AGGRESSIVE, 9900),
                          ("cons", P.PF_SIM_CONSERVATIVE, 10000)]:
        d = {k: (v.cuda() if torch.is_tensor(v) else v) for k, v in w.items()}
        sim = P.Simulator(req_off=d["req_off"], req_input=d["req_input"], req_output=d["req_output"],
                          max_new=d["max_new"], capacity=d["capacity"], policy=pol, param_bp=bp,
                          window=1000, max_len=w["max_len"], max_input_len=w["max_input_len"],
                          max_entries=128, init_history=d["init_history"], seed=3)
        sim.run(chunk=512)
        m = sim.metrics()[0].cpu().numpy().sum(0)
        res[name] = m
        assert m[3] == 8 * 120
        assert sim.device_error() == (0, 0)
    ev = {k: v[2] for k, v in res.items()}
    steps = {k: v[1] for k, v in res.items()}
    assert ev["opt"] == 0 and ev["cons"] == 0
    assert ev["ag99"] > ev["pf3"] >= ev["pf10"]
    assert steps["cons"] == max(steps.values())
