"""Pins for the CPU oracle (oracle/pf_oracle.cpp) against things OTHER than itself:
values printed by the paper (fig:peak narrative), SPEC.md worked examples, closed
forms, textbook/library special cases, invariants, and brute force on tiny inputs.
Each check is chosen so a plausible mistake (dropped term, wrong sign/index,
'>' vs '>=', transposed operand) fails at least one of them."""
import bisect
import json
import os
import random

import numpy as np
import pytest

import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")
U32 = 1 << 32


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ------------------------------------------------------------------ C-8 hash
def test_splitmix64_published_vector():
    # SplitMix64 (Steele/Lea/Flood 2014) from state 0: outputs are mix64(i*gamma), i = 1, 2, 3.
    g = 0x9E3779B97F4A7C15
    assert O.mix64(g) == 0xE220A8397B1DCDAF
    assert O.mix64((2 * g) & (2**64 - 1)) == 0x6E789E6AA1B965F4
    assert O.mix64((3 * g) & (2**64 - 1)) == 0x06C45D188009454F


def test_lowbias32_prototype_vectors():
    # from the survey prototype only (not a paper value).
    assert O.lowbias32(1) == 0x688990C0
    assert O.lowbias32(0xDEADBEEF) == 0xE628C683
    assert O.lowbias32(0) == 0


def test_p6_keys_and_draws():
    g = gold("config1_p5.json")["sampling_mode_P6"]
    seed = int(g["seed"], 16)
    for t in g["ticks"]:
        K = O.instance_key(seed, t["tick"], 0)
        assert K == int(t["K"], 16)
        assert [O.draw(K, s, 1, 0) for s in range(3)] == [int(x, 16) for x in t["u"]]


# ------------------------------------------------------------------ history, Eq.(eq:5)
def test_fifo_eviction_spec():
    ex = gold("spec_examples.json")["fifo_eviction"]
    orc = O.Oracle(1, 2, 100, 1, np.array([ex["window"]]))
    st, _ = orc.update_history([0, 1], [ex["record"]])
    assert st == 0
    assert list(orc.row(0)) == ex["expect"]


def test_history_more_completions_than_window_keeps_last_w():
    orc = O.Oracle(2, 3, 50, 1, np.array([[1, 2, 3], [4, 5, 6]]))
    st, _ = orc.update_history([0, 5, 6], [10, 11, 12, 13, 14, 20])
    assert st == 0
    assert list(orc.row(0)) == [12, 13, 14]
    assert list(orc.row(1)) == [5, 6, 20]


def test_history_rejects_out_of_range_row_unchanged():
    orc = O.Oracle(2, 2, 9, 1, np.array([[1, 2], [3, 4]]))
    st, bad = orc.update_history([0, 2, 3], [5, 10, 7])  # 10 > Lmax = 9 in row 0
    assert st == O.ORC_E_COMPLETION and bad == 0
    assert list(orc.row(0)) == [1, 2]
    assert list(orc.row(1)) == [4, 7]
    st, bad = orc.update_history([0, 1, 1], [0])  # 0 < 1
    assert st == O.ORC_E_COMPLETION and bad == 0


def test_default_init_is_max_len():
    # PAPER.md:295 "initialize the output length distribution using the preset maximum output length"
    orc = O.Oracle(1, 5, 77, 1, None)
    assert list(orc.row(0)) == [77] * 5


def test_eq5_probability_by_exact_u_counting():
    # P(2) = C(2, {2,2,3}) / 3 = 2/3. The inverse-CDF draw at u maps the
    # fraction of u in [0, 2^32) that returns 2 to P(2): count it exactly on the
    # boundary: ρ = floor(u*3/2^32) < 2  <=>  u < ceil(2*2^32/3).
    ex = gold("spec_examples.json")
    w = ex["eq5_window"]
    edge = -(-2 * U32 // 3)
    assert O.predict(w, 0, 100, edge - 1) == 2
    assert O.predict(w, 0, 100, edge) == 3
    assert abs(edge / U32 - ex["eq5_expect_P2_num"] / ex["eq5_expect_P2_den"]) < 1e-9


# ------------------------------------------------------------------ prediction, Alg.1 l.3-9
def test_conditional_spec_examples():
    ex = gold("spec_examples.json")
    rng = random.Random(1)
    for _ in range(200):
        u = rng.randrange(U32)
        c = ex["conditional_only_one"]
        assert O.predict(c["window"], c["l_t"], 100, u) == c["expect"]
        c = ex["conditional_empty"]
        assert O.predict(c["window"], c["l_t"], c["max_new"], u) == c["expect"]
        c = ex["conditional_clamp"]
        assert O.predict(c["window"], c["l_t"], c["max_new"], u) in c["expect_set"]
        c = ex["singleton"]
        assert O.predict(c["window"], 0, 100, u) == c["expect"]
    c = ex["conditional_clamp"]
    assert O.predict(c["window"], c["l_t"], c["max_new"], 0) == 5
    assert O.predict(c["window"], c["l_t"], c["max_new"], U32 - 1) == 6


def test_quantile_closed_forms():
    rng = random.Random(2)
    for _ in range(300):
        w = [rng.randint(1, 40) for _ in range(rng.randint(1, 30))]
        l_t = rng.randint(0, 45)
        mx = 64
        gt = sorted(h for h in w if h > l_t)
        # u = 0 -> smallest value > l_t: the textbook upper_bound (bisect_right)
        s = sorted(w)
        ub = bisect.bisect_right(s, l_t)
        exp0 = s[ub] if ub < len(s) else mx
        assert O.predict(w, l_t, mx, 0) == exp0
        # u = 2^32 - 1 -> max of the conditional support
        assert O.predict(w, l_t, mx, U32 - 1) == (max(gt) if gt else mx)
    # constant history v: v if l_t < v else max_new
    for v in (1, 5, 17):
        for l_t in range(0, 20):
            assert O.predict([v] * 9, l_t, 30, 12345) == (v if l_t < v else 30)


def test_quantile_matches_lookup_formulation():
    # O(1) lookup form of the same inverse CDF: base = #{h <= l_t} (numpy searchsorted
    # 'right' on the sorted window), rank ρ among the n_gt values above it.
    rng = np.random.default_rng(3)
    for _ in range(300):
        w = rng.integers(1, 200, size=rng.integers(1, 64))
        s = np.sort(w)
        l_t = int(rng.integers(0, 210))
        u = int(rng.integers(0, U32))
        mx = 180
        base = int(np.searchsorted(s, l_t, side="right"))
        n_gt = len(s) - base
        exp = mx if n_gt == 0 else min(int(s[base + ((u * n_gt) >> 32)]), mx)
        assert O.predict(w, l_t, mx, u) == exp


def test_prediction_strictly_above_generated_and_capped():
    rng = random.Random(4)
    for _ in range(500):
        w = [rng.randint(1, 50) for _ in range(rng.randint(1, 20))]
        mx = rng.randint(1, 60)
        l_t = rng.randint(0, mx - 1)
        v = O.predict(w, l_t, mx, rng.randrange(U32))
        assert l_t < v <= mx


def test_repetitions_max_equals_quantile_at_max_u():
    # C-9: max of R inverse-CDF samples == one inverse-CDF sample at max(u_r) (monotone).
    rng = random.Random(5)
    for _ in range(200):
        w = [rng.randint(1, 30) for _ in range(rng.randint(1, 25))]
        key = rng.randrange(2**64)
        R = rng.randint(1, 6)
        slot = rng.randint(0, 300)
        l_t = rng.randint(0, 20)
        umax = max(O.draw(key, slot, R, rep) for rep in range(R))
        assert O.predict_rep(w, l_t, 40, key, slot, R) == O.predict(w, l_t, 40, umax)


def test_sampling_frequencies_follow_conditional_distribution():
    # Statistical sanity (SPEC acceptance 2): hash draws give l̂ with
    # frequencies P(l | l > l_t).
    w = [1, 2, 2, 3, 3, 3, 5, 8, 8, 8]
    l_t = 2
    support = {3: 3, 5: 1, 8: 3}
    n = 20000
    counts = {}
    for i in range(n):
        key = O.instance_key(99, i, 7)
        v = O.predict_rep(w, l_t, 100, key, 0, 1)
        counts[v] = counts.get(v, 0) + 1
    assert set(counts) == set(support)
    tot = sum(support.values())
    chi2 = sum((counts[v] - n * c / tot) ** 2 / (n * c / tot) for v, c in support.items())
    assert chi2 < 20.0  # 2 dof; p ~ 5e-5


# ------------------------------------------------------------------ peak, Eq.(eq:1)-(eq:3)
def ar(entries):
    """SPEC (input, generated, predicted) triples -> (a, r)."""
    return [lp + lt for lp, lt, _ in entries], [lh - lt for _, lt, lh in entries]


def test_peak_spec_examples():
    ex = gold("spec_examples.json")
    for key in ("peak_one", "peak_two"):
        a, r = ar(ex[key]["entries"])
        for f in (O.peak_ticks, O.peak_sort, O.peak_brute):
            assert f(a, r) == ex[key]["expect"]
    for f in (O.peak_ticks, O.peak_sort, O.peak_brute):
        assert f([], []) == 0


def test_peak_closed_forms():
    rng = random.Random(6)
    for _ in range(100):
        lp, lt = rng.randint(0, 99), rng.randint(0, 50)
        lh = lt + rng.randint(0, 60)
        assert O.peak_ticks([lp + lt], [lh - lt]) == lp + lh  # one entry -> l_p + l̂
        n = rng.randint(1, 12)
        a = [rng.randint(0, 50) for _ in range(n)]
        rr = rng.randint(0, 40)
        assert O.peak_ticks(a, [rr] * n) == sum(a) + n * rr  # all r equal
        r = [rng.randint(0, 40) for _ in range(n)]
        rs = sorted(r, reverse=True)
        assert O.peak_ticks([0] * n, r) == max(i * rs[i - 1] for i in range(1, n + 1))  # all a = 0
    assert O.peak_ticks([0, 0, 0], [5, 4, 3]) == 9


def test_peak_formulations_agree_and_invariants():
    rng = random.Random(7)
    for _ in range(1500):
        n = rng.randint(0, 14)
        a = [rng.randint(0, 60) for _ in range(n)]
        r = [rng.randint(0, 25) for _ in range(n)]
        m = O.peak_ticks(a, r)
        assert m == O.peak_sort(a, r) == O.peak_brute(a, r)
        assert sum(a) <= m <= sum(a) + sum(r)  # current <= M* <= Σ(l_p + l̂)
        perm = list(range(n))
        rng.shuffle(perm)
        assert O.peak_ticks([a[i] for i in perm], [r[i] for i in perm]) == m  # permutation
        if n:
            assert O.peak_ticks(a + [rng.randint(0, 9)], r + [rng.randint(0, 25)]) >= m  # monotone


def test_fig_peak_narrative():
    g = gold("fig_peak.json")
    cap = g["capacity"]

    def entries(st):
        a = [x["l_p"] + x["l_t"] for x in st["running"]] + [st["candidate"]["l_p"]]
        r = [x["l_hat"] - x["l_t"] for x in st["running"]] + [st["candidate"]["l_hat"]]
        return a, r

    t = g["t"]
    a, r = entries(t)
    assert sum(a[:-1]) == t["expect_current_usage"]
    assert sum(a) == t["expect_aggressive_check"] and sum(a) <= cap  # aggressive admits at t
    m = O.peak_ticks(a, r)
    assert m == t["expect_M_star_with_candidate"] == 22 and m > cap  # "M_{t+2} = 22 > 21"
    occ = [sum(ai + tau for ai, ri in zip(a, r) if ri >= tau) for tau in range(max(r) + 1)]
    assert occ.index(max(occ)) == t["expect_argmax_tick"]
    p, _, _ = O.admit_one(a[:-1], r[:-1], a[-1:], r[-1:], cap, 0)
    assert (p == 1) == t["expect_admit"]
    t1 = g["t_plus_1"]
    a, r = entries(t1)
    assert O.peak_ticks(a, r) == t1["expect_M_star_with_candidate"]
    p, pk, _ = O.admit_one(a[:-1], r[:-1], a[-1:], r[-1:], cap, 0)
    assert (p == 1) == t1["expect_admit"] and pk == 21  # admitted "at t+1"


# ------------------------------------------------------------------ admission, Alg.1 l.7-14
def test_admission_spec_boundary():
    ex = gold("spec_examples.json")["admit_boundary"]
    lp, lh = ex["candidate"]
    p, pk, pr = O.admit_one([], [], [lp], [lh], ex["capacity"], ex["bp_admit"])
    assert (p, pk, pr) == (1, 9, 0)  # 9 <= 9: equality admits (C-12)
    p, pk, pr = O.admit_one([], [], [lp], [lh], ex["capacity"], ex["bp_reject"])
    assert (p, pk) == (0, 0)  # 9 > 0.9*9


def _brute_admit(ra, rr, qa, qr, cap, bp):
    """Definition: the longest FIFO prefix whose every prefix fits (early return)."""
    p = 0
    for j in range(1, len(qa) + 1):
        m = O.peak_brute(ra + qa[:j], rr + qr[:j])
        if m * 10000 <= (10000 - bp) * cap:
            p = j
        else:
            break
    return p, O.peak_brute(ra + qa[:p], rr + qr[:p])


def test_admission_brute_force_bsearch_and_invariants():
    rng = random.Random(8)
    for _ in range(600):
        k, q = rng.randint(0, 8), rng.randint(0, 6)
        ra = [rng.randint(0, 30) for _ in range(k)]
        rr = [rng.randint(1, 20) for _ in range(k)]
        qa = [rng.randint(0, 30) for _ in range(q)]
        qr = [rng.randint(1, 20) for _ in range(q)]
        cap = rng.randint(0, 400)
        bp = rng.choice([0, 300, 500, 1000])
        p, pk, pr = O.admit_one(ra, rr, qa, qr, cap, bp)
        assert (p, pk) == _brute_admit(ra, rr, qa, qr, cap, bp)
        assert (p, pk) == O.admit_one_bsearch(ra, rr, qa, qr, cap, bp)
        assert pr == O.peak_ticks(ra, rr)
        assert pk >= sum(ra) + sum(qa[:p])  # peak >= current usage of the admitted batch
        assert pk >= pr  # peak monotone in admitted requests
        assert O.admit_one(ra, rr, qa, qr, cap + rng.randint(0, 50), bp)[0] >= p  # monotone in M
        assert O.admit_one(ra, rr, qa, qr, cap, min(9999, bp + 700))[0] <= p  # anti-monotone in bp


# ------------------------------------------------------------------ batched oracle
def _config1(orc_mode, bp, tick=0, seed=0x2507101500000001):
    g = gold("config1_p5.json")
    win = np.repeat(np.array(g["window_values"], np.int32), g["window_each"])
    orc = O.Oracle(1, len(win), g["max_new"], 1, win[None, :])
    run = np.array(g["running"], np.int32)
    out = orc.admit(dist_of=[0], inst_id=[0], run_off=[0, len(run)], input_len=run[:, 0],
                    generated=run[:, 1], max_new=[g["max_new"]], q_off=[0, len(g["queue"])],
                    q_input_len=g["queue"], capacity=[g["capacity"]], mode=orc_mode,
                    quantile_u=0x80000000, reserved_bp=bp, seed=seed, tick=tick, want_pred=True)
    return g, out


def test_config1_hand_example_quantile_mode():
    for bp in (0, 300, 2000):
        g, out = _config1(1, bp)
        assert list(out["pred_run"]) == g["expect_pred_running"]
        assert list(out["pred_q"]) == g["expect_pred_queue"]
        assert int(out["peak_running"][0]) == g["expect_peak_running"]
        assert int(out["admitted"][0]) == g["expect_admitted"][str(bp)]
        assert int(out["peak"][0]) == g["expect_peak_admitted"][str(bp)]
    run = np.array(g["running"])
    a = run[:, 0] + run[:, 1]
    assert int(a.sum()) == g["expect_current_usage"]
    r = np.array(g["expect_pred_running"]) - run[:, 1]
    tau = g["expect_peak_running_tick"]
    assert int(a[r >= tau].sum() + tau * (r >= tau).sum()) == g["expect_peak_running"]
    qa = np.array(g["queue"])
    for p, exp in enumerate(g["expect_candidate_peaks"], 1):
        aa = np.concatenate([a, qa[:p]])
        rr = np.concatenate([r, np.array(g["expect_pred_queue"][:p])])
        assert O.peak_brute(aa, rr) == exp


def test_config1_sampling_mode_p6_table():
    for t in gold("config1_p5.json")["sampling_mode_P6"]["ticks"]:
        _, out = _config1(0, 0, tick=t["tick"])
        assert list(out["pred_run"]) == t["pred_running"]
        assert list(out["pred_q"]) == t["pred_queue"]
        assert int(out["peak_running"][0]) == t["peak_running"]
        assert int(out["admitted"][0]) == t["admitted"]
        assert int(out["peak"][0]) == t["peak_admitted"]


def test_batched_validation_sets_minus_one():
    win = np.full((3, 4), 5, np.int32)
    orc = O.Oracle(3, 4, 10, 1, win)
    common = dict(dist_of=[0, 1, 2], inst_id=[0, 1, 2], run_off=[0, 1, 2, 3], q_off=[0, 1, 2, 3],
                  q_input_len=[1, 1, 1], max_new=[10, 10, 10], capacity=[100, 100, 100], mode=1,
                  max_input_len=50, want_pred=True)
    out = orc.admit(input_len=[3, 3, 3], generated=[0, 10, 2], **common)  # l_t >= max_new in inst 1
    assert out["n_bad"] == 1 and out["first_error"] == O.ORC_E_GENERATED and out["first_error_inst"] == 1
    assert out["admitted"][1] == -1 and out["peak"][1] == -1 and out["pred_run"][1] == -1
    assert out["admitted"][0] >= 0 and out["admitted"][2] >= 0
    out = orc.admit(input_len=[3, 51, 3], generated=[0, 0, 0], **common)
    assert out["first_error"] == O.ORC_E_INPUT_LEN and out["peak"][1] == -1
    c2 = dict(common, max_new=[10, 11, 10])
    out = orc.admit(input_len=[3, 3, 3], generated=[0, 0, 0], **c2)
    assert out["first_error"] == O.ORC_E_MAX_NEW
    c3 = dict(common, capacity=[100, -1, 100])
    out = orc.admit(input_len=[3, 3, 3], generated=[0, 0, 0], **c3)
    assert out["first_error"] == O.ORC_E_CAPACITY
    out = orc.admit(input_len=[3, 3, 3], generated=[0, 0, 0], max_entries=1, **common)
    assert out["first_error"] == O.ORC_E_OFFSETS and out["n_bad"] == 3


def test_shared_distribution_is_concatenation_of_shards():
    # C-18: a group's window is the union of its 8 shard rings.
    rng = np.random.default_rng(9)
    rows = rng.integers(1, 30, size=(16, 5)).astype(np.int32)  # 2 groups x 8 shards
    orc = O.Oracle(16, 5, 40, 8, rows)
    lt = rng.integers(0, 39, size=20).astype(np.int32)
    out = orc.admit(dist_of=[1], inst_id=[123], run_off=[0, 20], input_len=np.ones(20, np.int32),
                    generated=lt, max_new=[40], mode=1, quantile_u=0x12345678, want_pred=True)
    win = rows[8:16].reshape(-1)
    exp = [O.predict(win, int(x), 40, 0x12345678) for x in lt]
    assert list(out["pred_run"]) == exp


# ------------------------------------------------------------------ baseline policies
def test_aggressive_spec_examples():
    # capacity 100, watermark 90 %, consumed 80: input 10 admitted
    # (90 ≤ 90), a further input 1 rejected (91 > 90).
    assert O.admit_aggressive([80], [0], [10], 100, 9000) == (1, 90)
    assert O.admit_aggressive([80], [0], [10, 1], 100, 9000) == (1, 90)
    assert O.admit_aggressive([70], [10], [10, 1], 100, 9000) == (1, 90)  # consumed = l_p + l_t


def test_conservative_spec_examples():
    # capacity 100, candidates (10, max_new 50): one fits without
    # overcommit (60 ≤ 100), the second does not (120 > 100); with 150 % both fit.
    assert O.admit_conservative([], [10, 10], 50, 100, 10000) == (1, 60)
    assert O.admit_conservative([], [10, 10], 50, 100, 15000) == (2, 120)
    assert O.admit_conservative([5], [10], 50, 100, 10000) == (0, 55)  # running budget l_p + max_new


def test_baseline_policies_brute_force():
    rng = random.Random(11)
    for _ in range(400):
        k, q = rng.randint(0, 6), rng.randint(0, 6)
        mx = rng.randint(1, 40)
        lp = [rng.randint(0, 30) for _ in range(k)]
        lt = [rng.randint(0, mx - 1) for _ in range(k)]
        ql = [rng.randint(0, 30) for _ in range(q)]
        cap = rng.randint(0, 300)
        wm = rng.choice([9000, 9500, 9900, 10000])
        p = 0
        while p < q and 10000 * (sum(lp) + sum(lt) + sum(ql[:p + 1])) <= wm * cap:
            p += 1
        assert O.admit_aggressive(lp, lt, ql, cap, wm) == (p, sum(lp) + sum(lt) + sum(ql[:p]))
        oc = rng.choice([10000, 12500, 15000])
        p = 0
        while p < q and 10000 * (sum(lp) + k * mx + sum(ql[:p + 1]) + (p + 1) * mx) <= oc * cap:
            p += 1
        assert O.admit_conservative(lp, ql, mx, cap, oc) == (p, sum(lp) + k * mx + sum(ql[:p]) + p * mx)


def test_adaptive_repetitions_rule():
    # R = max(1, ceil(64 / k)); prediction = max of the R samples. With a
    # 2-request batch R = 32: each prediction equals the quantile at the max of 32 draws.
    win = np.arange(1, 101, dtype=np.int32)
    orc = O.Oracle(1, 100, 200, 1, win[None, :])
    out = orc.admit(dist_of=[0], inst_id=[5], run_off=[0, 2], input_len=[3, 4], generated=[0, 50],
                    max_new=[200], mode=0, repetitions=0, seed=9, tick=2, want_pred=True)
    K = O.instance_key(9, 2, 5)
    for s, l_t in enumerate((0, 50)):
        umax = max(O.draw(K, s, 32, rep) for rep in range(32))
        assert out["pred_run"][s] == O.predict(win, l_t, 200, umax)


# ---- C-8 / C-9 re-derived in pure Python (independent of the oracle's C++ hash) ----------
_M64 = (1 << 64) - 1


def _py_mix64(z):
    z &= _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def _py_lowbias32(x):
    x &= 0xFFFFFFFF
    x ^= x >> 16
    x = (x * 0x7FEB352D) & 0xFFFFFFFF
    x ^= x >> 15
    x = (x * 0x846CA68B) & 0xFFFFFFFF
    return x ^ (x >> 16)


def _py_u(seed, tick, inst, slot, R):
    """C-8: K = mix64(seed ^ tick·C_T ^ inst·C_I); u_rep = lowbias32(lo32 K ^ hi32 K ^
    lo32((slot·R + rep)·0x9E3779B9)); C-9: u = max_rep u_rep (the inverse CDF is monotone)."""
    K = _py_mix64(seed ^ ((tick * 0xD1B54A32D192ED03) & _M64) ^ ((inst * 0x9E3779B97F4A7C15) & _M64))
    fold = (K & 0xFFFFFFFF) ^ (K >> 32)
    return max(_py_lowbias32(fold ^ (((slot * R + rep) * 0x9E3779B9) & 0xFFFFFFFF)) for rep in range(R))


def _py_predict(window, l_t, max_new, u):
    gt = sorted(h for h in window if h > l_t)          # C-3/C-4: values > l_t, ascending
    if not gt:
        return max_new                                  # C-5
    return min(gt[(u * len(gt)) >> 32], max_new)        # rank ⌊u·|gt|/2^32⌋, C-6


def test_py_c8_pins_splitmix_vector():
    # SplitMix64's published first output from state 0 (state += γ, then the finalizer)
    assert _py_mix64(0x9E3779B97F4A7C15) == 0xE220A8397B1DCDAF


@pytest.mark.parametrize("R", [2, 3, 7])
def test_repetitions_gt1_against_pure_python(R):
    """R > 1 draws (C-9 indexing (slot·R + rep)): every prediction of a small instance,
    running and queued, equals the pure-Python re-derivation."""
    rng = random.Random(R)
    win = [rng.randint(1, 60) for _ in range(40)]
    orc = O.Oracle(1, 40, 64, 1, np.array(win, dtype=np.int32)[None, :])
    lp = [rng.randint(0, 50) for _ in range(5)]
    lt = [rng.randint(0, 63) for _ in range(5)]
    ql = [rng.randint(0, 50) for _ in range(4)]
    seed, tick, inst = 0x1234567890ABCDEF, 7, 3
    out = orc.admit(dist_of=[0], inst_id=[inst], run_off=[0, 5], input_len=lp, generated=lt, max_new=[64],
                    q_off=[0, 4], q_input_len=ql, capacity=[10 ** 6], mode=0, repetitions=R, seed=seed,
                    tick=tick, want_pred=True)
    for s in range(5):
        assert out["pred_run"][s] == _py_predict(win, lt[s], 64, _py_u(seed, tick, inst, s, R))
    for j in range(4):  # queued slot k + j (0-based j), l_t = 0 (C-16)
        assert out["pred_q"][j] == _py_predict(win, 0, 64, _py_u(seed, tick, inst, 5 + j, R))


def test_adaptive_repetitions_at_k0_against_pure_python():
    """Reading of SPEC.md:161's R = max(1, ⌈64/k⌉) at k = 0 (no running batch): R = 64 (the
    k → 1 limit). Queued predictions of an instance with an empty running batch use 64 draws."""
    rng = random.Random(99)
    win = [rng.randint(1, 300) for _ in range(50)]
    orc = O.Oracle(1, 50, 300, 1, np.array(win, dtype=np.int32)[None, :])
    ql = [rng.randint(0, 100) for _ in range(6)]
    seed, tick, inst = 42, 3, 11
    out = orc.admit(dist_of=[0], inst_id=[inst], run_off=[0, 0], input_len=[], generated=[], max_new=[300],
                    q_off=[0, 6], q_input_len=ql, capacity=[10 ** 6], mode=0, repetitions=0, seed=seed,
                    tick=tick, want_pred=True)
    for j in range(6):
        assert out["pred_q"][j] == _py_predict(win, 0, 300, _py_u(seed, tick, inst, j, 64))
    # and k = 3 gives R = ⌈64/3⌉ = 22
    out = orc.admit(dist_of=[0], inst_id=[inst], run_off=[0, 3], input_len=[1, 2, 3], generated=[5, 0, 70],
                    max_new=[300], q_off=[0, 2], q_input_len=ql[:2], capacity=[10 ** 6], mode=0,
                    repetitions=0, seed=seed, tick=tick, want_pred=True)
    for s, l_t in enumerate((5, 0, 70)):
        assert out["pred_run"][s] == _py_predict(win, l_t, 300, _py_u(seed, tick, inst, s, 22))
    for j in range(2):
        assert out["pred_q"][j] == _py_predict(win, 0, 300, _py_u(seed, tick, inst, 3 + j, 22))
