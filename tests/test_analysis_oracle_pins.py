"""Pins for the window-similarity oracle (oracle/pf_analysis_oracle.cpp, NEXT-3;
fig:dist / fig:cos_win): SPEC's worked examples,
hand-built matrices, invariants, and numpy's bincount + matmul as an independent
formulation."""
import numpy as np
import pytest

import oracle as O
import workload.sim as S
from workload.gen import CHAT, D1, D2, D3


def test_spec_examples():
    g, c, _ = O.window_similarity([5, 7, 9, 5, 7, 9], 3, 10)  # identical windows
    assert np.all(c == 1.0)
    g, c, _ = O.window_similarity([1, 1, 9, 9], 2, 10)  # disjoint supports
    assert c[0, 1] == 0.0 and g[0, 1] == 0
    g, c, sm = O.window_similarity([2, 2, 3, 2, 3, 3], 3, 4)  # (2·1 + 1·2)/(√5·√5)
    assert g.tolist() == [[5, 4], [4, 5]] and c[0, 1] == 0.8 and sm == (0.8, 0.8)


def test_summary_hand_matrices():
    # all windows the same multiset -> (1, 1)
    _, _, sm = O.window_similarity([3, 4, 4] * 5, 3, 8)
    assert sm == (1.0, 1.0)
    # block-diagonal, two regimes A A B B with disjoint supports: adjacent 2/3, global 1/3
    _, c, sm = O.window_similarity([1, 2, 2, 1, 7, 8, 8, 7], 2, 8)
    assert np.allclose(c, [[1, 1, 0, 0], [1, 1, 0, 0], [0, 0, 1, 1], [0, 0, 1, 1]])
    assert abs(sm[0] - 2 / 3) < 1e-15 and abs(sm[1] - 1 / 3) < 1e-15


def test_against_numpy_and_invariants():
    rng = np.random.default_rng(5)
    x = rng.integers(1, 60, size=7 * 50 + 13)  # ragged tail dropped
    w, L = 50, 64
    g, c, sm = O.window_similarity(x, w, L)
    B = len(x) // w
    H = np.stack([np.bincount(x[b * w:(b + 1) * w], minlength=L + 1) for b in range(B)]).astype(np.int64)
    assert np.array_equal(g, H @ H.T)
    assert np.array_equal(c, c.T) and np.all((c >= 0) & (c <= 1 + 1e-15))
    assert np.allclose(np.diag(c), 1.0, rtol=0, atol=1e-15)
    n = np.sqrt(np.diag(H @ H.T).astype(np.float64))
    assert np.allclose(c, (H @ H.T) / np.outer(n, n), rtol=1e-14, atol=0)
    assert abs(sm[0] - np.mean([c[i, i + 1] for i in range(B - 1)])) < 1e-14
    assert abs(sm[1] - (c.sum() - np.trace(c)) / (B * (B - 1))) < 1e-14
    # permutation inside windows: unchanged; duplicating every request: unchanged
    xp = x[:B * w].reshape(B, w)
    xp = np.stack([rng.permutation(r) for r in xp]).reshape(-1)
    assert np.array_equal(O.window_similarity(xp, w, L)[1], c)
    xd = np.repeat(x[:B * w].reshape(B, w), 2, axis=1).reshape(-1)
    assert np.array_equal(O.window_similarity(xd, 2 * w, L)[1], c)


def test_adjacent_variant_matches_square_matrix():
    x = S.make_length_stream([CHAT, D1], 3000, div=4).numpy()
    w = 500
    _, c, _ = O.window_similarity(x, w, 2048)
    ck, mean = O.adjacent_similarity(x, w, w, 2048)
    B = len(x) // w
    assert len(ck) == B - 1
    assert np.array_equal(ck, np.array([c[i, i + 1] for i in range(B - 1)]))
    ck2, _ = O.adjacent_similarity(x, 1000, 250, 2048)  # historical 1000, running 250
    assert len(ck2) == (len(x) - 1000) // 250


def test_varying_load_adjacent_beats_global():
    """on concat(Distribution-1, 2, 3) adjacent windows are more similar
    than windows in general by >= 0.1 (PAPER.md:190 'the adjacent time windows (the
    diagonal pattern) have similar distributions')."""
    x = S.make_length_stream([D1, D2, D3], 4000, div=8).numpy()
    _, _, (adj, glob) = O.window_similarity(x, 1000, 640)
    assert adj - glob >= 0.1


def test_rejects_bad_input():
    assert O.window_similarity([1, 2, 3], 2, 8) is None  # one window
    assert O.window_similarity([1, 2, 0, 3], 2, 8) is None  # length 0
    assert O.window_similarity([1, 2, 9, 3], 2, 8) is None  # > Lmax
