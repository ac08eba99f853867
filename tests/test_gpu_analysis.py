"""GPU parity of the window-similarity analysis (pf_window_similarity /
pf_adjacent_similarity, NEXT-3) with the oracle: the integer Gram matrix bit for bit,
cosines bit for bit (same IEEE expression), means within 1e-12 (summation order)."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2507_10150_b200 as P
import workload.sim as S
from workload.gen import CHAT, D1, D2, D3

pytestmark = pytest.mark.gpu


def _streams():
    rng = np.random.default_rng(2)
    yield "random", rng.integers(1, 65, size=7 * 50 + 13).astype(np.int32), 50, 64
    yield "varying", S.make_length_stream([D1, D2, D3], 4000, div=8).numpy(), 1000, 640
    yield "chat", S.make_length_stream([CHAT], 40000).numpy(), 1000, 2048
    yield "wide", rng.integers(1, 32768, size=20 * 300).astype(np.int32), 300, 32767


@pytest.mark.parametrize("name,x,w,L", list(_streams()), ids=lambda v: v if isinstance(v, str) else "")
def test_window_similarity_parity(name, x, w, L):
    g, c, sm = P.window_similarity(torch.from_numpy(x).cuda(), w, L)
    og, oc, osm = O.window_similarity(x, w, L)
    assert np.array_equal(g.cpu().numpy(), og)
    assert np.array_equal(c.cpu().numpy(), oc)
    assert np.allclose(sm.cpu().numpy(), osm, rtol=1e-12, atol=0)


@pytest.mark.parametrize("hw,rw", [(1000, 1000), (1000, 250), (4000, 64), (100, 3000)])
def test_adjacent_similarity_parity(hw, rw):
    x = S.make_length_stream([CHAT, D1, D3], 8000, div=2).numpy()
    c, m = P.adjacent_similarity(torch.from_numpy(x).cuda(), hw, rw, 2048)
    oc, om = O.adjacent_similarity(x, hw, rw, 2048)
    assert np.array_equal(c.cpu().numpy(), oc)
    assert abs(float(m.item()) - om) <= 1e-12 * abs(om)


def test_burstgpt_scale_sampled():
    """A BurstGPT-sized trace (1.4 M requests, 1,400 windows of 1,000): symmetric, unit
    diagonal, and 64 sampled entries recomputed from numpy bincounts."""
    x = S.make_length_stream([CHAT, D1, D2, D3, CHAT, D3, D1], 200000).numpy()
    w, L = 1000, 5120
    g, c, sm = P.window_similarity(torch.from_numpy(x).cuda(), w, L)
    g, c = g.cpu().numpy(), c.cpu().numpy()
    B = len(x) // w
    assert g.shape == (B, B) and np.array_equal(g, g.T)
    assert np.all(np.diag(c) == 1.0)
    rng = np.random.default_rng(0)
    H = {}

    def h(b):
        if b not in H:
            H[b] = np.bincount(x[b * w:(b + 1) * w], minlength=L + 1).astype(np.int64)
        return H[b]

    for i, j in rng.integers(0, B, size=(64, 2)):
        assert g[i, j] == int(h(i) @ h(j))
    assert sm[0].item() > sm[1].item()  # adjacent windows are more alike than windows in general


def test_rejects_lengths_out_of_range():
    x = torch.tensor([1, 2, 3, 0], dtype=torch.int32, device="cuda")
    with pytest.raises(P.PFError):
        P.window_similarity(x, 2, 8)
    with pytest.raises(P.PFError):
        P.adjacent_similarity(torch.tensor([1, 2, 9, 3], dtype=torch.int32, device="cuda"), 2, 2, 8)
