"""Seeded request lists for the batched continuous-batching simulator (NEXT-2).

No method arithmetic: per instance, ``n_req`` requests drawn from one of the paper's
length classes (Distribution-1/2/3 or chat) with the same
SplitMix64 streams as ``gen.py``, lengths divided by ``div`` (a uniform down-scale
so the CPU oracle can replay whole runs; ``div = 1`` is the paper's scale), and a
KV capacity of ``slots`` worst-case requests: M = slots · (max_input + max_new) / div,
so every request fits on its own (SPEC.md engine, SimConfig invariant).
"""
from __future__ import annotations

import torch

from .gen import CHAT, D1, D2, D3, _draw, _key, _lengths, class_params

F_SIM_LP_B, F_SIM_LP, F_SIM_L_B, F_SIM_L, F_SIM_H_B, F_SIM_H = 40, 41, 42, 43, 44, 45


def make_sim_workload(cls: int, n_inst: int, n_req: int, *, div: int = 1, slots: int = 16,
                      window: int = 1000, seed: int = 0x2507101500000100, device="cpu"):
    """-> dict(req_off [n+1], req_input, req_output, max_new [n], capacity [n],
    init_history [n × window] (a steady-state window of the same class: w draws of L,
    oldest first), max_len, max_input_len); tensors are int32, the bounds ints."""
    assert cls in (CHAT, D1, D2, D3)
    max_new_full, max_in_full, _ = class_params(cls)
    max_new = max(1, max_new_full // div)
    max_in = max_in_full // div
    ids = torch.arange(n_inst * n_req, dtype=torch.int64)
    c = torch.full_like(ids, cls)

    def x(field):
        return _draw(_key(seed, ids, field), torch.zeros_like(ids))

    lp = _lengths(c, x(F_SIM_LP_B), x(F_SIM_LP), "lp") // div
    L = (_lengths(c, x(F_SIM_L_B), x(F_SIM_L), "L") // div).clamp(min=1, max=max_new)
    cap = slots * (max_in + max_new)
    hid = torch.arange(n_inst * window, dtype=torch.int64)
    hc = torch.full_like(hid, cls)
    hx = lambda field: _draw(_key(seed, hid, field), torch.zeros_like(hid))  # noqa: E731
    hist = (_lengths(hc, hx(F_SIM_H_B), hx(F_SIM_H), "L") // div).clamp(min=1, max=max_new)
    return {
        "req_off": (torch.arange(n_inst + 1, dtype=torch.int64) * n_req).to(torch.int32).to(device),
        "req_input": lp.to(torch.int32).to(device),
        "req_output": L.to(torch.int32).to(device),
        "max_new": torch.full((n_inst,), max_new, dtype=torch.int32, device=device),
        "capacity": torch.full((n_inst,), cap, dtype=torch.int32, device=device),
        "init_history": hist.to(torch.int32).reshape(n_inst, window).to(device),
        "max_len": max_new,
        "max_input_len": max_in,
    }


F_STREAM_B, F_STREAM = 46, 47


def make_length_stream(classes, per_class: int, *, div: int = 1, seed: int = 0x2507101500000200):
    """A synthetic trace of output lengths for the window-similarity analysis (NEXT-3):
    ``per_class`` requests of each class in ``classes`` concatenated in order (the paper's
    varying-load workload), lengths // div clamped to ≥ 1. -> int32 tensor."""
    parts = []
    for s, cls in enumerate(classes):
        ids = torch.arange(per_class, dtype=torch.int64) + s * per_class
        c = torch.full_like(ids, cls)
        x1 = _draw(_key(seed, ids, F_STREAM_B), torch.zeros_like(ids))
        x2 = _draw(_key(seed, ids, F_STREAM), torch.zeros_like(ids))
        parts.append((_lengths(c, x1, x2, "L") // div).clamp(min=1))
    return torch.cat(parts).to(torch.int32)
