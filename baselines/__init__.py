"""Optimized multithreaded CPU implementation of the hot path (cpu_fast.cpp), used by
bench.py only as a fairer CPU comparator next to the oracle-based cpu_baseline.
Not the oracle, not the product; tests/test_cpu_fast.py checks it against the oracle."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "cpu_fast.cpp")
_LIB = os.path.join(_HERE, "libcpufast.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O3", "-std=c++17", "-fPIC", "-shared", "-pthread",
                               _SRC, "-o", _LIB])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.pfc_admit.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(ctypes.POINTER(t))


def admit(batch, dist_rows, *, mode=0, quantile_u=0x80000000, bp=500, seed=0, tick=0, threads=None):
    """Alg.1 for every instance of a workload.Batch; dist_rows [D × window] int32 holds the
    distribution windows (per-instance rows, or a shared group's shard rows concatenated),
    indexed by batch.dist_of. -> (admitted, peak, peak_running) int32 arrays."""
    i32 = lambda t: np.ascontiguousarray(t.cpu().numpy() if hasattr(t, "cpu") else t, dtype=np.int32)
    n = batch.n
    rows = np.ascontiguousarray(dist_rows, dtype=np.int32)
    out = [np.empty(n, np.int32) for _ in range(3)]
    args = [i32(batch.dist_of), np.ascontiguousarray(batch.inst_ids.cpu().numpy(), dtype=np.int64),
            i32(batch.run_off), i32(batch.input_len), i32(batch.generated), i32(batch.q_off),
            i32(batch.q_input_len), i32(batch.max_new), i32(batch.capacity)]
    I32, I64 = ctypes.c_int32, ctypes.c_int64
    st = lib().pfc_admit(I32(n), _p(args[0], I32), _p(args[1], I64), *[_p(a, I32) for a in args[2:]],
                         I32(rows.shape[1]), I32(batch.cfg.max_len), _p(rows, I32), I32(mode),
                         ctypes.c_uint32(quantile_u & 0xFFFFFFFF), I32(bp), ctypes.c_uint64(seed & (2**64 - 1)),
                         ctypes.c_uint32(tick & 0xFFFFFFFF), I32(threads or os.cpu_count() or 1),
                         _p(out[0], I32), _p(out[1], I32), _p(out[2], I32))
    assert st == 0
    return out


def dist_rows_of(batch):
    """The distribution windows of a batch: per-instance rows, or each shared group's window
    (its shard rows concatenated, rows ordered group-major as in workload.gen)."""
    h = batch.hist_rows.cpu().numpy().astype(np.int32)
    cfg = batch.cfg
    if cfg.shared:
        return h.reshape(cfg.n_groups, -1)
    return h
