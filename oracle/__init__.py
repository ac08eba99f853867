"""CPU ORACLE for the Past-Future scheduler hot path (arXiv 2507.10150).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package. The product package ``paper_2507_10150_b200`` never imports it.

This is a thin ctypes loader for ``oracle/liborc.so`` (built from
``oracle/pf_oracle.cpp`` by ``__graft_entry__.build()`` or ``build_oracle()``
below). All arithmetic lives in the C++ file, which transcribes the paper's
definitions (Eq.(eq:5), Alg.1, Eq.(eq:1)-(eq:3)) — see its
header for the citations and pins.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pf_oracle.cpp")
_SRCS = [_SRC, os.path.join(_HERE, "pf_sim_oracle.cpp"), os.path.join(_HERE, "pf_analysis_oracle.cpp"),
         os.path.join(_HERE, "pf_forward_oracle.cpp")]
_LIB_PATH = os.path.join(_HERE, "liborc.so")
_lib = None

I32P = ctypes.POINTER(ctypes.c_int32)
I64P = ctypes.POINTER(ctypes.c_int64)

ORC_E_COMPLETION, ORC_E_OFFSETS, ORC_E_MAX_NEW = 1, 2, 3
ORC_E_INPUT_LEN, ORC_E_GENERATED, ORC_E_CAPACITY = 4, 5, 6


def build_oracle(force: bool = False) -> str:
    """Compile liborc.so with plain g++ (-O2, no SIMD intrinsics)."""
    stale = not os.path.exists(_LIB_PATH) or any(
        os.path.getmtime(_LIB_PATH) < os.path.getmtime(f) for f in _SRCS)
    if force or stale:
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-pthread",
                               *_SRCS, "-o", _LIB_PATH])
    return _LIB_PATH


class _AdmitArgs(ctypes.Structure):
    _fields_ = [
        ("n_inst", ctypes.c_int32),
        ("dist_of", I32P), ("inst_id", I64P),
        ("run_off", I32P), ("input_len", I32P), ("generated", I32P),
        ("q_off", I32P), ("q_input_len", I32P),
        ("max_new", I32P), ("capacity", I32P),
        ("mode", ctypes.c_int32), ("quantile_u", ctypes.c_uint32),
        ("repetitions", ctypes.c_int32), ("reserved_bp", ctypes.c_int32),
        ("seed", ctypes.c_uint64), ("tick", ctypes.c_uint32),
        ("max_input_len", ctypes.c_int32), ("max_entries", ctypes.c_int32),
        ("admitted_out", I32P), ("peak_out", I32P), ("peak_running_out", I32P),
        ("pred_run_out", I32P), ("pred_q_out", I32P),
        ("first_error", I32P), ("first_error_inst", I32P),
    ]


class _SimArgs(ctypes.Structure):
    _fields_ = [
        ("n_inst", ctypes.c_int32),
        ("req_off", I32P), ("req_input", I32P), ("req_output", I32P),
        ("max_new", I32P), ("capacity", I32P),
        ("policy", ctypes.c_int32), ("param_bp", ctypes.c_int32),
        ("window", ctypes.c_int32), ("max_len", ctypes.c_int32), ("init_history", I32P),
        ("max_entries", ctypes.c_int32),
        ("mode", ctypes.c_int32), ("quantile_u", ctypes.c_uint32), ("repetitions", ctypes.c_int32),
        ("seed", ctypes.c_uint64), ("instance_base", ctypes.c_int64), ("iterations", ctypes.c_int32),
        ("metrics_out", I64P), ("generated_out", I32P), ("evictions_out", I32P),
    ]


SIM_PAST_FUTURE, SIM_OPTIMUM, SIM_AGGRESSIVE, SIM_CONSERVATIVE = 0, 1, 2, 3
SIM_METRICS = ("iterations", "decode_steps", "evictions", "finished", "consumed_sum",
               "future_sum", "samples", "future_max", "forced", "admissions")


class _ForwardArgs(ctypes.Structure):
    _fields_ = [
        ("n_clusters", ctypes.c_int32), ("cluster_size", ctypes.c_int32),
        ("windows", I32P), ("window", ctypes.c_int32),
        ("run_off", I32P), ("input_len", I32P), ("generated", I32P),
        ("max_new", I32P), ("capacity", I32P), ("cq_off", I32P), ("cq_input_len", I32P),
        ("mode", ctypes.c_int32), ("quantile_u", ctypes.c_uint32), ("reserved_bp", ctypes.c_int32),
        ("seed", ctypes.c_uint64), ("tick", ctypes.c_uint32), ("instance_base", ctypes.c_int64),
        ("max_entries", ctypes.c_int32),
        ("dest_out", I32P), ("forwarded_out", I32P), ("peak_out", I32P),
    ]


def lib():
    global _lib
    if _lib is None:
        build_oracle()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_mix64.restype = ctypes.c_uint64
        L.orc_mix64.argtypes = [ctypes.c_uint64]
        L.orc_lowbias32.restype = ctypes.c_uint32
        L.orc_lowbias32.argtypes = [ctypes.c_uint32]
        L.orc_instance_key.restype = ctypes.c_uint64
        L.orc_instance_key.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int64]
        L.orc_draw.restype = ctypes.c_uint32
        L.orc_draw.argtypes = [ctypes.c_uint64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32]
        L.orc_predict.restype = ctypes.c_int32
        L.orc_predict.argtypes = [I32P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint32]
        L.orc_predict_rep.restype = ctypes.c_int32
        L.orc_predict_rep.argtypes = [I32P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                      ctypes.c_uint64, ctypes.c_int32, ctypes.c_int32]
        for fn in ("orc_peak_ticks", "orc_peak_sort", "orc_peak_brute"):
            getattr(L, fn).restype = ctypes.c_int64
            getattr(L, fn).argtypes = [ctypes.c_int32, I32P, I32P]
        L.orc_admit_one.restype = ctypes.c_int32
        L.orc_admit_one.argtypes = [ctypes.c_int32, I32P, I32P, ctypes.c_int32, I32P, I32P,
                                    ctypes.c_int64, ctypes.c_int32, I64P, I64P]
        L.orc_admit_one_bsearch.restype = ctypes.c_int32
        L.orc_admit_one_bsearch.argtypes = [ctypes.c_int32, I32P, I32P, ctypes.c_int32, I32P, I32P,
                                            ctypes.c_int64, ctypes.c_int32, I64P]
        L.orc_create.restype = ctypes.c_void_p
        L.orc_create.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, I32P]
        L.orc_destroy.restype = None
        L.orc_destroy.argtypes = [ctypes.c_void_p]
        L.orc_update_history.restype = ctypes.c_int32
        L.orc_update_history.argtypes = [ctypes.c_void_p, I32P, I32P, I32P]
        L.orc_get_row.restype = None
        L.orc_get_row.argtypes = [ctypes.c_void_p, ctypes.c_int32, I32P]
        L.orc_admit.restype = ctypes.c_int32
        L.orc_admit.argtypes = [ctypes.c_void_p, ctypes.POINTER(_AdmitArgs), ctypes.c_int32]
        L.orc_sizeof_admit_args.restype = ctypes.c_int32
        L.orc_admit_aggressive.restype = ctypes.c_int32
        L.orc_admit_aggressive.argtypes = [ctypes.c_int32, I32P, I32P, ctypes.c_int32, I32P, ctypes.c_int64,
                                           ctypes.c_int32, I64P]
        L.orc_admit_conservative.restype = ctypes.c_int32
        L.orc_admit_conservative.argtypes = [ctypes.c_int32, I32P, ctypes.c_int32, I32P, ctypes.c_int32,
                                             ctypes.c_int64, ctypes.c_int32, I64P]
        assert L.orc_sizeof_admit_args() == ctypes.sizeof(_AdmitArgs), "oracle ABI struct mismatch"
        L.orc_sim_run.restype = None
        L.orc_sim_run.argtypes = [ctypes.POINTER(_SimArgs), ctypes.c_int32]
        L.orc_sizeof_sim_args.restype = ctypes.c_int32
        F64P = ctypes.POINTER(ctypes.c_double)
        L.orc_forward.restype = None
        L.orc_forward.argtypes = [ctypes.POINTER(_ForwardArgs)]
        L.orc_sizeof_forward_args.restype = ctypes.c_int32
        assert L.orc_sizeof_forward_args() == ctypes.sizeof(_ForwardArgs), "oracle forward ABI mismatch"
        L.orc_window_similarity.restype = ctypes.c_int32
        L.orc_window_similarity.argtypes = [I32P, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, I64P,
                                            F64P, F64P]
        L.orc_adjacent_similarity.restype = ctypes.c_int32
        L.orc_adjacent_similarity.argtypes = [I32P, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                              ctypes.c_int32, F64P, F64P]
        assert L.orc_sizeof_sim_args() == ctypes.sizeof(_SimArgs), "oracle sim ABI struct mismatch"
        _lib = L
    return _lib


def _i32(x):
    a = np.ascontiguousarray(np.asarray(x, dtype=np.int32))
    return a


def _p32(a):
    return None if a is None else a.ctypes.data_as(I32P)


# ---------------------------------------------------------------- primitives
def mix64(z: int) -> int:
    return lib().orc_mix64(z & 0xFFFFFFFFFFFFFFFF)


def lowbias32(x: int) -> int:
    return lib().orc_lowbias32(x & 0xFFFFFFFF)


def instance_key(seed: int, tick: int, inst: int) -> int:
    return lib().orc_instance_key(seed & 0xFFFFFFFFFFFFFFFF, tick & 0xFFFFFFFF, inst)


def draw(key: int, slot: int, R: int, rep: int) -> int:
    return lib().orc_draw(key, slot, R, rep)


def predict(window, l_t: int, max_new: int, u: int) -> int:
    w = _i32(window)
    return lib().orc_predict(_p32(w), len(w), l_t, max_new, u & 0xFFFFFFFF)


def predict_rep(window, l_t: int, max_new: int, key: int, slot: int, R: int) -> int:
    w = _i32(window)
    return lib().orc_predict_rep(_p32(w), len(w), l_t, max_new, key, slot, R)


def peak_ticks(a, r) -> int:
    a, r = _i32(a), _i32(r)
    return lib().orc_peak_ticks(len(a), _p32(a), _p32(r))


def peak_sort(a, r) -> int:
    a, r = _i32(a), _i32(r)
    return lib().orc_peak_sort(len(a), _p32(a), _p32(r))


def peak_brute(a, r) -> int:
    a, r = _i32(a), _i32(r)
    return lib().orc_peak_brute(len(a), _p32(a), _p32(r))


def admit_one(run_a, run_r, q_a, q_r, capacity: int, bp: int = 0):
    """Literal Alg.1 admission for one instance -> (p*, M*(admitted), M*(R))."""
    ra, rr, qa, qr = _i32(run_a), _i32(run_r), _i32(q_a), _i32(q_r)
    pk, pr = ctypes.c_int64(), ctypes.c_int64()
    p = lib().orc_admit_one(len(ra), _p32(ra), _p32(rr), len(qa), _p32(qa), _p32(qr),
                            capacity, bp, ctypes.byref(pk), ctypes.byref(pr))
    return p, pk.value, pr.value


def admit_one_bsearch(run_a, run_r, q_a, q_r, capacity: int, bp: int = 0):
    ra, rr, qa, qr = _i32(run_a), _i32(run_r), _i32(q_a), _i32(q_r)
    pk = ctypes.c_int64()
    p = lib().orc_admit_one_bsearch(len(ra), _p32(ra), _p32(rr), len(qa), _p32(qa), _p32(qr),
                                    capacity, bp, ctypes.byref(pk))
    return p, pk.value


def admit_aggressive(run_lp, run_lt, q_lp, capacity: int, watermark_bp: int):
    """Baseline: watermark admission on input lengths only -> (p*, used)."""
    a, b, c = _i32(run_lp), _i32(run_lt), _i32(q_lp)
    used = ctypes.c_int64()
    p = lib().orc_admit_aggressive(len(a), _p32(a), _p32(b), len(c), _p32(c), capacity, watermark_bp,
                                   ctypes.byref(used))
    return p, used.value


def admit_conservative(run_lp, q_lp, max_new: int, capacity: int, overcommit_bp: int):
    """Baseline: input + max_new budget admission -> (p*, used)."""
    a, c = _i32(run_lp), _i32(q_lp)
    used = ctypes.c_int64()
    p = lib().orc_admit_conservative(len(a), _p32(a), len(c), _p32(c), max_new, capacity, overcommit_bp,
                                     ctypes.byref(used))
    return p, used.value


# ---------------------------------------------------------------- batched
class Oracle:
    """Batched oracle state: ``n_rows`` FIFO history rings of ``row_window``;
    an instance's distribution is ``rows_per_dist`` consecutive rows."""

    def __init__(self, n_rows: int, row_window: int, max_len: int, rows_per_dist: int = 1,
                 init_rows=None):
        self.n_rows, self.row_window, self.max_len = n_rows, row_window, max_len
        self.rows_per_dist = rows_per_dist
        init = None if init_rows is None else _i32(init_rows).reshape(-1)
        if init is not None:
            assert init.size == n_rows * row_window
        self._h = lib().orc_create(n_rows, row_window, max_len, rows_per_dist, _p32(init))
        if not self._h:
            raise ValueError("orc_create: invalid arguments")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            try:
                _lib.orc_destroy(h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None

    def update_history(self, comp_off, comp_len):
        co, cl = _i32(comp_off), _i32(comp_len)
        if cl.size == 0:
            cl = np.zeros(1, np.int32)
        bad = ctypes.c_int32(-1)
        st = lib().orc_update_history(self._h, _p32(co), _p32(cl), ctypes.byref(bad))
        return st, bad.value

    def row(self, i: int) -> np.ndarray:
        out = np.empty(self.row_window, np.int32)
        lib().orc_get_row(self._h, i, _p32(out))
        return out

    def admit(self, *, dist_of, inst_id, run_off, input_len, generated, max_new,
              q_off=None, q_input_len=None, capacity=None, mode=0, quantile_u=0x80000000,
              repetitions=1, reserved_bp=0, seed=0, tick=0, max_input_len=(1 << 30),
              max_entries=(1 << 30), want_pred=False, n_threads=None):
        n = len(max_new)
        keep = []

        def c32(x):
            a = _i32(x)
            if a.size == 0:
                a = np.zeros(1, np.int32)
            keep.append(a)
            return a

        dist_of_a = c32(dist_of)
        inst_id_a = np.ascontiguousarray(np.asarray(inst_id, dtype=np.int64))
        run_off_a = c32(run_off)
        il, gn = c32(input_len), c32(generated)
        mn = c32(max_new)
        estimate = capacity is None
        qo = None if estimate else c32(q_off)
        qi = None if estimate else c32(q_input_len)
        cap = None if estimate else c32(capacity)
        adm = None if estimate else np.empty(n, np.int32)
        peak = np.empty(n, np.int32)
        prun = None if estimate else np.empty(n, np.int32)
        n_run = int(np.asarray(run_off)[-1])
        n_q = 0 if estimate else int(np.asarray(q_off)[-1])
        pred_r = np.empty(max(n_run, 1), np.int32) if want_pred else None
        pred_q = np.empty(max(n_q, 1), np.int32) if (want_pred and not estimate) else None
        fe, fi = ctypes.c_int32(0), ctypes.c_int32(-1)
        args = _AdmitArgs(
            n, _p32(dist_of_a), inst_id_a.ctypes.data_as(I64P), _p32(run_off_a), _p32(il), _p32(gn),
            _p32(qo), _p32(qi), _p32(mn), _p32(cap), mode, quantile_u & 0xFFFFFFFF, repetitions,
            reserved_bp, seed & 0xFFFFFFFFFFFFFFFF, tick & 0xFFFFFFFF, max_input_len, max_entries,
            _p32(adm), _p32(peak), _p32(prun), _p32(pred_r), _p32(pred_q),
            ctypes.pointer(fe), ctypes.pointer(fi))
        nt = n_threads or os.cpu_count() or 1
        n_bad = lib().orc_admit(self._h, ctypes.byref(args), nt)
        out = {"peak": peak, "n_bad": n_bad, "first_error": fe.value, "first_error_inst": fi.value}
        if not estimate:
            out["admitted"], out["peak_running"] = adm, prun
        if want_pred:
            out["pred_run"] = pred_r[:n_run]
            if pred_q is not None:
                out["pred_q"] = pred_q[:n_q]
        return out


# ---------------------------------------------------------------- simulator (NEXT-2)
def sim_run(*, req_off, req_input, req_output, max_new, capacity, policy, param_bp, window,
            max_len, max_entries, iterations, init_history=None, mode=0, quantile_u=0x80000000,
            repetitions=1, seed=0, instance_base=0, n_threads=None):
    """Continuous-batching simulation of every instance for ``iterations`` iterations
    (pf_sim_oracle.cpp, readings S-1..S-9). Returns (metrics [n × 10] int64 with
    columns SIM_METRICS, generated per request, evictions per request)."""
    ro, ri, rq = _i32(req_off), _i32(req_input), _i32(req_output)
    ih = None if init_history is None else _i32(init_history).reshape(-1)
    mn, cap = _i32(max_new), _i32(capacity)
    n = len(mn)
    n_req = int(ro[-1])
    met = np.zeros((n, len(SIM_METRICS)), np.int64)
    gen = np.zeros(max(n_req, 1), np.int32)
    ev = np.zeros(max(n_req, 1), np.int32)
    if n_req == 0:
        ri = rq = np.zeros(1, np.int32)
    args = _SimArgs(n, _p32(ro), _p32(ri), _p32(rq), _p32(mn), _p32(cap), policy, param_bp, window,
                    max_len, _p32(ih), max_entries, mode, quantile_u & 0xFFFFFFFF, repetitions,
                    seed & 0xFFFFFFFFFFFFFFFF, instance_base, iterations,
                    met.ctypes.data_as(I64P), _p32(gen), _p32(ev))
    lib().orc_sim_run(ctypes.byref(args), n_threads or os.cpu_count() or 1)
    return met, gen[:n_req], ev[:n_req]


# ---------------------------------------------------------------- window similarity (NEXT-3)
def window_similarity(lengths, window: int, max_len: int):
    """-> (gram [B, B] int64, cos [B, B] float64, (mean_adjacent, mean_global)) or None."""
    x = _i32(lengths)
    B = len(x) // window if window > 0 else 0
    if B < 2:
        return None
    g = np.empty((B, B), np.int64)
    c = np.empty((B, B), np.float64)
    sm = np.empty(2, np.float64)
    F = ctypes.POINTER(ctypes.c_double)
    got = lib().orc_window_similarity(_p32(x), len(x), window, max_len, g.ctypes.data_as(I64P),
                                      c.ctypes.data_as(F), sm.ctypes.data_as(F))
    return None if got == 0 else (g, c, (float(sm[0]), float(sm[1])))


def adjacent_similarity(lengths, hist_window: int, run_window: int, max_len: int):
    """-> (cos per running window [K] float64, mean) or None."""
    x = _i32(lengths)
    if hist_window < 1 or run_window < 1 or len(x) < hist_window + run_window:
        return None
    K = (len(x) - hist_window) // run_window
    c = np.empty(K, np.float64)
    mean = ctypes.c_double()
    F = ctypes.POINTER(ctypes.c_double)
    got = lib().orc_adjacent_similarity(_p32(x), len(x), hist_window, run_window, max_len,
                                        c.ctypes.data_as(F), ctypes.byref(mean))
    return None if got == 0 else (c, mean.value)


# ---------------------------------------------------------------- forwarding (NEXT-4)
def forward(*, cluster_size, windows, run_off, input_len, generated, max_new, capacity, cq_off,
            cq_input_len, mode=0, quantile_u=0x80000000, reserved_bp=0, seed=0, tick=0,
            instance_base=0, max_entries=1 << 30):
    """Cross-instance forwarding (pf_forward_oracle.cpp, readings F-1..F-4).
    windows: [n, w] history per instance. -> (dest [Σq], forwarded [C], peak [n])."""
    win = np.ascontiguousarray(np.asarray(windows, dtype=np.int32))
    n, w = win.shape
    C = n // cluster_size
    keep = []

    def c32(x):
        a = _i32(x)
        if a.size == 0:
            a = np.zeros(1, np.int32)
        keep.append(a)
        return a

    nq = int(np.asarray(cq_off)[-1])
    dest = np.empty(max(nq, 1), np.int32)
    fwd = np.empty(C, np.int32)
    peak = np.empty(n, np.int32)
    args = _ForwardArgs(C, cluster_size, _p32(win), w, _p32(c32(run_off)), _p32(c32(input_len)),
                        _p32(c32(generated)), _p32(c32(max_new)), _p32(c32(capacity)), _p32(c32(cq_off)),
                        _p32(c32(cq_input_len)), mode, quantile_u & 0xFFFFFFFF, reserved_bp,
                        seed & 0xFFFFFFFFFFFFFFFF, tick & 0xFFFFFFFF, instance_base, max_entries,
                        _p32(dest), _p32(fwd), _p32(peak))
    lib().orc_forward(ctypes.byref(args))
    return dest[:nq], fwd, peak
