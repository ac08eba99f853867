"""Thin ctypes binding of libpfsched.so (include/pfsched.h).

Argument marshalling only: every step of the hot path runs in the CUDA kernels
behind the C-ABI. Tensors are passed as device pointers (``data_ptr()``) with
torch's current CUDA stream. There is no CPU fallback: if the library or a GPU
is missing, the calls raise.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpfsched.so")

PF_MODE_SAMPLE, PF_MODE_QUANTILE = 0, 1
PF_POLICY_AGGRESSIVE, PF_POLICY_CONSERVATIVE = 1, 2
DERR = {0: "none", 1: "completion", 2: "offsets", 3: "max_new", 4: "input_len", 5: "generated",
        6: "capacity", 7: "override"}

ABI_VERSION = 2
NCCL_UNIQUE_ID_BYTES = 128
_vp = ctypes.c_void_p
_i32 = ctypes.c_int32


class PFConfig(ctypes.Structure):
    _fields_ = [
        ("n_instances", _i32), ("window", _i32), ("max_len", _i32), ("max_input_len", _i32),
        ("max_entries", _i32), ("n_groups", _i32), ("group_off", _vp), ("instance_base", ctypes.c_int64),
        ("members_per_group", _i32), ("member_base", _i32), ("mode", _i32),
        ("quantile_u", ctypes.c_uint32), ("repetitions", _i32), ("reserved_bp", _i32),
        ("seed", ctypes.c_uint64), ("rank", _i32), ("nranks", _i32), ("nccl_unique_id", _vp),
    ]


class PFSimConfig(ctypes.Structure):
    _fields_ = [
        ("n_instances", _i32), ("window", _i32), ("max_len", _i32), ("max_input_len", _i32),
        ("max_entries", _i32), ("policy", _i32), ("param_bp", _i32), ("mode", _i32),
        ("quantile_u", ctypes.c_uint32), ("repetitions", _i32), ("seed", ctypes.c_uint64),
        ("instance_base", ctypes.c_int64),
    ]


PF_SIM_PAST_FUTURE, PF_SIM_OPTIMUM, PF_SIM_AGGRESSIVE, PF_SIM_CONSERVATIVE = 0, 1, 2, 3
SIM_METRICS = ("iterations", "decode_steps", "evictions", "finished", "consumed_sum",
               "future_sum", "samples", "future_max", "forced", "admissions")

_lib = None
SYMBOLS = ("pf_nccl_unique_id", "pf_create", "pf_destroy", "pf_update_history", "pf_exchange_buffer", "pf_commit_history",
           "pf_estimate_peak", "pf_admit", "pf_admit_override", "pf_admit_baseline", "pf_get_device_error",
           "pf_clear_device_error", "pf_export_history", "pf_last_error", "pf_abi_version",
           "pf_sim_create", "pf_sim_step", "pf_sim_done", "pf_sim_metrics", "pf_sim_context",
           "pf_sim_destroy", "pf_window_similarity", "pf_adjacent_similarity", "pf_forward")


def load(path: str = os.environ.get("PFSCHED_LIB", LIB_PATH)):
    """Load libpfsched.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} not found: run __graft_entry__.build() (no CPU fallback)")
    L = ctypes.CDLL(path)
    P = ctypes.POINTER
    L.pf_abi_version.restype = _i32
    L.pf_last_error.restype = ctypes.c_char_p
    L.pf_nccl_unique_id.argtypes = [_vp]
    L.pf_create.argtypes = [P(PFConfig), _vp, _vp, P(_vp)]
    L.pf_destroy.argtypes = [_vp]
    L.pf_update_history.argtypes = [_vp, _vp, _vp, _i32, _vp]
    L.pf_exchange_buffer.argtypes = [_vp, P(_vp), P(ctypes.c_int64)]
    L.pf_commit_history.argtypes = [_vp, _vp]
    L.pf_estimate_peak.argtypes = [_vp, _vp, _vp, _vp, _vp, ctypes.c_uint32, _vp, _vp, _vp]
    L.pf_admit.argtypes = [_vp] + [_vp] * 7 + [ctypes.c_uint32] + [_vp] * 6
    L.pf_admit_override.argtypes = [_vp] * 13
    L.pf_admit_baseline.argtypes = [_vp, _i32, _i32] + [_vp] * 10
    L.pf_get_device_error.argtypes = [_vp, P(_i32), P(_i32), _vp]
    L.pf_clear_device_error.argtypes = [_vp, _vp]
    L.pf_export_history.argtypes = [_vp, _vp, _vp]
    L.pf_sim_create.argtypes = [P(PFSimConfig)] + [_vp] * 7 + [P(_vp)]
    L.pf_sim_step.argtypes = [_vp, _i32, _vp]
    L.pf_sim_done.argtypes = [_vp, P(_i32), _vp]
    L.pf_sim_metrics.argtypes = [_vp] * 5
    L.pf_sim_context.argtypes = [_vp]
    L.pf_sim_context.restype = _vp
    L.pf_sim_destroy.argtypes = [_vp]
    L.pf_forward.argtypes = [_vp, _i32] + [_vp] * 7 + [ctypes.c_uint32] + [_vp] * 4
    L.pf_window_similarity.argtypes = [_vp, ctypes.c_int64, _i32, _i32, _vp, _vp, _vp, _vp]
    L.pf_adjacent_similarity.argtypes = [_vp, ctypes.c_int64, _i32, _i32, _i32, _vp, _vp, _vp]
    for s in SYMBOLS:
        if s not in ("pf_abi_version", "pf_last_error", "pf_sim_context"):
            getattr(L, s).restype = _i32
    assert L.pf_abi_version() == ABI_VERSION, f"{path}: ABI {L.pf_abi_version()} != {ABI_VERSION} (rebuild)"
    _lib = L
    return L


class PFError(RuntimeError):
    pass


def _check(st: int, what: str):
    if st != 0:
        raise PFError(f"{what} failed with status {st}: {load().pf_last_error().decode()}")


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not t.is_cuda or t.dtype != torch.int32 or not t.is_contiguous():
        raise PFError("expected a contiguous int32 CUDA tensor")
    return ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def nccl_unique_id() -> bytes:
    """pf_nccl_unique_id: a fresh 128-byte ncclUniqueId (send it to every rank)."""
    buf = ctypes.create_string_buffer(NCCL_UNIQUE_ID_BYTES)
    _check(load().pf_nccl_unique_id(buf), "pf_nccl_unique_id")
    return buf.raw


class Scheduler:
    """One pf_ctx: device history state for n instances (or G shared groups).
    nccl_id (shared mode): the 128-byte ncclUniqueId of a context-owned communicator; the
    context then all-reduces the group histograms itself inside update_history."""

    def __init__(self, *, n_instances: int, window: int, max_len: int, max_input_len: int,
                 max_entries: int, n_groups: int = 0, group_off: Optional[torch.Tensor] = None,
                 instance_base: int = 0, members_per_group: int = 0, member_base: int = 0,
                 mode: int = PF_MODE_SAMPLE, quantile_u: int = 0x80000000, repetitions: int = 1,
                 reserved_bp: int = 0, seed: int = 0, rank: int = 0, nranks: int = 1,
                 init_history: Optional[torch.Tensor] = None, nccl_id: Optional[bytes] = None):
        L = load()
        idbuf = None
        if nccl_id is not None:
            if len(nccl_id) != NCCL_UNIQUE_ID_BYTES:
                raise PFError("nccl_id must be 128 bytes (pf_nccl_unique_id)")
            idbuf = ctypes.create_string_buffer(bytes(nccl_id), NCCL_UNIQUE_ID_BYTES)
        self.cfg = PFConfig(n_instances, window, max_len, max_input_len, max_entries, n_groups,
                            None if group_off is None else group_off.data_ptr(), instance_base,
                            members_per_group, member_base, mode, quantile_u & 0xFFFFFFFF,
                            repetitions, reserved_bp, seed & 0xFFFFFFFFFFFFFFFF, rank, nranks,
                            None if idbuf is None else ctypes.cast(idbuf, _vp))
        self._keep = (group_off, init_history)
        h = ctypes.c_void_p()
        _check(L.pf_create(ctypes.byref(self.cfg), _ptr(init_history), _stream(), ctypes.byref(h)),
               "pf_create")
        self._h = h
        self.n = n_instances
        self.shared = n_groups > 0
        self.rows = n_groups * (8 // nranks) if self.shared else n_instances
        self.row_window = window // 8 if self.shared else window

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            load().pf_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- the three calls
    def update_history(self, comp_off: torch.Tensor, comp_len: torch.Tensor):
        _check(load().pf_update_history(self._h, _ptr(comp_off), _ptr(comp_len) if comp_len.numel() else None,
                                        int(comp_len.numel()), _stream()), "pf_update_history")

    def exchange_buffer(self) -> torch.Tensor:
        """Shared mode: the int32 [G, Lmax+1] device buffer to all-reduce (sum)."""
        buf, cnt = ctypes.c_void_p(), ctypes.c_int64()
        _check(load().pf_exchange_buffer(self._h, ctypes.byref(buf), ctypes.byref(cnt)), "pf_exchange_buffer")
        return _wrap_device_int32(buf.value, cnt.value)

    def commit_history(self):
        _check(load().pf_commit_history(self._h, _stream()), "pf_commit_history")

    def estimate_peak(self, run_off, input_len, generated, max_new, tick: int, *, peak_out=None,
                      pred_out=None):
        if peak_out is None:
            peak_out = torch.empty(self.n, dtype=torch.int32, device=run_off.device)
        _check(load().pf_estimate_peak(self._h, _ptr(run_off), _ptr(input_len), _ptr(generated),
                                       _ptr(max_new), tick & 0xFFFFFFFF, _ptr(peak_out), _ptr(pred_out),
                                       _stream()), "pf_estimate_peak")
        return peak_out

    def admit(self, run_off, input_len, generated, q_off, q_input_len, max_new, capacity, tick: int, *,
              admitted_out=None, peak_out=None, peak_running_out=None, pred_run_out=None,
              pred_q_out=None):
        dev = run_off.device
        if admitted_out is None:
            admitted_out = torch.empty(self.n, dtype=torch.int32, device=dev)
        if peak_out is None:
            peak_out = torch.empty(self.n, dtype=torch.int32, device=dev)
        _check(load().pf_admit(self._h, _ptr(run_off), _ptr(input_len), _ptr(generated), _ptr(q_off),
                               _ptr(q_input_len), _ptr(max_new), _ptr(capacity), tick & 0xFFFFFFFF,
                               _ptr(admitted_out), _ptr(peak_out), _ptr(peak_running_out),
                               _ptr(pred_run_out), _ptr(pred_q_out), _stream()), "pf_admit")
        return admitted_out, peak_out

    def admit_override(self, run_off, input_len, generated, lhat_run, q_off, q_input_len, lhat_q, capacity,
                       *, admitted_out=None, peak_out=None, peak_running_out=None):
        """A12 theoretical optimum: Alg.1 with the caller's l̂ (e.g. true output lengths)."""
        dev = run_off.device
        if admitted_out is None:
            admitted_out = torch.empty(self.n, dtype=torch.int32, device=dev)
        if peak_out is None:
            peak_out = torch.empty(self.n, dtype=torch.int32, device=dev)
        _check(load().pf_admit_override(self._h, _ptr(run_off), _ptr(input_len), _ptr(generated),
                                        _ptr(lhat_run), _ptr(q_off), _ptr(q_input_len), _ptr(lhat_q),
                                        _ptr(capacity), _ptr(admitted_out), _ptr(peak_out),
                                        _ptr(peak_running_out), _stream()), "pf_admit_override")
        return admitted_out, peak_out

    def admit_baseline(self, policy: int, ratio_bp: int, run_off, input_len, generated, q_off, q_input_len,
                       max_new, capacity, *, admitted_out=None, used_out=None):
        """The paper's aggressive (watermark) / conservative (overcommit) admission policies."""
        dev = run_off.device
        if admitted_out is None:
            admitted_out = torch.empty(self.n, dtype=torch.int32, device=dev)
        if used_out is None:
            used_out = torch.empty(self.n, dtype=torch.int32, device=dev)
        _check(load().pf_admit_baseline(self._h, policy, ratio_bp, _ptr(run_off), _ptr(input_len),
                                        _ptr(generated), _ptr(q_off), _ptr(q_input_len), _ptr(max_new),
                                        _ptr(capacity), _ptr(admitted_out), _ptr(used_out), _stream()),
               "pf_admit_baseline")
        return admitted_out, used_out

    def forward(self, cluster_size: int, run_off, input_len, generated, max_new, capacity, cq_off,
                cq_input_len, tick: int):
        """NEXT-4: forward each cluster's queue to its instances by M* headroom.
        -> (dest [Σq] int32, forwarded [C] int32, peak [n] int32)."""
        dev = run_off.device
        C = self.n // cluster_size
        dest = torch.empty(max(int(cq_input_len.numel()), 1), dtype=torch.int32, device=dev)
        fwd = torch.empty(C, dtype=torch.int32, device=dev)
        peak = torch.empty(self.n, dtype=torch.int32, device=dev)
        _check(load().pf_forward(self._h, cluster_size, _ptr(run_off), _ptr(input_len), _ptr(generated),
                                 _ptr(max_new), _ptr(capacity), _ptr(cq_off), _ptr(cq_input_len),
                                 tick & 0xFFFFFFFF, _ptr(dest), _ptr(fwd), _ptr(peak), _stream()),
               "pf_forward")
        return dest[:cq_input_len.numel()], fwd, peak

    def device_error(self):
        code, idx = _i32(), _i32()
        _check(load().pf_get_device_error(self._h, ctypes.byref(code), ctypes.byref(idx), _stream()),
               "pf_get_device_error")
        return code.value, idx.value

    def clear_device_error(self):
        _check(load().pf_clear_device_error(self._h, _stream()), "pf_clear_device_error")

    def export_history(self) -> torch.Tensor:
        out = torch.empty((self.rows, self.row_window), dtype=torch.int32, device="cuda")
        _check(load().pf_export_history(self._h, _ptr(out), _stream()), "pf_export_history")
        return out


class Simulator:
    """Batched continuous-batching simulator (pf_sim_*, NEXT-2): one serving simulation
    per instance, advanced together on the device (readings S-1..S-9, include/pfsched.h)."""

    def __init__(self, *, req_off, req_input, req_output, max_new, capacity, policy: int,
                 param_bp: int, window: int, max_len: int, max_input_len: int, max_entries: int,
                 init_history: Optional[torch.Tensor] = None, mode: int = PF_MODE_SAMPLE,
                 quantile_u: int = 0x80000000, repetitions: int = 1, seed: int = 0,
                 instance_base: int = 0):
        L = load()
        n = int(max_new.numel())
        self.cfg = PFSimConfig(n, window, max_len, max_input_len, max_entries, policy, param_bp, mode,
                               quantile_u & 0xFFFFFFFF, repetitions, seed & 0xFFFFFFFFFFFFFFFF,
                               instance_base)
        h = ctypes.c_void_p()
        _check(L.pf_sim_create(ctypes.byref(self.cfg), _ptr(req_off), _ptr(req_input), _ptr(req_output),
                               _ptr(max_new), _ptr(capacity), _ptr(init_history), _stream(),
                               ctypes.byref(h)), "pf_sim_create")
        self._h = h
        self.n = n
        self.n_req = int(req_input.numel())

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            load().pf_sim_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def step(self, iterations: int):
        _check(load().pf_sim_step(self._h, iterations, _stream()), "pf_sim_step")

    def n_done(self) -> int:
        d = _i32()
        _check(load().pf_sim_done(self._h, ctypes.byref(d), _stream()), "pf_sim_done")
        return d.value

    def run(self, chunk: int = 256, max_iterations: int = 1 << 30) -> int:
        """Step until every instance is done; returns the iterations launched."""
        it = 0
        while it < max_iterations and self.n_done() < self.n:
            c = min(chunk, max_iterations - it)
            self.step(c)
            it += c
        return it

    def metrics(self):
        """-> (metrics [n, 10] int64, generated [N] int32, evictions [N] int32) on the device."""
        m = torch.empty((self.n, len(SIM_METRICS)), dtype=torch.int64, device="cuda")
        g = torch.empty(max(self.n_req, 1), dtype=torch.int32, device="cuda")
        e = torch.empty_like(g)
        _check(load().pf_sim_metrics(self._h, ctypes.c_void_p(m.data_ptr()), _ptr(g), _ptr(e), _stream()),
               "pf_sim_metrics")
        return m, g[:self.n_req], e[:self.n_req]

    def device_error(self):
        code, idx = _i32(), _i32()
        ctx = load().pf_sim_context(self._h)
        _check(load().pf_get_device_error(ctx, ctypes.byref(code), ctypes.byref(idx), _stream()),
               "pf_get_device_error")
        return code.value, idx.value


def window_similarity(lengths: torch.Tensor, window: int, max_len: int):
    """fig:dist (NEXT-3): -> (gram [B, B] int64, cos [B, B] float64, summary [2] float64:
    mean adjacent, mean global) on the device."""
    B = lengths.numel() // window if window > 0 else 0
    dev = lengths.device
    g = torch.empty((max(B, 1), max(B, 1)), dtype=torch.int64, device=dev)
    c = torch.empty((max(B, 1), max(B, 1)), dtype=torch.float64, device=dev)
    sm = torch.empty(2, dtype=torch.float64, device=dev)
    _check(load().pf_window_similarity(_ptr(lengths), lengths.numel(), window, max_len,
                                       ctypes.c_void_p(g.data_ptr()), ctypes.c_void_p(c.data_ptr()),
                                       ctypes.c_void_p(sm.data_ptr()), _stream()), "pf_window_similarity")
    return g, c, sm


def adjacent_similarity(lengths: torch.Tensor, hist_window: int, run_window: int, max_len: int):
    """fig:cos_win (NEXT-3): -> (cos per running window [K] float64, mean [1] float64)."""
    n = lengths.numel()
    K = (n - hist_window) // run_window if (hist_window > 0 and run_window > 0 and n >= hist_window + run_window) else 0
    dev = lengths.device
    c = torch.empty(max(K, 1), dtype=torch.float64, device=dev)
    m = torch.empty(1, dtype=torch.float64, device=dev)
    _check(load().pf_adjacent_similarity(_ptr(lengths), n, hist_window, run_window, max_len,
                                         ctypes.c_void_p(c.data_ptr()), ctypes.c_void_p(m.data_ptr()),
                                         _stream()), "pf_adjacent_similarity")
    return c[:K], m


def _wrap_device_int32(ptr: int, count: int) -> torch.Tensor:
    """Zero-copy int32 CUDA tensor view of a context-owned device buffer."""
    class _CAI:
        __cuda_array_interface__ = {"shape": (count,), "typestr": "<i4", "data": (ptr, False),
                                    "version": 3, "strides": None}
    return torch.as_tensor(_CAI(), device="cuda")
