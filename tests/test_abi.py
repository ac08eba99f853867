"""The C-ABI library loads and exports every symbol include/pfsched.h declares, and
host-checkable argument errors return synchronously (no GPU needed for these)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "pfsched.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pf_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2507_10150_b200 import build
    build.build()
    import paper_2507_10150_b200 as P
    return P.load()


def test_exports_every_declared_symbol(lib):
    decl = _declared()
    assert {"pf_create", "pf_destroy", "pf_update_history", "pf_estimate_peak", "pf_admit"} <= set(decl)
    for name in decl:
        assert hasattr(lib, name), name
    import paper_2507_10150_b200 as P
    assert set(P.SYMBOLS) == set(decl)


def test_abi_version(lib):
    assert lib.pf_abi_version() == 2


def _cfg(**kw):
    from paper_2507_10150_b200.binding import PFConfig
    base = dict(n_instances=4, window=100, max_len=512, max_input_len=512, max_entries=64, n_groups=0,
                group_off=None, instance_base=0, members_per_group=0, member_base=0, mode=0,
                quantile_u=0, repetitions=1, reserved_bp=0, seed=0, rank=0, nranks=1, nccl_unique_id=None)
    base.update(kw)
    return PFConfig(**base)


@pytest.mark.parametrize("kw,status", [
    (dict(n_instances=0), -1), (dict(window=0), -1), (dict(max_len=0), -2), (dict(max_len=40000), -2),
    (dict(max_entries=5000), -2), (dict(repetitions=-1), -1), (dict(reserved_bp=10000), -1),
    (dict(mode=7), -1), (dict(max_input_len=10**7, max_entries=4096), -2),
    (dict(n_groups=2, window=100), -1), (dict(n_groups=2, window=96), -1),
    (dict(n_groups=2, window=96, group_off=1234, nranks=3), -1),
    (dict(nccl_unique_id=1234), -1),  # a communicator only exists in shared mode
])
def test_host_validation(lib, kw, status):
    h = ctypes.c_void_p()
    cfg = _cfg(**kw)
    st = lib.pf_create(ctypes.byref(cfg), None, None, ctypes.byref(h))
    assert st == status
    assert h.value is None
    assert len(lib.pf_last_error()) > 0


def test_null_arguments(lib):
    assert lib.pf_create(None, None, None, None) == -1
    assert lib.pf_destroy(None) == -1
    assert lib.pf_admit(*([None] * 8), 0, *([None] * 6)) == -1
    assert lib.pf_estimate_peak(None, None, None, None, None, 0, None, None, None) == -1
    assert lib.pf_update_history(None, None, None, 0, None) == -1


def test_sim_null_arguments(lib):
    assert lib.pf_sim_create(None, *([None] * 7), None) == -1
    assert lib.pf_sim_step(None, 1, None) == -1
    assert lib.pf_sim_done(None, None, None) == -1
    assert lib.pf_sim_metrics(None, None, None, None, None) == -1
    assert lib.pf_sim_destroy(None) == -1
    assert lib.pf_sim_context(None) is None


@pytest.mark.parametrize("kw", [dict(n_instances=0), dict(policy=9), dict(policy=0, param_bp=10000),
                                dict(policy=2, param_bp=0), dict(max_len=0)])
def test_sim_host_validation(lib, kw):
    from paper_2507_10150_b200.binding import PFSimConfig
    base = dict(n_instances=2, window=16, max_len=64, max_input_len=64, max_entries=16, policy=0,
                param_bp=300, mode=0, quantile_u=0, repetitions=1, seed=0, instance_base=0)
    base.update(kw)
    cfg = PFSimConfig(**base)
    h = ctypes.c_void_p()
    dummy = ctypes.c_void_p(16)  # never dereferenced: the config is rejected first
    assert lib.pf_sim_create(ctypes.byref(cfg), *([dummy] * 5), None, None, ctypes.byref(h)) == -1
    assert h.value is None


def test_analysis_host_validation(lib):
    assert lib.pf_window_similarity(None, 10, 2, 8, None, None, None, None) == -1
    dummy = ctypes.c_void_p(16)
    assert lib.pf_window_similarity(dummy, 3, 2, 8, None, None, None, None) == -1   # one window
    assert lib.pf_window_similarity(dummy, 10, 2, 40000, None, None, None, None) == -2
    assert lib.pf_adjacent_similarity(dummy, 10, 8, 4, 8, dummy, None, None) == -1  # no running window
    assert lib.pf_adjacent_similarity(dummy, 10, 2, 2, 8, None, None, None) == -1


def test_forward_null_arguments(lib):
    assert lib.pf_forward(None, 1, *([None] * 7), 0, *([None] * 4)) == -1


def test_nccl_unique_id(lib):
    """pf_nccl_unique_id: NULL output is rejected; otherwise NCCL is dlopen'ed at run time
    and writes 128 bytes (PF_ENCCL = -5 only if NCCL cannot be loaded)."""
    assert lib.pf_nccl_unique_id(None) == -1
    buf = ctypes.create_string_buffer(128)
    st = lib.pf_nccl_unique_id(buf)
    assert st in (0, -5), st
    if st == 0:
        assert any(buf.raw)
