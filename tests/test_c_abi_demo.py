"""include/pfsched.h is usable from plain C: examples/c_abi_demo.c (no torch, no Python in
the process) builds against libpfsched.so here, and on the GPU it reproduces the config-1
worked example (SURVEY P-5) through a per-instance context and through a
shared-mode context that owns a one-rank NCCL communicator."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "examples"))


def _build():
    from paper_2507_10150_b200 import build as B
    B.build()
    import build as EB  # examples/build.py
    return EB.build()


def test_c_demo_compiles_and_links():
    exe = _build()
    assert os.path.exists(exe)


@pytest.mark.gpu
def test_c_demo_runs_worked_example():
    exe = _build()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "c_abi_demo: ok" in r.stdout
    assert r.stdout.count("-> ok") == 4, r.stdout  # three per-instance contexts + the NCCL one
