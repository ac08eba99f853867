"""bench.py's N-rank path end to end on a one-GPU box: `bench.py --gpus 2` relaunches itself
under torch.distributed.run, both ranks run the timed cfg-5 schedule (side-stream history
exchange overlapping admit, max-over-ranks timing, e2e leg, output check) and rank 0 prints
one JSON line with n_gpus = 2. Test hook PFBENCH_SINGLE_DEVICE=1: both ranks on cuda:0 with a
gloo group and the caller-driven exchange, since NCCL refuses two ranks on one device (the
NCCL data plane itself is covered by the one-rank library communicator test)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("weak", [False, True])
def test_bench_two_ranks_one_device(weak):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["PFBENCH_SINGLE_DEVICE"] = "1"
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "4", "--warmup", "3",
           "--no-cpu-baseline", "--e2e-steps", "1", "--tick-pool", "4"] + (["--weak"] if weak else [])
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    d = json.loads(lines[-1])
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["scaling"] == ("weak" if weak else "strong")
    assert d["config"]["output_check"]["violations"] == 0
    assert d["config"]["instances"] == (2 if weak else 1) * (1 << 20)


def test_bench_two_ranks_replicas_cfg4():
    """Per-instance configs shard the instance range with no collective ("replicas"):
    two ranks each time half of cfg 4; the line reports the whole job."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["PFBENCH_SINGLE_DEVICE"] = "1"
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "4", "--steps", "4",
           "--warmup", "3", "--no-cpu-baseline", "--e2e-steps", "1", "--tick-pool", "4"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-4000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.strip()][-1])
    assert d["n_gpus"] == 2 and d["config"]["instances"] == 65536
    assert d["config"]["output_check"]["violations"] == 0
