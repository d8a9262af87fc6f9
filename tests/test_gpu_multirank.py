"""bench.py's multi-rank control path (f1 set-up) run end to end on a 1-GPU box.

Two ranks under torch.distributed.run with the control plane over gloo (BENCH_DIST_BACKEND=gloo), both on
cuda:0: the fused all-reduce set-up (with W4A16_NVLS=1 the NVLS multicast object is attempted first — two
ranks on one device cannot share one, so every rank falls back to CUDA-IPC peer regions together), the
start-up check of one
fused forward against the same forward op by op with the process-group all-reduce, the fallback when the
check fails on one rank (BENCH_FAIL_FUSED_CHECK=<rank>), and the hard failure of --allreduce fused. The
timed numbers of these runs mean nothing (two contexts time-slice one GPU); the JSON contract and the
branch taken are what is checked."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(extra_env, *args):
    env = dict(os.environ, BENCH_DIST_BACKEND="gloo", W4A16_NVLS="1", **extra_env)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--model", "8b",
           "--layers", "2", "--M", "8", "--sweep", "", "--sym-sweep", "", "--steps", "2", "--warmup", "3",
           "--no-kernels", "--no-lm-head", "--no-cpu-baseline", *args]
    return subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)


def _line(out):
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:] + out.stderr[-4000:]
    return json.loads(lines[0])


@pytest.mark.timeout(700)
def test_two_ranks_fused_allreduce_setup_and_check():
    out = _run({})
    assert out.returncode == 0, out.stderr[-4000:]
    d = _line(out)
    assert d["n_gpus"] == 2 and d["config"]["tp"] == 2
    assert d["config"]["allreduce"].startswith("fused"), d["config"]["allreduce"]
    assert d["value"] > 0


@pytest.mark.timeout(700)
def test_two_ranks_fall_back_together_when_the_check_fails_on_one():
    out = _run({"BENCH_FAIL_FUSED_CHECK": "1"})
    assert out.returncode == 0, out.stderr[-4000:]
    d = _line(out)
    assert d["config"]["allreduce"] == "gloo"           # the process-group all-reduce (NCCL in production)
    assert "falling back" in out.stderr


@pytest.mark.timeout(700)
def test_allreduce_fused_fails_hard_when_the_check_fails():
    out = _run({"BENCH_FAIL_FUSED_CHECK": "0"}, "--allreduce", "fused")
    assert out.returncode != 0
    assert "start-up check failed" in out.stderr
