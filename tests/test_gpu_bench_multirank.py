"""The bench's N > 1 flow, end to end, with two ranks on ONE GPU.

Covered: torchrun launch, identical slab partition on every rank, row-windowed uploads, the fused slab
gather (final-pass stores into rank 0's volume through CUDA IPC), the max-reduce of timings, and rank 0's
JSON line.

The control plane runs on gloo (BP_BENCH_BACKEND=gloo), because NCCL refuses two ranks on one device.
The two ranks' kernels are independent: neither waits on the other. This is a correctness test only and
produces no scaling number.
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_fused_gather_bitwise():
    env = dict(os.environ, BP_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29541", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--edge", "128", "--views", "64", "--batch", "32", "--steps", "1",
           "--warmup", "1", "--no-cpu", "--no-fdk", "--verify-gather"]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
    d = json.loads(line)
    assert d["n_gpus"] == 2
    assert "fused slab gather" in d["config"]["parallelism"]
    assert d["gather_bitwise_vs_single_context"] is True
    assert d["gpu_launches"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
