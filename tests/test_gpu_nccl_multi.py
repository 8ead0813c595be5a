"""Multi-GPU NCCL data plane (libperm-owned communicator, rank-0 planning and
plan broadcast) through bench.py under torchrun.  Needs >= 2 GPUs: skipped on
one-GPU boxes (the world-1 NCCL path is covered in test_gpu_parity.py)."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT, cuda_available


def _ngpu():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available() or _ngpu() < 2, reason="needs >= 2 GPUs")]


def run(cmd):
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900,
                         env={**os.environ, "PYTHONPATH": ROOT})
    assert out.returncode == 0, out.stderr[-3000:]
    return json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])


def test_two_gpus_nccl_bitwise():
    common = ["--dim", "34", "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--no-plain", "--no-cold"]
    one = run([sys.executable, "bench.py", *common])
    two = run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
               "--master-addr", "127.0.0.1", "--master-port", "29631", "bench.py", "--gpus", "2", *common])
    assert two["n_gpus"] == 2 and two["result"] == one["result"]
    assert "NCCL" in two["config"]["parallelism"]
