"""The multi-rank bench path (torchrun, shard sweep + all-gather + rank-order
fold + max-over-ranks timing) end to end on one B200: two ranks share the GPU
over gloo (NCCL refuses duplicate devices); the folded result must equal the
one-rank result bit for bit."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT, cuda_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_available(), reason="needs a B200")]


def run(cmd):
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900,
                         env={**os.environ, "PYTHONPATH": ROOT})
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    return json.loads(lines[-1])


def test_two_ranks_share_one_gpu_bitwise():
    common = ["--dim", "32", "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--no-plain", "--no-cold"]
    one = run([sys.executable, "bench.py", *common])
    two = run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
               "--master-addr", "127.0.0.1", "--master-port", "29613", "bench.py", "--gpus", "2",
               "--backend", "gloo", "--same-device", *common])
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert two["result"] == one["result"]
    # per step: sweep + tree passes over the rank's slots + fold (fewer passes per shard)
    assert 0 < two["gpu_launches"] <= one["gpu_launches"]
    assert two["value"] > 0 and two["e2e"]["value"] > 0
