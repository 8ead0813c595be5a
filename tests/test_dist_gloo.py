"""World-size-2 (and 4) CPU tests of the multi-rank host path over gloo:
shard geometry partitions the Gray range, the rank partials (here produced by
the CPU oracle over each rank's Gray range, standing in for the device sweep,
which needs a GPU) are all-gathered, and perm_fold_host's fixed-order fold and
scale reproduce the full permanent.  No GPU."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, p, seed, fc, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        import paper_2501_15126_b200 as pb
        from paper_2501_15126_b200.dist import gather_fold_host
        A = synth.erdos_renyi(n, p, seed)
        P = pb.Plan.from_dense(A, mode="reg", no_device=True, factor_cols=fc)
        info = P.info
        first, ntasks, gb, ge = P.shard_range(rank, world)
        B = A[np.ix_(info["row_perm"], info["col_perm"])]   # the plan's ordered matrix
        part, _ = oracle.nw_range(B, gb, ge)                   # Alg. 1 partial of this shard
        part *= -1.0 if info["K"] % 2 else 1.0                # unscaled h-space partial sign
        val = gather_fold_host(P, part, world)
        ranges = [None] * world
        dist.all_gather_object(ranges, (gb, ge))
        if rank == 0:
            q.put((val, ranges, info["K"]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,fc", [(2, 14, -1), (2, 16, 0), (4, 15, 0)])
def test_gloo_shards_fold_to_full_permanent(world, n, fc):
    import oracle
    import synth
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, n, 0.3, 7, fc, q), nprocs=world, join=True)
    val, ranges, K = q.get(timeout=60)
    # shards tile [0, 2^(n-1)) contiguously in rank order
    assert ranges[0][0] == 0 and ranges[-1][1] == 1 << (n - 1)
    for a, b in zip(ranges, ranges[1:]):
        assert a[1] == b[0]
    A = synth.erdos_renyi(n, 0.3, 7)
    exp, sabs = oracle.perm_nw(A)
    assert abs(val - exp) <= 1e-13 * sabs
