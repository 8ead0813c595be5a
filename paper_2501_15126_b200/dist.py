"""Multi-GPU plumbing (one process per GPU; torch.distributed only moves
host-side bytes: the NCCL unique id and the plan blob).

The Gray range is split into `world` power-of-two-aligned shards of whole
warp-tasks (perm_shard_range).  Production path (`init_comm` + `plan_on_rank0`):
rank 0 plans (search + NVRTC) once and broadcasts the exported plan, every
rank imports it with its own rank/world/NCCL communicator, and
perm_compute_async sweeps the rank's shard, all-gathers the 8/16-byte
partials over NCCL inside libperm (the path's single exchange step) and folds
them in rank order with the deterministic fold kernel -- bitwise identical to
the one-GPU result.  `ShardedPermanent` is the host-staged variant for gloo
tests (ranks sharing one GPU, where NCCL refuses duplicate devices).
"""
from __future__ import annotations

import hashlib


def plan_signature(plan):
    """Everything that decides the kernel bits: geometry, orderings and the
    hash of the generated source and cubin (codegen variant, caches, bounds)."""
    i = plan.info
    h = hashlib.sha256(plan.source.encode())
    h.update(plan.cubin())
    return (i["K"], i["B"], i["U"], i["M"], i["tasks"], tuple(i["col_perm"]), tuple(i["row_perm"]), h.hexdigest())


def _bcast_bytes(data, rank: int, group=None):
    import torch.distributed as dist
    box = [data if rank == 0 else None]
    dist.broadcast_object_list(box, src=0, group=group)
    return box[0]


def init_comm(rank: int, world: int, device: int, group=None):
    """libperm-owned NCCL communicator over the ranks of `group` (any world,
    including 1): rank 0's unique id is broadcast with torch.distributed."""
    from . import Comm
    uid = Comm.unique_id() if rank == 0 else None
    if world > 1:
        uid = _bcast_bytes(uid, rank, group)
    return Comm(world, rank, uid, device)


def plan_on_rank0(make_plan, group=None, **import_opts):
    """Rank 0 runs the planner (make_plan() -> Plan) and broadcasts its export;
    the other ranks import it (no search, no NVRTC) with `import_opts` (device,
    stream, rank, world, nccl_comm).  Every rank runs the same kernel bits."""
    from . import Plan
    rank, world = import_opts.get("rank", 0), max(1, import_opts.get("world", 1))
    if rank == 0:
        plan = make_plan()
        blob = plan.export()
    else:
        plan, blob = None, None
    if world > 1:
        blob = _bcast_bytes(blob, rank, group)
    if rank != 0:
        plan = Plan.from_blob(blob, **import_opts)
    return plan


def agree_plan(make_plan, world: int, group=None):
    """Plan on every rank (make_plan(autotune=...) -> Plan).  The planner's
    autotune may, on a near-tie, pick different kernels on different GPUs; the
    shards only form one reduction tree if all ranks run the same plan, so on
    any disagreement every rank re-plans with the deterministic model pick.
    Returns (plan, autotune setting used)."""
    plan = make_plan(autotune=0)
    if world == 1:
        return plan, 0
    import torch.distributed as dist
    sigs = [None] * world
    dist.all_gather_object(sigs, plan_signature(plan), group=group)
    if all(s == sigs[0] for s in sigs):
        return plan, 0
    plan.close()
    return make_plan(autotune=-1), -1


class ShardedPermanent:
    """Buffers + one-call step for a plan across the ranks of `group`."""

    def __init__(self, plan, rank: int, world: int, device, group=None):
        import torch
        self.plan, self.rank, self.world, self.group = plan, rank, world, group
        self.words = plan.partial_bytes // 8           # 1 (FP64) or 2 (INT01) 8-byte words
        self.part = torch.zeros(2, dtype=torch.float64, device=device)
        self.gathered = torch.zeros(2 * world, dtype=torch.float64, device=device)
        self.out = torch.zeros(2, dtype=torch.float64, device=device)
        if world > 1:
            # every rank plans on its own: the shards only form one reduction
            # tree if all ranks chose the same plan (ordering, K, geometry)
            import torch.distributed as dist
            sigs = [None] * world
            dist.all_gather_object(sigs, plan_signature(plan), group=group)
            if any(s != sigs[0] for s in sigs):
                raise RuntimeError(f"ranks planned different kernels: {sigs}")

    def step(self):
        """Enqueue shard sweep + all-gather + fold on the current stream."""
        import torch.distributed as dist
        self.plan.shard_async(self.rank, self.world, self.part.data_ptr())
        if self.world > 1:
            if dist.get_backend(self.group) == "gloo":   # test path (ranks sharing one GPU): host staging
                host = self.part[: self.words].cpu()
                outs = [host.clone() for _ in range(self.world)]
                dist.all_gather(outs, host, group=self.group)
                self.gathered[: self.world * self.words].copy_(
                    __import__("torch").cat(outs).to(self.gathered.device))
            else:
                dist.all_gather_into_tensor(self.gathered[: self.world * self.words], self.part[: self.words],
                                            group=self.group)
            src = self.gathered
        else:
            src = self.part
        self.plan.fold_async(src.data_ptr(), self.world, self.out.data_ptr())
        return self.out

    def value(self) -> float:
        return float(self.out[0].item())


def gather_fold_host(plan, partial: float, world: int, group=None) -> float:
    """Host-side variant (CPU / gloo): all-gather one FP64 partial per rank and
    fold with perm_fold_host (same fixed order and scale as the fold kernel)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([partial], dtype=torch.float64)
    if world > 1:
        out = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(out, t, group=group)
        parts = [float(x.item()) for x in out]
    else:
        parts = [partial]
    return plan.fold_host(parts)
