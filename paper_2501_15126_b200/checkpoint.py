"""Resumable long runs: the Gray range is swept as `pieces`
power-of-two shards in order (perm_compute_shard(piece, pieces)); after each
piece its unscaled partial (FP64 bits, or the exact INT01 T' partial) is
appended to a JSON checkpoint.  A restart skips the recorded pieces.  The
pieces are complete subtrees of the one-call reduction tree, so folding them
with perm_fold reproduces perm_compute bit for bit.
"""
from __future__ import annotations

import hashlib
import json
import os
import struct

from . import perm_result


def _bits(x: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def _float(b: int) -> float:
    return struct.unpack("<d", struct.pack("<Q", b))[0]


def _key(plan, pieces: int) -> dict:
    """Structure AND values: the generated kernel bakes every matrix value in
    as a literal, so the hash of its source and cubin tells two matrices with
    the same sparsity pattern apart (their partials must never be mixed)."""
    i = plan.info
    h = hashlib.sha256(plan.source.encode())
    h.update(plan.cubin())
    return {"n": i["n"], "nnz": i["nnz"], "K": i["K"], "B": i["B"], "M": i["M"], "tasks": i["tasks"],
            "row_perm": i["row_perm"], "col_perm": i["col_perm"], "mode": i["mode"], "pieces": pieces,
            "kernel_sha256": h.hexdigest()}


# warp-tasks a piece keeps at least: ~14 waves of the 1184 resident warps of a
# B200 (148 SMs x 2 blocks x 4 warps), so the last-wave tail of each piece
# stays small (a 2048-task piece, 1.7 waves, swept ER n=48 in 7.06 s against
# 6.02 s in one call)
MIN_TASKS_PER_PIECE = 1 << 14


def auto_pieces(plan) -> int:
    """The largest power of two <= 128 that leaves every piece
    MIN_TASKS_PER_PIECE warp-tasks (at least 1)."""
    tasks = int(plan.info["tasks"])
    p = 1
    while p < 128 and tasks // (2 * p) >= MIN_TASKS_PER_PIECE:
        p *= 2
    return p


def compute_resumable(plan, path: str, pieces: int | None = None, max_pieces: int | None = None):
    """Run (or resume) the permanent of `plan` in `pieces` shards (default:
    auto_pieces(plan)), checkpointing to `path` (JSON).  `max_pieces` bounds the
    pieces swept in this call (to emulate an interruption).  Returns the folded
    perm_result when complete, else None."""
    if pieces is None:
        pieces = auto_pieces(plan)
    state = {"key": _key(plan, pieces), "done": {}}
    if os.path.exists(path):
        with open(path) as f:
            old = json.load(f)
        if old.get("key") != state["key"]:
            raise ValueError(f"checkpoint {path} belongs to another plan/geometry")
        state = old
    swept = 0
    for r in range(pieces):
        if str(r) in state["done"]:
            continue
        if max_pieces is not None and swept >= max_pieces:
            return None
        s = plan.shard(r, pieces)
        state["done"][str(r)] = {"bits": _bits(s.value), "bits_im": _bits(s.value_im),
                                 "lo": s.exact_lo, "hi": s.exact_hi, "valid": s.exact_valid,
                                 "sweep_ms": s.sweep_ms}
        tmp = path + ".tmp"
        with open(tmp, "w") as f:
            json.dump(state, f)
        os.replace(tmp, path)  # atomic: a crash leaves the previous checkpoint
        swept += 1
    shards = []
    for r in range(pieces):
        d = state["done"][str(r)]
        s = perm_result()
        s.value = _float(d["bits"])
        s.value_im = _float(d["bits_im"])   # complex plans: imaginary partial (0 otherwise)
        s.exact_lo, s.exact_hi, s.exact_valid = d["lo"], d["hi"], d["valid"]
        s.sweep_ms = d["sweep_ms"]
        shards.append(s)
    return plan.fold(shards)
