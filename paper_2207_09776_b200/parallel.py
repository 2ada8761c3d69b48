"""Multi-GPU host logic: paths are sharded across ranks, statistics are combined once.

The reference runs every trajectory independently (OpenMP over paths,
proj/src/magnus.cpp:258-263, euler.cpp:142-145); there is no exchange inside the hot path.
On B200s each rank (one process per GPU, ``torch.distributed`` over NCCL) owns a
contiguous range of global path ids; Philox streams are keyed by the global id, so the
paths do not depend on the number of ranks.  The only collective is the final reduction
of the error/moment statistics:

* ``Err`` (analysis.cpp:93-130) is a sum over paths in ascending m divided by M.  To be
  bitwise independent of the rank count, the per-path ratios are all-gathered and summed
  in global path order (M doubles).
* the ME matrix, the moment sums (sum u, sum u^2) and the counts are all-reduced (sums).
"""
from __future__ import annotations

import math
from typing import Optional

import numpy as np


def shard(M_total: int, rank: int, world: int):
    """Contiguous path range of `rank`: (offset, count); the first M % world ranks get one
    more path."""
    base, extra = divmod(M_total, world)
    count = base + (1 if rank < extra else 0)
    offset = rank * base + min(rank, extra)
    return offset, count


def _t(x, device):
    import torch
    return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device=device)


def max_over_ranks(value: float, group=None, device="cpu") -> float:
    import torch
    import torch.distributed as dist
    if not dist.is_initialized():
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def combine_error_stats(per_path_rel: np.ndarray, me: np.ndarray, used: int, blowups: int,
                        M_total: int, moments: Optional[np.ndarray] = None, group=None,
                        device="cpu"):
    """Combine one rank's norms into the global RelError / MeanAbsError.

    per_path_rel: this rank's ||ref-app||_F/||ref||_F per path (NaN = blown), in path order.
    me: this rank's ME matrix (already divided by its `used`).
    Returns dict(err, blowups, ame, me, used[, sum_u, sum_u2]).
    """
    import torch
    import torch.distributed as dist
    rel = np.ascontiguousarray(per_path_rel, dtype=np.float64)
    if dist.is_initialized():
        world = dist.get_world_size(group)
        counts = torch.zeros(world, dtype=torch.int64, device=device)
        counts[dist.get_rank(group)] = len(rel)
        dist.all_reduce(counts, group=group)
        cmax = int(counts.max().item())
        buf = torch.full((cmax,), float("nan"), dtype=torch.float64, device=device)
        buf[:len(rel)] = _t(rel, device)
        parts = [torch.empty(cmax, dtype=torch.float64, device=device) for _ in range(world)]
        dist.all_gather(parts, buf, group=group)
        rel_all = np.concatenate([p[:int(c)].cpu().numpy() for p, c in zip(parts, counts.tolist())])
        packed = np.concatenate([np.asarray(me, np.float64).reshape(-1) * used,
                                 [float(used), float(blowups)],
                                 np.asarray(moments, np.float64).reshape(-1) if moments is not None else []])
        t = _t(packed, device)
        dist.all_reduce(t, group=group)
        packed = t.cpu().numpy()
        w2 = np.asarray(me).size
        me_sum, used_all, blow_all = packed[:w2], int(packed[w2]), int(packed[w2 + 1])
        mom = packed[w2 + 2:] if moments is not None else None
    else:
        rel_all = rel
        me_sum = np.asarray(me, np.float64).reshape(-1) * used
        used_all, blow_all = used, blowups
        mom = moments
    # ascending global m, the reference's accumulation order (analysis.cpp:99-127)
    s = 0.0
    for r in rel_all:
        if not math.isnan(r):
            s += float(r)
    err = math.inf if blow_all > 0 else s / float(M_total)
    me_all = (me_sum / used_all if used_all else me_sum).reshape(np.asarray(me).shape)
    out = {"err": err, "blowups": blow_all, "used": used_all, "me": me_all,
           "ame": float(me_all.mean()) if me_all.size else 0.0}
    if mom is not None:
        n = len(mom) // 2
        out["sum_u"], out["sum_u2"] = mom[:n], mom[n:]
    return out
