"""Row sharding across GPUs: decode rows (request x layer x draft token)
share nothing, so a batch splits into contiguous row blocks, one per rank, with no
collective on the hot path.  The optional gather of every rank's out_idx onto all ranks
(`gather_rows`, NCCL all-gather over NVLink / NVSwitch) is a single collective after the
selection and is not part of the per-row work.  Host-side logic only: the selection itself
is `gvr.topk` on each rank's own GPU.
"""
from __future__ import annotations

import numpy as np


def row_partition(row_lens, world: int) -> np.ndarray:
    """Split rows 0..R-1 into `world` contiguous blocks with near-equal total work.

    Work per row is its length (the row is read once; SURVEY.md §8e "balanced by
    Σ row_len").  Returns int64 bounds[world + 1] with bounds[0] = 0, bounds[-1] = R;
    rank w owns rows [bounds[w], bounds[w+1]).  Deterministic; blocks may be empty when
    R < world.
    """
    lens = np.asarray(row_lens, dtype=np.int64).reshape(-1)
    if world < 1:
        raise ValueError("world must be >= 1")
    R = lens.size
    bounds = np.zeros(world + 1, dtype=np.int64)
    bounds[-1] = R
    if R == 0:
        return bounds
    cum = np.concatenate([[0], np.cumsum(np.maximum(lens, 0) + 1)])  # +1: every row has a fixed cost
    total = cum[-1]
    for w in range(1, world):
        target = total * w / world
        b = int(np.searchsorted(cum, target, side="left"))
        # pick the closer of the two neighbouring cut points
        if b > 0 and abs(cum[b - 1] - target) <= abs(cum[min(b, R)] - target):
            b -= 1
        bounds[w] = min(max(b, bounds[w - 1]), R)
    return bounds


def gather_rows(local, bounds, group=None):
    """All-gather each rank's [rows_w, k] int32 block into the full [R, k] array on
    every rank (torch.distributed; NCCL on GPUs, gloo on CPU).  Blocks are padded to the
    largest block for the collective and trimmed afterwards."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    sizes = np.diff(np.asarray(bounds))
    if local.shape[0] != sizes[rank]:
        raise ValueError(f"rank {rank}: local block has {local.shape[0]} rows, partition says {sizes[rank]}")
    width = local.shape[1]
    mx = int(sizes.max()) if world else 0
    pad = torch.full((mx, width), -1, dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([parts[w][: int(sizes[w])] for w in range(world)], dim=0)


def sharded_topk(scores, row_lens, prev, k, bounds, gather=False, group=None, topk_fn=None):
    """Select this rank's block [bounds[rank], bounds[rank+1]) of a batch held by every
    rank (scores [R, S]; row_lens [R]; prev [R, k] or None) and optionally gather the
    full [R, k] result.  `topk_fn` defaults to the CUDA path (gvr.topk)."""
    import torch.distributed as dist

    if topk_fn is None:
        from . import topk as topk_fn
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    loc_prev = None if prev is None else prev[lo:hi].contiguous()
    out = topk_fn(scores[lo:hi].contiguous(), k, row_lens=row_lens[lo:hi].contiguous(), prev=loc_prev)
    return gather_rows(out, bounds, group) if gather else out
