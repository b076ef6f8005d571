"""Multi-GPU plumbing for the forward model: pairs are
independent and U depends only on the structure, so a batch is
sharded by CONTIGUOUS structure blocks (a structure's coefficient table is
built on one GPU only) with no collective on the data path; the only
communication is the final host gather of eta in row order (sweep.cpp:92-108
analogue), which keeps the output identical for any GPU count."""
from __future__ import annotations

import numpy as np


def shard_structures(n_structures: int, rank: int, world: int):
    """Contiguous block [lo, hi) of structures for `rank` (balanced, first
    ranks take the remainder)."""
    base, rem = divmod(n_structures, world)
    lo = rank * base + min(rank, rem)
    hi = lo + base + (1 if rank < rem else 0)
    return lo, hi


def shard_pairs(pairs, n_structures: int, rank: int, world: int):
    """The pairs (structure, theta0, theta1) owned by `rank`, with their
    structure index rebased to the shard, plus their positions in the batch."""
    lo, hi = shard_structures(n_structures, rank, world)
    idx = [i for i, p in enumerate(pairs) if lo <= int(p[0]) < hi]
    local = [(int(pairs[i][0]) - lo, float(pairs[i][1]), float(pairs[i][2])) for i in idx]
    return lo, hi, idx, local


def gather_rows(local_rows: np.ndarray, idx, total: int, group=None):
    """Assemble per-rank rows into the full batch in row order on every rank
    (all_gather_object over the process group: host-side, off the hot path)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    parts = [None] * world
    dist.all_gather_object(parts, (list(idx), np.asarray(local_rows)), group=group)
    out = None
    for ids, rows in parts:
        if out is None:
            out = np.zeros((total,) + rows.shape[1:], dtype=rows.dtype)
        if len(ids):
            out[np.asarray(ids)] = rows
    return out
