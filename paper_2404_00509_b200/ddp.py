"""DDP plumbing of the loader: samples are independent and
keyed by (seed, epoch, index), so rank r decodes perm[r::world] of the
(padded, DistributedSampler-style) epoch permutation computed identically on every rank -- there is no
collective on the data path.  The only collective is the reporting
reduction after a timed region (max time, summed work), over whatever
process group is initialised (NCCL on the GPU box, gloo in the CPU tests).
"""

from __future__ import annotations

import numpy as np

from .rng import epoch_permutation, shard


def rank_shard(seed: int, epoch: int, n: int, rank: int, world_size: int,
               mode: str = "pad") -> np.ndarray:
    """Indices rank `rank` decodes in `epoch` (pipeline.py:237-243 +
    DistributedSampler striding; rng.shard for the padding modes)."""
    return shard(epoch_permutation(seed, epoch, n), rank, world_size, mode)


def reduce_timing(values, device=None) -> tuple[float, float, float, float]:
    """(ms, images, e2e_ms, e2e_images) of this rank -> job totals: the max
    time over ranks and the summed images (one all_reduce each; identity
    when no process group is initialised)."""
    import torch
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_backend() == "gloo":
        device = "cpu"  # (gloo reduces host tensors)
    v = torch.tensor([float(x) for x in values], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        mx = v.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = v.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        return float(mx[0]), float(sm[1]), float(mx[2]), float(sm[3])
    return float(v[0]), float(v[1]), float(v[2]), float(v[3])
