"""Multi-GPU plumbing for the fused iteration (one process per GPU).

The reference is single-process; the B200 build shards the
iteration two ways, both ending in ONE collective exchange per
iteration:

* frame sharding (configs 2, 3, 5): the loss and gradient are sums over
  frames (reconstruction.py:303-316), so each rank runs deform -> forward ->
  adjoint -> deformation backward for a contiguous block of the selected
  frames and the flat float32 parameter gradients are all-reduced (SUM).
* sensor sharding (config 4): each rank owns a contiguous sensor block for
  every frame; ball states are recomputed on every rank (the "ball tiles
  broadcast": replicated parameters, a few ms of deform work), the adjoint
  gives per-rank partial state gradients, and because the deformation
  backward is linear in G the partial parameter gradients are all-reduced.

Every rank then applies the identical Adam step, so parameters stay
replicated without a parameter broadcast.
"""

from __future__ import annotations

import numpy as np


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of n items owned by `rank` of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    return (n * rank) // world, (n * (rank + 1)) // world


def frame_shard(selected, rank: int, world: int) -> np.ndarray:
    """This rank's frames out of the iteration's selected frames."""
    selected = np.asarray(selected, dtype=np.int64)
    lo, hi = shard_range(len(selected), rank, world)
    return selected[lo:hi]


def allreduce_iteration(grads, loss, coincident, group=None) -> None:
    """The iteration's exchange: SUM of the flat gradient buffer and of the
    loss, MIN of the coincidence word (INT64_MAX = none).  In place; works
    for NCCL (device tensors) and gloo (CPU tensors).

    Two collectives per iteration, none of which the host waits on: the f32
    gradients (all-reduce SUM) and a 16-byte status record per rank
    (all-gather of [loss bits, coincidence word] as int64), reduced on every
    rank in rank order -- the loss SUM and the coincidence MIN are identical
    on all ranks.  The host reads the results once, with the rest of the
    iteration's status after the guarded update."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return
    world = dist.get_world_size(group)
    if world == 1:
        return
    dist.all_reduce(grads, op=dist.ReduceOp.SUM, group=group)
    status = torch.stack([loss.reshape(1).view(torch.int64)[0],
                          coincident.reshape(1)[0]])
    gathered = torch.empty((world, 2), dtype=torch.int64, device=status.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(gathered, status, group=group)
    else:
        dist.all_gather(list(gathered.unbind(0)), status, group=group)
    loss.copy_(gathered[:, 0].contiguous().view(torch.float64).sum()
               .reshape(loss.shape))
    coincident.copy_(gathered[:, 1].min().reshape(coincident.shape))
