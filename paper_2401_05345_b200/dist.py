"""Data parallelism over camera views.

Every rank owns a contiguous block of the view batch, renders and
back-propagates its views into ONE local gradient buffer [P, 9] (the backward
accumulates), and the ranks then combine the buffers with a single all-reduce
(NCCL over NVLink on the GPU path; gloo in the CPU tests). Scene parameters are
replicated; there is no other exchange -- views are independent.
"""
from __future__ import annotations

from typing import Callable, Sequence


def shard_views(num_views: int, world: int, rank: int) -> range:
    """Contiguous block of view ids for `rank`; sizes differ by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("invalid world/rank")
    base, extra = divmod(num_views, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def view_parallel_backward(backward_view: Callable, views: Sequence, grad, group=None,
                           all_reduce: bool = True, chain: bool = False,
                           backward_views: Callable = None):
    """Run `backward_view(view, grad)` (which ADDS into grad) for this rank's
    shard of `views`, then sum `grad` over the group. Returns grad.
    chain: call `backward_view(view, grad, chained=k > 0)` -- the shard's
    backwards after the first may skip the wait for the previous launch
    (dw_render_backward_chained: the views are independent and rendered).
    backward_views: instead, ONE call `backward_views(shard, grad)` for the
    whole shard (dw_render_backward_views)."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    shard = [views[i] for i in shard_views(len(views), world, rank)]
    if backward_views is not None:
        backward_views(shard, grad)
    for k, v in enumerate(shard if backward_views is None else ()):
        if chain:
            backward_view(v, grad, chained=k > 0)
        else:
            backward_view(v, grad)
    if all_reduce and world > 1:
        dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=group)
    return grad


def view_parallel_train_step(grads_view: Callable, views: Sequence, grad3d, update: Callable,
                             group=None, all_reduce: Callable = None):
    """One data-parallel training step: for this rank's shard
    of `views`, `grads_view(view, grad3d)` ADDS the view's 3D parameter
    gradients (render backward + preprocess backward; the preprocess backward
    is view-dependent, so it runs per view) into grad3d [P, 14]; the ranks sum
    grad3d with ONE all-reduce; then every rank applies `update(grad3d)` (the
    optimizer step) to its replica -- identical sums keep the replicas equal.
    all_reduce (optional): a replacement for torch.distributed.all_reduce,
    e.g. the C ABI's dw_allreduce_grads over the group's NCCL communicator."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    for i in shard_views(len(views), world, rank):
        grads_view(views[i], grad3d)
    if world > 1:
        if all_reduce is not None:
            all_reduce(grad3d)
        else:
            dist.all_reduce(grad3d, op=dist.ReduceOp.SUM, group=group)
    update(grad3d)
    return grad3d
