"""Multi-GPU plumbing for the env-parallel hot path.

Envs are independent units: each rank owns a contiguous range of GLOBAL env
indices and every per-env random stream is keyed by that global index, so
env i evolves identically on 1, 2, 4 or 8 GPUs and a step needs no
communication.  The only collective is the BPTT reduction of config 4: the
scalar loss and the env-summed gradient of a shared action sequence,
all-reduced (SUM) over NCCL -- a few KB, latency-bound.
"""

from __future__ import annotations


def shard_range(rank: int, world: int, total: int) -> tuple:
    """Global index range [lo, hi) of `rank` among `world` shards of `total` envs."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    return rank * total // world, (rank + 1) * total // world


def is_initialized() -> bool:
    try:
        import torch.distributed as dist

        return dist.is_available() and dist.is_initialized()
    except ImportError:  # pragma: no cover
        return False


def allreduce_sum_(t):
    """In-place SUM over ranks (no-op single process)."""
    if is_initialized():
        import torch.distributed as dist

        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t


def max_over_ranks(x: float, device=None) -> float:
    if not is_initialized():
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_bptt(loss, action_grad_sum, out=None):
    """Pack [action_grad_sum (T*4), loss] into one buffer and all-reduce it:
    one collective per BPTT iteration.  Returns (loss, grad_sum)."""
    import torch

    n = action_grad_sum.numel()
    buf = out if out is not None else torch.empty(n + 1, dtype=torch.float64, device=action_grad_sum.device)
    buf[:n] = action_grad_sum.reshape(-1)
    buf[n] = loss
    allreduce_sum_(buf)
    return buf[n], buf[:n].reshape(action_grad_sum.shape)
