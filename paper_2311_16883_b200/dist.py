"""Multi-GPU plumbing of the hot path: one process per GPU,
torch.distributed for the process group.

The path shards by batch rows: rank r owns rows [r*M/P, (r+1)*M/P) of X and dY
(whole samples, a multiple of b), prunes them locally with per-rank selection
scope (reading R2 in DESIGN.md) and computes its partial dW = X_r,bsr^T dY_r.
The one exchange step is the sum of the partial dW over ranks (a7), an NCCL
all-reduce over NVLink on GPUs (gloo in the CPU tests).
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env_world() -> tuple[int, int, int]:
    """(rank, local_rank, world_size) from the torchrun environment (1 process: 0, 0, 1)."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def init(backend: str = "nccl") -> tuple[int, int, int]:
    rank, local, world = env_world()
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group(backend, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, local, world


def shard_rows(M: int, world: int, rank: int, align: int) -> tuple[int, int]:
    """Contiguous row range [r0, r1) of rank `rank`: the M/align aligned units
    (whole samples or whole block rows) are split as evenly as possible, lower
    ranks taking the remainder.  Every range is a multiple of `align`."""
    if M % align:
        raise ValueError(f"M={M} is not a multiple of {align}")
    units = M // align
    base, extra = divmod(units, world)
    u0 = rank * base + min(rank, extra)
    u1 = u0 + base + (1 if rank < extra else 0)
    return u0 * align, u1 * align


def allreduce_dw(dW: torch.Tensor, group=None) -> torch.Tensor:
    """a7: in-place sum of the per-rank partial weight gradients."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(dW, op=dist.ReduceOp.SUM, group=group)
    return dW


def max_over_ranks(x: float, device=None) -> float:
    """Device-timed step times are combined as the max over ranks."""
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, device=None) -> float:
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier():
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()


def finalize():
    if dist.is_initialized():
        dist.destroy_process_group()
