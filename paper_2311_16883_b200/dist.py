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


def plan_buckets(nbytes: list[int], cap_bytes: int) -> list[list[int]]:
    """Group consecutive gradients (in the order the backward pass produces them)
    into all-reduce buckets of at most cap_bytes each (a gradient larger than the
    cap gets a bucket of its own).  Buckets amortise the collective's launch and
    latency while the first ones overlap the rest of the backward pass."""
    if cap_bytes <= 0:
        raise ValueError("cap_bytes must be positive")
    buckets, cur, size = [], [], 0
    for i, n in enumerate(nbytes):
        if cur and size + n > cap_bytes:
            buckets.append(cur)
            cur, size = [], 0
        cur.append(i)
        size += n
    if cur:
        buckets.append(cur)
    return buckets


class BucketedAllReduce:
    """a7 overlapped with the backward pass: per-layer dW tensors are views into
    flat per-bucket buffers (bsr_wgrad writes straight into them); when the last
    gradient of a bucket has been issued, the bucket is all-reduced on a separate
    communication stream (NCCL; gloo on CPU) while the compute stream goes on
    with the next layers' dW.  wait() makes the caller's stream wait for every
    bucket.  shapes: (K, N) of each gradient in backward order."""

    def __init__(self, shapes, device, cap_bytes: int = 40 << 20, group=None, dtype=torch.float32):
        self.device = torch.device(device)
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        esz = torch.empty((), dtype=dtype).element_size()
        self.buckets = plan_buckets([int(k) * int(n) * esz for k, n in shapes], cap_bytes)
        self.flat, self.views, self.last = [], [None] * len(shapes), {}
        for bi, members in enumerate(self.buckets):
            total = sum(int(shapes[i][0]) * int(shapes[i][1]) for i in members)
            buf = torch.empty(total, dtype=dtype, device=self.device)
            off = 0
            for i in members:
                n = int(shapes[i][0]) * int(shapes[i][1])
                self.views[i] = buf[off:off + n].view(int(shapes[i][0]), int(shapes[i][1]))
                off += n
            self.flat.append(buf)
            self.last[members[-1]] = bi
        self.cuda = self.device.type == "cuda"
        self.comm = torch.cuda.Stream(self.device) if self.cuda else None
        self.works = []

    def view(self, i: int) -> torch.Tensor:
        return self.views[i]

    def ready(self, i: int) -> None:
        """Gradient i has been issued on the current stream; launch its bucket's
        all-reduce if i completes the bucket."""
        bi = self.last.get(i)
        if bi is None or self.world == 1:
            return
        if self.cuda:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(self.device))
            with torch.cuda.stream(self.comm):
                self.comm.wait_event(ev)
                self.works.append(dist.all_reduce(self.flat[bi], op=dist.ReduceOp.SUM, group=self.group,
                                                  async_op=True))
        else:
            self.works.append(dist.all_reduce(self.flat[bi], op=dist.ReduceOp.SUM, group=self.group, async_op=True))

    def wait(self) -> None:
        for w in self.works:
            w.wait()  # NCCL: the current stream waits for the collective
        self.works = []
        if self.cuda:
            torch.cuda.current_stream(self.device).wait_stream(self.comm)


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
