"""Cross-rank global top-k: keep the k = nearest(keep * N_total)
largest blocks of the CONCATENATED activation of all data-parallel ranks, so the
multi-GPU kept set equals the single-GPU one (P:L413-418 applied to the whole
batch; tie rule BJ: lower flat index first = lower rank first).

The device work is the library's (include/bsrprune.h: bsr_gselect_*, the
protocol state in device memory).  This module only issues the collectives
between those calls with torch.distributed:

  1. level-0 digit histogram (key bits 30..19) per rank  -> all-reduce -> boundary bin
  2. while the boundary bin is split: next digit (bits 18..9, then 8..0) of the
     keys in it -> all-reduce -> boundary sub-bin         (at most two more rounds)
  3. per rank (#keys above, #keys tied) at the final digit -> all-gather
  4. tie quota: r = k - sum(above); rank q keeps its first
     clamp(r - ties on ranks < q, 0, ties_q) tied blocks -> k_q = above_q + that.

`threshold_protocol` is the same protocol as pure host logic (injected
histogram / count / collective callables), unit-tested on CPU with gloo at world
size 2 and brute force; the device kernels follow it step by step
(csrc/select_global.cu, gselect_*).
"""
from __future__ import annotations

import ctypes
from typing import Callable, Sequence

import numpy as np

DIGITS = ((12, 19), (10, 9), (9, 0))  # (bits, shift) of the three key digits: 30..19, 18..9, 8..0


def select_bin(hist: Sequence[int], target: int) -> tuple[int, int, int]:
    """Bin holding the target-th largest key (1-based) of a histogram over
    ascending digit values: (bin, keys strictly above the bin, keys in the bin)."""
    h = np.asarray(hist, dtype=np.int64)[::-1]
    cum = np.cumsum(h)
    i = int(np.searchsorted(cum, target))  # first position with cum >= target
    return len(h) - 1 - i, int(cum[i] - h[i]), int(h[i])


def threshold_protocol(k_total: int, rank: int, hist_fn: Callable[[int, int], np.ndarray],
                       counts_fn: Callable[[int, int], tuple[int, int]],
                       allreduce: Callable[[np.ndarray], np.ndarray],
                       allgather: Callable[[np.ndarray], np.ndarray]) -> tuple[int, int, int, int]:
    """Returns (threshold, shift, tie_take, k_rank) for this rank.

    hist_fn(level, prefix) -> this rank's digit histogram; counts_fn(threshold,
    shift) -> this rank's (#(key >> shift) > threshold, #== threshold);
    allreduce sums an int64 vector over ranks; allgather returns the [world, ...]
    stack of every rank's vector."""
    if k_total == 0:
        return 0x7fffffff, 0, 0, 0
    prefix, shift = 0, 19
    hist = allreduce(np.asarray(hist_fn(0, 0), dtype=np.int64))
    b, above, cnt = select_bin(hist, k_total)
    prefix = b
    r = k_total - above
    for level in (1, 2):
        if r >= cnt:  # every key of the boundary bin is kept: no finer digit needed
            break
        bits, nshift = DIGITS[level]
        hist = allreduce(np.asarray(hist_fn(level, prefix), dtype=np.int64))
        b, a, cnt = select_bin(hist, r)
        prefix = (prefix << bits) | b
        above += a
        shift = nshift
        r = k_total - above
    above_q, tie_q = counts_fn(prefix, shift)
    allc = allgather(np.asarray([above_q, tie_q], dtype=np.int64))
    ties_before = int(allc[:rank, 1].sum())
    assert int(allc[:, 0].sum()) == above, "ranks disagree on the keys above the threshold"
    tie_take = int(min(max(r - ties_before, 0), tie_q))
    return prefix, shift, tie_take, int(above_q) + tie_take


def prune_global(X, b: int, keep: float, group=None, stream=None, total_rows: int | None = None):
    """bsr_prune with the whole data-parallel batch as selection scope.  Every rank
    calls it with its own rows; returns this rank's BSR (k_rank blocks).

    The protocol runs with its state in device memory (bsr_gselect_*): three
    histogram all-reduces and one all-gather on device buffers (NCCL; gloo stages
    through the host), no device->host copy until this rank's kept count is read
    at the very end to size the result.  total_rows: rows of the whole batch (the
    caller's sharding plan knows it); if None it is all-reduced once on the host."""
    import torch
    import torch.distributed as dist

    from . import BSR, _dt, _lib, _stream, alloc_bsr, keep_count, num_blocks, workspace

    lib = _lib.load()
    M, K = X.shape
    dev = X.device
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    cpu_coll = world > 1 and dist.get_backend(group) == "gloo"
    ws_bytes = lib.bsr_prune_workspace_bytes(M, K, b)
    ws = workspace(ws_bytes, dev, kind="prune", stream=stream)
    st = _stream(stream)

    def allreduce_(t):  # in place, on device buffers (gloo: through the host)
        if world == 1:
            return t
        if cpu_coll:
            h = t.cpu()
            dist.all_reduce(h, group=group)
            t.copy_(h)
        else:
            dist.all_reduce(t, group=group)
        return t

    def allgather(t):
        if world == 1:
            return t.reshape(1, -1).clone()
        src = t.cpu() if cpu_coll else t
        outs = [torch.empty_like(src) for _ in range(world)]
        dist.all_gather(outs, src, group=group)
        return torch.stack(outs).to(dev)

    N_rank = num_blocks(M, K, b)
    if total_rows is None:
        n_total = N_rank
        if world > 1:
            t = torch.tensor([N_rank], dtype=torch.int64)
            if not cpu_coll:
                t = t.to(dev)
            dist.all_reduce(t, group=group)
            n_total = int(t.item())
    else:
        n_total = num_blocks(int(total_rows), K, b)
    k_total = keep_count(n_total, keep)
    state = torch.empty(lib.bsr_gselect_state_bytes() // 8, dtype=torch.int64, device=dev)
    _lib.check(lib.bsr_gselect_init(k_total, state.data_ptr(), st))
    for level, nb in enumerate((4096, 1024, 512)):
        hist = torch.empty(nb, dtype=torch.int32, device=dev)  # uint32 counts (< 2^31)
        _lib.check(lib.bsr_gselect_hist(X.data_ptr(), M, K, b, _dt(X), level, state.data_ptr(), hist.data_ptr(),
                                        ws.data_ptr(), ws.numel(), st))
        allreduce_(hist)
        _lib.check(lib.bsr_gselect_update(hist.data_ptr(), level, state.data_ptr(), st))
    counts = torch.empty(2, dtype=torch.int64, device=dev)
    _lib.check(lib.bsr_gselect_counts(M, K, b, state.data_ptr(), counts.data_ptr(), ws.data_ptr(), ws.numel(), st))
    allc = allgather(counts).contiguous()
    _lib.check(lib.bsr_gselect_take(allc.data_ptr(), world, rank, state.data_ptr(), st))
    cap = min(N_rank, k_total)
    out = alloc_bsr(M, K, b, cap, X.dtype, dev)
    cs = out.c_struct()
    _lib.check(lib.bsr_prune_gselect(X.data_ptr(), M, K, b, _dt(X), state.data_ptr(), cap, ctypes.byref(cs),
                                     ws.data_ptr(), ws.numel(), st))
    k_rank = int(state[7].item())  # the one device -> host read: the size of this rank's result
    return BSR(rowptr=out.rowptr, colidx=out.colidx[:k_rank], values=out.values[:k_rank], M=M, K=K, b=b)
