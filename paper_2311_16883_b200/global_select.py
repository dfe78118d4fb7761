"""Cross-rank global top-k: keep the k = nearest(keep * N_total)
largest blocks of the CONCATENATED activation of all data-parallel ranks, so the
multi-GPU kept set equals the single-GPU one (P:L413-418 applied to the whole
batch; tie rule BJ: lower flat index first = lower rank first).

The device work is the library's (include/bsrprune.h: bsr_select_hist,
bsr_select_counts, bsr_prune_threshold).  This module only runs the exchange
protocol between those calls with torch.distributed:

  1. level-0 digit histogram (key bits 30..19) per rank  -> all-reduce -> boundary bin
  2. while the boundary bin is split: next digit (bits 18..9, then 8..0) of the
     keys in it -> all-reduce -> boundary sub-bin         (at most two more rounds)
  3. per rank (#keys above, #keys tied) at the final digit -> all-gather
  4. tie quota: r = k - sum(above); rank q keeps its first
     clamp(r - ties on ranks < q, 0, ties_q) tied blocks -> k_q = above_q + that.

`threshold_protocol` is the pure host logic (injected histogram / count /
collective callables), unit-tested on CPU with gloo at world size 2.
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


def prune_global(X, b: int, keep: float, group=None, stream=None):
    """bsr_prune with the whole data-parallel batch as selection scope.  Every rank
    calls it with its own rows; returns this rank's BSR (k_rank blocks)."""
    import torch
    import torch.distributed as dist

    from . import _lib, _dt, _stream, alloc_bsr, keep_count, num_blocks, workspace

    lib = _lib.load()
    M, K = X.shape
    dev = X.device
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    cpu_coll = world > 1 and dist.get_backend(group) == "gloo"
    ws_bytes = lib.bsr_prune_workspace_bytes(M, K, b)
    ws = workspace(ws_bytes, dev, kind="prune", stream=stream)
    st = _stream(stream)

    def coll_tensor(a: np.ndarray):
        t = torch.from_numpy(np.ascontiguousarray(a))
        return t if cpu_coll else t.to(dev)

    def allreduce(a):
        if world == 1:
            return a
        t = coll_tensor(a)
        dist.all_reduce(t, group=group)
        return t.cpu().numpy()

    def allgather(a):
        if world == 1:
            return a[None]
        t = coll_tensor(a)
        out = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(out, t, group=group)
        return np.stack([o.cpu().numpy() for o in out])

    def hist_fn(level, prefix):
        n = (4096, 1024, 512)[level]
        h = torch.empty(n, dtype=torch.int32, device=dev)
        _lib.check(lib.bsr_select_hist(X.data_ptr(), M, K, b, _dt(X), level, prefix, h.data_ptr(), ws.data_ptr(),
                                       ws.numel(), st))
        return h.cpu().numpy().astype(np.int64)

    def counts_fn(threshold, shift):
        c = torch.empty(2, dtype=torch.int64, device=dev)
        _lib.check(lib.bsr_select_counts(M, K, b, threshold, shift, c.data_ptr(), ws.data_ptr(), ws.numel(), st))
        return tuple(int(v) for v in c.cpu().tolist())

    n_total = int(allreduce(np.asarray([num_blocks(M, K, b)], dtype=np.int64))[0])
    k_total = keep_count(n_total, keep)
    if k_total == 0:
        hist_fn(0, 0)  # (the sums are not needed; keep the call sequence uniform across ranks)
    thr, shift, tie_take, k_rank = threshold_protocol(k_total, rank, hist_fn, counts_fn, allreduce, allgather)
    out = alloc_bsr(M, K, b, k_rank, X.dtype, dev)
    cs = out.c_struct()
    _lib.check(lib.bsr_prune_threshold(X.data_ptr(), M, K, b, _dt(X), thr, shift, tie_take, k_rank, ctypes.byref(cs),
                                       ws.data_ptr(), ws.numel(), st))
    return out
