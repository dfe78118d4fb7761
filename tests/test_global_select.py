"""Host logic of the cross-rank global top-k (include/bsrprune.h
bsr_select_*): the digit / tie-quota protocol of paper_2311_16883_b200.global_select
against brute-force global top-k on the concatenated keys (key desc, then flat
index asc -- the BJ tie rule), in process and with two gloo ranks."""
import os
import socket

import multiprocessing as mp
import numpy as np
import pytest

from paper_2311_16883_b200.global_select import select_bin, threshold_protocol

DIG = {0: (31, 19, 4096), 1: (19, 9, 1024), 2: (9, 0, 512)}  # level -> (prefix shift, digit shift, bins)


def local_hist(keys, level, prefix):
    sp, sh, nb = DIG[level]
    sel = keys if level == 0 else keys[(keys >> sp) == prefix]
    return np.bincount(((sel >> sh) & (nb - 1)).astype(np.int64), minlength=nb)


def local_counts(keys, thr, shift):
    kk = keys >> shift
    return int((kk > thr).sum()), int((kk == thr).sum())


def brute_mask(keys, k):
    order = np.lexsort((np.arange(len(keys)), -keys.astype(np.int64)))  # key desc, index asc
    m = np.zeros(len(keys), bool)
    m[order[:k]] = True
    return m


def rank_mask(keys, thr, shift, tie_take):
    kk = keys >> shift
    tie_idx = np.nonzero(kk == thr)[0][:tie_take]
    m = kk > thr
    m[tie_idx] = True
    return m


def make_keys(rng, n, family):
    if family == "float":
        v = rng.lognormal(3.0, 1.0, n).astype(np.float32)
    elif family == "ints":
        v = rng.integers(1, 6, n).astype(np.float32)  # heavy ties
    else:  # near-equal: same exponent, differ in the last mantissa bits
        v = (np.float32(1000.0) + rng.integers(0, 40, n).astype(np.float32) * np.float32(6.1e-5)).astype(np.float32)
    return v.view(np.uint32) & np.uint32(0x7FFFFFFF)


def test_select_bin_matches_sorted():
    rng = np.random.default_rng(0)
    for _ in range(50):
        h = rng.integers(0, 5, 64)
        if h.sum() == 0:
            continue
        t = int(rng.integers(1, h.sum() + 1))
        b, above, cnt = select_bin(h, t)
        assert h[b + 1:].sum() == above and h[b] == cnt and above < t <= above + cnt


class SimRank:
    """One rank of a simulated world: its collectives return what the real ones
    would (the sum / stack over every rank's local result of the same call)."""

    def __init__(self, keys_all, q):
        self.keys_all, self.q, self.last = keys_all, q, None

    def hist(self, level, prefix):
        self.last = (level, prefix)
        return local_hist(self.keys_all[self.q], level, prefix)

    def counts(self, thr, shift):
        self.last = (thr, shift)
        return local_counts(self.keys_all[self.q], thr, shift)

    def allreduce(self, a):
        return sum(local_hist(k, *self.last) for k in self.keys_all)

    def allgather(self, a):
        return np.stack([np.asarray(local_counts(k, *self.last)) for k in self.keys_all])


@pytest.mark.parametrize("family", ["float", "ints", "near"])
@pytest.mark.parametrize("world", [1, 2, 3, 5])
@pytest.mark.parametrize("keep", [0.0, 0.1, 0.5, 0.9, 1.0])
def test_protocol_equals_single_gpu_selection(family, world, keep):
    rng = np.random.default_rng(world * 100 + int(keep * 10))
    keys = [make_keys(rng, int(n), family) for n in rng.integers(5, 300, world)]
    allk = np.concatenate(keys)
    k = int(np.floor(keep * len(allk) + 0.5))
    masks = []
    for q in range(world):
        r = SimRank(keys, q)
        thr, shift, tie_take, kq = threshold_protocol(k, q, r.hist, r.counts, r.allreduce, r.allgather)
        masks.append(rank_mask(keys[q], thr, shift, tie_take))
        assert masks[-1].sum() == kq
    assert np.array_equal(np.concatenate(masks), brute_mask(allk, k))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, keys_all, k, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    keys = keys_all[rank]

    def allreduce(a):
        t = torch.from_numpy(a.copy())
        dist.all_reduce(t)
        return t.numpy()

    def allgather(a):
        t = torch.from_numpy(a.copy())
        out = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(out, t)
        return np.stack([o.numpy() for o in out])

    thr, shift, tie_take, kq = threshold_protocol(k, rank, lambda lv, pf: local_hist(keys, lv, pf),
                                                  lambda t, s: local_counts(keys, t, s), allreduce, allgather)
    q.put((rank, rank_mask(keys, thr, shift, tie_take), kq))
    dist.destroy_process_group()


@pytest.mark.parametrize("family", ["float", "ints"])
def test_gloo_two_ranks_protocol(family):
    rng = np.random.default_rng(7)
    keys = [make_keys(rng, 400, family), make_keys(rng, 250, family)]
    allk = np.concatenate(keys)
    k = int(np.floor(0.37 * len(allk) + 0.5))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, keys, k, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = np.concatenate([r[1] for r in res])
    assert np.array_equal(got, brute_mask(allk, k))
    assert sum(r[2] for r in res) == k
