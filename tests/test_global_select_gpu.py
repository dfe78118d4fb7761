"""GPU parity of the cross-rank global top-k: bsr_select_hist /
bsr_select_counts / bsr_prune_threshold driven by paper_2311_16883_b200.prune_global.

* one rank: identical (bit for bit) to bsr_prune on the same X;
* two ranks (two processes on cuda:0, gloo collectives): every rank's BSR equals
  the oracle's selection on the CONCATENATED X restricted to that rank's rows
  (P:L413-418 over the whole batch; BJ tie rule across ranks)."""
import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

import oracle
import synth
from helpers import enforce_gap, to_torch

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2311_16883_b200 as bp  # noqa: E402


def _x(family, M, K, seed, b, k):
    if family == "ints":  # exact fp32 block sums, many ties
        return synth.ints(M, K, seed)
    X, _ = enforce_gap(synth.f_aff(M, K, seed), b, k)
    return X


@pytest.mark.parametrize("b", [4, 16, 32, 64])
@pytest.mark.parametrize("keep", [0.0, 0.1, 0.5, 0.93, 1.0])
@pytest.mark.parametrize("family", ["aff", "ints"])
def test_single_rank_equals_prune(b, keep, family):
    M, K = 40 * b, 6 * b if b >= 32 else 256
    k = oracle.keep_count(oracle.num_blocks(M, K, b), keep)
    Xt = to_torch(_x(family, M, K, 11 + b, b, max(k, 1)))
    A = bp.prune(Xt, b, keep=keep)
    G = bp.prune_global(Xt, b, keep)
    torch.cuda.synchronize()
    assert G.nnzb == A.nnzb == k
    assert torch.equal(G.rowptr, A.rowptr)
    assert torch.equal(G.colidx, A.colidx)
    assert torch.equal(G.values.view(torch.int32), A.values.view(torch.int32))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, X, b, keep, rows, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r0, r1 = rows[rank]
    G = bp.prune_global(torch.from_numpy(X[r0:r1]).cuda(), b, keep)
    torch.cuda.synchronize()
    q.put((rank, G.rowptr.cpu().numpy(), G.colidx.cpu().numpy(), G.values.cpu().numpy().view(np.int32)))
    dist.destroy_process_group()


@pytest.mark.parametrize("family,b,keep,shape", [("ints", 16, 0.37, None), ("aff", 32, 0.5, None), ("ints", 4, 0.8, None),
                                                 ("aff", 32, 0.5, (25088, 384))])  # the last: C2 at full size
def test_two_ranks_equal_concatenated_oracle(family, b, keep, shape):
    M, K = shape if shape else (48 * b, 8 * b)
    rows = [(0, (M // b * 5 // 12) * b), ((M // b * 5 // 12) * b, M)]  # unequal shards
    k = oracle.keep_count(oracle.num_blocks(M, K, b), keep)
    X = _x(family, M, K, 5, b, k)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, X, b, keep, rows, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    mask = oracle.prune(X, b, k)["mask"].reshape(M // b, K // b)
    assert sum(len(r[2]) for r in res) == k
    for rank, rowptr, colidx, values in res:
        r0, r1 = rows[rank]
        m = mask[r0 // b:r1 // b].reshape(-1)
        rp, ci, vals = oracle.build_bsr(X[r0:r1], m, b)
        np.testing.assert_array_equal(rowptr, rp)
        np.testing.assert_array_equal(colidx, ci)
        np.testing.assert_array_equal(values, vals.view(np.int32))
