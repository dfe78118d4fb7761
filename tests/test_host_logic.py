"""Host-side logic on CPU: the algorithmic-work formulas bench.py reports against
(SURVEY §8d / Appendix A.3 numbers), and the multi-rank plumbing of the path
(row sharding, dW all-reduce, max/sum over ranks) with world-size-2 gloo."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
import synth
from paper_2311_16883_b200 import dist as D
from paper_2311_16883_b200 import metrics


def test_bsr_bytes_closed_form():
    # BJ closed form k*b^2*4 + k*4 + (M/b+1)*4 at C1 / C2
    assert metrics.bsr_bytes(256, 16, 128, 4) == 131_652
    assert metrics.bsr_bytes(25088, 32, 4704, 4) == 19_289_540
    assert metrics.bsr_bytes(25088, 32, 4704, 4) == oracle.storage_bytes(25088, 32, 32, 4704)


def test_step_work_c2():
    M, K, N, b = 25088, 384, 1536, 32
    k = oracle.keep_count(oracle.num_blocks(M, K, b), 0.5)
    assert k == 4704
    assert metrics.prune_bytes(M, K, b, k, 4) == 38_535_168 + 19_289_540      # 57.8 MB (A.3)
    assert metrics.wgrad_flops(b, k, N) == 14_797_504_512                     # 14.80 GFLOP (A.3)
    assert metrics.act_bytes_saved(M, K, b, k, 4) == 19_245_628               # 49.9 % (§8a)
    # every block row keeps something: dY is read whole (b*N*R_ne*4 = 154 MB)
    w = metrics.wgrad_bytes(M, K, b, k, N, 4, 4, M // b)
    assert w == 19_289_540 + 4 * M * N + 4 * K * N
    assert metrics.prune_bytes(M, K, b, 0, 4) == 4 * (M // b + 1)
    assert metrics.decompress_bytes(M, K, b, k, 4) == metrics.prune_bytes(M, K, b, k, 4)


def test_wgrad_bound_c2_vs_b24():
    # S12 fc1 (C2) is HBM-bound, B24 per rank is tensor-bound (SURVEY finding 6)
    peak_tc, peak_bw = 2250.0, 8000.0
    M, K, N, b = 25088, 384, 1536, 32
    k = 4704
    assert metrics.wgrad_bound(metrics.wgrad_flops(b, k, N), metrics.wgrad_bytes(M, K, b, k, N, 2, 2, M // b),
                               peak_tc, peak_bw) == "hbm"
    M, K, N = 25088, 768, 3072
    k = oracle.keep_count(oracle.num_blocks(M, K, b), 0.5)
    assert metrics.wgrad_bound(metrics.wgrad_flops(b, k, N), metrics.wgrad_bytes(M, K, b, k, N, 2, 2, M // b),
                               peak_tc, peak_bw) == "tensor"


def test_allreduce_bus_bytes():
    assert metrics.allreduce_bus_bytes(384, 1536, 1) == 0.0
    assert metrics.allreduce_bus_bytes(384, 1536, 8) == pytest.approx(2 * 7 / 8 * 4 * 384 * 1536)


@pytest.mark.parametrize("M,world,align", [(25088, 2, 196 * 32), (200704, 8, 196), (25088, 3, 32), (64, 4, 16)])
def test_shard_rows_partition(M, world, align):
    ranges = [D.shard_rows(M, world, r, align) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == M
    for (a0, a1), (b0, _) in zip(ranges, ranges[1:]):
        assert a1 == b0
    for r0, r1 in ranges:
        assert r0 % align == 0 and r1 % align == 0 and r1 >= r0
    sizes = [r1 - r0 for r0, r1 in ranges]
    assert max(sizes) - min(sizes) <= align


def test_shard_rows_rejects_misaligned():
    with pytest.raises(ValueError):
        D.shard_rows(100, 2, 0, 32)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, M, K, N, b, keep, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    D.init("gloo")
    X = synth.f_aff(M, K, synth.seed_for(4))
    dY = synth.grad_out(M, N, synth.seed_for(4))
    r0, r1 = D.shard_rows(M, world, rank, b)
    Xr, dYr = X[r0:r1], dY[r0:r1]
    k = oracle.keep_count(oracle.num_blocks(r1 - r0, K, b), keep)  # per-rank scope (R2)
    ref = oracle.prune(Xr, b, k)
    dW = torch.from_numpy(oracle.wgrad(ref["rowptr"], ref["colidx"], ref["values"], r1 - r0, K, b, dYr))
    D.allreduce_dw(dW)
    tmax = D.max_over_ranks(float(rank + 1))
    tsum = D.sum_over_ranks(float(rank + 1))
    q.put((rank, dW.numpy(), ref["mask"], tmax, tsum))
    D.finalize()


def test_gloo_two_ranks_allreduce_equals_concatenated_oracle():
    """P7 (multi-rank pin): sum over ranks of the per-rank oracle dW equals the
    oracle dW of the whole X with the union of the per-rank masks."""
    M, K, N, b, keep, world = 8 * 16, 64, 48, 16, 0.4, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, M, K, N, b, keep, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    X = synth.f_aff(M, K, synth.seed_for(4))
    dY = synth.grad_out(M, N, synth.seed_for(4))
    mask = np.concatenate([r[2] for r in res])  # per-rank masks in flat (row-major block) order
    rowptr, colidx, values = oracle.build_bsr(X, mask, b)
    want = oracle.wgrad(rowptr, colidx, values, M, K, b, dY)
    for rank, dW, _, tmax, tsum in res:
        np.testing.assert_allclose(dW, want, rtol=1e-12, atol=1e-15)
        assert tmax == 2.0 and tsum == 3.0
    # per-rank scope (R2): each rank keeps nearest(keep * its own block count)
    assert mask.sum() == sum(oracle.keep_count(oracle.num_blocks(M // 2, K, b), keep) for _ in range(2))


def test_plan_buckets():
    assert D.plan_buckets([10, 10, 10, 10], 25) == [[0, 1], [2, 3]]
    assert D.plan_buckets([30, 5, 5], 25) == [[0], [1, 2]]  # an oversized gradient gets its own bucket
    assert D.plan_buckets([], 8) == []
    sizes = [9437184] * 48  # ResMLP-B24: 24 x (fc1, fc2) dW of 768 x 3072 fp32
    b = D.plan_buckets(sizes, 40 << 20)
    assert [i for bk in b for i in bk] == list(range(48))  # order preserved, every gradient once
    assert all(sum(sizes[i] for i in bk) <= 40 << 20 for bk in b)
    with pytest.raises(ValueError):
        D.plan_buckets([1], 0)


def _bucket_worker(rank, world, port, shapes, cap, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    D.init("gloo")
    br = D.BucketedAllReduce(shapes, "cpu", cap_bytes=cap, dtype=torch.float64)
    rng = np.random.default_rng(100 + rank)
    local = []
    for i, (k, n) in enumerate(shapes):  # "backward": write each gradient, then mark it ready
        g = torch.from_numpy(rng.standard_normal((k, n)))
        br.view(i).copy_(g)
        local.append(g.clone())
        br.ready(i)
    br.wait()
    q.put((rank, [br.view(i).clone().numpy() for i in range(len(shapes))], [g.numpy() for g in local],
           len(br.buckets)))
    D.finalize()


def test_gloo_two_ranks_bucketed_allreduce():
    """The bucket scheduler (a7 overlapped with the backward pass) at world size 2:
    every gradient ends up as the sum over ranks, whatever bucket it sat in."""
    shapes = [(8, 16), (4, 4), (16, 16), (2, 8), (8, 8)]
    cap = 8 * 16 * 8  # bytes: float64 views, so ~1-2 gradients per bucket
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bucket_worker, args=(r, world, port, shapes, cap, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][3] >= 3  # several buckets were in flight
    for i in range(len(shapes)):
        want = res[0][2][i] + res[1][2][i]
        for r in range(world):
            np.testing.assert_allclose(res[r][1][i], want, rtol=1e-15, atol=0)


def test_default_prec_choices():
    """The layer's default dW arithmetic for each storage type and shape."""
    import torch
    from paper_2311_16883_b200.sparse_linear import _default_prec
    f32, bf16 = torch.float32, torch.bfloat16
    assert _default_prec(f32, 32, 1536, 25088, 384) == "fp32"
    assert _default_prec(bf16, 32, 1536, 25088, 384) == "bf16"
    assert _default_prec(bf16, 4, 1536, 25088, 384) == "bf16"    # dense rebuild: 32 | rows, 32 | in
    assert _default_prec(bf16, 4, 1536, 25080, 384) == "fp32"    # rows not a multiple of 32
    assert _default_prec(bf16, 8, 200, 25088, 384) == "fp32"     # N not a multiple of 128
    assert _default_prec(bf16, 16, 200, 25088, 384) == "fp32"
