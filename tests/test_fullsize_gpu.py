"""Full-size and edge-case GPU parity (VERDICT r01 "Next round" item 1).

* dW element by element against the FULL oracle at C2 (quadruple loop) and at
  the per-rank ResMLP-B24 shards (fc1 25088x768 -> 3072, fc2 25088x3072 -> 768,
  b = 32, keep 0.5; oracle = decompress + one fp64 BLAS matmul, pinned to the
  loop in test_oracle.py), on every dW kernel family.
* prune at C5 size (1 GiB fp32, b = 4 and 32) and decompress at C2 / C3_fc2 /
  C5 size: bit-exact.
* tie overflow: integer-valued full-size inputs whose boundary radix bin holds
  far more than the 4096-key candidate list (the global-refinement path).
* decompress with K/b >= 64 (multi-chunk colidx scan, early break).
* two prunes and two dWs in flight on two streams: bit-identical to serial runs.
* data-parallel dW (a7): two processes on cuda:0, per-rank prune -> dW ->
  all-reduce == the sum of the per-rank oracles.
"""
import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

import oracle
import synth
from helpers import bits, enforce_gap, gap_k, to_torch

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2311_16883_b200 as bp  # noqa: E402

TOL = {"fp32": 1e-5, "tf32": 5e-3, "bf16": 1e-4}


def assert_bsr_equal(A, ref, bf16=False):
    np.testing.assert_array_equal(A.rowptr.cpu().numpy(), ref["rowptr"])
    np.testing.assert_array_equal(A.colidx.cpu().numpy(), ref["colidx"])
    np.testing.assert_array_equal(bits(A.values).reshape(-1), ref["values"].view(np.int16 if bf16 else np.int32).reshape(-1))


# ----------------------------------------------------------------------------- dW, full size
_REF_CACHE = {}


def _layer(name, bf16):
    """(X, dY, k, oracle BSR, oracle dW) of a full-size layer, cached per (layer, dtype)."""
    key = (name, bf16)
    if key not in _REF_CACHE:
        if name == "C2":
            c = synth.CONFIGS["C2"]
            M, K, N, b, fam, seed = c["M"], c["K"], c["N"], c["b"], c["family"], synth.seed_for(2)
        else:  # B24 per-rank shard at P = 8: batch 128 x 196 tokens
            c = synth.CONFIGS["C4_" + name]
            M, K, N, b, fam, seed = 25088, c["K"], c["N"], c["b"], c["family"], synth.seed_for(4, 0, 3)
        X = synth.activation(fam, M, K, seed)
        dY = synth.grad_out(M, N, seed)
        k = oracle.keep_count(oracle.num_blocks(M, K, b), 0.5)
        if bf16:
            X, dY = synth.to_bf16_bits(X), synth.to_bf16_bits(dY)
            k = gap_k(X, b, k)
        else:
            X, _ = enforce_gap(X, b, k)
        ref = oracle.prune(X, b, k)
        fn = oracle.wgrad if name == "C2" else oracle.wgrad_masked
        dW = fn(ref["rowptr"], ref["colidx"], ref["values"], M, K, b, dY)
        _REF_CACHE.clear()  # keep one layer's arrays alive at a time
        _REF_CACHE[key] = (X, dY, k, b, ref, dW)
    return _REF_CACHE[key]


@pytest.mark.parametrize("layer", ["C2", "fc1", "fc2"])
@pytest.mark.parametrize("prec", ["fp32", "tf32", "bf16"])
@pytest.mark.parametrize("algo", ["auto", "runs", "span"])
def test_dw_full_elementwise(layer, prec, algo):
    bf = prec == "bf16"
    X, dY, k, b, ref, ref_dW = _layer(layer, bf)
    A = bp.prune(to_torch(X, bf16=bf), b, k=k)
    torch.cuda.synchronize()
    assert_bsr_equal(A, ref, bf16=bf)
    if prec == "fp32" and algo == "span":
        with pytest.raises(bp.BsrError):
            bp.wgrad(A, to_torch(dY, bf16=bf), prec=prec, algo=algo)
        return
    out = torch.full(ref_dW.shape, float("nan"), device="cuda")
    bp.wgrad(A, to_torch(dY, bf16=bf), prec=prec, algo=algo, out=out)
    got = out.cpu().numpy()
    assert np.isfinite(got).all()
    err = oracle.rel_frobenius(got, ref_dW)
    assert err <= TOL[prec], err
    # element-wise: no single entry may be off by more than the tolerance times the
    # largest |dW| of its row (a dropped block shows up even when rel-F is small)
    scale = np.abs(ref_dW).max(axis=1, keepdims=True) + 1e-30
    assert (np.abs(got - ref_dW) / scale).max() <= 20 * TOL[prec]


@pytest.mark.parametrize("layer", ["C2", "fc2"])
def test_dw_nk_full(layer):
    """bsr_wgrad_nk at full size (the FP32-grade native transposing split-K reduce):
    bit-identical to bsr_wgrad's dW transposed, and against the full oracle."""
    X, dY, k, b, ref, ref_dW = _layer(layer, False)
    A = bp.prune(to_torch(X), b, k=k)
    dYt = to_torch(dY)
    kn = bp.wgrad(A, dYt, prec="fp32")
    nk = torch.full((ref_dW.shape[1], ref_dW.shape[0]), float("nan"), device="cuda")
    bp.wgrad(A, dYt, prec="fp32", layout="nk", out=nk)
    torch.cuda.synchronize()
    assert torch.equal(nk, kn.t())
    assert oracle.rel_frobenius(nk.t().cpu().numpy(), ref_dW) <= TOL["fp32"]


# ----------------------------------------------------------------------------- prune / decompress, full size
@pytest.mark.parametrize("b", [4, 32])
def test_prune_c5_1gib(b):
    """C5 (prune/pack bandwidth sweep) at 1 GiB fp32 (K = 1536, F_unif), keep 0.5:
    16.8 M blocks at b = 4 -- 32-bit slot/count paths, many CTAs per row range."""
    K = 1536
    M = (1 << 30) // (4 * K) // 64 * 64
    X = synth.f_unif(M, K, seed=5_000 + b)
    k = oracle.keep_count(oracle.num_blocks(M, K, b), 0.5)
    X, _ = enforce_gap(X, b, k)
    ref = oracle.prune(X, b, k)
    Xt = to_torch(X)
    A = bp.prune(Xt, b, k=k)
    torch.cuda.synchronize()
    assert_bsr_equal(A, ref)
    D = bp.decompress(A)
    torch.cuda.synchronize()
    dense = oracle.decompress(ref["rowptr"], ref["colidx"], ref["values"], M, K, b)
    assert np.array_equal(bits(D), dense.view(np.int32))


@pytest.mark.parametrize("name", ["C2", "C3_fc2"])
@pytest.mark.parametrize("bf16", [False, True])
def test_decompress_full(name, bf16):
    c = synth.CONFIGS[name]
    M, K, b = c["M"], c["K"], c["b"]
    X = synth.activation(c["family"], M, K, synth.seed_for(c["id"]))
    if bf16:
        X = synth.to_bf16_bits(X)
    k = oracle.keep_count(oracle.num_blocks(M, K, b), c["keep"])
    k = gap_k(X, b, k)
    ref = oracle.prune(X, b, k)
    A = bp.prune(to_torch(X, bf16=bf16), b, k=k)
    D = bp.decompress(A)
    torch.cuda.synchronize()
    assert_bsr_equal(A, ref, bf16=bf16)
    dense = oracle.decompress(ref["rowptr"], ref["colidx"], ref["values"], M, K, b)
    assert np.array_equal(bits(D), dense.view(np.int16 if bf16 else np.int32))


@pytest.mark.parametrize("b", [16, 32])
@pytest.mark.parametrize("keep", [0.5, 0.9])
@pytest.mark.parametrize("bf16", [False, True])
def test_decompress_wide_rows(b, keep, bf16):
    """K/b = 96 block columns (rows with > 32 stored blocks): the decompress walks a
    row's colidx in several 32-entry chunks and stops early once past its unit."""
    M, K = 64 * b, 96 * b
    X = synth.f_gelu(M, K, seed=31 + b)
    if bf16:
        X = synth.to_bf16_bits(X)
    k = gap_k(X, b, oracle.keep_count(oracle.num_blocks(M, K, b), keep))
    ref = oracle.prune(X, b, k)
    A = bp.prune(to_torch(X, bf16=bf16), b, k=k)
    D = bp.decompress(A)
    torch.cuda.synchronize()
    assert_bsr_equal(A, ref, bf16=bf16)
    dense = oracle.decompress(ref["rowptr"], ref["colidx"], ref["values"], M, K, b)
    assert np.array_equal(bits(D), dense.view(np.int16 if bf16 else np.int32))


# ----------------------------------------------------------------------------- tie overflow
@pytest.mark.parametrize("b", [4, 32])
@pytest.mark.parametrize("path", ["prune", "presummed", "global1"])
def test_tie_overflow_full_size(b, path):
    """S12 fc1-sized integer X: b = 32 blocks each hold exactly 100..103 entries of
    +-1 (sum of squares 100..103: all 9408 keys in ONE 12-bit radix bin, > the
    4096-key candidate list); b = 4 entries in {-2..2} (sums 0..64: ~10^5 keys per
    value).  k sits inside a tie run: the global refinement rounds and the
    flat-order tie quota decide.  Exact integers: the oracle's keys equal the GPU's."""
    M, K = 25088, 384
    if b == 32:
        X = synth.block_count_ints(M, K, b, [100, 101, 102, 103], seed=61)
    else:
        X = synth.ints(M, K, seed=62)
    N = oracle.num_blocks(M, K, b)
    s = oracle.block_sumsq(X, b)
    k = N // 2
    srt = np.sort(s)[::-1]
    assert srt[k - 1] == srt[k]  # the boundary is inside a tie
    digit = s.astype(np.float32).view(np.uint32) >> 19  # first radix digit of the fp32 key
    assert (digit == (np.float32(srt[k - 1]).view(np.uint32) >> 19)).sum() > 4096  # boundary bin > the list
    ref = oracle.prune(X, b, k)
    Xt = to_torch(X)
    if path == "prune":
        A = bp.prune(Xt, b, k=k)
    elif path == "presummed":
        _, A = bp.act_prune(Xt, b, k=k, act="identity")
    else:
        keep = k / N
        assert oracle.keep_count(N, keep) == k
        A = bp.prune_global(Xt, b, keep)
    torch.cuda.synchronize()
    assert_bsr_equal(A, ref)


# ----------------------------------------------------------------------------- streams
def test_two_streams_bit_identical():
    """Per-stream workspaces: two prunes and two dWs in flight on two streams give
    the same bits as the same calls run one after another."""
    b, M, K, N = 32, 6272, 384, 1536
    Xs = [to_torch(synth.f_aff(M, K, seed=s)) for s in (71, 72)]
    dYs = [to_torch(synth.grad_out(M, N, seed=s)) for s in (71, 72)]
    serial = []
    for X, dY in zip(Xs, dYs):
        A = bp.prune(X, b, keep=0.5)
        serial.append((A, bp.wgrad(A, dY, prec="fp32"), bp.wgrad(A, dY, prec="tf32")))
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for s in streams:
        s.wait_stream(torch.cuda.current_stream())
    outs = []
    for _ in range(3):  # repeat: the workspaces are reused while the other stream runs
        for X, dY, s in zip(Xs, dYs, streams):
            with torch.cuda.stream(s):
                A = bp.prune(X, b, keep=0.5, stream=s)
                outs.append((A, bp.wgrad(A, dY, prec="fp32", stream=s), bp.wgrad(A, dY, prec="tf32", stream=s)))
    torch.cuda.synchronize()
    for i, (A, w3, w1) in enumerate(outs):
        Ar, r3, r1 = serial[i % 2]
        assert torch.equal(A.rowptr, Ar.rowptr) and torch.equal(A.colidx, Ar.colidx)
        assert torch.equal(A.values.view(torch.int32), Ar.values.view(torch.int32))
        assert torch.equal(w3.view(torch.int32), r3.view(torch.int32))
        assert torch.equal(w1.view(torch.int32), r1.view(torch.int32))


# ----------------------------------------------------------------------------- data-parallel dW (a7)
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _dp_worker(rank, world, port, shards, b, keep, prec, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2311_16883_b200 import dist as D
    X, dY = shards[rank]
    A = bp.prune(torch.from_numpy(X).cuda(), b, keep=keep)
    dW = bp.wgrad(A, torch.from_numpy(dY).cuda(), prec=prec)
    D.allreduce_dw(dW)
    torch.cuda.synchronize()
    q.put((rank, dW.cpu().numpy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("prec", ["fp32", "tf32"])
def test_two_ranks_dw_allreduce(prec):
    """a7 end to end: each rank prunes its own rows (per-rank scope, R2), computes
    its partial dW on the GPU and the partials are summed by the all-reduce
    (gloo on CUDA tensors here; NCCL on the multi-GPU box).  Against the sum of
    the per-rank oracles (P7)."""
    b, K, N, keep = 32, 384, 1536, 0.5
    shards = []
    ref = 0.0
    for r, Mr in enumerate((196 * 32, 196 * 16)):  # unequal shards
        X = synth.f_aff(Mr, K, seed=81 + r)
        dY = synth.grad_out(Mr, N, seed=81 + r)
        k = oracle.keep_count(oracle.num_blocks(Mr, K, b), keep)
        X, _ = enforce_gap(X, b, k)
        o = oracle.prune(X, b, k)
        ref = ref + oracle.wgrad(o["rowptr"], o["colidx"], o["values"], Mr, K, b, dY)
        shards.append((X, dY))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dp_worker, args=(r, 2, port, shards, b, keep, prec, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.array_equal(res[0][1].view(np.int32), res[1][1].view(np.int32))  # every rank holds the same sum
    assert oracle.rel_frobenius(res[0][1], ref) <= TOL[prec]


@pytest.mark.parametrize("b", [4, 16])
def test_dense_rebuild_fp32_grade_full_size(b):
    """The dense-rebuild tensor-core path (AUTO for the FP32 grade below b = 32) at the
    full S12 fc1 size, element-wise against the oracle (masked-X BLAS form)."""
    c = synth.CONFIGS["C2"]
    M, K, N = c["M"], c["K"], c["N"]
    X = synth.activation(c["family"], M, K, synth.seed_for(2, 1))
    dY = synth.grad_out(M, N, synth.seed_for(2, 1))
    k = oracle.keep_count(oracle.num_blocks(M, K, b), 0.5)
    k = gap_k(X, b, k)
    ref = oracle.prune(X, b, k)
    want = oracle.wgrad_masked(ref["rowptr"], ref["colidx"], ref["values"], M, K, b, dY)
    A = bp.prune(to_torch(X), b, k=k)
    out = torch.full((K, N), float("nan"), device="cuda")
    bp.wgrad(A, to_torch(dY), prec="fp32", algo="dense", out=out)
    auto = bp.wgrad(A, to_torch(dY), prec="fp32")  # AUTO picks the same path here
    got = out.cpu().numpy()
    assert oracle.rel_frobenius(got, want) <= 1e-5
    assert torch.equal(auto.view(torch.int32), out.view(torch.int32))


@pytest.mark.parametrize("prec,algo", [("fp32", "runs"), ("fp32", "simt"), ("fp32", "dense"), ("tf32", "runs"),
                                       ("tf32", "span"), ("bf16", "runs"), ("bf16", "span"), ("bf16", "dense")])
def test_dw_deterministic(prec, algo):
    """Every dW family is deterministic: split partials are summed in split order, so
    repeated launches (and a launch on another stream) give the same bits."""
    c = synth.CONFIGS["C2"]
    M, K, N, b = c["M"], c["K"], c["N"], c["b"]
    bf = prec == "bf16"
    X = synth.activation(c["family"], M, K, 7)
    dY = synth.grad_out(M, N, 7)
    if bf:
        X, dY = synth.to_bf16_bits(X), synth.to_bf16_bits(dY)
    A = bp.prune(to_torch(X, bf16=bf), b, keep=0.5)
    dYt = to_torch(dY, bf16=bf)
    first = bp.wgrad(A, dYt, prec=prec, algo=algo)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        other = bp.wgrad(A, dYt, prec=prec, algo=algo, stream=s)
    torch.cuda.synchronize()
    for _ in range(3):
        again = bp.wgrad(A, dYt, prec=prec, algo=algo)
        assert torch.equal(again.view(torch.int32), first.view(torch.int32))
    assert torch.equal(other.view(torch.int32), first.view(torch.int32))


def test_rows_tensor_cores_full_s12_batch():
    """The 1 x b variant's tensor-core dW at the full S12 fc1 batch (128 samples),
    against the oracle's own per-sample selection (integer-valued X: exact fp32 sums,
    ties by the flat-index rule, so the GPU must select exactly the oracle's set)."""
    S, K, N, b = 196, 384, 1536, 16
    M = S * 128
    X = synth.ints(M, K, 57)
    dY = synth.grad_out(M, N, 57)
    ks = oracle.keep_count(S * K // b, 0.5)
    ref = oracle.prune_per_sample(X, b, ks, S)
    A = bp.prune_rows(to_torch(X), b, 0.5, sample_rows=S)
    got = bp.wgrad_rows(A, to_torch(dY), tensor_cores=True).cpu().numpy()
    np.testing.assert_array_equal(A.rowptr.cpu().numpy(), ref["rowptr"])
    np.testing.assert_array_equal(A.colidx.cpu().numpy(), ref["colidx"])
    Xm = oracle.decompress(ref["rowptr"], ref["colidx"], ref["values"].reshape(-1, 1, b), M, K, 1, b)
    want = Xm.astype(np.float64).T @ dY.astype(np.float64)  # (X * mask)^T dY in fp64 (pinned form)
    assert oracle.rel_frobenius(got, want) <= 1e-5
