"""GPU parity of bsr_wgrad_nk (BSR_DW_NK: dW^T, N x K, nn.Linear.weight.grad's
layout) against bsr_wgrad's K x N dW and the fp64 oracle.

The native path (FP32-grade per-run kernel with a chain-capped split-K reduce)
sums the same partials in the same order as bsr_wgrad: bit-identical to dW^T,
also when accumulating.  Every other path computes dW and transposes it: bit-
identical at accumulate = 0, one rounding of old + dW when accumulating.
"""
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

CASES = [  # (M, K, N, b, prec, algo, bf16 storage, native)
    (4096, 384, 256, 32, "fp32", "auto", False, True),    # 3xTF32, 3 chain-capped splits
    (4096, 256, 384, 64, "fp32", "runs", False, True),
    (2048, 256, 256, 16, "fp32", "auto", False, False),   # dense rebuild
    (1024, 96, 200, 8, "fp32", "simt", False, False),     # FFMA, N not a multiple of 128
    (2048, 256, 256, 32, "tf32", "auto", False, False),
    (2048, 256, 256, 32, "bf16", "auto", True, False),
    (1024, 128, 128, 32, "fp32", "auto", False, False),   # one split: transposed afterwards
]


def _inputs(M, K, N, b, bf16, seed):
    X = synth.f_aff(M, K, seed=seed)
    dY = synth.grad_out(M, N, seed + 1)
    if bf16:
        return to_torch(synth.to_bf16_bits(X), bf16=True), to_torch(synth.to_bf16_bits(dY), bf16=True)
    return to_torch(X), to_torch(dY)


@pytest.mark.parametrize("M,K,N,b,prec,algo,bf16,native", CASES)
def test_nk_is_transposed_dw(M, K, N, b, prec, algo, bf16, native):
    Xt, dYt = _inputs(M, K, N, b, bf16, seed=100 + b)
    A = bp.prune(Xt, b, keep=0.5)
    kn = bp.wgrad(A, dYt, prec=prec, algo=algo)
    nk = torch.full((N, K), float("nan"), device="cuda")
    bp.wgrad(A, dYt, prec=prec, algo=algo, layout="nk", out=nk)
    torch.cuda.synchronize()
    assert torch.equal(nk, kn.t()), (prec, algo, (nk - kn.t()).abs().max().item())
    if prec == "fp32":  # and against the oracle on the same BSR
        vals = A.values.float().cpu().numpy()
        ref = oracle.wgrad(A.rowptr.cpu().numpy(), A.colidx.cpu().numpy(), vals, M, K, b, dYt.float().cpu().numpy())
        assert oracle.rel_frobenius(nk.t().cpu().numpy(), ref) <= 1e-5


@pytest.mark.parametrize("M,K,N,b,prec,algo,bf16,native", CASES)
def test_nk_accumulate(M, K, N, b, prec, algo, bf16, native):
    Xt, dYt = _inputs(M, K, N, b, bf16, seed=200 + b)
    A = bp.prune(Xt, b, keep=0.4)
    base = torch.randn(K, N, device="cuda")
    kn = base.clone()
    bp.wgrad(A, dYt, prec=prec, algo=algo, out=kn, accumulate=True)
    nk = base.t().contiguous()
    bp.wgrad(A, dYt, prec=prec, algo=algo, layout="nk", out=nk, accumulate=True)
    torch.cuda.synchronize()
    if native:
        assert torch.equal(nk, kn.t())
    else:
        torch.testing.assert_close(nk, kn.t(), rtol=2e-6, atol=1e-6)


def test_nk_empty_bsr():
    Xt = torch.zeros(2048, 256, device="cuda")
    dYt = to_torch(synth.grad_out(2048, 256, 3))
    A = bp.prune(Xt, 32, k=0)
    nk = torch.full((256, 256), 7.0, device="cuda")
    bp.wgrad(A, dYt, prec="fp32", layout="nk", out=nk)
    torch.cuda.synchronize()
    assert torch.count_nonzero(nk).item() == 0


def test_sparse_linear_uses_nk_and_matches_dense_masked():
    """SparseLinear's weight.grad (N x K, no transpose in the layer) equals the
    gradient of the input masked by the oracle's own top-k selection."""
    torch.manual_seed(0)
    M, K, N, b = 4096, 384, 256, 32
    k = oracle.keep_count(oracle.num_blocks(M, K, b, b), 0.5)
    Xn, _ = enforce_gap(synth.f_aff(M, K, seed=9), b, k)
    layer = bp.SparseLinear(K, N, sparsity=0.5, block=b).cuda()
    y = layer(torch.from_numpy(Xn).cuda())
    g = synth.grad_out(M, N, 10)
    y.backward(torch.from_numpy(g).cuda())
    ref_bsr = oracle.prune(Xn, b, k)
    Xm = oracle.decompress(ref_bsr["rowptr"], ref_bsr["colidx"], ref_bsr["values"], M, K, b).astype(np.float64)
    ref = g.astype(np.float64).T @ Xm  # N x K
    assert layer.weight.grad.is_contiguous() and tuple(layer.weight.grad.shape) == (N, K)
    assert oracle.rel_frobenius(layer.weight.grad.cpu().numpy(), ref) <= 1e-5


@pytest.mark.parametrize("prec,algo,b,K", [("fp32", "auto", 32, 384), ("tf32", "runs", 32, 384),
                                           ("tf32", "span", 16, 2048)])
@pytest.mark.parametrize("layout", ["kn", "nk"])
def test_tma_paths_from_a_fresh_thread(prec, algo, b, K, layout):
    """A thread whose first CUDA work is a dW call (cached workspace and output
    allocations: no runtime call made the context current -- PyTorch's autograd
    worker in SparseLinear's backward) must still encode its TMA descriptors."""
    import threading
    M, N = 2048, 256
    X = to_torch(synth.f_aff(M, K, seed=5))
    dY = to_torch(synth.grad_out(M, N, 6))
    A = bp.prune(X, b, keep=0.5)
    ref = bp.wgrad(A, dY, prec=prec, algo=algo, layout=layout)  # workspace cached on the default stream
    out = torch.empty_like(ref)
    torch.cuda.synchronize()
    err = []

    def body():
        try:
            bp.wgrad(A, dY, prec=prec, algo=algo, layout=layout, out=out)
            torch.cuda.synchronize()
        except Exception as e:  # pragma: no cover - reported below
            err.append(repr(e))

    t = threading.Thread(target=body)
    t.start()
    t.join()
    assert not err, err[0]
    assert torch.equal(out, ref)
