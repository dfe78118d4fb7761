"""GPU parity of the block-sparse affine scaling layer:
bsr_affine_wgrad against the fp64 oracle (orc_affine_wgrad), rel-F <= 1e-5 (fp32
FMAs, round-to-nearest, fixed order), plus the SparseAffine module end to end."""
import numpy as np
import pytest

import oracle
import synth
from helpers import gap_k, to_torch

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2311_16883_b200 as bp  # noqa: E402


@pytest.mark.parametrize("b", [4, 8, 16, 32, 64])
@pytest.mark.parametrize("keep", [0.0, 0.3, 1.0])
@pytest.mark.parametrize("bf16", [False, True])
def test_affine_wgrad_parity(b, keep, bf16):
    M, K = 49 * b, 12 * b  # 49 block rows: ragged split ranges
    X = synth.f_aff(M, K, seed=40 + b)
    dY = synth.grad_out(M, K, seed=40 + b)
    if bf16:
        X, dY = synth.to_bf16_bits(X), synth.to_bf16_bits(dY)
    k = gap_k(X, b, oracle.keep_count(oracle.num_blocks(M, K, b), keep))
    ref = oracle.prune(X, b, k)
    want = oracle.affine_wgrad(ref["rowptr"], ref["colidx"], ref["values"], M, K, b, dY)
    A = bp.prune(to_torch(X, bf16=bf16), b, k=k)
    got = bp.affine_wgrad(A, to_torch(dY, bf16=bf16)).cpu().numpy()
    if k == 0:
        assert not got.any()
    else:
        assert oracle.rel_frobenius(got, want) <= 1e-5
    # accumulate
    base = torch.randn(K, device="cuda")
    out = base.clone()
    bp.affine_wgrad(A, to_torch(dY, bf16=bf16), out=out, accumulate=True)
    assert oracle.rel_frobenius(out.cpu().numpy() - base.cpu().numpy(), want) <= 1e-5 or k == 0


def test_affine_wgrad_s12_size():
    """ResMLP-S12 residual stream at batch 128 (25088 x 384), b = 16, keep 0.5."""
    M, K, b = 25088, 384, 16
    X = synth.f_aff(M, K, seed=44)
    dY = synth.grad_out(M, K, seed=44)
    k = gap_k(X, b, oracle.keep_count(oracle.num_blocks(M, K, b), 0.5))
    ref = oracle.prune(X, b, k)
    want = oracle.affine_wgrad(ref["rowptr"], ref["colidx"], ref["values"], M, K, b, dY)
    A = bp.prune(to_torch(X), b, k=k)
    got = bp.affine_wgrad(A, to_torch(dY)).cpu().numpy()
    assert oracle.rel_frobenius(got, want) <= 1e-5


def test_sparse_affine_module():
    """SparseAffine: forward dense (alpha * x + beta), backward dx = alpha * dy and
    dbeta = sum(dy) dense, dalpha from the BSR of x."""
    M, K, b = 196 * 8, 384, 32
    layer = bp.SparseAffine(K, sparsity=0.5, block=b, device="cuda")
    with torch.no_grad():
        layer.alpha.copy_(torch.linspace(0.5, 1.5, K))
        layer.beta.copy_(torch.linspace(-0.1, 0.1, K))
    xn = synth.f_aff(M, K, seed=45)
    dyn = synth.grad_out(M, K, seed=45)
    k = oracle.keep_count(oracle.num_blocks(M, K, b), 0.5)
    assert gap_k(xn, b, k) == k
    x = to_torch(xn).requires_grad_(True)
    y = layer(x)
    y.backward(to_torch(dyn))
    torch.cuda.synchronize()
    alpha = layer.alpha.detach().double().cpu().numpy()
    np.testing.assert_allclose(y.detach().cpu().numpy(), xn * alpha + layer.beta.detach().double().cpu().numpy(),
                               rtol=1e-6, atol=1e-6)
    np.testing.assert_allclose(x.grad.cpu().numpy(), dyn * alpha, rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose(layer.beta.grad.cpu().numpy(), dyn.astype(np.float64).sum(0), rtol=1e-4, atol=1e-6)
    ref = oracle.prune(xn, b, k)
    want = oracle.affine_wgrad(ref["rowptr"], ref["colidx"], ref["values"], M, K, b, dyn)
    assert oracle.rel_frobenius(layer.alpha.grad.cpu().numpy(), want) <= 1e-5
