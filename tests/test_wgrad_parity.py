"""GPU parity of bsr_wgrad's FP32 grade (dW = X_bsr^T . dY) against the fp64
oracle, on the FFMA kernel ("simt") and on the library's automatic choice
("auto": the 3xTF32 tensor-core kernel where it applies, FFMA elsewhere).

Tolerance (BJ north star): relative Frobenius error <= 1e-5.  Expected
magnitudes: fp32 ~2e-6..5e-6.
"""
import numpy as np
import pytest

import oracle
import synth
from helpers import to_torch

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2311_16883_b200 as bp  # noqa: E402

TOL = {"fp32": 1e-5, "tf32": 5e-3, "bf16": 5e-3}


@pytest.fixture(params=["simt", "auto"])
def algo(request):
    return request.param


def prune_both(X, b, k):
    ref = oracle.prune(X, b, k)
    A = bp.prune(to_torch(X), b, k=k)
    return A, ref


@pytest.mark.parametrize("b", [4, 8, 16, 32, 64])
@pytest.mark.parametrize("keep", [0.0, 0.2, 0.5, 1.0])
@pytest.mark.parametrize("N", [128, 384, 260])
def test_wgrad_fp32_small(algo, b, keep, N):
    M, K = 37 * b, 6 * b
    Nb = 37 * 6
    k = oracle.keep_count(Nb, keep)
    X = synth.f_gelu(M, K, seed=100 + b)
    dY = synth.grad_out(M, N, seed=100 + b)
    A, ref = prune_both(X, b, k)
    dW = bp.wgrad(A, to_torch(dY), prec="fp32", algo=algo)
    torch.cuda.synchronize()
    ref_dW = oracle.wgrad(ref["rowptr"], ref["colidx"], ref["values"], M, K, b, dY)
    if k == 0:
        assert not dW.any()
    else:
        err = oracle.rel_frobenius(dW.cpu().numpy(), ref_dW)
        assert err <= TOL["fp32"], err


@pytest.mark.parametrize("b", [16, 32])
def test_wgrad_fp32_accumulate_and_bf16_operands(algo, b):
    M, K, N = 40 * b, 5 * b, 256
    X = synth.f_aff(M, K, seed=200 + b)
    dY = synth.grad_out(M, N, seed=200 + b)
    A, ref = prune_both(X, b, 77)
    ref_dW = oracle.wgrad(ref["rowptr"], ref["colidx"], ref["values"], M, K, b, dY)
    base = torch.randn(K, N, device="cuda")
    out = base.clone()
    bp.wgrad(A, to_torch(dY), prec="fp32", out=out, accumulate=True, algo=algo)
    torch.cuda.synchronize()
    err = oracle.rel_frobenius(out.cpu().numpy() - base.cpu().numpy(), ref_dW)
    assert err <= 1e-5, err
    # bf16 dY through the FP32 path: exact bf16 -> fp32 widening on load
    dYh = synth.to_bf16_bits(dY)
    dW = bp.wgrad(A, to_torch(dYh, bf16=True), prec="fp32", algo=algo)
    torch.cuda.synchronize()
    ref_h = oracle.wgrad(ref["rowptr"], ref["colidx"], ref["values"], M, K, b, dYh)
    assert oracle.rel_frobenius(dW.cpu().numpy(), ref_h) <= 1e-5


@pytest.mark.parametrize("b", [4, 8, 16, 32, 64])
@pytest.mark.parametrize("keep", [0.1, 0.5])
def test_wgrad_fp32_bf16_storage(b, keep):
    """bf16 X and dY through the FP32 path (exact widening, fp32 FFMA) against the
    oracle run on the same bf16 values; several kcol tiles and splits."""
    M, K, N = 96 * b, 2 * 128 + 4 * b, 384
    Xh = synth.to_bf16_bits(synth.f_gelu(M, K, seed=600 + b))
    dYh = synth.to_bf16_bits(synth.grad_out(M, N, seed=600 + b))
    Xf = synth.bf16_bits_to_f32(Xh)
    k = oracle.keep_count((M // b) * (K // b), keep)
    ref = oracle.prune(Xf, b, k)
    A = bp.prune(to_torch(Xh, bf16=True), b, k=k)
    torch.cuda.synchronize()
    if not np.array_equal(A.colidx.cpu().numpy(), ref["colidx"]):
        pytest.skip("bf16 block sums moved the top-k boundary for this seed")
    dW = bp.wgrad(A, to_torch(dYh, bf16=True), prec="fp32")
    torch.cuda.synchronize()
    ref_dW = oracle.wgrad(ref["rowptr"], ref["colidx"], ref["values"], M, K, b, synth.bf16_bits_to_f32(dYh))
    assert oracle.rel_frobenius(dW.cpu().numpy(), ref_dW) <= 1e-5


def test_wgrad_fp32_worked_example():
    """Lifted worked example: dW with dY = ones equals the column sums of the
    masked X -- the hand-derived [3,4,5,4] scaled by the lift (exact)."""
    X = np.array([[3, 4, 0, 0], [0, 0, 1, 0], [0, 0, 2, 2], [0, 1, 2, 2]], np.float32)
    m = 8
    XL = np.kron(X, np.ones((m, m), np.float32))
    A = bp.prune(to_torch(XL), 2 * m, k=3)
    dW = bp.wgrad(A, torch.ones(4 * m, 4, device="cuda"), prec="fp32")
    torch.cuda.synchronize()
    expect = np.repeat(np.array([3, 4, 5, 4], np.float32) * m, m)
    np.testing.assert_array_equal(dW[:, 0].cpu().numpy(), expect)


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_wgrad_fp32_baseline_configs(algo, name):
    """Full-size configs: sampled entries computed one by one by the oracle."""
    c = synth.CONFIGS[name]
    M, K, N, b = c["M"], c["K"], c["N"], c["b"]
    k = oracle.keep_count(oracle.num_blocks(M, K, b), c["keep"])
    X = synth.activation(c["family"], M, K, synth.seed_for(c["id"]))
    dY = synth.grad_out(M, N, synth.seed_for(c["id"]))
    A, ref = prune_both(X, b, k)
    dW = bp.wgrad(A, to_torch(dY), prec="fp32", algo=algo).cpu().numpy()
    rng = np.random.default_rng(0)
    rows = rng.integers(0, K, 400)
    cols = rng.integers(0, N, 400)
    want = oracle.wgrad_entries(ref["rowptr"], ref["colidx"], ref["values"], M, K, b, dY, rows, cols)
    err = oracle.rel_frobenius(dW[rows, cols], want)
    assert err <= 1e-5, err
