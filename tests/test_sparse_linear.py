"""SparseLinear: the paper's block-sparse linear operator built on
the hot path -- dense forward, top-k BSR saved for backward, dW from the BSR.
Gradients are checked against the fp64 oracle on the same pruned activation."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2311_16883_b200 import SparseLinear  # noqa: E402


def run(prec, sparsity, block, M=196 * 16, K=384, N=256, dtype=torch.float32, seed=0):
    torch.manual_seed(seed)
    x_np = synth.f_gelu(M, K, seed)
    dy_np = synth.grad_out(M, N, seed)
    layer = SparseLinear(K, N, sparsity=sparsity, block=block, prec=prec, device="cuda", dtype=dtype)
    x = torch.from_numpy(x_np).to("cuda", dtype).requires_grad_(True)
    y = layer(x)
    dy = torch.from_numpy(dy_np).to("cuda", dtype)
    y.backward(dy)
    torch.cuda.synchronize()
    return layer, x, y, x_np, dy_np


@pytest.mark.parametrize("prec,block,tol", [("tf32", 32, 5e-3), ("fp32", 16, 1e-5), ("tf32", 64, 5e-3)])
@pytest.mark.parametrize("sparsity", [0.0, 0.5, 0.8])
def test_grad_weight_matches_oracle(prec, block, tol, sparsity):
    layer, x, y, x_np, dy_np = run(prec, sparsity, block)
    M, K = x_np.shape
    k = oracle.keep_count(oracle.num_blocks(M, K, block), 1.0 - sparsity)
    ref = oracle.prune(x_np, block, k)
    dw_ref = oracle.wgrad(ref["rowptr"], ref["colidx"], ref["values"], M, K, block, dy_np)  # K x N
    got = layer.weight.grad.detach().t().cpu().numpy()
    assert oracle.rel_frobenius(got, dw_ref) <= tol
    # the input / bias gradients and the forward stay dense
    W = layer.weight.detach().double().cpu().numpy()
    np.testing.assert_allclose(x.grad.cpu().numpy(), dy_np.astype(np.float64) @ W, rtol=0, atol=2e-4)
    np.testing.assert_allclose(layer.bias.grad.cpu().numpy(), dy_np.astype(np.float64).sum(0), rtol=1e-4, atol=1e-5)
    y_ref = x_np.astype(np.float64) @ W.T + layer.bias.detach().double().cpu().numpy()
    np.testing.assert_allclose(y.detach().cpu().numpy(), y_ref, rtol=0, atol=5e-2)


def test_bf16_layer():
    layer, x, y, x_np, dy_np = run(None, 0.5, 32, dtype=torch.bfloat16)
    assert layer.weight.grad is not None and torch.isfinite(layer.weight.grad).all()
    xb = synth.to_bf16_bits(x_np)
    dyb = synth.to_bf16_bits(dy_np)
    M, K = x_np.shape
    k = oracle.keep_count(oracle.num_blocks(M, K, 32), 0.5)
    ref = oracle.prune(xb, 32, k)
    dw_ref = oracle.wgrad(ref["rowptr"], ref["colidx"], ref["values"], M, K, 32, dyb)
    got = layer.weight.grad.detach().float().t().cpu().numpy()
    assert oracle.rel_frobenius(got, dw_ref) <= 5e-3  # bf16 weight.grad rounding included


def test_eval_mode_is_dense_and_leading_dims():
    layer = SparseLinear(64, 128, sparsity=0.9, block=16, device="cuda").eval()
    x = torch.randn(2, 49, 64, device="cuda")
    with torch.no_grad():
        y = layer(x)
    torch.testing.assert_close(y, x @ layer.weight.t() + layer.bias)
    layer.train()
    x = torch.randn(2, 48, 64, device="cuda", requires_grad=True)
    y = layer(x)
    assert y.shape == (2, 48, 128)
    y.sum().backward()
    assert x.grad.shape == x.shape


def test_saved_activation_is_the_bsr():
    """Memory: the dense input is not kept for backward -- only its BSR."""
    M, K, N, b = 196 * 32, 384, 1536, 32
    layer = SparseLinear(K, N, sparsity=0.8, block=b, device="cuda")
    torch.cuda.synchronize()
    x = torch.randn(M, K, device="cuda", requires_grad=False)
    layer(x.clone())  # warm-up: cuBLAS / prune workspaces are allocated once, outside the measurement
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    y = layer(x.clone())  # the clone is the activation; it must be freed after forward
    torch.cuda.synchronize()
    held = torch.cuda.memory_allocated() - base - y.numel() * 4
    k = oracle.keep_count(oracle.num_blocks(M, K, b), 0.2)
    bsr_bytes = oracle.storage_bytes(M, b, b, k)
    # the caching allocator rounds blocks > 1 MiB to 2 MiB and keeps small pools: allow 1 MiB of slack
    assert held <= bsr_bytes + (1 << 20), (held, bsr_bytes)
    assert held < 0.5 * M * K * 4


@pytest.mark.parametrize("block", [4, 8])
def test_bf16_small_blocks(block):
    """bf16 activations with b < 16: no block tensor-core kernel at that size, so the
    layer's default is the bf16 dense rebuild where the shape allows it and the FP32
    FFMA path otherwise -- never a bf16 call the library rejects."""
    layer, x, y, x_np, dy_np = run(None, 0.5, block, N=256, dtype=torch.bfloat16)
    assert layer.weight.grad is not None and torch.isfinite(layer.weight.grad).all()
    xb, dyb = synth.to_bf16_bits(x_np), synth.to_bf16_bits(dy_np)
    M, K = x_np.shape
    k = oracle.keep_count(oracle.num_blocks(M, K, block), 0.5)
    ref = oracle.prune(xb, block, k)
    dw_ref = oracle.wgrad(ref["rowptr"], ref["colidx"], ref["values"], M, K, block, dyb)
    got = layer.weight.grad.detach().float().t().cpu().numpy()
    assert oracle.rel_frobenius(got, dw_ref) <= 5e-3  # bf16 weight.grad rounding included


def test_fp32_layer_defaults_to_fp32_grade():
    """fp32 activations: the default dW is the FP32 grade (<= 1e-5), as nn.Linear's
    fp32 weight gradient would be -- not a silent tf32 downgrade."""
    layer, x, y, x_np, dy_np = run(None, 0.5, 32)
    M, K = x_np.shape
    k = oracle.keep_count(oracle.num_blocks(M, K, 32), 0.5)
    ref = oracle.prune(x_np, 32, k)
    dw_ref = oracle.wgrad(ref["rowptr"], ref["colidx"], ref["values"], M, K, 32, dy_np)
    got = layer.weight.grad.detach().t().cpu().numpy()
    assert oracle.rel_frobenius(got, dw_ref) <= 1e-5

