"""Block-sparse linear operator of the paper, built on the hot path.

"The block-sparse linear operator is designed to be a plug-in replacement for
PyTorch's nn.linear layer with two additional parameters: the level of sparsity,
and the block size of the sparse structure".  The forward stays
dense "to ensure an accurate loss computation"; after it, the
input activation is pruned to its top-k b x b blocks and saved as BSR instead of
the dense tensor (fig:operator P:L313-321).  In the backward pass
the weight gradient comes from the BSR while "the input and bias
gradients do not depend on activations" and are computed densely.

    layer = SparseLinear(384, 1536, sparsity=0.5, block=32)   # keep = 1 - sparsity
    y = layer(x)            # x: (..., 384) CUDA tensor; rows = prod(leading dims)

Only the dense forward GEMM, dX = dY.W and db = sum(dY) use cuBLAS / PyTorch
ops (not part of the hot path, BJ "dX stays dense"); block norms, top-k, the
BSR pack and dW = X_bsr^T . dY run in libbsrprune's sm_100a kernels.
"""
from __future__ import annotations

import math

import torch

from . import BSR, affine_wgrad, prune, wgrad

__all__ = ["SparseLinear", "sparse_linear", "SparseAffine"]


class _SparseLinearFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x2d: torch.Tensor, weight: torch.Tensor, bias, keep: float, block: int, prec: str):
        y = x2d @ weight.t()
        if bias is not None:
            y = y + bias
        # prune AFTER the dense forward; only the BSR is kept for backward
        bsr = prune(x2d.detach(), block, keep=keep)
        ctx.bsr = bsr
        ctx.prec = prec
        ctx.has_bias = bias is not None
        ctx.save_for_backward(weight)
        return y

    @staticmethod
    def backward(ctx, dy: torch.Tensor):
        (weight,) = ctx.saved_tensors
        bsr: BSR = ctx.bsr
        dy = dy.contiguous()
        dx = dy @ weight if ctx.needs_input_grad[0] else None
        dw = None
        if ctx.needs_input_grad[1]:
            dy_w = dy.to(torch.bfloat16) if ctx.prec == "bf16" and dy.dtype != torch.bfloat16 else dy
            # nn.Linear stores weight as N x K: the library writes dW^T directly (bsr_wgrad_nk)
            dw = wgrad(bsr, dy_w, prec=ctx.prec, layout="nk").to(weight.dtype)
        db = dy.sum(0) if ctx.has_bias and ctx.needs_input_grad[2] else None
        ctx.bsr = None
        return dx, dw, db, None, None, None


def _default_prec(dtype: torch.dtype, block: int, out_features: int, rows: int = 0, in_features: int = 0) -> str:
    """dW arithmetic matching what nn.Linear would give: fp32 activations get the
    FP32-grade path (rel-F <= 1e-5: 3xTF32 tensor cores where the library has them,
    FFMA otherwise -- the library picks), bf16 activations the bf16 tensor cores
    where they apply: N % 128 == 0 and either b >= 16 (the block kernels) or rows
    and in_features multiples of 32 (b < 16: the dense rebuild of the masked X,
    measured 3-20x faster than the FFMA kernel on S12 at b = 4/8,
    profiles/r02g/c3.jsonl); the FP32 FFMA path (which reads bf16 storage) elsewhere."""
    if dtype == torch.bfloat16 and out_features % 128 == 0:
        if block >= 16 or (rows % 32 == 0 and in_features % 32 == 0 and rows > 0):
            return "bf16"
    return "fp32"


def sparse_linear(x: torch.Tensor, weight: torch.Tensor, bias=None, sparsity: float = 0.5, block: int = 16,
                  prec: str | None = None) -> torch.Tensor:
    """Functional form: y = x W^T + b with the input activation saved as top-k BSR."""
    lead = x.shape[:-1]
    x2d = x.reshape(-1, x.shape[-1]).contiguous()
    p = prec or _default_prec(x.dtype, block, weight.shape[0], x2d.shape[0], x2d.shape[1])
    y = _SparseLinearFn.apply(x2d, weight, bias, 1.0 - float(sparsity), int(block), p)
    return y.reshape(*lead, weight.shape[0])


class SparseLinear(torch.nn.Module):
    """nn.Linear with two extra parameters, `sparsity` (fraction of blocks pruned,
    s in the paper) and `block` (b): the saved input activation keeps its
    round((1 - s) * N) largest-l2-norm b x b blocks."""

    def __init__(self, in_features: int, out_features: int, sparsity: float = 0.5, block: int = 16,
                 bias: bool = True, prec: str | None = None, device=None, dtype=None):
        super().__init__()
        if in_features % block:
            raise ValueError(f"in_features={in_features} must be a multiple of block={block}")
        if not 0.0 <= sparsity <= 1.0:
            raise ValueError("sparsity must be in [0, 1]")
        self.in_features, self.out_features = in_features, out_features
        self.sparsity, self.block, self.prec = float(sparsity), int(block), prec
        kw = dict(device=device, dtype=dtype)
        self.weight = torch.nn.Parameter(torch.empty(out_features, in_features, **kw))
        self.bias = torch.nn.Parameter(torch.empty(out_features, **kw)) if bias else None
        torch.nn.init.kaiming_uniform_(self.weight, a=math.sqrt(5))
        if self.bias is not None:
            bound = 1.0 / math.sqrt(in_features)
            torch.nn.init.uniform_(self.bias, -bound, bound)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        if not self.training or not torch.is_grad_enabled():
            out = x @ self.weight.t()
            return out + self.bias if self.bias is not None else out
        return sparse_linear(x, self.weight, self.bias, self.sparsity, self.block, self.prec)

    def extra_repr(self) -> str:
        return (f"in_features={self.in_features}, out_features={self.out_features}, sparsity={self.sparsity}, "
                f"block={self.block}, bias={self.bias is not None}")


class _SparseAffineFn(torch.autograd.Function):
    """y = alpha * x + beta per channel; x saved as the BSR of its top-k blocks."""

    @staticmethod
    def forward(ctx, x2d: torch.Tensor, alpha: torch.Tensor, beta: torch.Tensor, keep: float, block: int):
        y = torch.addcmul(beta, x2d, alpha)
        ctx.bsr = prune(x2d.detach(), block, keep=keep)
        ctx.save_for_backward(alpha)
        return y

    @staticmethod
    def backward(ctx, dy: torch.Tensor):
        (alpha,) = ctx.saved_tensors
        dy = dy.contiguous()
        dx = dy * alpha if ctx.needs_input_grad[0] else None
        dalpha = affine_wgrad(ctx.bsr, dy).to(alpha.dtype) if ctx.needs_input_grad[1] else None
        dbeta = dy.sum(0) if ctx.needs_input_grad[2] else None
        ctx.bsr = None
        return dx, dalpha, dbeta, None, None


class SparseAffine(torch.nn.Module):
    """ResMLP's affine scaling layer Aff(x) = alpha * x + beta in its
    block-sparse version: the input activation is saved as the BSR of
    its round((1 - s) * N) largest-l2-norm b x b blocks and the scale gradient is
    computed from it (bsr_affine_wgrad); dx = alpha * dy and dbeta = sum(dy) need
    no activation and stay dense."""

    def __init__(self, dim: int, sparsity: float = 0.5, block: int = 16, device=None, dtype=None):
        super().__init__()
        if dim % block:
            raise ValueError(f"dim={dim} must be a multiple of block={block}")
        self.dim, self.sparsity, self.block = dim, float(sparsity), int(block)
        self.alpha = torch.nn.Parameter(torch.ones(dim, device=device, dtype=dtype))
        self.beta = torch.nn.Parameter(torch.zeros(dim, device=device, dtype=dtype))

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        if not self.training or not torch.is_grad_enabled():
            return torch.addcmul(self.beta, x, self.alpha)
        lead = x.shape[:-1]
        x2d = x.reshape(-1, self.dim).contiguous()
        y = _SparseAffineFn.apply(x2d, self.alpha, self.beta, 1.0 - self.sparsity, self.block)
        return y.reshape(*lead, self.dim)
