"""B200-native hot path of structured activation pruning (arXiv 2311.16883).

Thin Python layer over the C-ABI library ``libbsrprune.so`` (include/bsrprune.h).
PyTorch supplies device memory and the current CUDA stream only; every step --
block norms, top-k, BSR packing, decompression and the block-sparse weight
gradient -- runs in the library's hand-written sm_100a kernels.

    bsr = prune(X, b=32, keep=0.5)          # forward: X (M x K, cuda) -> BSR
    dW  = wgrad(bsr, dY, prec="fp32")       # backward: dW = X_bsr^T . dY (K x N)
    Xm  = decompress(bsr)                   # X masked to the kept blocks
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import ALGO, BsrError, DT_BF16, DT_F32, PREC

__all__ = ["BSR", "BsrError", "prune", "prune_stochastic", "validate", "decompress", "wgrad", "block_sumsq", "num_blocks", "keep_count",
           "storage_bytes", "workspace", "version", "set_pdl", "wgrad_multicast", "affine_wgrad", "SparseAffine", "SparseLinear", "sparse_linear", "prune_global",
           "RowBSR", "prune_rows", "decompress_rows", "wgrad_rows", "act_prune"]

_DT = {torch.float32: DT_F32, torch.bfloat16: DT_BF16}


def _dt(t: torch.Tensor) -> int:
    try:
        return _DT[t.dtype]
    except KeyError:
        raise TypeError(f"unsupported dtype {t.dtype} (float32 or bfloat16)") from None


def _stream(stream) -> ctypes.c_void_p:
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _cuda2d(t: torch.Tensor, name: str) -> torch.Tensor:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dim() != 2 or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous 2-D tensor")
    return t


@dataclass
class BSR:
    """Block Sparse Row matrix: device tensors + logical shape."""
    rowptr: torch.Tensor   # int32 [M/b + 1]
    colidx: torch.Tensor   # int32 [nnzb]
    values: torch.Tensor   # dtype [nnzb, b, b]
    M: int
    K: int
    b: int

    @property
    def nnzb(self) -> int:
        return self.colidx.numel()

    @property
    def dtype(self) -> torch.dtype:
        return self.values.dtype

    def nbytes(self) -> int:
        return storage_bytes(self.M, self.b, self.nnzb, self.dtype)

    def c_struct(self) -> _lib.BsrT:
        return _lib.BsrT(self.M, self.K, self.b, _dt(self.values), self.nnzb, self.rowptr.data_ptr(),
                         self.colidx.data_ptr() if self.nnzb else None,
                         self.values.data_ptr() if self.nnzb else None)


def version() -> str:
    return _lib.load().bsr_version().decode()


def num_blocks(M: int, K: int, b: int) -> int:
    return int(_lib.load().bsr_num_blocks(M, K, b))


def keep_count(N: int, keep: float) -> int:
    k = int(_lib.load().bsr_keep_count(N, float(keep)))
    if k < 0:
        raise ValueError("keep must be in [0, 1]")
    return k


def storage_bytes(M: int, b: int, k: int, dtype=torch.float32) -> int:
    return int(_lib.load().bsr_storage_bytes(M, b, k, _DT[dtype]))


_WS: dict = {}


def _stream_obj(device: torch.device, stream=None):
    return torch.cuda.current_stream(device) if stream is None else stream


def workspace(nbytes: int, device: torch.device, kind: str = "wgrad", stream=None) -> torch.Tensor:
    """Cached device workspace of at least nbytes, one per (device, kind, stream).

    Keyed on the launch stream so that calls in flight on different streams never
    share a workspace (the prune keeps its grid-barrier counter and histograms
    there, the dW its split-K partials).  The buffer is allocated -- and, for the
    prune, zero-filled -- ON that stream, so the first launch is ordered after the
    fill.  bsr_prune needs a zero-filled workspace on first use and leaves it that
    way (include/bsrprune.h), so the prune workspace is used for nothing else."""
    s = _stream_obj(device, stream)
    key = (device.type, device.index, kind, s.cuda_stream)
    ws = _WS.get(key)
    if ws is None or ws.numel() < nbytes:
        with torch.cuda.stream(s):
            alloc = torch.zeros if kind == "prune" else torch.empty
            ws = alloc(max(nbytes, 256), dtype=torch.uint8, device=device)
        _WS[key] = ws
    return ws


def _check_out_bsr(out: "BSR", M: int, K: int, b: int, k: int, dtype: torch.dtype, device) -> None:
    """The caller-supplied output BSR must match the call exactly (the kernel writes
    k colidx entries, k*b*b values and M/b+1 rowptr entries)."""
    if (out.M, out.K, out.b) != (M, K, b):
        raise ValueError(f"out BSR is for M={out.M} K={out.K} b={out.b}, the call has M={M} K={K} b={b}")
    for name, t, n, dt in (("rowptr", out.rowptr, M // b + 1, torch.int32), ("colidx", out.colidx, k, torch.int32)):
        if t.dtype != dt or t.numel() != n or not t.is_contiguous() or t.device != device:
            raise ValueError(f"out.{name} must be a contiguous {dt} tensor of {n} elements on {device}")
    v = out.values
    if v.dtype != dtype or tuple(v.shape) != (k, b, b) or not v.is_contiguous() or v.device != device:
        raise ValueError(f"out.values must be a contiguous {dtype} tensor of shape ({k}, {b}, {b}) on {device}")


def _check_dense_out(t: torch.Tensor, shape, dtype, device, name: str) -> None:
    if t.dtype != dtype or tuple(t.shape) != tuple(shape) or not t.is_contiguous() or t.device != device:
        raise ValueError(f"{name} must be a contiguous {dtype} tensor of shape {tuple(shape)} on {device}")


def alloc_bsr(M: int, K: int, b: int, k: int, dtype: torch.dtype, device) -> BSR:
    return BSR(rowptr=torch.empty(M // b + 1, dtype=torch.int32, device=device),
               colidx=torch.empty(k, dtype=torch.int32, device=device),
               values=torch.empty((k, b, b), dtype=dtype, device=device), M=M, K=K, b=b)


def prune(X: torch.Tensor, b: int, keep: float | None = None, k: int | None = None, out: BSR | None = None,
          stream=None) -> BSR:
    """Keep the top-k b x b blocks of X by l2 norm and pack them into BSR.

    Exactly one of ``keep`` (ratio, k = nearest(keep*N)) or ``k`` is given."""
    lib = _lib.load()
    X = _cuda2d(X, "X")
    M, K = X.shape
    N = num_blocks(M, K, b)
    if N < 0:
        raise _lib.BsrError(2, f"b={b} must divide M={M} and K={K}")
    if (keep is None) == (k is None):
        raise ValueError("give exactly one of keep or k")
    if k is None:
        k = keep_count(N, keep)
    if out is None:
        out = alloc_bsr(M, K, b, k, X.dtype, X.device)
    else:
        _check_out_bsr(out, M, K, b, k, X.dtype, X.device)
    ws_bytes = lib.bsr_prune_workspace_bytes(M, K, b)
    ws = workspace(ws_bytes, X.device, kind="prune", stream=stream)
    cs = out.c_struct()
    _lib.check(lib.bsr_prune_k(X.data_ptr(), M, K, b, k, _dt(X), ctypes.byref(cs), ws.data_ptr(), ws.numel(),
                               _stream(stream)))
    return out


def prune_stochastic(X: torch.Tensor, b: int, keep: float | None = None, k: int | None = None, window: int = 0,
                     p: float = 0.5, seed: int = 0, out: BSR | None = None, stream=None) -> BSR:
    """Top-k with stochastic boundary swapping (DESIGN reading R19):
    pair i < min(window, k, N-k) of (rank k-1-i, rank k+i) swaps kept/pruned iff
    the counter-based uniform u_i(seed) < p.  Exactly k blocks kept; same seed,
    same selection."""
    lib = _lib.load()
    X = _cuda2d(X, "X")
    M, K = X.shape
    N = num_blocks(M, K, b)
    if N < 0:
        raise _lib.BsrError(2, f"b={b} must divide M={M} and K={K}")
    if (keep is None) == (k is None):
        raise ValueError("give exactly one of keep or k")
    if k is None:
        k = keep_count(N, keep)
    if out is None:
        out = alloc_bsr(M, K, b, k, X.dtype, X.device)
    else:
        _check_out_bsr(out, M, K, b, k, X.dtype, X.device)
    ws = workspace(lib.bsr_prune_stochastic_workspace_bytes(M, K, b), X.device, kind="prune", stream=stream)
    cs = out.c_struct()
    _lib.check(lib.bsr_prune_stochastic(X.data_ptr(), M, K, b, k, int(window), float(p), int(seed) & (2**64 - 1),
                                        _dt(X), ctypes.byref(cs), ws.data_ptr(), ws.numel(), _stream(stream)))
    return out


def validate(A: BSR, stream=None) -> int:
    """Structural check of a BSR on the device (bsr_validate): -1 when rowptr / colidx
    hold the BSR invariants, else the lowest offending block row.  Reads the result
    back (one device-to-host copy of an int32)."""
    lib = _lib.load()
    bad = torch.empty(1, dtype=torch.int32, device=A.rowptr.device)
    cs = A.c_struct()
    _lib.check(lib.bsr_validate(ctypes.byref(cs), bad.data_ptr(), _stream(stream)))
    return int(bad.item())


def act_prune(Z: torch.Tensor, b: int, keep: float | None = None, k: int | None = None, act: str = "gelu",
              X_out: torch.Tensor | None = None, out: BSR | None = None, stream=None) -> tuple[torch.Tensor, BSR]:
    """Producer fusion: X = act(Z) with the block norms computed in
    the same pass, then the prune reads X only for the kept blocks.  Returns
    (X, BSR); identical to X = act(Z); prune(X, b, ...)."""
    lib = _lib.load()
    Z = _cuda2d(Z, "Z")
    M, K = Z.shape
    N = num_blocks(M, K, b)
    if k is None:
        if keep is None:
            raise ValueError("give keep or k")
        k = keep_count(N, keep)
    if X_out is None:
        X_out = torch.empty_like(Z)
    else:
        _check_dense_out(X_out, (M, K), Z.dtype, Z.device, "X_out")
    if out is None:
        out = alloc_bsr(M, K, b, k, Z.dtype, Z.device)
    else:
        _check_out_bsr(out, M, K, b, k, Z.dtype, Z.device)
    ws_bytes = lib.bsr_prune_workspace_bytes(M, K, b)
    ws = workspace(ws_bytes, Z.device, kind="prune", stream=stream)
    a = {"identity": 0, "gelu": 1}[act]
    _lib.check(lib.bsr_act_block_sumsq(Z.data_ptr(), X_out.data_ptr(), M, K, b, _dt(Z), a, ws.data_ptr(), ws.numel(),
                                       _stream(stream)))
    cs = out.c_struct()
    _lib.check(lib.bsr_prune_presummed(X_out.data_ptr(), M, K, b, k, _dt(Z), ctypes.byref(cs), ws.data_ptr(),
                                       ws.numel(), _stream(stream)))
    return X_out, out


def block_sumsq(X: torch.Tensor, b: int, stream=None) -> torch.Tensor:
    lib = _lib.load()
    X = _cuda2d(X, "X")
    M, K = X.shape
    N = num_blocks(M, K, b)
    out = torch.empty(max(N, 0), dtype=torch.float32, device=X.device)
    _lib.check(lib.bsr_block_sumsq(X.data_ptr(), M, K, b, _dt(X), out.data_ptr(), _stream(stream)))
    return out


def decompress(A: BSR, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    lib = _lib.load()
    if out is None:
        out = torch.empty((A.M, A.K), dtype=A.dtype, device=A.rowptr.device)
    else:
        _check_dense_out(out, (A.M, A.K), A.dtype, A.rowptr.device, "out")
    cs = A.c_struct()
    _lib.check(lib.bsr_decompress(ctypes.byref(cs), out.data_ptr(), _stream(stream)))
    return out


def wgrad(A: BSR, dY: torch.Tensor, prec: str = "fp32", out: torch.Tensor | None = None,
          accumulate: bool = False, stream=None, algo: str = "auto", layout: str = "kn") -> torch.Tensor:
    """dW = X_bsr^T . dY (K x N fp32) over the kept blocks only.

    prec: "fp32" (FP32 grade, rel-F <= 1e-5: 3xTF32 tensor cores or FFMA), "tf32"
    or "bf16" (tensor cores, <= 5e-3).  algo: "auto" (the library's per-shape
    choice), "runs", "span" (the two tcgen05 kernels) or "simt" (FFMA).
    layout: "kn" (K x N) or "nk" (dW^T, N x K: nn.Linear.weight.grad's layout,
    bsr_wgrad_nk)."""
    lib = _lib.load()
    dY = _cuda2d(dY, "dY")
    if dY.shape[0] != A.M:
        raise ValueError(f"dY has {dY.shape[0]} rows, BSR has M={A.M}")
    if layout not in ("kn", "nk"):
        raise ValueError(f"layout must be 'kn' or 'nk', got {layout!r}")
    N = dY.shape[1]
    shape = (A.K, N) if layout == "kn" else (N, A.K)
    if out is None:
        out = torch.empty(shape, dtype=torch.float32, device=dY.device)
    else:
        _check_dense_out(out, shape, torch.float32, dY.device, "out")
    p = PREC[prec]
    if layout == "kn":
        fn, ws_bytes = lib.bsr_wgrad_algo, lib.bsr_wgrad_algo_workspace_bytes(A.M, A.K, A.b, N, p, ALGO[algo])
    else:
        fn, ws_bytes = lib.bsr_wgrad_nk, lib.bsr_wgrad_nk_workspace_bytes(A.M, A.K, A.b, N, p, ALGO[algo])
    ws = workspace(ws_bytes, dY.device, stream=stream) if ws_bytes else None
    cs = A.c_struct()
    _lib.check(fn(ctypes.byref(cs), dY.data_ptr(), _dt(dY), N, out.data_ptr(), int(accumulate), p, ALGO[algo],
                  ws.data_ptr() if ws is not None else None, ws.numel() if ws is not None else 0, _stream(stream)))
    return out


def affine_wgrad(A: BSR, dY: torch.Tensor, out: torch.Tensor | None = None, accumulate: bool = False,
                 stream=None) -> torch.Tensor:
    """Scale gradient of the block-sparse affine layer: dalpha[c] = sum of
    x * dY over the kept blocks of column c (K fp32).  dY: M x K, like X."""
    lib = _lib.load()
    dY = _cuda2d(dY, "dY")
    if tuple(dY.shape) != (A.M, A.K):
        raise ValueError(f"dY must be {A.M} x {A.K} like the pruned activation, got {tuple(dY.shape)}")
    if out is None:
        out = torch.empty(A.K, dtype=torch.float32, device=dY.device)
    else:
        _check_dense_out(out, (A.K,), torch.float32, dY.device, "out")
    ws = workspace(lib.bsr_affine_wgrad_workspace_bytes(A.M, A.K, A.b), dY.device, stream=stream)
    cs = A.c_struct()
    _lib.check(lib.bsr_affine_wgrad(ctypes.byref(cs), dY.data_ptr(), _dt(dY), out.data_ptr(), int(accumulate),
                                    ws.data_ptr(), ws.numel(), _stream(stream)))
    return out


def wgrad_multicast(A: BSR, dY: torch.Tensor, mc_ptr: int, prec: str = "fp32", algo: str = "auto",
                    stream=None) -> None:
    """Fused a6 + a7 (SURVEY §8f f3 ii): ADD this rank's dW = X_bsr^T . dY into the
    K x N fp32 buffer behind the multimem (NVLS multicast) address mc_ptr, from the
    dW kernel itself (multimem.red.add); the NVSwitch sums the ranks.  The caller
    zeroes the buffer on every rank first and synchronises the ranks afterwards
    (paper_2311_16883_b200.dist.NvlsGradient)."""
    lib = _lib.load()
    dY = _cuda2d(dY, "dY")
    if dY.shape[0] != A.M:
        raise ValueError(f"dY has {dY.shape[0]} rows, BSR has M={A.M}")
    N = dY.shape[1]
    p = PREC[prec]
    ws_bytes = lib.bsr_wgrad_workspace_bytes(A.M, A.K, A.b, N, p)
    ws = workspace(ws_bytes, dY.device, stream=stream) if ws_bytes else None
    cs = A.c_struct()
    _lib.check(lib.bsr_wgrad_multicast(ctypes.byref(cs), dY.data_ptr(), _dt(dY), N, ctypes.c_void_p(mc_ptr), p,
                                       ALGO[algo], ws.data_ptr() if ws is not None else None,
                                       ws.numel() if ws is not None else 0, _stream(stream)))


def set_pdl(mask: int) -> int:
    """Process-wide programmatic-dependent-launch mask (include/bsrprune.h); returns the old one."""
    return int(_lib.load().bsr_set_pdl(int(mask)))


from .sparse_linear import SparseAffine, SparseLinear, sparse_linear  # noqa: E402  (uses the functions above)
from .global_select import prune_global  # noqa: E402
from .rows import RowBSR, decompress_rows, prune_rows, wgrad_rows  # noqa: E402
