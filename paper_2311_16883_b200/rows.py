"""The paper-faithful variant: 1 x b row-segment blocks
selected per sample.  Argument marshalling over the C
ABI (include/bsrprune.h: bsr_prune_rows, bsr_decompress_rows, bsr_wgrad_rows);
every step runs in the library's kernels (csrc/prune_rows.cu)."""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _dt, _lib, _stream, workspace


@dataclass
class RowBSR:
    """BSR with br = 1, bc = b: rowptr[M + 1], colidx[k], values[k, b] (device)."""
    rowptr: torch.Tensor
    colidx: torch.Tensor
    values: torch.Tensor
    M: int
    K: int
    b: int
    sample_rows: int

    @property
    def nnz(self) -> int:
        return int(self.colidx.numel())


def keep_per_sample(sample_rows: int, K: int, b: int, keep: float) -> int:
    return int(_lib.load().bsr_rows_keep_per_sample(sample_rows, K, b, float(keep)))


def prune_rows(X: torch.Tensor, b: int, keep: float, sample_rows: int = 196, stream=None) -> RowBSR:
    """Keep, in every sample of `sample_rows` rows, the nearest(keep * sample_rows * K / b)
    1 x b segments of largest l2 norm (ties -> lower flat index)."""
    lib = _lib.load()
    M, K = X.shape
    ks = keep_per_sample(sample_rows, K, b, keep)
    if ks < 0 or M % sample_rows:
        raise ValueError(f"sample_rows={sample_rows} must divide M={M} and b={b} must divide K={K}")
    k = (M // sample_rows) * ks
    out = RowBSR(rowptr=torch.empty(M + 1, dtype=torch.int32, device=X.device),
                 colidx=torch.empty(k, dtype=torch.int32, device=X.device),
                 values=torch.empty((k, b), dtype=X.dtype, device=X.device), M=M, K=K, b=b, sample_rows=sample_rows)
    ws = workspace(lib.bsr_prune_rows_workspace_bytes(M, K, b), X.device, kind="rows", stream=stream)
    _lib.check(lib.bsr_prune_rows(X.data_ptr(), M, K, b, sample_rows, float(keep), _dt(X), out.rowptr.data_ptr(),
                                  out.colidx.data_ptr() if k else None, out.values.data_ptr() if k else None,
                                  ws.data_ptr(), ws.numel(), _stream(stream)))
    return out


def decompress_rows(A: RowBSR, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    lib = _lib.load()
    if out is None:
        out = torch.empty(A.M, A.K, dtype=A.values.dtype, device=A.rowptr.device)
    _lib.check(lib.bsr_decompress_rows(A.rowptr.data_ptr(), A.colidx.data_ptr() if A.nnz else None,
                                       A.values.data_ptr() if A.nnz else None, A.M, A.K, A.b, _dt(A.values),
                                       out.data_ptr(), _stream(stream)))
    return out


def wgrad_rows(A: RowBSR, dY: torch.Tensor, out: torch.Tensor | None = None, accumulate: bool = False,
               stream=None, tensor_cores: bool | None = None) -> torch.Tensor:
    """dW = X_bsr^T . dY (K x N fp32) over the kept segments.  FP32 FFMA
    (deterministic), or -- tensor_cores=True, or None when the shape allows it --
    the tcgen05 kernel on the densely rebuilt kept rows (FP32 grade for f32, bf16
    for bf16 storage; include/bsrprune.h bsr_wgrad_rows_tc)."""
    lib = _lib.load()
    N = dY.shape[1]
    if dY.shape[0] != A.M:
        raise ValueError(f"dY has {dY.shape[0]} rows, the BSR has M={A.M}")
    if out is None:
        out = torch.empty(A.K, N, dtype=torch.float32, device=dY.device)
    tc_ws = lib.bsr_wgrad_rows_tc_workspace_bytes(A.M, A.K, A.b, N, _dt(A.values))
    if tensor_cores is None:
        tensor_cores = bool(tc_ws) and dY.dtype == A.values.dtype
    if tensor_cores:
        ws = workspace(tc_ws, dY.device, kind="rows_tc", stream=stream)
        _lib.check(lib.bsr_wgrad_rows_tc(A.rowptr.data_ptr(), A.colidx.data_ptr() if A.nnz else None,
                                         A.values.data_ptr() if A.nnz else None, A.nnz, A.M, A.K, A.b, _dt(A.values),
                                         dY.data_ptr(), _dt(dY), N, out.data_ptr(), int(accumulate), ws.data_ptr(),
                                         ws.numel(), _stream(stream)))
        return out
    ws_bytes = lib.bsr_wgrad_rows_workspace_bytes(A.M, A.K, A.b, N)
    ws = workspace(ws_bytes, dY.device, stream=stream) if ws_bytes else None
    _lib.check(lib.bsr_wgrad_rows(A.rowptr.data_ptr(), A.colidx.data_ptr() if A.nnz else None,
                                  A.values.data_ptr() if A.nnz else None, A.nnz, A.M, A.K, A.b, _dt(A.values),
                                  dY.data_ptr(), _dt(dY), N, out.data_ptr(), int(accumulate),
                                  ws.data_ptr() if ws is not None else None, ws.numel() if ws is not None else 0,
                                  _stream(stream)))
    return out
