"""Test-side helpers: boundary-gap enforcement (uses the oracle's norms),
numpy <-> torch moves, and BSR comparison."""
from __future__ import annotations

import numpy as np

import oracle
import synth


def enforce_gap(X: np.ndarray, b: int, k: int, rel: float = 1e-5, max_iter: int = 20) -> tuple[np.ndarray, int]:
    """BJ: "the generator guarantees a >= 1e-5 relative norm gap at the k-th
    boundary".  Pruned blocks whose fp64 norm is within 2*rel of the k-th largest
    norm tau are scaled (in fp32) to tau*(1 - 3*rel).  Returns (X', adjusted)."""
    X = np.array(X, dtype=np.float32, copy=True)
    M, K = X.shape
    N = (M // b) * (K // b)
    if k <= 0 or k >= N:
        return X, 0
    adjusted = 0
    blocks = X.reshape(M // b, b, K // b, b)
    for _ in range(max_iter):
        norm = np.sqrt(oracle.block_sumsq(X, b))
        order = np.lexsort((np.arange(N), -norm))  # norm desc, index asc
        tau = norm[order[k - 1]]
        pruned = order[k:]
        bad = pruned[norm[pruned] > tau * (1.0 - 2.0 * rel)]
        if bad.size == 0:
            return X, adjusted
        I, J = np.divmod(bad, K // b)
        c = (tau * (1.0 - 3.0 * rel) / np.maximum(norm[bad], 1e-300)).astype(np.float32)
        blocks[I, :, J, :] *= c[:, None, None]
        adjusted += bad.size
    raise RuntimeError("gap enforcement did not converge")


def gap_ok(X: np.ndarray, b: int, k: int, rel: float = 1e-5) -> bool:
    norm = np.sqrt(oracle.block_sumsq(X, b))
    N = norm.size
    if k <= 0 or k >= N:
        return True
    s = np.sort(norm)[::-1]
    return s[k - 1] >= s[k] * (1.0 + rel)


def gap_k(X: np.ndarray, b: int, k: int, rel: float = 2e-4) -> int:
    """The kept count nearest to k whose boundary has a natural relative gap
    >= rel between the k-th and (k+1)-th largest fp64 block sums of squares, so
    that the fp32 sums of the GPU select the same set as the oracle's fp64 ones
    without rescaling X (used for bf16 inputs, where rescaling would leave the
    bf16 grid).  X: fp32 array or bf16 bit patterns (uint16)."""
    if X.dtype == np.uint16:
        X = synth.bf16_bits_to_f32(X)
    s = np.sort(oracle.block_sumsq(X, b))[::-1]
    N = s.size
    if k <= 0 or k >= N:
        return k
    for d in range(N):
        for kk in (k - d, k + d):
            if 0 < kk < N and s[kk - 1] > s[kk] * (1.0 + rel):
                return kk
    return k


def make_x(family: str, M: int, K: int, seed: int, b: int, k: int, gap: bool = True) -> np.ndarray:
    X = synth.activation(family, M, K, seed)
    if gap:
        X, _ = enforce_gap(X, b, k)
    return X


def to_torch(a: np.ndarray, device="cuda", bf16: bool = False):
    import torch
    if bf16:  # a holds bf16 bit patterns (uint16)
        return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).to(device)
    return torch.from_numpy(np.ascontiguousarray(a)).to(device)


def bits(t) -> np.ndarray:
    """Raw bit patterns of a CUDA/CPU tensor as a numpy integer array."""
    import torch
    t = t.detach().cpu().contiguous()
    if t.dtype == torch.float32:
        return t.view(torch.int32).numpy()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy()
    return t.numpy()
