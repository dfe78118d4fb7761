"""CPU oracle for the hot path of arXiv 2311.16883 -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
and ``--impl reference`` legs may import this package.  The product path
(``paper_2311_16883_b200``) never imports, links or calls it and shares no code
with it.  The arithmetic lives in plain C (``bsr_oracle.c``, fp64, single
thread); this module only marshals numpy arrays through ctypes, plus two tiny
pure-Python routines (brute-force top-k, relative Frobenius error) used to pin
the oracle and to grade parity.

Citations: ``P:L<n>`` = line n of /root/reference/PAPER.md; ``BJ`` =
BASELINE.json ``north_star``; readings R1..R14 are listed in DESIGN.md §3.

Pins (tests/test_oracle.py) -- every function here is pinned by something
other than itself:
  keep_count / storage_bytes  Table II, 48 printed cells, and the
                              BJ closed form at C1/C2.
  block_sumsq                 hand-computed worked examples; numpy.linalg.norm
                              on each block; constant-block closed form.
  select_topk                 brute force over all k-subsets (N <= 14) with the
                              BJ tie rule; invariants (min kept >= max pruned).
  build_bsr                   torch ``to_sparse_bsr`` (library) on the masked
                              matrix; hand-derived worked example.
  decompress                  equals X * kron(mask, ones) (numpy).
  wgrad / wgrad_entries       keep=1 -> numpy X^T @ dY; any keep ->
                              (X*mask)^T @ dY (numpy matmul); linearity.
  wgrad_masked                the same definition with a library matmul as its
                              one step: decompress (the C oracle) then numpy's
                              fp64 (X*mask)^T @ dY.  Used where the quadruple
                              loop is too slow (B24 shards, 59 GFLOP); pinned
                              to wgrad within 1e-12 (tests/test_oracle.py).
  prune_per_sample            SPEC's per-sample examples (golden
                              fixture), brute force per sample, count
                              exactness per sample, numpy segment norms.
  wgrad_rect                  (X*mask)^T @ dY (numpy matmul) for 1 x b.
  affine_wgrad                keep=1 -> numpy sum(X * dY, axis 0); any keep ->
                              sum((X*mask) * dY, axis 0); keep=0 -> 0; a
                              hand-computed 4 x 4 example.
"""
from __future__ import annotations

import ctypes
import itertools
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bsr_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

DT_F32, DT_BF16 = 0, 1

_lib = None


def build(force: bool = False) -> str:
    """Compile bsr_oracle.c with gcc (-O2, no fast-math) into liboracle.so."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        i64, i32, vp, dbl = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_double
        lib.orc_num_blocks.restype = i64
        lib.orc_num_blocks.argtypes = [i64, i64, i64, i64]
        lib.orc_keep_count.restype = i64
        lib.orc_keep_count.argtypes = [i64, dbl]
        lib.orc_storage_bytes.restype = i64
        lib.orc_storage_bytes.argtypes = [i64, i64, i64, i64, i64, i64]
        lib.orc_block_sumsq.restype = i32
        lib.orc_block_sumsq.argtypes = [vp, i32, i64, i64, i64, i64, vp]
        lib.orc_select_topk.restype = i32
        lib.orc_select_topk.argtypes = [vp, i64, i64, vp]
        lib.orc_build_bsr.restype = i32
        lib.orc_build_bsr.argtypes = [vp, i32, i64, i64, i64, i64, vp, vp, vp, vp]
        lib.orc_prune.restype = i32
        lib.orc_prune.argtypes = [vp, i32, i64, i64, i64, i64, vp, vp, vp, vp, vp]
        lib.orc_decompress.restype = i32
        lib.orc_decompress.argtypes = [vp, vp, vp, i32, i64, i64, i64, i64, vp]
        lib.orc_wgrad.restype = i32
        lib.orc_wgrad.argtypes = [vp, vp, vp, i32, i64, i64, i64, i64, vp, i32, i64, vp]
        lib.orc_wgrad_entries.restype = i32
        lib.orc_wgrad_entries.argtypes = [vp, vp, vp, i32, i64, i64, i64, i64, vp, i32, i64,
                                          vp, vp, i64, vp]
        lib.orc_swap_uniform.restype = dbl
        lib.orc_swap_uniform.argtypes = [ctypes.c_uint64, i64]
        lib.orc_select_topk_stochastic.restype = i32
        lib.orc_select_topk_stochastic.argtypes = [vp, i64, i64, i64, dbl, ctypes.c_uint64, vp]
        lib.orc_affine_wgrad.restype = i32
        lib.orc_affine_wgrad.argtypes = [vp, vp, vp, i32, i64, i64, i64, i64, vp, i32, vp]
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _dtype_code(a: np.ndarray) -> int:
    if a.dtype == np.float32:
        return DT_F32
    if a.dtype == np.uint16:  # raw bfloat16 bit patterns
        return DT_BF16
    raise TypeError(f"oracle takes float32 or uint16 (bf16 bits), got {a.dtype}")


def _check(rc: int, what: str):
    if rc != 0:
        raise ValueError(f"oracle {what} failed with code {rc}")


# ---------------------------------------------------------------- bookkeeping
def num_blocks(M: int, K: int, br: int, bc: int | None = None) -> int:
    """N = (M/br)(K/bc); -1 if the blocks do not tile the matrix."""
    return int(_load().orc_num_blocks(M, K, br, br if bc is None else bc))


def keep_count(N: int, keep: float) -> int:
    """Kept blocks k = nearest(keep*N) (reading R3, pinned by Table II)."""
    k = int(_load().orc_keep_count(N, float(keep)))
    if k < 0:
        raise ValueError("keep must be in [0, 1]")
    return k


def storage_bytes(M: int, br: int, bc: int, k: int, value_bytes: int = 4, index_bytes: int = 4) -> int:
    """BSR stored bytes: k*br*bc*vb + k*ib + (M/br+1)*ib (BJ)."""
    return int(_load().orc_storage_bytes(M, br, bc, k, value_bytes, index_bytes))


# ---------------------------------------------------------------- the path
def block_sumsq(X: np.ndarray, br: int, bc: int | None = None) -> np.ndarray:
    """fp64 sum of squares of every block, flat order f = I*(K/bc)+J."""
    bc = br if bc is None else bc
    X = np.ascontiguousarray(X)
    M, K = X.shape
    N = num_blocks(M, K, br, bc)
    if N < 0:
        raise ValueError("blocks do not tile X")
    out = np.empty(N, dtype=np.float64)
    _check(_load().orc_block_sumsq(_ptr(X), _dtype_code(X), M, K, br, bc, _ptr(out)), "block_sumsq")
    return out


def block_norms(X: np.ndarray, br: int, bc: int | None = None) -> np.ndarray:
    return np.sqrt(block_sumsq(X, br, bc))


def select_topk(sumsq: np.ndarray, k: int) -> np.ndarray:
    """uint8 mask of the k KEPT blocks: largest norm first, ties -> lower flat index (BJ)."""
    sumsq = np.ascontiguousarray(sumsq, dtype=np.float64)
    mask = np.empty(sumsq.size, dtype=np.uint8)
    _check(_load().orc_select_topk(_ptr(sumsq), sumsq.size, int(k), _ptr(mask)), "select_topk")
    return mask


def build_bsr(X: np.ndarray, mask: np.ndarray, br: int, bc: int | None = None):
    """(rowptr int32, colidx int32, values [k, br, bc]) of the masked matrix."""
    bc = br if bc is None else bc
    X = np.ascontiguousarray(X)
    M, K = X.shape
    mask = np.ascontiguousarray(mask, dtype=np.uint8)
    k = int(mask.sum())
    rowptr = np.empty(M // br + 1, dtype=np.int32)
    colidx = np.empty(max(k, 0), dtype=np.int32)
    values = np.empty((k, br, bc), dtype=X.dtype)
    _check(_load().orc_build_bsr(_ptr(X), _dtype_code(X), M, K, br, bc, _ptr(mask),
                                 _ptr(rowptr), _ptr(colidx), _ptr(values)), "build_bsr")
    return rowptr, colidx, values


def prune(X: np.ndarray, b: int, k: int):
    """Full forward-side step on b x b blocks with k kept blocks.

    Returns dict(rowptr, colidx, values, sumsq, mask)."""
    X = np.ascontiguousarray(X)
    M, K = X.shape
    N = num_blocks(M, K, b, b)
    if N < 0:
        raise ValueError("b must divide M and K")
    rowptr = np.empty(M // b + 1, dtype=np.int32)
    colidx = np.empty(k, dtype=np.int32)
    values = np.empty((k, b, b), dtype=X.dtype)
    sumsq = np.empty(N, dtype=np.float64)
    mask = np.empty(N, dtype=np.uint8)
    _check(_load().orc_prune(_ptr(X), _dtype_code(X), M, K, b, int(k), _ptr(rowptr), _ptr(colidx),
                             _ptr(values), _ptr(sumsq), _ptr(mask)), "prune")
    return dict(rowptr=rowptr, colidx=colidx, values=values, sumsq=sumsq, mask=mask)


def decompress(rowptr, colidx, values, M: int, K: int, br: int, bc: int | None = None) -> np.ndarray:
    bc = br if bc is None else bc
    values = np.ascontiguousarray(values)
    out = np.empty((M, K), dtype=values.dtype)
    _check(_load().orc_decompress(_ptr(np.ascontiguousarray(rowptr, np.int32)),
                                  _ptr(np.ascontiguousarray(colidx, np.int32)), _ptr(values),
                                  _dtype_code(values), M, K, br, bc, _ptr(out)), "decompress")
    return out


def wgrad(rowptr, colidx, values, M: int, K: int, b: int, dY: np.ndarray) -> np.ndarray:
    """fp64 dW = X_bsr^T . dY, K x Nout (BJ)."""
    values = np.ascontiguousarray(values)
    dY = np.ascontiguousarray(dY)
    Nout = dY.shape[1]
    assert dY.shape[0] == M
    dW = np.empty((K, Nout), dtype=np.float64)
    _check(_load().orc_wgrad(_ptr(np.ascontiguousarray(rowptr, np.int32)),
                             _ptr(np.ascontiguousarray(colidx, np.int32)), _ptr(values),
                             _dtype_code(values), M, K, b, b, _ptr(dY), _dtype_code(dY), Nout,
                             _ptr(dW)), "wgrad")
    return dW


def wgrad_entries(rowptr, colidx, values, M: int, K: int, b: int, dY: np.ndarray,
                  rows: np.ndarray, cols: np.ndarray) -> np.ndarray:
    """dW[rows[t], cols[t]] each computed on its own (full-size sampled parity)."""
    values = np.ascontiguousarray(values)
    dY = np.ascontiguousarray(dY)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    cols = np.ascontiguousarray(cols, dtype=np.int64)
    out = np.empty(rows.size, dtype=np.float64)
    _check(_load().orc_wgrad_entries(_ptr(np.ascontiguousarray(rowptr, np.int32)),
                                     _ptr(np.ascontiguousarray(colidx, np.int32)), _ptr(values),
                                     _dtype_code(values), M, K, b, b, _ptr(dY), _dtype_code(dY),
                                     dY.shape[1], _ptr(rows), _ptr(cols), rows.size, _ptr(out)),
           "wgrad_entries")
    return out


def _as_f64(a: np.ndarray) -> np.ndarray:
    """fp32 values, or bf16 stored as uint16 bit patterns (exact 16-bit shift)."""
    if a.dtype == np.uint16 or a.dtype == np.int16:
        return (a.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    return a.astype(np.float64)


def wgrad_masked(rowptr, colidx, values, M: int, K: int, b: int, dY: np.ndarray) -> np.ndarray:
    """fp64 dW = (X*mask)^T . dY (BJ): the dense masked X rebuilt by
    the C oracle's decompress (O6), then ONE library matmul in fp64.  Same
    definition as `wgrad`, summed by BLAS instead of the quadruple loop."""
    Xm = _as_f64(decompress(rowptr, colidx, values, M, K, b))
    return Xm.T @ _as_f64(np.ascontiguousarray(dY))


def affine_wgrad(rowptr, colidx, values, M: int, K: int, b: int, dY: np.ndarray) -> np.ndarray:
    """fp64 scale gradient of the block-sparse affine layer:
    dalpha[c] = sum over kept blocks of x * dY in column c (dY is M x K)."""
    values = np.ascontiguousarray(values)
    dY = np.ascontiguousarray(dY)
    assert dY.shape == (M, K)
    out = np.empty(K, dtype=np.float64)
    _check(_load().orc_affine_wgrad(_ptr(np.ascontiguousarray(rowptr, np.int32)),
                                    _ptr(np.ascontiguousarray(colidx, np.int32)), _ptr(values),
                                    _dtype_code(values), M, K, b, b, _ptr(dY), _dtype_code(dY), _ptr(out)),
           "affine_wgrad")
    return out


def swap_uniform(seed: int, i: int) -> float:
    """The counter-based uniform u_i of the stochastic boundary swap (reading R19)."""
    return float(_load().orc_swap_uniform(seed, i))


def prune_stochastic(X: np.ndarray, b: int, k: int, window: int, p: float, seed: int):
    """Top-k with stochastic boundary swapping (reading R19): pair i of
    the w' = min(window, k, N-k) pairs (rank k-1-i, rank k+i) swaps kept/pruned iff
    swap_uniform(seed, i) < p.  Returns dict(rowptr, colidx, values, mask)."""
    X = np.ascontiguousarray(X)
    M, K = X.shape
    sumsq = block_sumsq(X, b)
    N = sumsq.size
    mask = np.empty(N, dtype=np.uint8)
    _check(_load().orc_select_topk_stochastic(_ptr(np.ascontiguousarray(sumsq)), N, k, window, float(p), seed,
                                             _ptr(mask)), "select_topk_stochastic")
    rowptr, colidx, values = build_bsr(X, mask, b)
    return {"rowptr": rowptr, "colidx": colidx, "values": values, "mask": mask}


def wgrad_rect(rowptr, colidx, values, M: int, K: int, br: int, bc: int, dY: np.ndarray) -> np.ndarray:
    """fp64 dW = X_bsr^T . dY for br x bc blocks (1 x b row segments for the
    per-sample variant)."""
    values = np.ascontiguousarray(values)
    dY = np.ascontiguousarray(dY)
    Nout = dY.shape[1]
    assert dY.shape[0] == M
    dW = np.empty((K, Nout), dtype=np.float64)
    _check(_load().orc_wgrad(_ptr(np.ascontiguousarray(rowptr, np.int32)),
                             _ptr(np.ascontiguousarray(colidx, np.int32)), _ptr(values),
                             _dtype_code(values), M, K, br, bc, _ptr(dY), _dtype_code(dY), Nout,
                             _ptr(dW)), "wgrad")
    return dW


def prune_per_sample(X: np.ndarray, b: int, k: int, sample_rows: int):
    """The paper-faithful variant: 1 x b row-segment blocks
    (Table II geometry) compared only within one sample --
    "Blocks are only compared locally, not among other activations in the
    mini-batch", every sample keeping the same number of blocks.
    Each run of `sample_rows` rows keeps exactly its k largest-norm segments
    (ties -> lower flat index, BJ); one BSR (br = 1, bc = b) over all rows.

    Returns dict(rowptr, colidx, values, mask)."""
    X = np.ascontiguousarray(X)
    M, K = X.shape
    if M % sample_rows or K % b:
        raise ValueError("sample_rows must divide M and b must divide K")
    masks = [select_topk(block_sumsq(X[s0:s0 + sample_rows], 1, b), k) for s0 in range(0, M, sample_rows)]
    mask = np.concatenate(masks) if masks else np.zeros(0, np.uint8)
    rowptr, colidx, values = build_bsr(X, mask, 1, b)
    return dict(rowptr=rowptr, colidx=colidx, values=values, mask=mask)


# ---------------------------------------------------------------- pins / grading
def brute_force_topk(sumsq, k: int) -> np.ndarray:
    """O9: enumerate every k-subset, keep the one with the largest total squared
    norm ("maximal retained energy"); among equal totals, the
    lexicographically smallest sorted index tuple (BJ tie rule, lower index
    kept).  Exponential -- tiny N only."""
    N = len(sumsq)
    best, best_set = None, None
    for subset in itertools.combinations(range(N), k):  # lexicographic order
        total = sum(float(sumsq[i]) for i in subset)
        if best is None or total > best:
            best, best_set = total, subset
    mask = np.zeros(N, dtype=np.uint8)
    if best_set:
        mask[list(best_set)] = 1
    return mask


def rel_frobenius(A, B) -> float:
    """O10: ||A - B||_F / ||B||_F in fp64 (B = oracle); 0 iff equal when B == 0."""
    A = np.asarray(A, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    nb = float(np.sqrt(np.sum(B * B)))
    nd = float(np.sqrt(np.sum((A - B) ** 2)))
    if nb == 0.0:
        return 0.0 if nd == 0.0 else float("inf")
    return nd / nb
