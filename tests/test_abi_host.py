"""The C-ABI library on the host (no GPU): it loads, exports every symbol that
include/bsrprune.h declares, its pure helpers agree with the oracle, and every
validation error is reported before any CUDA call."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
from paper_2311_16883_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2311_16883_b200.build import build
    build()
    return _lib.load()


def declared_symbols():
    names = []
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if fn.endswith(".h"):
            src = open(os.path.join(ROOT, "include", fn)).read()
            names += re.findall(r"BSR_API\s+[\w\s\*]+?\b(bsr_\w+)\s*\(", src)
    return sorted(set(names))


def test_exports_every_declared_symbol(lib):
    names = declared_symbols()
    assert len(names) >= 13
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(names) == sorted(_lib.EXPORTED)
    assert lib.bsr_version().decode().startswith("bsrprune")


def test_library_is_sm100a():
    so = os.path.join(ROOT, "paper_2311_16883_b200", "libbsrprune.so")
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {so} 2>&1").read()
    assert "sm_100a" in out, out


@pytest.mark.parametrize("M,K,b", [(256, 256, 16), (25088, 384, 32), (64, 48, 4), (196, 384, 32), (0, 4, 4)])
def test_num_blocks_matches_oracle(lib, M, K, b):
    assert lib.bsr_num_blocks(M, K, b) == oracle.num_blocks(M, K, b, b)


@pytest.mark.parametrize("N", [0, 1, 7, 256, 9408, 37632])
@pytest.mark.parametrize("keep", [0.0, 0.1, 0.25, 0.5, 0.7, 0.9, 1.0])
def test_keep_count_matches_oracle(lib, N, keep):
    assert lib.bsr_keep_count(N, keep) == oracle.keep_count(N, keep)


def test_keep_count_rejects_bad_keep(lib):
    assert lib.bsr_keep_count(10, float("nan")) == -1
    assert lib.bsr_keep_count(10, -0.1) == -1
    assert lib.bsr_keep_count(10, 1.01) == -1


@pytest.mark.parametrize("M,b,k", [(256, 16, 128), (25088, 32, 4704), (64, 4, 0), (128, 64, 2)])
def test_storage_bytes_matches_oracle(lib, M, b, k):
    assert lib.bsr_storage_bytes(M, b, k, _lib.DT_F32) == oracle.storage_bytes(M, b, b, k, 4, 4)
    assert lib.bsr_storage_bytes(M, b, k, _lib.DT_BF16) == oracle.storage_bytes(M, b, b, k, 2, 4)


def test_workspace_query(lib):
    assert lib.bsr_prune_workspace_bytes(256, 256, 16) >= 2 * 256 * 4
    assert lib.bsr_prune_workspace_bytes(100, 256, 16) == 0
    # FP32 grade at b = 16: the FFMA kernel's split partials (2 x K x N) or the dense
    # rebuild's masked X + 32 x 32 values + indices + tensor-core partials, whichever is larger
    need = lib.bsr_wgrad_workspace_bytes(256, 256, 16, 256, 0)
    assert need >= 2 * 256 * 256 * 4 and need >= 2 * 256 * 256 * 4 + 4 * (256 // 32 + 1)
    # N = 200 (not a multiple of 128): FFMA only; one block row: no split
    assert lib.bsr_wgrad_workspace_bytes(16, 256, 16, 200, 0) == 0
    assert lib.bsr_wgrad_workspace_bytes(256, 256, 16, 200, 0) == 2 * 256 * 200 * 4


# ------------------------------------------------------------ validation errors
FAKE = 0x10000  # 16-byte aligned fake device address: never dereferenced (validation fails first)


def prune_status(lib, X=FAKE, M=256, K=256, b=16, keep=0.5, dtype=0, rowptr=FAKE + 0x100000,
                 colidx=FAKE + 0x200000, values=FAKE + 0x300000, ws=FAKE + 0x800000, ws_bytes=1 << 20):
    out = _lib.BsrT(0, 0, 0, 0, 0, rowptr, colidx, values)
    st = lib.bsr_prune(X, M, K, b, keep, dtype, ctypes.byref(out), ws, ws_bytes, None)
    return st, out, lib.bsr_last_error().decode()


@pytest.mark.parametrize("kw,status", [
    (dict(b=5), 3), (dict(b=128), 3), (dict(M=250), 2), (dict(K=200, b=16), 2), (dict(M=0), 2),
    (dict(keep=float("nan")), 1), (dict(keep=1.5), 1), (dict(keep=-0.01), 1), (dict(X=0), 1),
    (dict(rowptr=0), 1), (dict(values=0), 1), (dict(colidx=0), 1), (dict(dtype=7), 1),
    (dict(X=FAKE + 4), 4), (dict(values=FAKE + 0x300008), 4), (dict(ws_bytes=16), 5), (dict(ws=0), 5),
    (dict(X=FAKE + 0x300000, values=FAKE + 0x300000), 1),
    (dict(M=2 ** 40, K=2 ** 20, b=4), 2),
])
def test_prune_validation(lib, kw, status):
    st, out, msg = prune_status(lib, **kw)
    assert st == status, (st, msg)
    assert msg  # a human-readable reason
    assert out.nnzb == 0 and out.M == 0  # descriptor untouched


def test_prune_k_validation(lib):
    out = _lib.BsrT(0, 0, 0, 0, 0, FAKE, FAKE, FAKE)
    assert lib.bsr_prune_k(FAKE, 256, 256, 16, 257, 0, ctypes.byref(out), FAKE, 1 << 20, None) == 1
    assert lib.bsr_prune_k(FAKE, 256, 256, 16, -1, 0, ctypes.byref(out), FAKE, 1 << 20, None) == 1
    assert lib.bsr_prune_k(FAKE, 256, 256, 16, 5, 0, None, FAKE, 1 << 20, None) == 1


def test_decompress_and_wgrad_validation(lib):
    good = _lib.BsrT(256, 256, 16, 0, 10, FAKE, FAKE, FAKE)
    assert lib.bsr_decompress(None, FAKE, None) == 1
    assert lib.bsr_decompress(ctypes.byref(good), 0, None) == 1
    assert lib.bsr_decompress(ctypes.byref(good), FAKE + 8, None) == 4
    bad_b = _lib.BsrT(256, 256, 12, 0, 10, FAKE, FAKE, FAKE)
    assert lib.bsr_decompress(ctypes.byref(bad_b), FAKE, None) == 3
    too_many = _lib.BsrT(256, 256, 16, 0, 257, FAKE, FAKE, FAKE)
    assert lib.bsr_decompress(ctypes.byref(too_many), FAKE, None) == 1
    W = FAKE + 0x1000000
    assert lib.bsr_wgrad(ctypes.byref(good), FAKE, 0, 0, W, 0, 0, None, 0, None) == 2       # N = 0
    assert lib.bsr_wgrad(ctypes.byref(good), FAKE, 0, 6, W, 0, 0, None, 0, None) == 4       # pitch 24 B
    assert lib.bsr_wgrad(ctypes.byref(good), FAKE, 0, 256, W, 2, 0, None, 0, None) == 1     # accumulate
    assert lib.bsr_wgrad(ctypes.byref(good), FAKE, 0, 256, W, 0, 9, None, 0, None) == 1     # prec
    assert lib.bsr_wgrad(ctypes.byref(good), FAKE, 1, 256, W, 0, 2, None, 0, None) == 3     # bf16 TC + f32 X
    assert lib.bsr_wgrad(ctypes.byref(good), 0, 0, 256, W, 0, 0, None, 0, None) == 1
    assert lib.bsr_wgrad(ctypes.byref(good), FAKE, 0, 256, FAKE, 0, 0, None, 0, None) == 1  # dW overlaps dY


def test_status_strings(lib):
    for code, name in _lib.STATUS_NAMES.items():
        assert lib.bsr_status_string(code).decode() == name


def test_variant_calls_validation(lib):
    """Argument checks of the §8f variants' entry points (host-side, before any launch)."""
    WS, BIG = FAKE + 0x800000, 1 << 30
    H = FAKE + 0x2000000
    # global selection (f4)
    assert lib.bsr_select_hist(FAKE, 256, 256, 16, 0, 3, 0, H, WS, BIG, None) == 1          # level
    assert lib.bsr_select_hist(FAKE, 256, 256, 16, 0, 0, 0, None, WS, BIG, None) == 1       # hist
    assert lib.bsr_select_hist(FAKE, 256, 256, 5, 0, 0, 0, H, WS, BIG, None) == 3           # b
    assert lib.bsr_select_hist(FAKE, 256, 256, 16, 0, 0, 0, H, WS, 16, None) == 5           # workspace
    assert lib.bsr_select_counts(256, 256, 16, 0, 5, H, WS, BIG, None) == 1                 # shift
    out = _lib.BsrT(0, 0, 0, 0, 0, FAKE + 0x100000, FAKE + 0x200000, FAKE + 0x300000)
    assert lib.bsr_prune_threshold(FAKE, 256, 256, 16, 0, 0, 0, 11, 10, ctypes.byref(out), WS, BIG, None) == 1
    assert lib.bsr_prune_threshold(FAKE, 256, 256, 16, 0, 0, 0, 0, 257, ctypes.byref(out), WS, BIG, None) == 1
    # 1 x b per-sample variant (f2)
    assert lib.bsr_rows_keep_per_sample(196, 384, 16, 0.5) == 2352
    assert lib.bsr_rows_keep_per_sample(196, 383, 16, 0.5) == -1
    assert lib.bsr_prune_rows_workspace_bytes(392, 384, 16) == 392 * 24 * 4
    assert lib.bsr_prune_rows(FAKE, 392, 384, 16, 100, 0.5, 0, FAKE, FAKE, FAKE, WS, BIG, None) == 2  # sample_rows
    assert lib.bsr_prune_rows(FAKE, 392, 384, 16, 196, 1.5, 0, FAKE, FAKE, FAKE, WS, BIG, None) == 1  # keep
    assert lib.bsr_prune_rows(FAKE, 392, 12, 4, 196, 0.5, 1, FAKE, FAKE, FAKE, WS, BIG, None) == 4    # bf16 pitch 24 B
    assert lib.bsr_prune_rows(FAKE, 392, 384, 16, 196, 0.5, 0, FAKE, FAKE, FAKE, WS, 8, None) == 5    # workspace
    assert lib.bsr_wgrad_rows(FAKE, FAKE, FAKE, 10, 392, 384, 16, 0, FAKE, 0, 6, FAKE, 0, None, 0, None) == 4  # N pitch
    assert lib.bsr_wgrad_rows(FAKE, FAKE, FAKE, 10, 392, 384, 16, 0, FAKE, 0, 256, FAKE, 2, None, 0, None) == 1
    # producer fusion (f3)
    assert lib.bsr_act_block_sumsq(FAKE, FAKE, 256, 256, 16, 0, 2, WS, BIG, None) == 1       # act
    assert lib.bsr_act_block_sumsq(FAKE, FAKE + 8, 256, 256, 16, 0, 1, WS, BIG, None) == 4   # alignment
    assert lib.bsr_act_block_sumsq(FAKE, FAKE, 256, 256, 16, 0, 1, WS, 8, None) == 5         # workspace
    assert lib.bsr_prune_presummed(FAKE, 256, 256, 16, 10, 0, ctypes.byref(out), None, 0, None) == 5


def test_wgrad_algo_set_pdl_and_affine_validation(lib):
    """bsr_wgrad_algo (explicit kernel family), bsr_set_pdl and the block-sparse
    affine layer's entry point: host-side checks before any launch."""
    good = _lib.BsrT(256, 256, 16, 0, 10, FAKE, FAKE, FAKE)
    W, WS, BIG = FAKE + 0x1000000, FAKE + 0x800000, 1 << 30
    assert lib.bsr_wgrad_algo(ctypes.byref(good), FAKE, 0, 256, W, 0, 0, 7, WS, BIG, None) == 1    # algo
    assert lib.bsr_wgrad_algo(ctypes.byref(good), FAKE, 0, 256, W, 0, 1, 3, WS, BIG, None) == 3    # tf32 on FFMA
    assert lib.bsr_wgrad_algo(ctypes.byref(good), FAKE, 0, 256, W, 0, 0, 2, WS, BIG, None) == 3    # fp32 on span
    assert lib.bsr_wgrad_algo(ctypes.byref(good), FAKE, 0, 256, W, 0, 0, 1, WS, BIG, None) == 3    # fp32 runs b=16
    assert lib.bsr_wgrad_algo(ctypes.byref(good), FAKE, 0, 256, W, 0, 1, 1, WS, BIG, None) == 3    # tf32 runs b=16
    b32 = _lib.BsrT(25088, 384, 32, 0, 4704, FAKE, FAKE, FAKE)
    need = lib.bsr_wgrad_workspace_bytes(25088, 384, 32, 1536, 0)
    assert need >= 17 * 384 * 1536 * 4  # FP32 grade: the chain cap sets >= 17 splits at C2
    W2, WS2 = FAKE + (1 << 30), FAKE + (1 << 31)  # clear of dY (154 MB)
    assert lib.bsr_wgrad_algo(ctypes.byref(b32), FAKE, 0, 1536, W2, 0, 0, 1, WS2, need - 16, None) == 5  # workspace
    old = lib.bsr_set_pdl(0)
    assert lib.bsr_set_pdl(old) == 0
    assert lib.bsr_affine_wgrad_workspace_bytes(256, 256, 16) > 0
    assert lib.bsr_affine_wgrad_workspace_bytes(256, 256, 12) == 0
    assert lib.bsr_affine_wgrad(None, FAKE, 0, W, 0, WS, BIG, None) == 1
    assert lib.bsr_affine_wgrad(ctypes.byref(good), FAKE, 5, W, 0, WS, BIG, None) == 1             # dy dtype
    assert lib.bsr_affine_wgrad(ctypes.byref(good), FAKE, 0, W, 3, WS, BIG, None) == 1             # accumulate
    assert lib.bsr_affine_wgrad(ctypes.byref(good), FAKE + 4, 0, W, 0, WS, BIG, None) == 4         # alignment
    assert lib.bsr_affine_wgrad(ctypes.byref(good), FAKE, 0, W, 0, WS, 16, None) == 5             # workspace


def test_wgrad_multicast_validation(lib):
    good = _lib.BsrT(256, 256, 16, 0, 10, FAKE, FAKE, FAKE)
    MC, WS, BIG = FAKE + 0x1000000, FAKE + 0x800000, 1 << 30
    assert lib.bsr_wgrad_multicast(ctypes.byref(good), FAKE, 0, 256, None, 0, 0, WS, BIG, None) == 1       # mc
    assert lib.bsr_wgrad_multicast(ctypes.byref(good), FAKE, 0, 256, MC, 0, 2, WS, BIG, None) == 3         # span
    assert lib.bsr_wgrad_multicast(ctypes.byref(good), FAKE, 0, 256, MC, 1, 0, WS, BIG, None) == 3         # tf32 b=16
    assert lib.bsr_wgrad_multicast(ctypes.byref(good), FAKE, 0, 256, MC, 2, 0, WS, BIG, None) == 3         # bf16 + f32 X
    assert lib.bsr_wgrad_multicast(ctypes.byref(good), FAKE + 4, 0, 256, MC, 0, 0, WS, BIG, None) == 4     # align
