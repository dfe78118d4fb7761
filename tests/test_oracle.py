"""Pins of the CPU oracle against things other than itself.

No GPU.  Each test names the passage or mathematical fact it pins.
"""
import itertools
import os

import numpy as np
import pytest
import torch

import oracle
import synth


# ------------------------------------------------------------------ P1 Table II
def test_table2_all_48_cells(golden):
    """P1: Table II -- every printed cell, to 2 decimals, from the
    oracle's byte accounting with 1 x b blocks and nearest-integer k (R3)."""
    rows = golden("table2_bsr_overhead.txt")
    bs = [int(v) for v in rows[0][1:]]
    R, C = 196, 384
    checked = 0
    for row in rows[1:]:
        s = int(row[0]) / 100.0
        for b, printed in zip(bs, row[1:]):
            N = oracle.num_blocks(R, C, 1, b)
            k = oracle.keep_count(N, 1.0 - s)
            stored = oracle.storage_bytes(R, 1, b, k, 4, 4)
            overhead = 100.0 * (stored / (R * C * 4) - (1.0 - s))
            assert abs(overhead - float(printed)) <= 0.005 + 1e-9, (s, b, overhead, printed)
            checked += 1
    assert checked == 48


@pytest.mark.parametrize("rounding", ["floor", "ceil"])
def test_table2_rejects_other_roundings(golden, rounding):
    """P1 corollary: floor/ceil of keep*N do NOT reproduce Table II, so the
    table really pins nearest rounding (12 / 14 cells fail)."""
    rows = golden("table2_bsr_overhead.txt")
    bs = [int(v) for v in rows[0][1:]]
    R, C = 196, 384
    bad = 0
    for row in rows[1:]:
        s = int(row[0]) / 100.0
        for b, printed in zip(bs, row[1:]):
            N = R * C // b
            x = (1.0 - s) * N
            k = int(np.floor(x + 1e-9)) if rounding == "floor" else int(np.ceil(x - 1e-9))
            ov = 100.0 * ((k * b * 4 + k * 4 + (R + 1) * 4) / (R * C * 4) - (1.0 - s))
            bad += abs(ov - float(printed)) > 0.005 + 1e-9
    assert bad >= 10


# ------------------------------------------------------------------ P2 closed form
def test_storage_bytes_north_star_closed_form():
    """P2: BJ closed form k*b^2*4 + k*4 + (M/b+1)*4 at C1 and C2."""
    N1 = oracle.num_blocks(256, 256, 16)
    k1 = oracle.keep_count(N1, 0.5)
    assert (N1, k1) == (256, 128)
    assert oracle.storage_bytes(256, 16, 16, k1) == 131_652
    N2 = oracle.num_blocks(25088, 384, 32)
    k2 = oracle.keep_count(N2, 0.5)
    assert (N2, k2) == (9408, 4704)
    assert oracle.storage_bytes(25088, 32, 32, k2) == 19_289_540


def test_keep_count_edges():
    assert oracle.keep_count(10, 0.0) == 0
    assert oracle.keep_count(10, 1.0) == 10
    assert oracle.keep_count(7, 0.5) == 4  # 3.5 -> 4 (half up; unpinned by the paper, R3)
    assert oracle.keep_count(0, 0.3) == 0
    with pytest.raises(ValueError):
        oracle.keep_count(10, 1.5)
    with pytest.raises(ValueError):
        oracle.keep_count(10, float("nan"))
    assert oracle.num_blocks(196, 384, 32) == -1  # not tileable (R10)


# ------------------------------------------------------------------ worked examples
def _floats(row):
    return np.array([float(v) for v in row], dtype=np.float32)


def test_worked_example_b2(golden):
    """P8: hand-derived 4x4, b=2 example (tests/golden/worked_example_b2.txt)."""
    rows = {tuple(r[:2]) if r[0].startswith("keep") else (r[0],): r for r in golden("worked_example_b2.txt")}
    X = _floats(rows[("X",)][1:]).reshape(4, 4)
    np.testing.assert_array_equal(oracle.block_sumsq(X, 2), _floats(rows[("sumsq",)][1:]))
    N = oracle.num_blocks(4, 4, 2)
    for tag in ("keep0.5", "keep0.75"):
        keep = float(tag[4:])
        k = oracle.keep_count(N, keep)
        assert k == int(rows[(tag, "k")][2])
        out = oracle.prune(X, 2, k)
        np.testing.assert_array_equal(out["rowptr"], [int(v) for v in rows[(tag, "rowptr")][2:]])
        np.testing.assert_array_equal(out["colidx"], [int(v) for v in rows[(tag, "colidx")][2:]])
        np.testing.assert_array_equal(out["values"].ravel(), _floats(rows[(tag, "values")][2:]))
        assert oracle.storage_bytes(4, 2, 2, k) == int(rows[(tag, "bytes")][2])
    out = oracle.prune(X, 2, 3)
    dW = oracle.wgrad(out["rowptr"], out["colidx"], out["values"], 4, 4, 2, np.ones((4, 1), np.float32))
    np.testing.assert_array_equal(dW.ravel(), _floats(rows[("keep0.75", "dW_onesN1")][2:]))
    full = oracle.prune(X, 2, 4)
    dW = oracle.wgrad(full["rowptr"], full["colidx"], full["values"], 4, 4, 2, np.ones((4, 1), np.float32))
    np.testing.assert_array_equal(dW.ravel(), _floats(rows[("keep1.0", "dW_onesN1")][2:]))


def test_spec_norm_example_b3(golden):
    """Hand-computed 1x3 norms (fig:pruning setup P:L434-441)."""
    rows = {r[0]: r[1:] for r in golden("spec_norm_example_b3.txt")}
    X = _floats(rows["row"]).reshape(1, 12)
    norms = oracle.block_norms(X, 1, 3)
    np.testing.assert_allclose(norms, [float(v) for v in rows["norms"]], rtol=1e-7)
    mask = oracle.select_topk(oracle.block_sumsq(X, 1, 3), oracle.keep_count(4, 0.5))
    assert list(np.nonzero(mask)[0]) == [int(v) for v in rows["kept"]]


def test_kronecker_lift_preserves_selection():
    """P8 lifted: X kron 1_{m x m} with b' = 2m scales norms by m and keeps the
    same blocks, rowptr and colidx (including the tie)."""
    X = np.array([[3, 4, 0, 0], [0, 0, 1, 0], [0, 0, 2, 2], [0, 1, 2, 2]], np.float32)
    base = oracle.prune(X, 2, 3)
    for m in (2, 4, 8):
        XL = np.kron(X, np.ones((m, m), np.float32))
        lifted = oracle.prune(XL, 2 * m, 3)
        np.testing.assert_array_equal(lifted["rowptr"], base["rowptr"])
        np.testing.assert_array_equal(lifted["colidx"], base["colidx"])
        np.testing.assert_allclose(np.sqrt(lifted["sumsq"]), m * np.sqrt(base["sumsq"]))


# ------------------------------------------------------------------ norms
@pytest.mark.parametrize("br,bc", [(1, 4), (2, 2), (4, 4), (3, 5), (16, 16)])
def test_block_sumsq_matches_numpy_norm(br, bc):
    """O2 vs numpy.linalg.norm (Frobenius, library) applied block by block."""
    M, K = br * 5, bc * 3
    X = synth.f_aff(M, K, seed=11)
    got = oracle.block_sumsq(X, br, bc)
    ref = []
    for I in range(M // br):
        for J in range(K // bc):
            ref.append(np.linalg.norm(X[I * br:(I + 1) * br, J * bc:(J + 1) * bc].astype(np.float64), "fro") ** 2)
    np.testing.assert_allclose(got, ref, rtol=1e-13)


def test_block_sumsq_constant_blocks():
    """Closed form: a block filled with c has sumsq = c^2 * b^2."""
    b = 8
    vals = np.array([[0.5, -3.0], [2.0, 0.0]], np.float32)
    X = np.kron(vals, np.ones((b, b), np.float32))
    np.testing.assert_array_equal(oracle.block_sumsq(X, b), (vals.ravel().astype(np.float64) ** 2) * b * b)


def test_block_sumsq_bf16_input():
    X = synth.f_aff(32, 32, seed=5)
    h = synth.to_bf16_bits(X)
    np.testing.assert_array_equal(oracle.block_sumsq(h, 8), oracle.block_sumsq(synth.bf16_bits_to_f32(h), 8))


# ------------------------------------------------------------------ P3 brute force top-k
@pytest.mark.parametrize("seed", range(6))
def test_select_topk_equals_brute_force_random(seed):
    rng = np.random.default_rng(seed)
    N = int(rng.integers(1, 13))
    s = rng.random(N) * 10
    for k in range(N + 1):
        np.testing.assert_array_equal(oracle.select_topk(s, k), oracle.brute_force_topk(s, k))


def test_select_topk_equals_brute_force_ties():
    """P3/P10 with constructed ties: tie rule = lower flat index kept (BJ)."""
    cases = [[1, 1, 1, 1, 1, 1], [2, 1, 2, 1, 2, 1, 0], [0, 0, 0], [5, 3, 3, 3, 5, 1, 3, 3]]
    for s in cases:
        s = np.array(s, np.float64)
        for k in range(len(s) + 1):
            np.testing.assert_array_equal(oracle.select_topk(s, k), oracle.brute_force_topk(s, k))


def test_select_topk_all_equal_keeps_prefix():
    s = np.full(10, 4.0)
    for k in range(11):
        assert list(np.nonzero(oracle.select_topk(s, k))[0]) == list(range(k))


def test_select_invariants_large():
    """P11: |kept| = k; min kept norm >= max pruned norm."""
    X = synth.f_gelu(64 * 8, 64, seed=3)
    ss = oracle.block_sumsq(X, 8)
    for keep in (0.1, 0.3, 0.5, 0.8):
        k = oracle.keep_count(ss.size, keep)
        m = oracle.select_topk(ss, k).astype(bool)
        assert m.sum() == k
        assert ss[m].min() >= ss[~m].max()


# ------------------------------------------------------------------ P4 library BSR
@pytest.mark.parametrize("b,keep", [(4, 0.5), (8, 0.3), (16, 1.0), (2, 0.9)])
def test_build_bsr_matches_torch_to_sparse_bsr(b, keep):
    """P4: torch.Tensor.to_sparse_bsr on the masked matrix (no kept all-zero block)."""
    M, K = b * 6, b * 5
    X = synth.f_aff(M, K, seed=b)
    ss = oracle.block_sumsq(X, b)
    k = oracle.keep_count(ss.size, keep)
    out = oracle.prune(X, b, k)
    mask = out["mask"].reshape(M // b, K // b).astype(np.float32)
    masked = X * np.kron(mask, np.ones((b, b), np.float32))
    t = torch.from_numpy(masked).to_sparse_bsr((b, b))
    np.testing.assert_array_equal(out["rowptr"], t.crow_indices().numpy().astype(np.int32))
    np.testing.assert_array_equal(out["colidx"], t.col_indices().numpy().astype(np.int32))
    np.testing.assert_array_equal(out["values"], t.values().numpy())


def test_bsr_invariants():
    """P11: rowptr[0]=0, non-decreasing, rowptr[-1]=k, colidx strictly increasing per row."""
    X = synth.f_unif(16 * 9, 16 * 7, seed=2)
    N = oracle.num_blocks(*X.shape, 16)
    k = oracle.keep_count(N, 0.4)
    out = oracle.prune(X, 16, k)
    rp, ci = out["rowptr"], out["colidx"]
    assert rp[0] == 0 and rp[-1] == k and np.all(np.diff(rp) >= 0)
    for I in range(len(rp) - 1):
        row = ci[rp[I]:rp[I + 1]]
        assert np.all(np.diff(row) > 0) and np.all((row >= 0) & (row < 7))


def test_kept_zero_block_is_stored():
    """R6: a kept all-zero block is stored (nnzb = k exactly)."""
    X = np.zeros((8, 8), np.float32)
    out = oracle.prune(X, 4, 3)
    assert out["rowptr"][-1] == 3 and list(out["colidx"]) == [0, 1, 0]


# ------------------------------------------------------------------ P5 decompress / dW
@pytest.mark.parametrize("b,keep", [(4, 0.5), (8, 0.25), (16, 0.75)])
def test_decompress_equals_masked_x(b, keep):
    M, K = b * 7, b * 4
    X = synth.f_aff(M, K, seed=b + 100)
    out = oracle.prune(X, b, oracle.keep_count(oracle.num_blocks(M, K, b), keep))
    mask = out["mask"].reshape(M // b, K // b).astype(np.float32)
    ref = np.where(np.kron(mask, np.ones((b, b), np.float32)) > 0, X, np.float32(0))  # +0.0 fill
    got = oracle.decompress(out["rowptr"], out["colidx"], out["values"], M, K, b)
    np.testing.assert_array_equal(got.view(np.uint32), ref.view(np.uint32))


def test_wgrad_keep1_equals_dense_matmul():
    """P5: keep = 1 => dW = X^T dY (numpy fp64 matmul)."""
    M, K, Nout, b = 64, 48, 40, 8
    X = synth.f_aff(M, K, seed=7)
    dY = synth.grad_out(M, Nout, seed=7)
    out = oracle.prune(X, b, oracle.num_blocks(M, K, b))
    dW = oracle.wgrad(out["rowptr"], out["colidx"], out["values"], M, K, b, dY)
    ref = X.astype(np.float64).T @ dY.astype(np.float64)
    np.testing.assert_allclose(dW, ref, rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("keep", [0.0, 0.2, 0.5, 0.9])
def test_wgrad_equals_masked_matmul(keep):
    """P5/P6: dW = (X * mask)^T dY; keep = 0 => exactly zero."""
    M, K, Nout, b = 96, 64, 24, 16
    X = synth.f_gelu(M, K, seed=8)
    dY = synth.grad_out(M, Nout, seed=8)
    out = oracle.prune(X, b, oracle.keep_count(oracle.num_blocks(M, K, b), keep))
    mask = out["mask"].reshape(M // b, K // b).astype(np.float64)
    ref = (X.astype(np.float64) * np.kron(mask, np.ones((b, b)))).T @ dY.astype(np.float64)
    dW = oracle.wgrad(out["rowptr"], out["colidx"], out["values"], M, K, b, dY)
    np.testing.assert_allclose(dW, ref, rtol=1e-12, atol=1e-15)
    if keep == 0.0:
        assert not dW.any()


def test_wgrad_linearity():
    """P7: dW(X, dY1 + dY2) = dW(X, dY1) + dW(X, dY2); sum over row shards = whole."""
    M, K, Nout, b = 64, 32, 16, 8
    X = synth.f_aff(M, K, seed=9)
    d1, d2 = synth.ints(M, Nout, 1, -9, 9), synth.ints(M, Nout, 2, -9, 9)  # exact fp32 sums
    out = oracle.prune(X, b, 20)
    args = (out["rowptr"], out["colidx"], out["values"], M, K, b)
    lhs = oracle.wgrad(*args, d1 + d2)
    rhs = oracle.wgrad(*args, d1) + oracle.wgrad(*args, d2)
    np.testing.assert_allclose(lhs, rhs, rtol=1e-12, atol=1e-12)
    # row shards with the same mask: per-shard BSR = row slices of the whole BSR
    half = M // 2
    nb = half // b
    rp = out["rowptr"]
    top = (rp[:nb + 1], out["colidx"][:rp[nb]], out["values"][:rp[nb]])
    bot = (rp[nb:] - rp[nb], out["colidx"][rp[nb]:], out["values"][rp[nb]:])
    s = oracle.wgrad(*top, half, K, b, d1[:half]) + oracle.wgrad(*bot, half, K, b, d1[half:])
    np.testing.assert_allclose(s, oracle.wgrad(*args, d1), rtol=1e-12, atol=1e-15)


def test_wgrad_entries_match_full():
    M, K, Nout, b = 64, 32, 48, 16
    X = synth.f_aff(M, K, seed=10)
    dY = synth.grad_out(M, Nout, seed=10)
    out = oracle.prune(X, b, 5)
    args = (out["rowptr"], out["colidx"], out["values"], M, K, b, dY)
    full = oracle.wgrad(*args)
    rows, cols = np.array([0, 5, 31, 17, 16]), np.array([0, 47, 3, 20, 1])
    np.testing.assert_allclose(oracle.wgrad_entries(*args, rows, cols), full[rows, cols], rtol=1e-13)


def test_wgrad_bf16_operands():
    M, K, Nout, b = 32, 32, 16, 8
    X = synth.f_aff(M, K, seed=12)
    dY = synth.grad_out(M, Nout, seed=12)
    Xh, dYh = synth.to_bf16_bits(X), synth.to_bf16_bits(dY)
    out = oracle.prune(Xh, b, 10)
    dW = oracle.wgrad(out["rowptr"], out["colidx"], out["values"], M, K, b, dYh)
    Xf, dYf = synth.bf16_bits_to_f32(Xh), synth.bf16_bits_to_f32(dYh)
    mask = out["mask"].reshape(M // b, K // b).astype(np.float64)
    ref = (Xf.astype(np.float64) * np.kron(mask, np.ones((b, b)))).T @ dYf.astype(np.float64)
    np.testing.assert_allclose(dW, ref, rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("bf16", [False, True])
@pytest.mark.parametrize("keep", [0.0, 0.3, 1.0])
def test_wgrad_masked_equals_quadruple_loop(bf16, keep):
    """wgrad_masked (decompress + one BLAS matmul) is the same definition as the
    quadruple loop: equal to ~1e-12 relative on every keep, f32 and bf16 operands."""
    M, K, Nout, b = 128, 96, 40, 16
    X = synth.f_gelu(M, K, seed=13)
    dY = synth.grad_out(M, Nout, seed=13)
    if bf16:
        X, dY = synth.to_bf16_bits(X), synth.to_bf16_bits(dY)
    out = oracle.prune(X, b, oracle.keep_count(oracle.num_blocks(M, K, b), keep))
    args = (out["rowptr"], out["colidx"], out["values"], M, K, b, dY)
    loop = oracle.wgrad(*args)
    np.testing.assert_allclose(oracle.wgrad_masked(*args), loop, rtol=1e-12, atol=1e-15)
    if keep == 0.0:
        assert not oracle.wgrad_masked(*args).any()


@pytest.mark.parametrize("keep", [0.0, 0.4, 1.0])
def test_affine_wgrad_equals_masked_column_dot(keep):
    """Block-sparse affine layer: dalpha = sum over rows of (X*mask) * dY;
    keep = 1 -> the dense affine gradient sum(X * dY, axis 0)."""
    M, K, b = 96, 64, 16
    X = synth.f_aff(M, K, seed=14)
    dY = synth.grad_out(M, K, seed=14)
    out = oracle.prune(X, b, oracle.keep_count(oracle.num_blocks(M, K, b), keep))
    mask = np.kron(out["mask"].reshape(M // b, K // b), np.ones((b, b)))
    ref = (X.astype(np.float64) * mask * dY.astype(np.float64)).sum(axis=0)
    got = oracle.affine_wgrad(out["rowptr"], out["colidx"], out["values"], M, K, b, dY)
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-15)
    if keep == 1.0:
        np.testing.assert_allclose(got, (X.astype(np.float64) * dY).sum(0), rtol=1e-12, atol=1e-15)
    if keep == 0.0:
        assert not got.any()


def test_affine_wgrad_hand_example():
    """The 4 x 4 worked example (b = 2, keep 0.75: kept B00, B01, B11) with dY = 1:
    dalpha = column sums of the masked X = [3, 4+1... ] computed by hand."""
    X = np.array([[3, 4, 0, 0], [0, 0, 1, 0], [0, 0, 2, 2], [0, 1, 2, 2]], np.float32)
    out = oracle.prune(X, 2, 3)
    got = oracle.affine_wgrad(out["rowptr"], out["colidx"], out["values"], 4, 4, 2, np.ones((4, 4), np.float32))
    # masked X = [[3,4,0,0],[0,0,1,0],[0,0,2,2],[0,0,2,2]] (B10 = [[0,0],[0,1]] pruned)
    np.testing.assert_array_equal(got, [3.0, 4.0, 5.0, 4.0])
    dY = np.array([[1, 2, 3, 4]] * 4, np.float32)  # per-column weights
    got = oracle.affine_wgrad(out["rowptr"], out["colidx"], out["values"], 4, 4, 2, dY)
    np.testing.assert_array_equal(got, [3.0, 8.0, 15.0, 16.0])


def test_rel_frobenius():
    B = np.array([[3.0, 4.0]])
    assert oracle.rel_frobenius(B, B) == 0.0
    assert abs(oracle.rel_frobenius(B * 1.01, B) - 0.01) < 1e-12
    assert oracle.rel_frobenius(np.zeros(2), np.zeros(2)) == 0.0


def test_brute_force_itself_on_hand_case():
    """Brute force on a hand case: {5,1,1,4} keep 3 -> {0,1,3} (tie -> index 1)."""
    assert list(np.nonzero(oracle.brute_force_topk([25, 1, 1, 16], 3))[0]) == [0, 1, 3]
    assert list(itertools.compress(range(4), oracle.brute_force_topk([25, 1, 1, 16], 2))) == [0, 3]


# ---------------------------------------------------------------- f2: 1 x b, per-sample scope
def _golden_per_sample():
    rows = {}
    with open(os.path.join(os.path.dirname(__file__), "golden", "spec_per_sample_b3.txt")) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                key, *vals = line.split()
                rows[key] = vals
    return np.array([float(v) for v in rows["X"]], dtype=np.float32)[None, :], [int(v) for v in rows["kept"]]


def test_per_sample_spec_example():
    """segments 1 and 3 pruned, nnzb = 2."""
    X, kept = _golden_per_sample()
    ref = oracle.prune_per_sample(X, 3, oracle.keep_count(4, 0.5), 1)
    assert list(np.nonzero(ref["mask"])[0]) == kept
    assert list(ref["rowptr"]) == [0, 2] and list(ref["colidx"]) == kept
    np.testing.assert_allclose(oracle.block_norms(X, 1, 3), [3.7417, 0.1732, 4.0, 1.7321], atol=1e-4)


def test_per_sample_no_cross_sample_starvation():
    """sample 0 all large, sample 1 all tiny, keep 0.5 -> each keeps half."""
    S, K, b = 4, 12, 3
    X = np.concatenate([np.full((S, K), 10.0, np.float32), np.full((S, K), 1e-3, np.float32)])
    X += np.arange(2 * S * K, dtype=np.float32).reshape(2 * S, K) * 1e-6  # distinct norms
    k = oracle.keep_count(S * K // b, 0.5)
    ref = oracle.prune_per_sample(X, b, k, S)
    per = ref["mask"].reshape(2, -1).sum(axis=1)
    assert list(per) == [k, k]


@pytest.mark.parametrize("seed", range(6))
def test_per_sample_brute_force(seed):
    rng = np.random.default_rng(seed)
    S, nsamp, K, b = 3, 3, 8, 2  # 12 segments per sample
    X = rng.integers(-2, 3, size=(S * nsamp, K)).astype(np.float32)  # exact norms, ties
    keep = [0.0, 0.25, 0.5, 0.75, 1.0, 0.4][seed]
    k = oracle.keep_count(S * K // b, keep)
    ref = oracle.prune_per_sample(X, b, k, S)
    for s in range(nsamp):
        seg = (X[s * S:(s + 1) * S].reshape(S, K // b, b) ** 2).sum(-1).reshape(-1).astype(np.float64)
        want = oracle.brute_force_topk(seg, k)
        np.testing.assert_array_equal(ref["mask"].reshape(nsamp, -1)[s], want)


def test_wgrad_rect_equals_masked_matmul():
    rng = np.random.default_rng(3)
    S, nsamp, K, b, N = 5, 4, 24, 4, 7
    X = rng.standard_normal((S * nsamp, K)).astype(np.float32)
    dY = rng.standard_normal((S * nsamp, N)).astype(np.float32)
    ref = oracle.prune_per_sample(X, b, 9, S)
    dW = oracle.wgrad_rect(ref["rowptr"], ref["colidx"], ref["values"], S * nsamp, K, 1, b, dY)
    Xm = X.astype(np.float64) * np.repeat(ref["mask"].reshape(S * nsamp, K // b), b, axis=1)
    np.testing.assert_allclose(dW, Xm.T @ dY.astype(np.float64), rtol=1e-12, atol=1e-12)


# ------------------------------------------------------------------ P13 stochastic boundary swapping (R19)
def _rank_order(s):
    """Flat indices by (value desc, index asc): numpy lexsort, not the oracle's qsort."""
    s = np.asarray(s, np.float64)
    return np.lexsort((np.arange(s.size), -s))


def test_swap_uniform_is_splitmix64():
    """u_i = (splitmix64 output >> 11) * 2^-53 with the generator's state starting
    at `seed`: the published first outputs of splitmix64 from state 0 are
    0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F."""
    for i, v in enumerate((0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F)):
        assert oracle.swap_uniform(0, i) == (v >> 11) / 2.0 ** 53
    u = np.array([oracle.swap_uniform(12345, i) for i in range(20000)])
    assert u.min() >= 0.0 and u.max() < 1.0
    assert abs(u.mean() - 0.5) < 0.01 and abs(u.var() - 1 / 12) < 0.005


def test_stochastic_p0_is_topk():
    """p = 0: no pair swaps, the selection is the deterministic top-k."""
    rng = np.random.default_rng(5)
    X = synth.ints(16 * 8, 12 * 8, seed=5, lo=-9, hi=9)
    for k, w in ((10, 3), (96, 50), (0, 4), (192, 4), (50, 0)):
        r = oracle.prune_stochastic(X, 8, k, w, 0.0, int(rng.integers(1 << 62)))
        np.testing.assert_array_equal(r["mask"], oracle.prune(X, 8, k)["mask"])


@pytest.mark.parametrize("k,w", [(10, 3), (100, 50), (5, 9), (190, 9), (96, 96)])
def test_stochastic_p1_swaps_whole_window(k, w):
    """p = 1: every pair swaps -- kept = ranks [0, k-w') and [k, k+w'), w' = min(w, k, N-k)."""
    X = synth.ints(16 * 4, 12 * 4, seed=k + w, lo=-3, hi=3)  # ties: the rank order decides
    N = 16 * 12
    s = oracle.block_sumsq(X, 4)
    order = _rank_order(s)
    wp = min(w, k, N - k)
    want = np.zeros(N, np.uint8)
    want[order[: k - wp]] = 1
    want[order[k: k + wp]] = 1
    r = oracle.prune_stochastic(X, 4, k, w, 1.0, 77)
    np.testing.assert_array_equal(r["mask"], want)


def test_stochastic_pairs_and_counts():
    """Any p: exactly k kept; ranks < k - w' always kept, ranks >= k + w' never;
    a kept rank k+i comes with a pruned rank k-1-i (pairs), and the swapped pairs
    are the i with u_i < p."""
    X = synth.ints(40 * 8, 30 * 8, seed=9, lo=-20, hi=20)
    s = oracle.block_sumsq(X, 8)
    N = s.size
    order = _rank_order(s)
    rank = np.empty(N, np.int64)
    rank[order] = np.arange(N)
    for k, w, p, seed in ((600, 200, 0.3, 1), (300, 1000, 0.7, 2), (1100, 100, 0.5, 3)):
        m = oracle.prune_stochastic(X, 8, k, w, p, seed)["mask"].astype(bool)
        wp = min(w, k, N - k)
        assert m.sum() == k
        assert m[rank < k - wp].all() and not m[rank >= k + wp].any()
        for i in range(wp):
            sw = oracle.swap_uniform(seed, i) < p
            assert m[order[k - 1 - i]] == (not sw) and m[order[k + i]] == sw


def test_stochastic_swap_fraction():
    """The swapped fraction of the w' pairs is p within 5 binomial sigmas."""
    X = synth.f_aff(200 * 8, 40 * 8, seed=4)
    k, w = 4000, 3000
    for p in (0.1, 0.5, 0.9):
        m = oracle.prune_stochastic(X, 8, k, w, p, 11)["mask"].astype(bool)
        top = oracle.prune(X, 8, k)["mask"].astype(bool)
        swapped = int((top & ~m).sum())
        assert abs(swapped - p * w) < 5 * np.sqrt(w * p * (1 - p)), (p, swapped)


def test_stochastic_bsr_is_masked_x():
    """The BSR of the stochastic selection decompresses to X masked by it (O5/O6)."""
    X = synth.ints(12 * 4, 9 * 4, seed=2, lo=-5, hi=5)
    r = oracle.prune_stochastic(X, 4, 50, 20, 0.5, 3)
    D = oracle.decompress(r["rowptr"], r["colidx"], r["values"], X.shape[0], X.shape[1], 4)
    m = np.kron(r["mask"].reshape(12, 9), np.ones((4, 4))).astype(bool)
    np.testing.assert_array_equal(D, np.where(m, X, 0))
