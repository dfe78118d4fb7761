"""GPU parity of bsr_prune / bsr_block_sumsq / bsr_decompress against the oracle.

Bit-exact: the kept set, rowptr, colidx and values (raw bits) -- BJ.  Inputs
carry a >= 1e-5 relative norm gap at the k-th boundary (helpers.enforce_gap)
except in the exact-integer tie tests, where fp32 sums of squares are exact
and the tie rule itself is checked.
"""
import numpy as np
import pytest

import oracle
import synth
from helpers import bits, enforce_gap, gap_ok, to_torch

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2311_16883_b200 as bp  # noqa: E402


def run_and_compare(Xn: np.ndarray, b: int, k: int, bf16: bool = False):
    """Xn: float32 matrix or uint16 bf16 bit patterns."""
    M, K = Xn.shape
    ref = oracle.prune(Xn, b, k)
    X = to_torch(Xn, bf16=bf16)
    out = bp.prune(X, b, k=k)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out.rowptr.cpu().numpy(), ref["rowptr"])
    np.testing.assert_array_equal(out.colidx.cpu().numpy(), ref["colidx"])
    got_vals = bits(out.values)
    ref_vals = ref["values"].view(np.int32 if not bf16 else np.int16)
    np.testing.assert_array_equal(got_vals, ref_vals)
    assert out.nnzb == k
    return out, ref


SHAPES = [(37, 13), (8, 5), (1, 1), (64, 3), (5, 40)]  # (block rows, block cols): tiles + ragged tails


@pytest.mark.parametrize("b", [4, 8, 16, 32, 64])
@pytest.mark.parametrize("keep", [0.1, 0.5, 0.9])
@pytest.mark.parametrize("shape", SHAPES)
def test_prune_f32_random(b, keep, shape):
    M, K = shape[0] * b, shape[1] * b
    N = shape[0] * shape[1]
    k = oracle.keep_count(N, keep)
    X, _ = enforce_gap(synth.f_aff(M, K, seed=1000 + b + shape[0]), b, k)
    assert gap_ok(X, b, k)
    run_and_compare(X, b, k)


@pytest.mark.parametrize("b", [4, 8, 16, 32, 64])
@pytest.mark.parametrize("keep", [0.3, 0.7])
def test_prune_bf16_random(b, keep):
    M, K = 23 * b, 12 * b  # bf16 rows must be a multiple of 16 bytes
    k = oracle.keep_count(23 * 12, keep)
    X = synth.f_gelu(M, K, seed=2000 + b)
    # gap enforced on the bf16-rounded values, then re-checked after rounding
    for _ in range(5):
        Xh = synth.to_bf16_bits(X)
        Xf = synth.bf16_bits_to_f32(Xh)
        if gap_ok(Xf, b, k, rel=1e-5):
            break
        X, _ = enforce_gap(Xf, b, k, rel=1e-2)
    assert gap_ok(synth.bf16_bits_to_f32(Xh), b, k)
    run_and_compare(Xh, b, k, bf16=True)


@pytest.mark.parametrize("b", [4, 16, 32, 64])
def test_prune_keep_0_and_1(b):
    M, K = 9 * b, 7 * b
    X = synth.f_unif(M, K, seed=3000 + b)
    run_and_compare(X, b, 0)
    run_and_compare(X, b, 63)  # k = N: every block, single copy pass


@pytest.mark.parametrize("b", [4, 8, 16, 32, 64])
def test_prune_every_k_small(b):
    """Every k in [0, N] on a small integer-valued matrix (exact fp32 keys, many ties)."""
    M, K = 3 * b, 4 * b
    X = synth.ints(M, K, seed=4000 + b, lo=-1, hi=1)
    for k in range(0, 13):
        run_and_compare(X, b, k)


@pytest.mark.parametrize("b", [4, 16, 64])
def test_prune_all_equal_ties(b):
    """All blocks tie: the first k in flat order are kept (BJ tie rule)."""
    M, K = 20 * b, 9 * b
    X = np.ones((M, K), np.float32)
    for k in (1, 17, 90, 179):
        out, _ = run_and_compare(X, b, k)
    Z = np.zeros((M, K), np.float32)  # all-zero blocks: kept zero blocks are stored
    run_and_compare(Z, b, 33)


@pytest.mark.parametrize("b", [8, 32])
def test_prune_two_level_ties(b):
    """Integer input with two tie levels straddling the boundary."""
    nbr, nbc = 30, 10
    lev = np.random.default_rng(b).choice([1.0, 2.0, 3.0], size=(nbr, nbc)).astype(np.float32)
    X = np.kron(lev, np.ones((b, b), np.float32))
    for k in (50, 100, 150, 299):
        run_and_compare(X, b, k)


def test_prune_kronecker_lift_worked_example():
    """The hand-derived 4x4 example lifted to b' = 4, 16, 64 (tests/golden)."""
    X = np.array([[3, 4, 0, 0], [0, 0, 1, 0], [0, 0, 2, 2], [0, 1, 2, 2]], np.float32)
    for m in (2, 8, 32):
        XL = np.kron(X, np.ones((m, m), np.float32))
        out, _ = run_and_compare(XL, 2 * m, 3)
        assert list(out.rowptr.cpu().numpy()) == [0, 2, 3]
        assert list(out.colidx.cpu().numpy()) == [0, 1, 1]


def test_prune_scale_invariance():
    """P9: X * 2^e gives the same kept set (sumsq scales exactly by 4^e)."""
    b = 16
    X = synth.ints(16 * b, 8 * b, seed=5, lo=-2, hi=2)
    base = bp.prune(to_torch(X), b, k=40)
    for e in (-3, 5):
        o = bp.prune(to_torch(X * np.float32(2.0 ** e)), b, k=40)
        torch.cuda.synchronize()
        assert torch.equal(o.rowptr, base.rowptr) and torch.equal(o.colidx, base.colidx)


@pytest.mark.parametrize("name", ["C1", "C2", "C3_fc2"])
def test_prune_baseline_configs(name):
    """BASELINE.json configs at full size, bit-exact against the oracle."""
    c = synth.CONFIGS[name]
    N = oracle.num_blocks(c["M"], c["K"], c["b"])
    k = oracle.keep_count(N, c["keep"])
    X, _ = enforce_gap(synth.activation(c["family"], c["M"], c["K"], synth.seed_for(c["id"])), c["b"], k)
    out, _ = run_and_compare(X, c["b"], k)
    assert out.nbytes() == oracle.storage_bytes(c["M"], c["b"], c["b"], k)


@pytest.mark.parametrize("b", [4, 8, 16, 32, 64])
@pytest.mark.parametrize("keep", [0.1, 0.5, 1.0])
def test_prune_s12_sweep_shapes(b, keep):
    """C3 sweep shapes (S12 fc1, batch 128) at every block size."""
    M, K = 25088, 384
    k = oracle.keep_count(oracle.num_blocks(M, K, b), keep)
    X, _ = enforce_gap(synth.f_aff(M, K, seed=synth.seed_for(3, b)), b, k)
    run_and_compare(X, b, k)


@pytest.mark.parametrize("b", [4, 8, 16, 32, 64])
def test_block_sumsq_hook(b):
    """a1 alone: fp32 sums of squares vs the fp64 oracle (relative error
    <= (b + 8) * 2^-24, the sequential-plus-tree bound), exact on integers."""
    M, K = 19 * b, 9 * b
    X = synth.f_aff(M, K, seed=6000 + b)
    got = bp.block_sumsq(to_torch(X), b).cpu().numpy().astype(np.float64)
    ref = oracle.block_sumsq(X, b)
    assert np.all(np.abs(got - ref) <= (b + 8) * 2.0 ** -24 * ref)
    Xi = synth.ints(M, K, seed=6100 + b, lo=-3, hi=3)
    np.testing.assert_array_equal(bp.block_sumsq(to_torch(Xi), b).cpu().numpy(), oracle.block_sumsq(Xi, b))


@pytest.mark.parametrize("b", [4, 8, 16, 32, 64])
@pytest.mark.parametrize("bf16", [False, True])
def test_decompress_roundtrip(b, bf16):
    """a5: decompress(prune(X)) == oracle decompress, bit for bit."""
    M, K = 21 * b, 12 * b
    X = synth.f_aff(M, K, seed=7000 + b)
    Xn = synth.to_bf16_bits(X) if bf16 else X
    k = oracle.keep_count(21 * 12, 0.4)
    ref = oracle.prune(Xn, b, k)
    A = bp.prune(to_torch(Xn, bf16=bf16), b, k=k)
    D = bp.decompress(A)
    torch.cuda.synchronize()
    ref_dense = oracle.decompress(ref["rowptr"], ref["colidx"], ref["values"], M, K, b)
    np.testing.assert_array_equal(bits(D), ref_dense.view(np.int16 if bf16 else np.int32))


def test_decompress_empty():
    b = 16
    X = synth.f_unif(4 * b, 4 * b, seed=1)
    A = bp.prune(to_torch(X), b, k=0)
    D = bp.decompress(A)
    torch.cuda.synchronize()
    assert not bits(D).any()  # +0.0 everywhere


def test_prune_is_deterministic_and_stream_ordered():
    b = 32
    X = to_torch(synth.f_aff(100 * b, 12 * b, seed=9))
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        a = bp.prune(X, b, keep=0.5)
        c = bp.prune(X, b, keep=0.5)
    s.synchronize()
    assert torch.equal(a.colidx, c.colidx) and torch.equal(a.values, c.values)
