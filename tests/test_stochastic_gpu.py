"""GPU parity of bsr_prune_stochastic against the oracle.

Bit-exact: kept set, rowptr, colidx, values.  Inputs are small integers, so the
fp32 block sums of squares (GPU keys) and the oracle's fp64 ones are exact and
rank identically -- the whole boundary's order matters here, not only the k-th
key -- and ties are plentiful (the tie rule inside the boundary is exercised).
"""
import numpy as np
import pytest

import oracle
import synth
from helpers import bits, to_torch

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2311_16883_b200 as bp  # noqa: E402


def compare(Xn, b, k, window, p, seed, bf16=False):
    ref = oracle.prune_stochastic(Xn, b, k, window, p, seed)  # bf16: the oracle reads the bit patterns
    out = bp.prune_stochastic(to_torch(Xn, bf16=bf16), b, k=k, window=window, p=p, seed=seed)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out.rowptr.cpu().numpy(), ref["rowptr"])
    np.testing.assert_array_equal(out.colidx.cpu().numpy(), ref["colidx"])
    np.testing.assert_array_equal(bits(out.values), ref["values"].view(np.int16 if bf16 else np.int32))
    assert out.nnzb == k
    return ref


@pytest.mark.parametrize("b", [4, 8, 16, 32, 64])
@pytest.mark.parametrize("window,p", [(1, 1.0), (7, 0.5), (100, 0.3), (4096, 0.5), (50, 0.0)])
def test_stochastic_f32(b, window, p):
    nbr, nbc = 37, 13  # ragged tails of the warp units / CTAs
    X = synth.ints(nbr * b, nbc * b, seed=b + window, lo=-20, hi=20)
    N = nbr * nbc
    for k in (1, N // 3, N // 2, N - 1):
        compare(X, b, k, window, p, seed=1000 * b + k)


@pytest.mark.parametrize("b", [4, 16, 32])
def test_stochastic_bf16(b):
    nbr, nbc = 24, 16
    X = synth.ints(nbr * b, nbc * b, seed=b, lo=-100, hi=100)
    h = synth.to_bf16_bits(X)
    for k, w, p in ((100, 30, 0.5), (200, 300, 0.8), (5, 5, 1.0)):
        compare(h, b, k, w, p, seed=k, bf16=True)


@pytest.mark.parametrize("b", [8, 32])
def test_stochastic_heavy_ties(b):
    """Thousands of blocks tied on each key value (block_count_ints): the ranks
    inside the boundary are decided by the flat index alone."""
    M, K = 96 * b, 48 * b
    X = synth.block_count_ints(M, K, b, counts=[0, 1, 2, 3], seed=b)
    N = 96 * 48
    for k, w, p in ((N // 2, 1000, 0.5), (N // 4, 4096, 0.9), (N - 10, 4096, 0.5)):
        compare(X, b, k, w, p, seed=w + k)


def test_stochastic_all_equal():
    X = np.ones((64 * 8, 32 * 8), np.float32)
    compare(X, 8, 700, 300, 0.5, seed=3)


def test_stochastic_large_n_multi_cta():
    """N = 150528 keys (S12 fc2 at b = 16: 25088 x 1536): several CTAs per kernel,
    the boundary list at its 8192-entry maximum."""
    b, M, K = 16, 25088, 1536
    X = synth.ints(M, K, seed=7, lo=-6, hi=6)
    N = (M // b) * (K // b)
    compare(X, b, N // 2, 4096, 0.5, seed=99)


def test_stochastic_degenerate():
    """w' = 0 (window 0, k = 0, k = N) is bsr_prune_k; window larger than k or N-k is capped."""
    b = 8
    X = synth.ints(10 * b, 10 * b, seed=1, lo=-9, hi=9)
    for k, w in ((0, 5), (100, 5), (40, 0), (3, 50), (97, 50)):
        compare(X, b, k, w, 1.0, seed=5)


def test_stochastic_seed_changes_selection_and_repeats():
    b = 8
    X = to_torch(synth.ints(32 * b, 32 * b, seed=2, lo=-20, hi=20))
    a1 = bp.prune_stochastic(X, b, k=512, window=200, p=0.5, seed=1)
    a2 = bp.prune_stochastic(X, b, k=512, window=200, p=0.5, seed=1)
    a3 = bp.prune_stochastic(X, b, k=512, window=200, p=0.5, seed=2)
    assert torch.equal(a1.colidx, a2.colidx) and torch.equal(a1.values, a2.values)
    assert not (torch.equal(a1.colidx, a3.colidx) and torch.equal(a1.rowptr, a3.rowptr))


def test_stochastic_rejects():
    X = to_torch(synth.ints(64, 64, seed=1))
    with pytest.raises(bp.BsrError):
        bp.prune_stochastic(X, 8, k=32, window=8, p=1.5)
    with pytest.raises(bp.BsrError):
        bp.prune_stochastic(X, 8, k=32, window=-1, p=0.5)
    Xl = to_torch(np.ones((512, 512 * 4), np.float32))  # N = 16384 at b = 8
    with pytest.raises(bp.BsrError):
        bp.prune_stochastic(Xl, 8, k=8192, window=5000, p=0.5)


def test_stochastic_graph_capture():
    """Stream-ordered with no host sync: capturable, and the replay gives the same BSR."""
    b = 16
    Xn = synth.ints(64 * b, 24 * b, seed=3, lo=-20, hi=20)
    X = to_torch(Xn)
    ref = oracle.prune_stochastic(Xn, b, 700, 300, 0.5, 8)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        out = bp.prune_stochastic(X, b, k=700, window=300, p=0.5, seed=8)  # warm: workspace allocated
        g = torch.cuda.CUDAGraph()
        out.values.zero_()
        with torch.cuda.graph(g, stream=s):
            bp.prune_stochastic(X, b, k=700, window=300, p=0.5, seed=8, out=out)
        out.values.fill_(float("nan"))
        g.replay()
    s.synchronize()
    np.testing.assert_array_equal(out.colidx.cpu().numpy(), ref["colidx"])
    np.testing.assert_array_equal(bits(out.values), ref["values"].view(np.int32))


def test_stochastic_workspace_reuse_across_shapes():
    """One cached workspace serves calls of different N: the zero-filled state the
    kernels rely on sits at offsets that do not move with N (a larger call's key /
    slot arrays must not leave garbage there for a smaller one)."""
    big = synth.ints(200 * 8, 64 * 8, seed=11, lo=-20, hi=20)
    compare(big, 8, 6000, 3000, 0.5, seed=1)
    bp.prune(to_torch(big), 8, k=5000)
    for nbr in (30, 9, 50):
        X = synth.ints(nbr * 4, 16 * 4, seed=nbr, lo=-20, hi=20)
        compare(X, 4, nbr * 8, 100, 0.7, seed=nbr)


def test_stochastic_small_n_limit_b64():
    """N = kSmallN = 24576 keys at b = 64 with the largest window: the largest
    shared-memory footprint of the one-kernel finishing path (all keys + the
    8192-entry boundary list per CTA)."""
    b, nbr, nbc = 64, 96, 256
    X = synth.ints(nbr * b, nbc * b, seed=12, lo=-3, hi=3)
    h = synth.to_bf16_bits(X)
    compare(h, b, 12288, 4096, 0.5, seed=4, bf16=True)
    compare(h, b, 12288, 1000, 0.5, seed=4, bf16=True)


def test_stochastic_large_n_bf16():
    """The multi-kernel path (N = 150528 keys: S12 fc1 at b = 4) on bf16 storage."""
    b, M, K = 4, 25088, 384
    X = synth.ints(M, K, seed=8, lo=-6, hi=6)
    h = synth.to_bf16_bits(X)
    N = (M // b) * (K // b)
    compare(h, b, N // 3, 2048, 0.4, seed=5, bf16=True)
