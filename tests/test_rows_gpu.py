"""GPU parity of the paper-faithful per-sample 1 x b variant:
bsr_prune_rows / bsr_decompress_rows / bsr_wgrad_rows against the oracle's
prune_per_sample / decompress / wgrad_rect."""
import numpy as np
import pytest

import oracle
import synth
from helpers import to_torch

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2311_16883_b200 as bp  # noqa: E402


def _gap_ok(X, b, k, S, rel=1e-5):
    """Every sample's k-th / (k+1)-th segment sums differ by >= rel (fp32 keys decide the same set)."""
    for s0 in range(0, X.shape[0], S):
        ss = np.sort(oracle.block_sumsq(X[s0:s0 + S], 1, b))[::-1]
        if 0 < k < len(ss) and ss[k - 1] - ss[k] < rel * ss[k - 1]:
            return False
    return True


def oracle_rows_ref(X, b, keep, S, A, bf16=False):
    """The oracle's own per-sample selection of X (never the GPU's): skips the case if
    fp32 segment sums could rank differently from the oracle's fp64 ones, else
    requires the GPU's BSR to equal it bit for bit and returns it (values as fp32)."""
    K = X.shape[1]
    Xf = synth.bf16_bits_to_f32(X) if bf16 else X
    ks = oracle.keep_count(S * K // b, keep)
    if not _gap_ok(Xf, b, ks, S, rel=1e-5):  # fp32 sums of <= 64 squares: error < 4e-6 relative
        pytest.skip("fp32 segment sums too close at the boundary for this seed")
    ref = oracle.prune_per_sample(X, b, ks, S)
    np.testing.assert_array_equal(A.rowptr.cpu().numpy(), ref["rowptr"])
    np.testing.assert_array_equal(A.colidx.cpu().numpy(), ref["colidx"])
    vals = ref["values"].reshape(-1, 1, b)
    return ref["rowptr"], ref["colidx"], (synth.bf16_bits_to_f32(vals) if bf16 else vals)


def _x(family, M, K, seed):
    return synth.ints(M, K, seed) if family == "ints" else synth.f_aff(M, K, seed, tokens=14)


@pytest.mark.parametrize("b", [4, 8, 16, 32, 64])
@pytest.mark.parametrize("keep", [0.0, 0.1, 0.5, 0.9, 1.0])
@pytest.mark.parametrize("family", ["ints", "aff"])
def test_prune_rows_parity(b, keep, family):
    S, nsamp, K = 14, 5, 4 * b if b >= 32 else 128
    M = S * nsamp
    X = _x(family, M, K, 300 + b)
    ks = oracle.keep_count(S * K // b, keep)
    if family == "aff" and not _gap_ok(X, b, ks, S):
        pytest.skip("fp32 segment sums too close at the boundary for this seed")
    ref = oracle.prune_per_sample(X, b, ks, S)
    A = bp.prune_rows(to_torch(X), b, keep, sample_rows=S)
    D = bp.decompress_rows(A)
    torch.cuda.synchronize()
    assert A.nnz == nsamp * ks == int(ref["mask"].sum())
    np.testing.assert_array_equal(A.rowptr.cpu().numpy(), ref["rowptr"])
    np.testing.assert_array_equal(A.colidx.cpu().numpy(), ref["colidx"])
    np.testing.assert_array_equal(A.values.cpu().numpy().view(np.int32), ref["values"].reshape(-1, b).view(np.int32))
    dense = oracle.decompress(ref["rowptr"], ref["colidx"], ref["values"], M, K, 1, b)
    np.testing.assert_array_equal(D.cpu().numpy().view(np.int32), dense.view(np.int32))


@pytest.mark.parametrize("b", [4, 8, 16, 32, 64])
@pytest.mark.parametrize("keep", [0.1, 0.5, 1.0])
@pytest.mark.parametrize("N", [128, 384, 200])
def test_wgrad_rows_parity(b, keep, N):
    S, nsamp, K = 14, 7, 256 + 2 * b
    M = S * nsamp
    X = synth.f_gelu(M, K, 400 + b)
    dY = synth.grad_out(M, N, 400 + b)
    A = bp.prune_rows(to_torch(X), b, keep, sample_rows=S)
    torch.cuda.synchronize()
    rp, ci, vals = oracle_rows_ref(X, b, keep, S, A)
    want = oracle.wgrad_rect(rp, ci, vals, M, K, 1, b, dY)
    got = bp.wgrad_rows(A, to_torch(dY)).cpu().numpy()
    assert oracle.rel_frobenius(got, want) <= 1e-5
    base = torch.randn(K, N, device="cuda")
    out = base.clone()
    bp.wgrad_rows(A, to_torch(dY), out=out, accumulate=True)
    assert oracle.rel_frobenius(out.cpu().numpy() - base.cpu().numpy(), want) <= 1e-5


@pytest.mark.parametrize("b", [4, 16])
def test_rows_bf16_storage(b):
    S, nsamp, K, N = 14, 4, 128, 256
    M = S * nsamp
    Xh = synth.to_bf16_bits(synth.f_aff(M, K, 77, tokens=14))
    dYh = synth.to_bf16_bits(synth.grad_out(M, N, 77))
    A = bp.prune_rows(to_torch(Xh, bf16=True), b, 0.5, sample_rows=S)
    torch.cuda.synchronize()
    rp, ci, vals = oracle_rows_ref(Xh, b, 0.5, S, A, bf16=True)
    want = oracle.wgrad_rect(rp, ci, vals, M, K, 1, b, synth.bf16_bits_to_f32(dYh))
    got = bp.wgrad_rows(A, to_torch(dYh, bf16=True)).cpu().numpy()
    assert oracle.rel_frobenius(got, want) <= 1e-5


def test_rows_s12_fc1_shape():
    """S12 fc1 geometry (196 tokens x 384 channels per sample, b = 16, keep 0.5)
    on 8 samples: exact per-sample counts and dW parity at full K and N."""
    S, nsamp, K, N, b = 196, 8, 384, 1536, 16
    M = S * nsamp
    X = synth.f_aff(M, K, 5)
    dY = synth.grad_out(M, N, 5)
    A = bp.prune_rows(to_torch(X), b, 0.5, sample_rows=S)
    dW = bp.wgrad_rows(A, to_torch(dY))
    torch.cuda.synchronize()
    rp = A.rowptr.cpu().numpy()
    ks = oracle.keep_count(S * K // b, 0.5)
    assert all(rp[(s + 1) * S] - rp[s * S] == ks for s in range(nsamp))
    orp, oci, ovals = oracle_rows_ref(X, b, 0.5, S, A)
    want = oracle.wgrad_rect(orp, oci, ovals, M, K, 1, b, dY)
    assert oracle.rel_frobenius(dW.cpu().numpy(), want) <= 1e-5


def test_rows_selection_full_s12_batch():
    """C3 geometry at the full batch (128 samples x 196 tokens x 384 channels,
    b = 16, keep 0.5): every sample's selection and packed values bit-exact
    against the oracle (integer-valued X: exact fp32 sums, ties resolved by the
    BJ rule)."""
    S, nsamp, K, b = 196, 128, 384, 16
    M = S * nsamp
    X = synth.ints(M, K, 21)
    ks = oracle.keep_count(S * K // b, 0.5)
    ref = oracle.prune_per_sample(X, b, ks, S)
    A = bp.prune_rows(to_torch(X), b, 0.5, sample_rows=S)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(A.rowptr.cpu().numpy(), ref["rowptr"])
    np.testing.assert_array_equal(A.colidx.cpu().numpy(), ref["colidx"])
    np.testing.assert_array_equal(A.values.cpu().numpy().view(np.int32), ref["values"].reshape(-1, b).view(np.int32))


@pytest.mark.parametrize("S,K,b", [(128, 384, 4), (128, 768, 8), (416, 512, 4), (208, 2048, 8), (196, 1536, 4)])
def test_rows_select_keys_at_shared_memory_limit(S, K, b):
    """Samples of 12288 segment keys (48 KB: beyond the default dynamic shared
    memory limit, so the launch must opt in -- ADVICE r01), exactly 53248 (208 KB,
    the on-chip threshold) and 75264 (S12 fc2 at b = 4: the keys stay in global
    memory, 4 loads in flight per thread)."""
    assert S * K // b in (12288, 53248, 75264)
    M = 2 * S
    X = synth.ints(M, K, 77)  # exact sums; ties decided by the flat-index rule
    ks = oracle.keep_count(S * K // b, 0.5)
    ref = oracle.prune_per_sample(X, b, ks, S)
    A = bp.prune_rows(to_torch(X), b, 0.5, sample_rows=S)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(A.rowptr.cpu().numpy(), ref["rowptr"])
    np.testing.assert_array_equal(A.colidx.cpu().numpy(), ref["colidx"])
    np.testing.assert_array_equal(A.values.cpu().numpy().view(np.int32), ref["values"].reshape(-1, b).view(np.int32))


@pytest.mark.parametrize("bf16", [False, True])
@pytest.mark.parametrize("keep", [0.1, 0.5, 1.0])
def test_wgrad_rows_tensor_cores(bf16, keep):
    """The 1 x b variant's dW on the tensor cores (kept rows rebuilt densely, keep-all
    32 x 32 BSR, per-run tcgen05 kernel: FP32 grade for f32, bf16 for bf16) against
    the oracle on its own selection (which the GPU's must equal), and the FFMA kernel."""
    S, nsamp, K, N, b = 196, 8, 384, 256, 16  # M = 1568 = 49 x 32
    M = S * nsamp
    X = synth.f_aff(M, K, 55)
    dY = synth.grad_out(M, N, 55)
    if bf16:
        X, dY = synth.to_bf16_bits(X), synth.to_bf16_bits(dY)
    A = bp.prune_rows(to_torch(X, bf16=bf16), b, keep, sample_rows=S)
    torch.cuda.synchronize()
    rp, ci, vals = oracle_rows_ref(X, b, keep, S, A, bf16=bf16)
    want = oracle.wgrad_rect(rp, ci, vals, M, K, 1, b, synth.bf16_bits_to_f32(dY) if bf16 else dY)
    tc = bp.wgrad_rows(A, to_torch(dY, bf16=bf16), tensor_cores=True).cpu().numpy()
    ff = bp.wgrad_rows(A, to_torch(dY, bf16=bf16), tensor_cores=False).cpu().numpy()
    assert oracle.rel_frobenius(tc, want) <= 1e-5
    assert oracle.rel_frobenius(ff, want) <= 1e-5
