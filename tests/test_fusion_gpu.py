"""GPU parity of the producer fusion: bsr_act_block_sumsq writes
X = act(Z) and the block sums in one pass, bsr_prune_presummed prunes from those
sums.  The result must be bit-identical to act(Z) followed by bsr_prune on the
written X (same fp32 sums, hence the same selection), and match the oracle."""
import numpy as np
import pytest

import oracle
import synth
from helpers import enforce_gap, to_torch

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2311_16883_b200 as bp  # noqa: E402


def _same(A, B):
    assert A.nnzb == B.nnzb
    assert torch.equal(A.rowptr, B.rowptr) and torch.equal(A.colidx, B.colidx)
    assert torch.equal(A.values.view(torch.int16 if A.values.dtype == torch.bfloat16 else torch.int32),
                       B.values.view(torch.int16 if B.values.dtype == torch.bfloat16 else torch.int32))


@pytest.mark.parametrize("b", [4, 8, 16, 32, 64])
@pytest.mark.parametrize("keep", [0.1, 0.5, 0.9])
@pytest.mark.parametrize("bf16", [False, True])
def test_gelu_fusion_equals_unfused(b, keep, bf16):
    M, K = 24 * b, 256 if b < 64 else 384
    Z = synth.f_aff(M, K, 900 + b)
    Zt = to_torch(synth.to_bf16_bits(Z), bf16=True) if bf16 else to_torch(Z)
    X, A = bp.act_prune(Zt, b, keep=keep, act="gelu")
    torch.cuda.synchronize()
    ref_x = torch.nn.functional.gelu(Zt.float(), approximate="tanh")
    if bf16:
        assert (X.float() - ref_x).abs().max().item() <= 2 ** -7 * ref_x.abs().max().item()
    else:
        torch.testing.assert_close(X, ref_x, rtol=2e-6, atol=2e-6)
    _same(A, bp.prune(X, b, keep=keep))  # the presummed sums are the ones the prune computes from X


@pytest.mark.parametrize("b", [4, 16, 32, 64])
@pytest.mark.parametrize("keep", [0.0, 0.3, 1.0])
def test_identity_fusion_equals_oracle(b, keep):
    M, K = 32 * b, 128 if b < 64 else 256
    k = oracle.keep_count(oracle.num_blocks(M, K, b), keep)
    Z, _ = enforce_gap(synth.f_gelu(M, K, 31 + b), b, max(k, 1))
    Zt = to_torch(Z)
    X, A = bp.act_prune(Zt, b, k=k, act="identity")
    torch.cuda.synchronize()
    assert torch.equal(X.view(torch.int32), Zt.view(torch.int32))
    ref = oracle.prune(Z, b, k)
    np.testing.assert_array_equal(A.rowptr.cpu().numpy(), ref["rowptr"])
    np.testing.assert_array_equal(A.colidx.cpu().numpy(), ref["colidx"])
    np.testing.assert_array_equal(A.values.cpu().numpy().view(np.int32), ref["values"].view(np.int32))


def test_gelu_fusion_in_place_c3_shape():
    """S12 fc2 input (25088 x 1536), in place (X_out is Z), b = 32, keep 0.5."""
    M, K, b = 25088, 1536, 32
    Zt = to_torch(synth.f_aff(M, K, 3))
    ref_x = torch.nn.functional.gelu(Zt, approximate="tanh")
    X, A = bp.act_prune(Zt, b, keep=0.5, act="gelu", X_out=Zt)
    torch.cuda.synchronize()
    torch.testing.assert_close(X, ref_x, rtol=2e-6, atol=2e-6)
    _same(A, bp.prune(X, b, keep=0.5))
