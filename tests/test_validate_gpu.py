"""bsr_validate: the device-side structural check of a BSR (SURVEY §5 validation
hook) -- valid on every prune output and on the oracle's BSR, and it names the
first broken block row for each kind of corruption."""
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


@pytest.mark.parametrize("b,keep", [(4, 0.3), (16, 0.5), (32, 0.5), (32, 0.0), (32, 1.0), (64, 0.9)])
def test_prune_outputs_are_valid(b, keep):
    X = to_torch(synth.f_aff(40 * b, 24 * b, seed=b))
    A = bp.prune(X, b, keep=keep)
    assert bp.validate(A) == -1


def test_oracle_bsr_is_valid():
    X = synth.ints(30 * 8, 20 * 8, seed=3, lo=-5, hi=5)
    ref = oracle.prune(X, 8, 230)
    A = bp.BSR(torch.from_numpy(ref["rowptr"]).cuda(), torch.from_numpy(ref["colidx"]).cuda(),
               torch.from_numpy(ref["values"]).cuda(), 30 * 8, 20 * 8, 8)
    assert bp.validate(A) == -1


def _bsr(b=8, nbr=30, nbc=20, k=230):
    X = to_torch(synth.ints(nbr * b, nbc * b, seed=4, lo=-5, hi=5))
    return bp.prune(X, b, k=k)


def test_detects_corruption():
    A = _bsr()
    rp = A.rowptr.cpu().numpy()
    ci = A.colidx.cpu().numpy()
    rows = [r for r in range(len(rp) - 1) if rp[r + 1] - rp[r] >= 2]
    r = rows[len(rows) // 2]
    # colidx not ascending inside row r
    B = _bsr()
    B.colidx[rp[r]], B.colidx[rp[r] + 1] = int(ci[rp[r] + 1]), int(ci[rp[r]])
    assert bp.validate(B) == r
    # colidx out of range in row r
    B = _bsr()
    B.colidx[rp[r + 1] - 1] = 20
    assert bp.validate(B) == r
    # rowptr[0] != 0
    B = _bsr()
    B.rowptr[0] = 1
    assert bp.validate(B) == 0
    # rowptr decreasing between rows r and r + 1: row r is reported
    B = _bsr()
    B.rowptr[r + 1] = int(rp[r]) - 1
    assert bp.validate(B) == r
    # last entry != nnzb
    B = _bsr()
    B.rowptr[-1] = int(rp[-1]) - 1
    assert bp.validate(B) == len(rp) - 2
