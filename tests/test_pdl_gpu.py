"""Programmatic dependent launch (PDL, csrc/launch.h): the bsr_set_pdl bit mask only
changes WHEN the wgrad / split-K reduce / decompress CTAs are scheduled, never
what they compute.  Every kernel waits (griddepcontrol.wait) for its stream
predecessor before its first global access, so prune -> wgrad -> decompress
chained back to back must give bit-identical BSR, dW and decompressed X under
every mask, captured in a CUDA graph or launched eagerly.  Each mask runs in its
own subprocess (fresh graph, fresh workspaces)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2311_16883_b200 as bp, synth
out, M, K, N, b, dt, prec, graph = sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]), int(sys.argv[6]), sys.argv[7], sys.argv[8], sys.argv[9] == "1"
bp.set_pdl(int(sys.argv[10]))
tdt = torch.bfloat16 if dt == "bf16" else torch.float32
X = torch.from_numpy(synth.f_aff(M, K, 4242)).to("cuda", tdt)
dY = torch.from_numpy(synth.f_aff(M, N, 4343)).to("cuda", tdt)
A = bp.prune(X, b, keep=0.5)
dW = bp.wgrad(A, dY, prec=prec)
Xd = bp.decompress(A)
def step():
    bp.prune(X, b, keep=0.5, out=A)
    bp.wgrad(A, dY, prec=prec, out=dW)
    bp.decompress(A, out=Xd)
torch.cuda.synchronize()
if graph:
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for _ in range(5):
        g.replay()
else:
    for _ in range(5):
        step()
torch.cuda.synchronize()
iv = lambda t: t.view(torch.int16 if t.dtype == torch.bfloat16 else torch.int32).cpu().numpy()
np.savez(out, rowptr=A.rowptr.cpu().numpy(), colidx=A.colidx.cpu().numpy(), values=iv(A.values),
         dW=dW.view(torch.int32).cpu().numpy(), Xd=iv(Xd))
"""


def _run(tmp_path, mask, args):
    f = tmp_path / f"pdl_{mask}.npz"
    r = subprocess.run([sys.executable, "-c", _SCRIPT, ROOT, str(f), *map(str, args), str(mask)], cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(f)


@pytest.mark.parametrize("dt,prec", [("f32", "tf32"), ("bf16", "bf16"), ("f32", "fp32")])
@pytest.mark.parametrize("graph", [0, 1])
def test_pdl_masks_bit_identical(tmp_path, dt, prec, graph):
    # C2-like shape with split-K (reduce kernel in the chain): 6272 x 384 -> 1536, b = 32
    args = (6272, 384, 1536, 32, dt, prec, graph)
    ref = _run(tmp_path, 0, args)
    for mask in (1 | 4 | 16 | 32 | 64, 1 | 2 | 8 | 16 | 32 | 64):
        got = _run(tmp_path, mask, args)
        for k in ref.files:
            assert np.array_equal(ref[k], got[k]), (mask, k)
