"""Small calls of every kernel family, for compute-sanitizer (tools/sanitize.sh):
prune (multi-barrier + candidate exchange, tie-overflow refinement, k = N), decompress,
dW (FP32 grade 3xTF32, tf32 / bf16 per-run and span, FFMA), the 1 x b variant,
producer fusion, device-side global selection and the affine layer -- C1 sizes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2311_16883_b200 as bp  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda")
for dt in (torch.float32, torch.bfloat16):
    for b in (4, 16, 32, 64):
        M, K, N = 8 * 64, 4 * 64, 256
        X = torch.from_numpy(synth.f_aff(M, K, 1)).to(dev, dt)
        Xi = torch.from_numpy(synth.ints(M, K, 2)).to(dev, dt)  # tie-heavy: refinement path
        dY = torch.from_numpy(synth.grad_out(M, N, 1)).to(dev, dt)
        for src in (X, Xi):
            for keep in (0.0, 0.3, 1.0):
                A = bp.prune(src, b, keep=keep)
                bp.decompress(A)
                precs = ["fp32"] + (["bf16"] if dt == torch.bfloat16 else ["tf32"])
                for prec in precs:
                    for algo in ("auto", "runs", "span", "simt"):
                        try:
                            bp.wgrad(A, dY, prec=prec, algo=algo)
                        except bp.BsrError:
                            pass
                bp.affine_wgrad(A, torch.from_numpy(synth.grad_out(M, K, 3)).to(dev, dt))
        bp.act_prune(X, b, keep=0.5, act="gelu")
        bp.prune_global(X, b, 0.5)
        R = bp.prune_rows(X, b, 0.5, sample_rows=64)
        bp.decompress_rows(R)
        bp.wgrad_rows(R, dY)
torch.cuda.synchronize()
print("sanitize calls done")
