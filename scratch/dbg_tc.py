import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import oracle, synth
from helpers import to_torch
import paper_2311_16883_b200 as bp
for prec in ["tf32", "bf16"]:
    for b in [16, 32, 64]:
        for (nbr, nbc, N, keep) in [(4, 2, 128, 1.0), (37, 6, 128, 0.5)]:
            M, K = nbr*b, nbc*b
            k = oracle.keep_count(nbr*nbc, keep)
            X = synth.f_gelu(M, K, 1); dY = synth.grad_out(M, N, 1)
            if prec == "bf16":
                X, dY = synth.to_bf16_bits(X), synth.to_bf16_bits(dY)
            ref = oracle.prune(X, b, k)
            A = bp.prune(to_torch(X, bf16=prec=="bf16"), b, k=k)
            try:
                out = torch.full((K, N), float('nan'), device='cuda')
                bp.wgrad(A, to_torch(dY, bf16=prec=="bf16"), prec=prec, out=out)
                torch.cuda.synchronize()
                got = out.cpu().numpy()
            except Exception as e:
                print(prec, b, nbr, nbc, N, "EXC", e); continue
            r = oracle.wgrad(ref["rowptr"], ref["colidx"], ref["values"], M, K, b, dY)
            nan = np.isnan(got).sum()
            g = np.nan_to_num(got)
            err = oracle.rel_frobenius(g, r)
            # best-fit scale and transposition hints
            ratio = (g*r).sum()/max((r*r).sum(),1e-30)
            print(f"{prec} b={b} {nbr}x{nbc} N={N} k={k} err={err:.3e} nan={nan} zero={int((g==0).sum())}/{g.size} proj={ratio:.3f} gmax={np.abs(g).max():.3e} rmax={np.abs(r).max():.3e}", flush=True)
            if err > 0.01 and nbr == 4:
                print(" got[:4,:4]", g[:4,:4]); print(" ref[:4,:4]", r[:4,:4])
