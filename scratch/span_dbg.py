"""Directed CG=2 / CG=1 span-kernel checks vs a float64 torch reference (one subprocess per case)."""
import os, subprocess, sys, json
import os as _o, sys as _s; _s.path.insert(0, _o.path.dirname(_o.path.dirname(_o.path.abspath(__file__))))
if len(sys.argv) > 1:
    import torch
    import paper_2311_16883_b200 as bp
    b, nbr, nbc, N, keep, prec = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), float(sys.argv[5]), sys.argv[6]
    g = torch.Generator(device="cuda").manual_seed(0)
    dt = torch.bfloat16 if prec == "bf16" else torch.float32
    X = torch.randn(nbr * b, nbc * b, device="cuda", generator=g).to(dt)
    dY = torch.randn(nbr * b, N, device="cuda", generator=g).to(dt)
    A = bp.prune(X, b, keep=keep)
    dW = bp.wgrad(A, dY, prec=prec)
    D = bp.decompress(A)
    ref = D.double().T @ dY.double()
    torch.cuda.synchronize()
    err = ((dW.double() - ref).norm() / ref.norm().clamp_min(1e-30)).item()
    print(json.dumps(dict(err=err)))
    sys.exit(0)
cases = []
for prec in ["tf32", "bf16"]:
    for (nbr, nbc, N) in [(3136, 12, 256), (784, 12, 1536), (200, 12, 512), (98, 48, 512)]:
        for keep in [0.5, 0.1, 0.9]:
            cases.append((32, nbr, nbc, N, keep, prec))
cases += [(16, 1568, 24, 1536, 0.5, "bf16"), (16, 1568, 24, 1536, 0.1, "bf16"), (64, 392, 6, 1536, 0.5, "tf32"), (64, 392, 6, 1536, 0.5, "bf16"), (64, 392, 6, 1536, 0.2, "bf16")]
for dbg in ["0"]:
    for c in cases:
        env = dict(os.environ, BSRP_WGRAD_CG="2", BSRP_SPAN_DBG=dbg)
        r = subprocess.run([sys.executable, __file__, *map(str, c)], env=env, capture_output=True, text=True, timeout=120)
        out = r.stdout.strip().splitlines()[-1] if r.returncode == 0 else "FAIL " + " | ".join(l for l in r.stderr.splitlines() if "cta" in l or "timeouts" in l)[:1500]
        print(f"dbg={dbg} case={c}: {out}", flush=True)
