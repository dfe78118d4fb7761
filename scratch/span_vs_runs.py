"""dW time of the per-run and the span tcgen05 kernels on the S12 layers (b 16/32/64, keep 0.1/0.5/0.9)."""
import os, sys, json, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1:
    import torch
    import paper_2311_16883_b200 as bp
    lname, prec = sys.argv[1], sys.argv[2]
    M, K, N = (25088, 384, 1536) if lname == "fc1" else (25088, 1536, 384)
    dt = torch.bfloat16 if prec == "bf16" else torch.float32
    g = torch.Generator(device="cuda").manual_seed(0)
    X = torch.randn(M, K, device="cuda", generator=g).to(dt)
    dYs = [torch.randn(M, N, device="cuda", generator=g).to(dt) for _ in range(3)]
    out = {}
    for b in (16, 32, 64):
        if prec == "tf32" and b < 32:
            continue
        for keep in (0.1, 0.5, 0.9):
            A = bp.prune(X, b, keep=keep)
            dW = torch.empty(K, N, device="cuda")
            for i in range(3): bp.wgrad(A, dYs[i], prec=prec, out=dW)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for r in range(30): bp.wgrad(A, dYs[r % 3], prec=prec, out=dW)
            e1.record(); torch.cuda.synchronize()
            out[f"{b}/{keep}"] = round(e0.elapsed_time(e1) / 30 * 1e3, 1)
    print(json.dumps(out))
    sys.exit(0)
for lname in ("fc1", "fc2"):
    for prec in ("tf32", "bf16"):
        res = {}
        for kern in ("runs", "span"):
            env = dict(os.environ, BSRP_WGRAD=kern)
            r = subprocess.run([sys.executable, __file__, lname, prec], env=env, capture_output=True, text=True)
            res[kern] = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-300:]
        print(lname, prec, json.dumps(res), flush=True)
