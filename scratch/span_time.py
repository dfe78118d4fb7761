"""Time bsr_wgrad alone at C2 (CUDA events, back-to-back launches) for the library BSRP_LIB points at."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2311_16883_b200 as bp
prec = sys.argv[1] if len(sys.argv) > 1 else "tf32"
keep = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
M, K, N, b = 25088, 384, 1536, 32
dt = torch.bfloat16 if prec == "bf16" else torch.float32
g = torch.Generator(device="cuda").manual_seed(0)
Xs = [torch.randn(M, K, device="cuda", generator=g).to(dt) for _ in range(3)]
dYs = [torch.randn(M, N, device="cuda", generator=g).to(dt) for _ in range(3)]
As = [bp.prune(X, b, keep=keep) for X in Xs]
outs = [torch.empty(K, N, device="cuda") for _ in range(3)]
for i in range(3): bp.wgrad(As[i], dYs[i], prec=prec, out=outs[i])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
R = 60
e0.record()
for r in range(R):
    i = r % 3
    bp.wgrad(As[i], dYs[i], prec=prec, out=outs[i])
e1.record(); torch.cuda.synchronize()
print(json.dumps(dict(lib=os.path.basename(os.environ.get("BSRP_LIB", "default")), prec=prec, keep=keep, us=e0.elapsed_time(e1) / R * 1e3)))
if os.environ.get("SPAN_TRACE"):
    import ctypes, numpy as np
    lib = bp._lib.load()
    buf = (ctypes.c_ulonglong * (160 * 16))()
    torch.cuda.synchronize()
    bp.wgrad(As[0], dYs[0], prec=prec, out=outs[0]); torch.cuda.synchronize()
    lib.bsr_dev_span_trace(buf)
    tt = np.array(buf, dtype=np.float64).reshape(160, 16)[:144]; t = tt[:, :8]
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3
    names = ["start", "setup", "prod_done", "acc_full", "epi_done", "end"]
    for i, n in enumerate(names):
        print(f"{n:10s} min {rel[:, i].min():7.2f} med {np.median(rel[:, i]):7.2f} max {rel[:, i].max():7.2f} us")
    for i, n in [(8, "prod plan-wait cyc"), (9, "prod empty-wait cyc"), (10, "prod issue cyc"), (11, "rows"), (12, "mma full-wait cyc"), (13, "mma issue cyc")]:
        v = tt[:, i]; v = v[v > 0]
        if len(v): print(f"{n:22s} med {np.median(v):10.0f} max {v.max():10.0f}")
