#!/usr/bin/env python
"""Measurement sweeps of SURVEY §8(d) on one B200 (run through gpurun):

  c3  ResMLP-S12 linear layers at batch 128 (BASELINE configs[2]): fc1 (X 25088 x 384,
      dY 25088 x 1536) and fc2 (X 25088 x 1536, dY 25088 x 384), block size
      4/8/16/32/64 x keep 0.1..1.0 (sparsity 90%..0%), fp32 and bf16 storage.  Per
      (layer, b, keep, dtype): prune / wgrad / decompress device time, GB/s,
      TFLOP/s and roofline fractions; plus the 12-block model totals.
  c5  prune/pack bandwidth sweep (configs[4]): X of 256 MiB, 1 GiB and 4 GiB
      (K = 1536 fp32), blocks 4/16/32/64, keep 0.1/0.5/1.0.

    python tools/sweep.py c3 c5 --out-dir profiles/r01_sweep

Timing: CUDA events around back-to-back launches on the current stream over
rotating input sets (each set larger than the 126 MB L2 for c3; c5 inputs are
larger than L2 by themselves), after warm-up.  Inputs are seeded synthetic
activations generated on the device with the shape/distribution recipe of
DESIGN.md §4 (per-channel affine + per-sample scale; GELU for fc2 inputs).
`check` is a self-consistency check of every measured dW against float64 torch
on the decompressed BSR (parity against the oracle is the job of tests/).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2311_16883_b200 as bp  # noqa: E402
from paper_2311_16883_b200 import metrics  # noqa: E402

SEED = 231116883


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1800.0, "fallback (B200_PROFILING.md)"


def activation(M, K, family, seed, dtype):
    """F_aff / F_gelu of DESIGN.md §4 on the device: sigma_s * f(alpha_c z + beta_c),
    sigma_s per 196-row sample, alpha_c / beta_c per channel."""
    g = torch.Generator(device="cuda").manual_seed(seed)
    z = torch.randn(M, K, device="cuda", generator=g)
    alpha = torch.exp(0.5 * torch.randn(K, device="cuda", generator=g))
    beta = (0.1 if family == "aff" else 0.5) * torch.randn(K, device="cuda", generator=g)
    sig = torch.exp(0.25 * torch.randn((M + 195) // 196, device="cuda", generator=g)).repeat_interleave(196)[:M]
    x = z.mul_(alpha).add_(beta)
    if family == "gelu":
        x = torch.nn.functional.gelu(x, approximate="tanh")
    x.mul_(sig[:, None])
    return x.to(dtype)


def grad_out(M, N, seed, dtype):
    g = torch.Generator(device="cuda").manual_seed(seed + 1)
    return (0.01 * torch.randn(M, N, device="cuda", generator=g)).to(dtype)


def timed(fn, sets, reps):
    """Mean device time (ms) of one launch: reps x len(sets) back-to-back launches."""
    for j in range(len(sets)):
        fn(j)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        for j in range(len(sets)):
            fn(j)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (reps * len(sets))


def prec_for(dtype, b):
    """bf16 storage: the bf16 tensor cores (block kernels at b >= 16, the dense rebuild
    below); fp32 storage: the FP32 grade (3xTF32 tensor cores at b >= 32, the dense
    rebuild below) -- the library's defaults."""
    if dtype == torch.bfloat16:
        return "bf16"
    return "fp32"


def sweep_c3(out, hbm, bf16_tf, nsets=3, reps=6):
    layers = [("fc1", 25088, 384, 1536, "aff"), ("fc2", 25088, 1536, 384, "gelu")]
    rows = []
    for dtype in (torch.float32, torch.bfloat16):
        s = 4 if dtype == torch.float32 else 2
        for lname, M, K, N, fam in layers:
            Xs = [activation(M, K, fam, SEED + 10 * i + (lname == "fc2"), dtype) for i in range(nsets)]
            dYs = [grad_out(M, N, SEED + 10 * i + 5, dtype) for i in range(nsets)]
            for b in (4, 8, 16, 32, 64):
                nblocks = bp.num_blocks(M, K, b)
                for keep in (0.1, 0.3, 0.5, 0.7, 0.9, 1.0):
                    k = bp.keep_count(nblocks, keep)
                    prec = prec_for(dtype, b)
                    As = [bp.alloc_bsr(M, K, b, k, dtype, "cuda") for _ in range(nsets)]
                    dWs = [torch.empty(K, N, device="cuda") for _ in range(nsets)]
                    Ds = [torch.empty(M, K, dtype=dtype, device="cuda") for _ in range(nsets)]
                    t_p = timed(lambda j: bp.prune(Xs[j], b, k=k, out=As[j]), Xs, reps)
                    t_w = timed(lambda j: bp.wgrad(As[j], dYs[j], prec=prec, out=dWs[j]), Xs, reps)
                    t_d = timed(lambda j: bp.decompress(As[j], out=Ds[j]), Xs, reps)
                    rp = As[0].rowptr
                    r_ne = int((rp[1:] > rp[:-1]).sum().item())
                    ref = Ds[0].double().T @ dYs[0].double()
                    err = ((dWs[0].double() - ref).norm() / ref.norm().clamp_min(1e-300)).item()
                    pb = metrics.prune_bytes(M, K, b, k, s)
                    wb = metrics.wgrad_bytes(M, K, b, k, N, s, s, r_ne)
                    wf = metrics.wgrad_flops(b, k, N)
                    db = metrics.decompress_bytes(M, K, b, k, s)
                    tc_peak = bf16_tf if prec == "bf16" else bf16_tf / 2 if prec == "tf32" else (
                        bf16_tf / 6 if b >= 32 else None)  # FP32 grade: 3xTF32 (useful flops) or FFMA
                    w_tf = wf / (t_w * 1e-3) / 1e12
                    w_gbs = wb / (t_w * 1e-3) / 1e9
                    roof_t = max(wb / (hbm * 1e9), wf / (tc_peak * 1e12) if tc_peak else 0.0)
                    row = dict(config="C3", layer=lname, M=M, K=K, N=N, b=b, keep=keep, k=k, dtype=str(dtype)[6:],
                               prec=prec, prune_ms=t_p, prune_gbs=pb / (t_p * 1e-3) / 1e9,
                               prune_hbm_frac=pb / (t_p * 1e-3) / 1e9 / hbm, wgrad_ms=t_w, wgrad_tflops=w_tf,
                               wgrad_gbs=w_gbs, wgrad_tc_frac=(w_tf / tc_peak) if tc_peak else None,
                               wgrad_roofline_frac=roof_t / (t_w * 1e-3),
                               wgrad_bound="tensor" if tc_peak and wf / (tc_peak * 1e12) > wb / (hbm * 1e9) else "hbm",
                               decompress_ms=t_d, decompress_gbs=db / (t_d * 1e-3) / 1e9,
                               act_bytes_saved=metrics.act_bytes_saved(M, K, b, k, s),
                               act_saved_frac=metrics.act_bytes_saved(M, K, b, k, s) / (s * M * K),
                               check_rel_err=err)
                    rows.append(row)
                    print(json.dumps(row), flush=True)
                    out.write(json.dumps(row) + "\n")
                    del As, dWs, Ds
            del Xs, dYs
            torch.cuda.empty_cache()
    # the whole S12 model: 12 blocks x (fc1 + fc2)
    model = []
    for dt in ("float32", "bfloat16"):
        for b in (4, 8, 16, 32, 64):
            for keep in (0.1, 0.3, 0.5, 0.7, 0.9, 1.0):
                sel = [r for r in rows if r["dtype"] == dt and r["b"] == b and r["keep"] == keep]
                if len(sel) != 2:
                    continue
                tot = {x: 12 * sum(r[x] for r in sel) for x in ("prune_ms", "wgrad_ms", "decompress_ms")}
                m = dict(config="C3-model", model="ResMLP-S12 (12 blocks x fc1+fc2)", dtype=dt, b=b, keep=keep,
                         **{f"model_{x}": v for x, v in tot.items()},
                         model_act_bytes_saved=12 * sum(r["act_bytes_saved"] for r in sel))
                model.append(m)
                out.write(json.dumps(m) + "\n")
    return rows, model


def sweep_c5(out, hbm, reps=4):
    K = 1536
    rows = []
    for size in (256 << 20, 1 << 30, 4 << 30):
        M = (size // (K * 4)) // 64 * 64
        Xs = [activation(M, K, "aff", SEED + 500 + i, torch.float32) for i in range(2)]
        for b in (4, 16, 32, 64):
            nblocks = bp.num_blocks(M, K, b)
            for keep in (0.1, 0.5, 1.0):
                k = bp.keep_count(nblocks, keep)
                As = [bp.alloc_bsr(M, K, b, k, torch.float32, "cuda") for _ in range(2)]
                t_p = timed(lambda j: bp.prune(Xs[j], b, k=k, out=As[j]), Xs, reps)
                pb = metrics.prune_bytes(M, K, b, k, 4)
                D = torch.empty(M, K, device="cuda")
                t_d = timed(lambda j: bp.decompress(As[j], out=D), Xs, reps)
                db = metrics.decompress_bytes(M, K, b, k, 4)
                row = dict(config="C5", x_bytes=4 * M * K, M=M, K=K, b=b, keep=keep, k=k, prune_ms=t_p,
                           prune_gbs=pb / (t_p * 1e-3) / 1e9, prune_hbm_frac=pb / (t_p * 1e-3) / 1e9 / hbm,
                           decompress_ms=t_d, decompress_gbs=db / (t_d * 1e-3) / 1e9,
                           decompress_hbm_frac=db / (t_d * 1e-3) / 1e9 / hbm)
                rows.append(row)
                print(json.dumps(row), flush=True)
                out.write(json.dumps(row) + "\n")
                del As, D
                torch.cuda.empty_cache()
        del Xs
        torch.cuda.empty_cache()
    return rows


def sweep_global(out, hbm, reps=20):
    """f4 at one rank: prune_global (digit-histogram protocol with host round trips,
    the collectives being no-ops) vs bsr_prune on the same X -- the protocol's
    fixed cost, and a check that both select the same blocks."""
    rows = []
    for lname, M, K, fam in (("fc1", 25088, 384, "aff"), ("fc2", 25088, 1536, "gelu")):
        X = activation(M, K, fam, SEED + 900, torch.float32)
        for b in (16, 32):
            for keep in (0.1, 0.5):
                A = bp.prune(X, b, keep=keep)
                t_p = timed(lambda j: bp.prune(X, b, keep=keep, out=A), [0], reps)
                G = bp.prune_global(X, b, keep)
                same = bool(torch.equal(G.colidx, A.colidx) and torch.equal(G.rowptr, A.rowptr))
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                for _ in range(reps):
                    bp.prune_global(X, b, keep)
                torch.cuda.synchronize()
                t_g = (time.perf_counter() - t0) / reps * 1e3
                row = dict(config="f4-global-1rank", layer=lname, M=M, K=K, b=b, keep=keep, prune_ms=t_p,
                           prune_global_ms_wall=t_g, same_selection=same)
                rows.append(row)
                print(json.dumps(row), flush=True)
                out.write(json.dumps(row) + "\n")
    return rows


def sweep_rows(out, hbm, reps=6, nsets=3):
    """f2: the paper-faithful 1 x b per-sample variant on the S12 layers at batch 128
    (196-row samples): prune_rows / wgrad_rows / decompress_rows device time."""
    rows = []
    S = 196
    for lname, M, K, N, fam in (("fc1", 25088, 384, 1536, "aff"), ("fc2", 25088, 1536, 384, "gelu")):
        Xs = [activation(M, K, fam, SEED + 20 * i + 7, torch.float32) for i in range(nsets)]
        dYs = [grad_out(M, N, SEED + 20 * i + 9, torch.float32) for i in range(nsets)]
        for b in (4, 8, 16, 32, 64):
            for keep in (0.1, 0.5, 0.9):
                As = [bp.prune_rows(X, b, keep, sample_rows=S) for X in Xs]
                k = As[0].nnz
                t_p = timed(lambda j: bp.prune_rows(Xs[j], b, keep, sample_rows=S), Xs, reps)
                dW = torch.empty(K, N, device="cuda")
                t_w = timed(lambda j: bp.wgrad_rows(As[j], dYs[j], out=dW), Xs, reps)
                t_wf = timed(lambda j: bp.wgrad_rows(As[j], dYs[j], out=dW, tensor_cores=False), Xs, reps)
                D = torch.empty(M, K, device="cuda")
                t_d = timed(lambda j: bp.decompress_rows(As[j], out=D), Xs, reps)
                ref = bp.decompress_rows(As[0]).double().T @ dYs[0].double()
                err = ((bp.wgrad_rows(As[0], dYs[0]).double() - ref).norm() / ref.norm()).item()
                bsr = k * b * 4 + 4 * k + 4 * (M + 1)
                pb = 4 * M * K + bsr
                row = dict(config="f2-rows", layer=lname, M=M, K=K, N=N, b=b, keep=keep, k=k, sample_rows=S,
                           prune_ms=t_p, prune_gbs=pb / (t_p * 1e-3) / 1e9, prune_hbm_frac=pb / (t_p * 1e-3) / 1e9 / hbm,
                           wgrad_ms=t_w, wgrad_tflops=2 * k * b * N / (t_w * 1e-3) / 1e12,
                           wgrad_path="tensor cores (dense rebuild, FP32 grade)" if
                           bp._lib.load().bsr_wgrad_rows_tc_workspace_bytes(M, K, b, N, 0) else "FFMA",
                           wgrad_ffma_ms=t_wf,
                           decompress_ms=t_d, decompress_gbs=(bsr + 4 * M * K) / (t_d * 1e-3) / 1e9,
                           act_bytes_saved=4 * M * K - bsr, check_rel_err=err)
                rows.append(row)
                print(json.dumps(row), flush=True)
                out.write(json.dumps(row) + "\n")
                del As
        del Xs, dYs
        torch.cuda.empty_cache()
    return rows


def sweep_fusion(out, hbm, reps=20, nsets=3):
    """f3 (norm in the producer): GELU(Z) + bsr_prune vs the fused
    bsr_act_block_sumsq + bsr_prune_presummed, S12 fc2 input (25088 x 1536) and
    the C2 shape (25088 x 384), b 16/32, keep 0.1/0.5."""
    rows = []
    for lname, M, K in (("fc2-input", 25088, 1536), ("fc1-input", 25088, 384)):
        Zs = [activation(M, K, "aff", SEED + 40 + i, torch.float32) for i in range(nsets)]
        Xs = [torch.empty_like(Z) for Z in Zs]
        for b in (16, 32):
            for keep in (0.1, 0.5):
                k = bp.keep_count(bp.num_blocks(M, K, b), keep)
                As = [bp.alloc_bsr(M, K, b, k, torch.float32, "cuda") for _ in range(nsets)]

                def unfused(j):  # PyTorch's GELU kernel (one read of Z, one write of X), then the prune
                    bp.prune(torch.nn.functional.gelu(Zs[j], approximate="tanh"), b, k=k, out=As[j])

                def gelu_only(j):
                    torch.nn.functional.gelu(Zs[j], approximate="tanh")

                t_u = timed(unfused, Zs, reps)
                t_g = timed(gelu_only, Zs, reps)
                t_f = timed(lambda j: bp.act_prune(Zs[j], b, k=k, act="gelu", X_out=Xs[j], out=As[j]), Zs, reps)
                row = dict(config="f3-fusion", layer=lname, M=M, K=K, b=b, keep=keep,
                           unfused_ms=t_u, torch_gelu_ms=t_g, fused_ms=t_f, saved_ms=t_u - t_f)
                rows.append(row)
                print(json.dumps(row), flush=True)
                out.write(json.dumps(row) + "\n")
        del Zs, Xs
        torch.cuda.empty_cache()
    return rows


def sweep_stoch(out, hbm, reps=20, nsets=4):
    """f4 stochastic boundary swapping (R19) vs the deterministic prune on the S12
    layers at batch 128: device time and algorithmic GB/s of each (same bytes:
    X read once, k blocks written)."""
    rows = []
    for lname, M, K, fam in (("fc1", 25088, 384, "aff"), ("fc2", 25088, 1536, "gelu")):
        Xs = [activation(M, K, fam, SEED + 40 * i + 3, torch.float32) for i in range(nsets)]
        for b in (16, 32):
            keep = 0.5
            N = bp.num_blocks(M, K, b)
            k = bp.keep_count(N, keep)
            alg = metrics.prune_bytes(M, K, b, k, 4)
            outs = [bp.prune(X, b, k=k) for X in Xs]
            t_p = timed(lambda j: bp.prune(Xs[j], b, k=k, out=outs[j]), Xs, reps)
            for window in (64, 1024, 4096):
                t_s = timed(lambda j: bp.prune_stochastic(Xs[j], b, k=k, window=window, p=0.5, seed=j, out=outs[j]),
                            Xs, reps)
                row = dict(config="f4-stochastic", layer=lname, M=M, K=K, b=b, keep=keep, N=N, k=k, window=window,
                           p=0.5, prune_ms=t_p, stoch_ms=t_s, prune_hbm_frac=alg / (t_p * 1e-3) / 1e9 / hbm,
                           stoch_hbm_frac=alg / (t_s * 1e-3) / 1e9 / hbm)
                rows.append(row)
                print(json.dumps(row), flush=True)
                out.write(json.dumps(row) + "\n")
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", nargs="+", choices=["c3", "c5", "global", "rows", "fusion", "stoch"])
    ap.add_argument("--out-dir", default=os.path.join(ROOT, "gpurun_out", "sweep"))
    a = ap.parse_args()
    os.makedirs(a.out_dir, exist_ok=True)
    hbm, bf16_tf, src = peaks()
    meta = dict(gpu=torch.cuda.get_device_name(0), hbm_gbs=hbm, bf16_tflops=bf16_tf, peak_source=src,
                when=time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()), lib=bp.version())
    for w in a.which:
        with open(os.path.join(a.out_dir, f"{w}.jsonl"), "w") as out:
            out.write(json.dumps(dict(meta=meta)) + "\n")
            if w == "c3":
                sweep_c3(out, hbm, bf16_tf)
            elif w == "c5":
                sweep_c5(out, hbm)
            elif w == "global":
                sweep_global(out, hbm)
            elif w == "rows":
                sweep_rows(out, hbm)
            elif w == "stoch":
                sweep_stoch(out, hbm)
            else:
                sweep_fusion(out, hbm)


if __name__ == "__main__":
    main()
