#!/usr/bin/env python
"""Benchmark of the B200 hot path of structured activation pruning (arXiv 2311.16883).

One step = one pass of the whole hot path over one layer's batch:
    a1-a4  bsr_prune      X (M x K) -> top-k b x b blocks by l2 norm -> BSR
    a6     bsr_wgrad      dW = X_bsr^T . dY  (K x N fp32, kept blocks only)
    a5     bsr_decompress BSR -> masked dense X
    a7     all-reduce(dW) over ranks (N > 1 only; NCCL)
Workload at N = 1: BASELINE.json configs[1], ResMLP-S12 fc1 (X 25088 x 384 = batch
128 x 196 tokens, dY 25088 x 1536, b = 32, keep 0.5).  At N > 1 every rank runs
its own such shard (weak scaling) and the partial dW are all-reduced.

Printed: ONE JSON line (rank 0).  `value` = algorithmic bytes of the whole step
(SURVEY §8d formulas, paper_2311_16883_b200/metrics.py) summed over ranks / the
max-over-ranks device time of the K timed steps, in GB/s; per-kernel GB/s,
TFLOP/s and roofline fractions are in `kernels` / `roofline`.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--dtype f32|bf16]
    python bench.py --impl reference ...   # the CPU oracle arm
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402
from paper_2311_16883_b200 import metrics  # noqa: E402

METRIC = "prune GB/s & BSR-dW TFLOP/s vs roofline at 1/2/4/8 B200; act bytes saved"
NSETS = 3  # rotating device input sets: X+dY = 193 MB per set at C2, > the 126 MB L2
PROFILE_SUMMARY = os.path.join(ROOT, "profiles", "ncu_traffic.json")


def parse():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["native", "reference"], default="native")
    ap.add_argument("--config", default="C2", choices=sorted(synth.CONFIGS))
    ap.add_argument("--dtype", choices=["f32", "bf16"], default="f32", help="element type of X and dY")
    ap.add_argument("--prec", choices=["fp32", "tf32", "bf16"], default=None,
                    help="dW arithmetic (default: tf32 for f32 inputs, bf16 for bf16 inputs)")
    ap.add_argument("--b", type=int, default=None)
    ap.add_argument("--keep", type=float, default=None)
    ap.add_argument("--no-graph", action="store_true", help="launch eagerly instead of CUDA-graph replays")
    ap.add_argument("--order", choices=["pwd", "pdw"], default="pwd",
                    help="kernel order inside a step: prune-wgrad-decompress or prune-decompress-wgrad")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=50)
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="cpu_baseline sample budget")
    ap.add_argument("--ref-budget", type=float, default=120.0, help="--impl reference: seconds for all steps")
    a = ap.parse_args()
    if a.warmup < 3:
        ap.error("--warmup must be >= 3")
    if a.prec is None:
        a.prec = "bf16" if a.dtype == "bf16" else "tf32"
    return a


def workload(a):
    c = dict(synth.CONFIGS[a.config])
    if a.b is not None:
        c["b"] = a.b
    if a.keep is not None:
        c["keep"] = a.keep
    return c


def host_inputs(c, rank, dtype):
    """Seeded synthetic X and dY for this rank (synth recipe)."""
    seed = synth.seed_for(c["id"], 0, rank)
    X = synth.activation(c["family"], c["M"], c["K"], seed)
    dY = synth.grad_out(c["M"], c["N"], seed)
    if dtype == "bf16":
        X, dY = synth.to_bf16_bits(X), synth.to_bf16_bits(dY)
    return X, dY


def config_json(c, a, world):
    return {"workload": f"{a.config}: {c['desc']}", "M": c["M"], "K": c["K"], "N": c["N"], "b": c["b"],
            "keep": c["keep"], "x_dtype": a.dtype, "dw_prec": a.prec, "global_batch_rows": c["M"] * world,
            "parallelism": f"dp{world}" if world > 1 else "single",
            "l2": f"{NSETS} rotating device input sets (X+dY per set larger than the 126 MB L2)"}


# ----------------------------------------------------------------------------- CPU oracle legs
def _oracle_step(X, dY, b, keep):
    """The oracle's version of one step on (a slice of) the workload; returns
    (seconds, algorithmic bytes, flops)."""
    import oracle
    M, K = X.shape
    N = dY.shape[1]
    k = oracle.keep_count(oracle.num_blocks(M, K, b), keep)
    t0 = time.perf_counter()
    ref = oracle.prune(X, b, k)
    oracle.wgrad(ref["rowptr"], ref["colidx"], ref["values"], M, K, b, dY)
    oracle.decompress(ref["rowptr"], ref["colidx"], ref["values"], M, K, b)
    dt = time.perf_counter() - t0
    s_x = X.dtype.itemsize
    r_ne = int(np.count_nonzero(np.diff(ref["rowptr"])))
    w = metrics.step_work(M, K, N, b, k, s_x, dY.dtype.itemsize, r_ne)
    return dt, w.bytes, w.wgrad_flops


def _oracle_rows_for(X, dY, b, keep, seconds):
    """Rows of the bounded sample: calibrate on 4 block rows, scale linearly."""
    Ms0 = min(4 * b, X.shape[0])
    t, _, _ = _oracle_step(X[:Ms0], dY[:Ms0], b, keep)
    rows = int(seconds / max(t, 1e-6) * Ms0) // b * b
    return max(b, min(rows, X.shape[0]))


def cpu_baseline(X, dY, c, seconds):
    Ms = _oracle_rows_for(X, dY, c["b"], c["keep"], seconds)
    dt, nbytes, _ = _oracle_step(np.ascontiguousarray(X[:Ms]), np.ascontiguousarray(dY[:Ms]), c["b"], c["keep"])
    return {"value": nbytes / dt / 1e9, "unit": "GB/s", "cores": 1, "kind": "oracle",
            "seconds": round(dt, 3),
            "sample": f"one oracle step (fp64 C, 1 thread: norms, qsort top-k, BSR, triple-loop dW, decompress) "
                      f"on the first {Ms} of {X.shape[0]} rows of the same seeded workload, "
                      f"k = nearest(keep * blocks of the slice)"}


def run_reference(a):
    """--impl reference: the CPU oracle as it stands, on the same config/metric."""
    from paper_2311_16883_b200.dist import env_world
    rank, _, world = env_world()
    if rank != 0:
        return 0
    c = workload(a)
    X, dY = host_inputs(c, 0, a.dtype)
    per_step = a.ref_budget / (a.steps + a.warmup)
    Ms = _oracle_rows_for(X, dY, c["b"], c["keep"], per_step)
    Xs, dYs = np.ascontiguousarray(X[:Ms]), np.ascontiguousarray(dY[:Ms])
    for _ in range(a.warmup):
        _oracle_step(Xs, dYs, c["b"], c["keep"])
    tot_t, tot_b = 0.0, 0.0
    for _ in range(a.steps):
        dt, nb, _ = _oracle_step(Xs, dYs, c["b"], c["keep"])
        tot_t += dt
        tot_b += nb
    value = tot_b / tot_t / 1e9
    sample = (f"each step: one oracle step on the first {Ms} of {c['M']} rows of the workload "
              f"(fp64 C, single thread)")
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": a.gpus,
           "steps": a.steps, "warmup": a.warmup, "ms_per_step": tot_t / a.steps * 1e3, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64 (oracle)", "data": "synthetic",
           "config": config_json(c, a, 1),
           "cpu_baseline": {"value": value, "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": sample},
           "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


# ----------------------------------------------------------------------------- clocks
_REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
            0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting", 0x10: "sync_boost"}


class ClockSampler:
    """NVML samples of the SM clock and clock-event reasons while the timed
    region runs (the recipe's nvidia-smi clocks line, at ms resolution)."""

    def __init__(self, device_index: int):
        self.samples, self.ok = [], False
        try:
            import pynvml
            pynvml.nvmlInit()
            import torch
            h = None
            try:
                p = torch.cuda.get_device_properties(device_index)
                bus = f"{p.pci_domain_id:08X}:{p.pci_bus_id:02X}:{p.pci_device_id:02X}.0"
                h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.nv, self.h = pynvml, h
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - no NVML
            self.err = repr(e)
        self._stop = threading.Event()

    def sample(self):
        if not self.ok:
            return
        try:
            mhz = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
            reasons = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            util = self.nv.nvmlDeviceGetUtilizationRates(self.h).gpu
            self.samples.append((mhz, reasons, util))
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self.sample()
            time.sleep(0.002)

    def start(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        self._t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "error": getattr(self, "err", "")}
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        mhz = [s[0] for s in self.samples]
        bits = 0
        for s in self.samples:
            bits |= s[1]
        reasons = sorted({name for bit, name in _REASONS.items() if bits & bit})
        return {"sm_mhz": statistics.median(mhz), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.samples), "sm_mhz_min": min(mhz)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


def ncu_traffic(kernel: str, c, a):
    """dram bytes per launch of `kernel` from the committed ncu --set full summary, if it
    was captured on this exact workload; else None."""
    if not os.path.exists(PROFILE_SUMMARY):
        return None
    with open(PROFILE_SUMMARY) as f:
        d = json.load(f)
    key = f"{kernel}|{a.config}|b{c['b']}|keep{c['keep']}|{a.dtype}|{a.prec}"
    e = d.get(key)
    return None if e is None else e.get("dram_bytes_per_launch")


# ----------------------------------------------------------------------------- the GPU arm
def run_native(a):
    import torch

    import paper_2311_16883_b200 as bp
    from paper_2311_16883_b200 import dist as D

    rank, local, world = D.init("nccl")
    if world != a.gpus:
        print(f"warning: --gpus {a.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    c = workload(a)
    M, K, N, b, keep = c["M"], c["K"], c["N"], c["b"], c["keep"]
    tdt = torch.bfloat16 if a.dtype == "bf16" else torch.float32
    s_x = s_dy = 2 if a.dtype == "bf16" else 4
    nblocks = bp.num_blocks(M, K, b)
    k = bp.keep_count(nblocks, keep)

    Xh, dYh = host_inputs(c, rank, a.dtype)

    def to_dev(h):
        t = torch.from_numpy(h.view(np.int16) if a.dtype == "bf16" else h)
        t = t.view(torch.bfloat16) if a.dtype == "bf16" else t
        return t.to(dev)

    X0, dY0 = to_dev(Xh), to_dev(dYh)
    Xs = [X0] + [X0.clone() for _ in range(NSETS - 1)]
    dYs = [dY0] + [dY0.clone() for _ in range(NSETS - 1)]
    bsrs = [bp.alloc_bsr(M, K, b, k, tdt, dev) for _ in range(NSETS)]
    dWs = [torch.empty(K, N, dtype=torch.float32, device=dev) for _ in range(NSETS)]
    Xds = [torch.empty(M, K, dtype=tdt, device=dev) for _ in range(NSETS)]

    phases = ["prune", "wgrad", "decompress"] if a.order == "pwd" else ["prune", "decompress", "wgrad"]

    def phase_fn(j, p):
        if p == "prune":
            return lambda: bp.prune(Xs[j], b, k=k, out=bsrs[j])
        if p == "wgrad":
            return lambda: bp.wgrad(bsrs[j], dYs[j], prec=a.prec, out=dWs[j])
        return lambda: bp.decompress(bsrs[j], out=Xds[j])

    # eager warm-up (allocates the cached workspace, sets kernel attributes)
    for j in range(NSETS):
        for p in phases:
            phase_fn(j, p)()
    torch.cuda.synchronize()
    ref_colidx = bsrs[0].colidx.clone()
    ref_dw = dWs[0].clone()

    lib = bp._lib.load()
    launches_per_step = {}
    use_graph = not a.no_graph
    step_graphs, phase_graphs = None, None
    REP = 4  # launches of one phase per input set inside a per-kernel timing graph

    def full_step(j):
        for p in phases:
            phase_fn(j, p)()

    if use_graph:
        try:
            s = torch.cuda.Stream(device=dev)
            s.wait_stream(torch.cuda.current_stream())
            # one graph per input set holding the whole step (prune -> wgrad -> decompress)
            step_graphs = []
            for j in range(NSETS):
                g = torch.cuda.CUDAGraph()
                n0 = lib.bsr_kernel_launches()
                with torch.cuda.graph(g, stream=s):
                    full_step(j)
                step_graphs.append(g)
                launches_per_step["step"] = lib.bsr_kernel_launches() - n0
            # per-kernel timing graphs: REP x NSETS back-to-back launches of one phase
            phase_graphs = {}
            for p in phases:
                g = torch.cuda.CUDAGraph()
                n0 = lib.bsr_kernel_launches()
                with torch.cuda.graph(g, stream=s):
                    for _ in range(REP):
                        for j in range(NSETS):
                            phase_fn(j, p)()
                launches_per_step[p] = (lib.bsr_kernel_launches() - n0) // (REP * NSETS)
                phase_graphs[p] = g
            torch.cuda.current_stream().wait_stream(s)
            for j in range(NSETS):
                step_graphs[j].replay()
            torch.cuda.synchronize()
            # the replays reproduce the eager result (dW: split-K partials summed in split order)
            if not torch.equal(bsrs[0].colidx, ref_colidx):
                raise RuntimeError("graph replay prune differs from eager launch")
            if not torch.allclose(dWs[0], ref_dw, rtol=1e-4, atol=1e-6):
                raise RuntimeError("graph replay dW differs from eager launch")
        except Exception as e:  # capture unsupported: launch eagerly
            print(f"note: CUDA-graph capture failed ({e!r}); launching eagerly", file=sys.stderr)
            use_graph, step_graphs, phase_graphs = False, None, None
    if not use_graph:
        for p in phases:
            n0 = lib.bsr_kernel_launches()
            phase_fn(0, p)()
            launches_per_step[p] = lib.bsr_kernel_launches() - n0
        launches_per_step["step"] = sum(launches_per_step[p] for p in phases)
        torch.cuda.synchronize()

    stream = torch.cuda.current_stream()

    def step(j):
        if use_graph:
            step_graphs[j].replay()
        else:
            full_step(j)
        if world > 1:
            D.allreduce_dw(dWs[j])

    for i in range(a.warmup):
        step(i % NSETS)
    torch.cuda.synchronize()

    # per-rank work of one step (R_ne from the device rowptr, outside the timed region)
    r_ne = int((bsrs[0].rowptr[1:] != bsrs[0].rowptr[:-1]).sum().item())
    work = metrics.step_work(M, K, N, b, k, s_x, s_dy, r_ne)

    # ---- the timed region: K whole steps, barrier + synchronize on both sides, clocks sampled
    t0e, t1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = ClockSampler(local)
    D.barrier()
    torch.cuda.synchronize()
    clk.start()
    t0e.record(stream)
    for i in range(a.steps):
        step(i % NSETS)
    t1e.record(stream)
    while not t1e.query():  # the GPU is still busy: keep sampling clocks
        time.sleep(0.0005)
    torch.cuda.synchronize()
    clk.stop()
    D.barrier()
    t_ms = t0e.elapsed_time(t1e)
    t_ms_max = D.max_over_ranks(t_ms, dev)
    bytes_all = D.sum_over_ranks(work.bytes, dev) * a.steps
    flops_all = D.sum_over_ranks(work.wgrad_flops, dev) * a.steps
    value = bytes_all / (t_ms_max * 1e-3) / 1e9

    # ---- per-kernel durations: each phase launched back to back (REP x NSETS launches per
    # graph replay, rotating input sets), CUDA events on the launching stream around the replays
    ph_ms = {}
    n_rep = max(3, min(200, a.steps // 4))
    for p in phases:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if use_graph:
            phase_graphs[p].replay()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(n_rep):
            if use_graph:
                phase_graphs[p].replay()
            else:
                for _ in range(REP):
                    for j in range(NSETS):
                        phase_fn(j, p)()
        e1.record(stream)
        torch.cuda.synchronize()
        ph_ms[p] = e0.elapsed_time(e1) / (n_rep * REP * NSETS)
    if world > 1:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        D.barrier()
        e0.record(stream)
        for i in range(n_rep):
            D.allreduce_dw(dWs[i % NSETS])
        e1.record(stream)
        torch.cuda.synchronize()
        ph_ms["allreduce"] = D.max_over_ranks(e0.elapsed_time(e1) / n_rep, dev)

    # ---- e2e: the public API with host buffers; H2D of the step's inputs and D2H of dW timed
    pin_X = torch.from_numpy(Xh.view(np.int16) if a.dtype == "bf16" else Xh).pin_memory()
    pin_dY = torch.from_numpy(dYh.view(np.int16) if a.dtype == "bf16" else dYh).pin_memory()
    if a.dtype == "bf16":
        pin_X, pin_dY = pin_X.view(torch.bfloat16), pin_dY.view(torch.bfloat16)
    pin_dW = torch.empty(K, N, dtype=torch.float32).pin_memory()
    e2e_steps = max(1, min(a.e2e_steps, a.steps))

    def e2e_step(j):
        Xs[j].copy_(pin_X, non_blocking=True)
        dYs[j].copy_(pin_dY, non_blocking=True)
        bp.prune(Xs[j], b, k=k, out=bsrs[j])
        bp.wgrad(bsrs[j], dYs[j], prec=a.prec, out=dWs[j])
        bp.decompress(bsrs[j], out=Xds[j])
        D.allreduce_dw(dWs[j])
        pin_dW.copy_(dWs[j], non_blocking=True)

    for i in range(3):
        e2e_step(i % NSETS)
    torch.cuda.synchronize()
    D.barrier()
    n_l0 = lib.bsr_kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(e2e_steps):
        e2e_step(i % NSETS)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_launches = lib.bsr_kernel_launches() - n_l0
    e2e_ms = D.max_over_ranks(e0.elapsed_time(e1), dev)
    e2e_value = D.sum_over_ranks(work.bytes, dev) * e2e_steps / (e2e_ms * 1e-3) / 1e9

    if rank != 0:
        D.finalize()
        return 0

    # ---- per-kernel numbers and the roofline of the dominant kernel
    pk = measured_peaks()
    tc_peak = pk["bf16_tflops"] * (0.5 if a.prec == "tf32" else 1.0)  # tf32 = bf16 x nominal 1.1/2.25
    per_kernel = {
        "prune": {"ms": ph_ms["prune"], "alg_bytes": work.prune_bytes,
                  "GB/s": work.prune_bytes / (ph_ms["prune"] * 1e-3) / 1e9},
        "wgrad": {"ms": ph_ms["wgrad"], "alg_bytes": work.wgrad_bytes, "flops": work.wgrad_flops,
                  "GB/s": work.wgrad_bytes / (ph_ms["wgrad"] * 1e-3) / 1e9,
                  "TFLOP/s": work.wgrad_flops / (ph_ms["wgrad"] * 1e-3) / 1e12},
        "decompress": {"ms": ph_ms["decompress"], "alg_bytes": work.decompress_bytes,
                       "GB/s": work.decompress_bytes / (ph_ms["decompress"] * 1e-3) / 1e9},
    }
    for kname in ("prune", "decompress"):
        per_kernel[kname]["hbm_frac"] = per_kernel[kname]["GB/s"] / pk["hbm_gbs"]
    wk = per_kernel["wgrad"]
    wk["tc_peak_tflops"] = tc_peak
    wk["tc_frac"] = wk["TFLOP/s"] / tc_peak
    t_roof = max(work.wgrad_flops / (tc_peak * 1e12), work.wgrad_bytes / (pk["hbm_gbs"] * 1e9))
    wk["roofline_frac"] = t_roof / (ph_ms["wgrad"] * 1e-3)
    wk["bound"] = metrics.wgrad_bound(work.wgrad_flops, work.wgrad_bytes, tc_peak, pk["hbm_gbs"])
    if world > 1:
        bus = metrics.allreduce_bus_bytes(K, N, world)
        per_kernel["allreduce"] = {"ms": ph_ms["allreduce"], "bus_bytes": bus,
                                   "busbw_GB/s": bus / (ph_ms["allreduce"] * 1e-3) / 1e9}
    dom = max(("prune", "wgrad", "decompress"), key=lambda n: per_kernel[n]["ms"])
    dk = per_kernel[dom]
    if dom == "wgrad" and wk["bound"] == "tensor":
        roof = {"bound": "tensor", "achieved": wk["TFLOP/s"], "peak": tc_peak, "unit": "TFLOP/s",
                "frac": wk["tc_frac"]}
    else:
        roof = {"bound": "hbm", "achieved": dk["GB/s"], "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": dk["GB/s"] / pk["hbm_gbs"]}
    traffic = ncu_traffic(dom, c, a)
    roof.update({"kernel": dom, "traffic": traffic, "alg_bytes_per_launch": dk["alg_bytes"],
                 "launch_ms": dk["ms"], "peak_source": f"{pk['source']} (MEASURED_PEAKS.json)"
                 if pk["source"] == "measured" else "fallback (B200_PROFILING.md)"})

    per_step_launches = launches_per_step["step"]
    out = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": t_ms_max / a.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": ("bf16" if a.dtype == "bf16" else "f32") + f" (dW {a.prec})", "data": "synthetic",
        "config": config_json(c, a, world),
        "roofline": roof,
        "kernels": per_kernel,
        "wgrad_tflops": wk["TFLOP/s"],
        "prune_gbs": per_kernel["prune"]["GB/s"],
        "act_bytes_saved": {"bytes_per_layer": metrics.act_bytes_saved(M, K, b, k, s_x),
                            "frac": metrics.act_bytes_saved(M, K, b, k, s_x) / (s_x * M * K),
                            "bsr_bytes": metrics.bsr_bytes(M, b, k, s_x)},
        "work_per_step": {"alg_bytes": work.bytes, "wgrad_flops": work.wgrad_flops, "k": k, "nblocks": nblocks,
                          "r_ne": r_ne, "wgrad_flops_all_ranks_per_s": flops_all / (t_ms_max * 1e-3)},
        "launch": "one CUDA graph per step (prune -> wgrad -> decompress)" if use_graph else "eager",
        "kernel_timing": "per phase: back-to-back launches inside one graph over the rotating input sets, "
                         "CUDA events around the replays (a second timed region after the step loop)",
        "gpu_launches": per_step_launches * a.steps,
        "gpu_launches_per_step": launches_per_step,
        "clocks": clk.summary(),
        "e2e": {"value": e2e_value, "unit": "GB/s", "h2d_bytes_per_step": int(Xh.nbytes + dYh.nbytes),
                "d2h_bytes_per_step": int(K * N * 4), "steps": e2e_steps, "ms_per_step": e2e_ms / e2e_steps,
                "gpu_launches": int(e2e_launches),
                "how": "pinned host X, dY -> device, bp.prune/wgrad/decompress (C-ABI), [all-reduce], dW -> pinned host"},
        "peaks": pk,
    }
    if not a.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(Xh, dYh, c, a.cpu_seconds)
    print(json.dumps(out), flush=True)
    D.finalize()
    return 0


def main():
    a = parse()
    if a.impl == "reference":
        return run_reference(a)
    return run_native(a)


if __name__ == "__main__":
    sys.exit(main())
