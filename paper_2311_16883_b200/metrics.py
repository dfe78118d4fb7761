"""Algorithmic work of each step of the hot path -- what the method
must move or compute, not what an implementation happens to move.

These are pure host formulas used by bench.py to turn measured times into
GB/s, TFLOP/s and roofline fractions.  Notation: M x K activation X with
element size s_x, b x b blocks, k kept blocks, dY M x N with element size s_dy,
R_ne = block rows that keep at least one block (read from rowptr), P ranks.
"""
from __future__ import annotations

from dataclasses import dataclass


def bsr_bytes(M: int, b: int, k: int, s_x: int) -> int:
    """Stored BSR bytes: values k*b*b*s_x + colidx 4k + rowptr 4(M/b+1)
    (BJ closed form with s_x = 4)."""
    return k * b * b * s_x + 4 * k + 4 * (M // b + 1)


def prune_bytes(M: int, K: int, b: int, k: int, s_x: int) -> int:
    """a1-a4: read X once, write the BSR.  k = 0 writes rowptr only (X need
    not be read); the norm array, histograms and per-CTA counts are
    implementation overhead and count against the achieved fraction."""
    if k == 0:
        return 4 * (M // b + 1)
    return s_x * M * K + bsr_bytes(M, b, k, s_x)


def decompress_bytes(M: int, K: int, b: int, k: int, s_x: int) -> int:
    """a5: read the BSR, write the dense M x K result."""
    return bsr_bytes(M, b, k, s_x) + s_x * M * K


def wgrad_flops(b: int, k: int, N: int) -> int:
    """a6: 2 * k * b^2 * N multiply-adds over the kept blocks only."""
    return 2 * k * b * b * N


def wgrad_bytes(M: int, K: int, b: int, k: int, N: int, s_x: int, s_dy: int, r_ne: int,
                accumulate: bool = False) -> int:
    """a6: read the BSR, the dY rows of non-empty block rows (b*N each), write
    dW (K x N fp32; read it too when accumulating)."""
    return bsr_bytes(M, b, k, s_x) + s_dy * b * N * r_ne + 4 * K * N * (2 if accumulate else 1)


def allreduce_bus_bytes(K: int, N: int, P: int) -> float:
    """a7: ring / NVLS bus bytes of an fp32 K x N all-reduce over P ranks."""
    return 0.0 if P <= 1 else 2.0 * (P - 1) / P * 4 * K * N


def act_bytes_saved(M: int, K: int, b: int, k: int, s_x: int) -> int:
    """Dense activation bytes minus the stored BSR bytes (the paper's memory
    saving, tab:memory_saved P:L526-552, b x b analogue)."""
    return s_x * M * K - bsr_bytes(M, b, k, s_x)


@dataclass
class StepWork:
    """Algorithmic work of one step (prune -> wgrad -> decompress) on one rank."""
    prune_bytes: int
    wgrad_bytes: int
    wgrad_flops: int
    decompress_bytes: int

    @property
    def bytes(self) -> int:
        return self.prune_bytes + self.wgrad_bytes + self.decompress_bytes


def step_work(M: int, K: int, N: int, b: int, k: int, s_x: int, s_dy: int, r_ne: int) -> StepWork:
    return StepWork(prune_bytes(M, K, b, k, s_x), wgrad_bytes(M, K, b, k, N, s_x, s_dy, r_ne),
                    wgrad_flops(b, k, N), decompress_bytes(M, K, b, k, s_x))


def wgrad_bound(flops: float, nbytes: float, peak_tflops: float, peak_gbs: float) -> str:
    """Which roofline bounds a dW launch: 'tensor' if the tensor-core time
    exceeds the HBM time, else 'hbm'."""
    return "tensor" if flops / (peak_tflops * 1e12) >= nbytes / (peak_gbs * 1e9) else "hbm"
