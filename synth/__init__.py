"""Seeded synthetic inputs shared by the tests, the oracle legs and bench.py.

This module holds NO arithmetic of the method (no norms, no selection, no
packing, no products): it only draws random activations/gradients with the
shapes and value distributions of the paper's workloads, and names the
BASELINE.json configurations.  Recipe:

* F_aff  -- post-affine residual stream (input of fc1 and of the cross-patch
  layer): x = sigma_s * (alpha_c * z + beta_c), z ~ N(0,1),
  alpha_c ~ LogNormal(0, 0.5), beta_c ~ N(0, 0.1^2) per channel,
  sigma_s ~ LogNormal(0, 0.25) per sample of ``tokens`` rows (the "darker
  image" effect).
* F_gelu -- input of fc2: x = sigma_s * gelu_tanh(alpha_c * z + beta_c),
  beta_c ~ N(0, 0.5^2).
* F_unif -- U(-1, 1) (bandwidth sweeps).
* dY     -- i.i.d. N(0, 1e-2^2).
* ints   -- integers in [lo, hi] (exact fp32 sums of squares: tie tests).

Seeds: 231116883 + 1000*config_id + 10*layer_id + rank.
"""
from __future__ import annotations

import numpy as np

SEED_BASE = 231116883
TOKENS = 196  # ResMLP patches per image (14 x 14)


def seed_for(config_id: int, layer_id: int = 0, rank: int = 0) -> int:
    return SEED_BASE + 1000 * config_id + 10 * layer_id + rank


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def _per_sample(M: int, tokens: int, rng, sigma: float) -> np.ndarray:
    n_samples = -(-M // tokens)
    s = rng.lognormal(0.0, sigma, size=n_samples).astype(np.float64)
    return np.repeat(s, tokens)[:M, None]


def f_aff(M: int, K: int, seed: int, tokens: int = TOKENS) -> np.ndarray:
    rng = _rng(seed)
    alpha = rng.lognormal(0.0, 0.5, size=K)
    beta = rng.normal(0.0, 0.1, size=K)
    sig = _per_sample(M, tokens, rng, 0.25)
    z = rng.standard_normal((M, K), dtype=np.float32)
    return (sig * (alpha * z + beta)).astype(np.float32)


def _gelu_tanh(v):
    return 0.5 * v * (1.0 + np.tanh(0.7978845608028654 * (v + 0.044715 * v ** 3)))


def f_gelu(M: int, K: int, seed: int, tokens: int = TOKENS) -> np.ndarray:
    rng = _rng(seed)
    alpha = rng.lognormal(0.0, 0.5, size=K)
    beta = rng.normal(0.0, 0.5, size=K)
    sig = _per_sample(M, tokens, rng, 0.25)
    z = rng.standard_normal((M, K), dtype=np.float32)
    return (sig * _gelu_tanh(alpha * z + beta)).astype(np.float32)


def f_unif(M: int, K: int, seed: int) -> np.ndarray:
    return _rng(seed).uniform(-1.0, 1.0, size=(M, K)).astype(np.float32)


def grad_out(M: int, N: int, seed: int, scale: float = 1e-2) -> np.ndarray:
    z = _rng(seed ^ 0x5EED).standard_normal((M, N), dtype=np.float32)
    return (z * np.float32(scale)).astype(np.float32)


def ints(M: int, K: int, seed: int, lo: int = -2, hi: int = 2) -> np.ndarray:
    return _rng(seed).integers(lo, hi + 1, size=(M, K)).astype(np.float32)


def block_count_ints(M: int, K: int, b: int, counts, seed: int) -> np.ndarray:
    """Tie family at full size: every b x b block holds exactly c entries of +-1
    (the rest 0), c drawn uniformly from `counts`, so every block's sum of squares
    is the integer c -- exact in fp32 and in fp64, with few distinct values, i.e.
    thousands of blocks tied on each value."""
    rng = _rng(seed)
    nbr, nbc = M // b, K // b
    c = rng.choice(np.asarray(counts), size=(nbr, nbc))
    r = rng.random((nbr, nbc, b * b))
    order = np.argsort(r, axis=2)  # a random permutation of the block's slots
    slots = np.arange(b * b)[None, None, :]
    sel = np.zeros((nbr, nbc, b * b), dtype=bool)
    np.put_along_axis(sel, order, slots < c[..., None], axis=2)
    sign = np.where(rng.random((nbr, nbc, b * b)) < 0.5, -1.0, 1.0).astype(np.float32)
    blk = (sel * sign).reshape(nbr, nbc, b, b).astype(np.float32)
    return np.ascontiguousarray(blk.transpose(0, 2, 1, 3).reshape(M, K))


def to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """fp32 -> bfloat16 bit patterns (uint16), round-to-nearest-even (data prep)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    rounded = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return rounded.astype(np.uint16)


def bf16_bits_to_f32(h: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(h, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


# BASELINE.json "configs" (ids 1..5 = C1..C5)
CONFIGS = {
    "C1": dict(id=1, M=256, K=256, N=256, b=16, keep=0.5, family="aff",
               desc="single linear layer: X 256x256 fp32, dY 256x256, block 16, keep 50%"),
    "C2": dict(id=2, M=25088, K=384, N=1536, b=32, keep=0.5, family="aff",
               desc="ResMLP-S12 fc1: X 25088x384 (batch 128 x 196 tokens), dY 25088x1536, block 32, keep 50%"),
    "C3_fc2": dict(id=3, M=25088, K=1536, N=384, b=32, keep=0.5, family="gelu",
                   desc="ResMLP-S12 fc2: X 25088x1536, dY 25088x384"),
    "C4_fc1": dict(id=4, M=200704, K=768, N=3072, b=32, keep=0.5, family="aff",
                   desc="ResMLP-B24 fc1 at batch 1024 (sharded over ranks)"),
    "C4_fc2": dict(id=4, M=200704, K=3072, N=768, b=32, keep=0.5, family="gelu",
                   desc="ResMLP-B24 fc2 at batch 1024 (sharded over ranks)"),
}


def activation(family: str, M: int, K: int, seed: int) -> np.ndarray:
    if family == "aff":
        return f_aff(M, K, seed)
    if family == "gelu":
        return f_gelu(M, K, seed)
    if family == "unif":
        return f_unif(M, K, seed)
    if family == "ints":
        return ints(M, K, seed)
    raise ValueError(family)
