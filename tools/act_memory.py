#!/usr/bin/env python
"""Measured activation memory of ResMLP-S12-shaped MLP stacks with SparseLinear
vs nn.Linear (the b x b analogue of the paper's tab:memory_saved).

Each of the 12 blocks is fc1 (384 -> 1536) -> GELU -> fc2 (1536 -> 384) with a
residual add, on batch x 196 tokens.  The saved-for-backward memory is read from
torch.cuda.memory_allocated() after the forward pass (weights, the input and the
output excluded), once with nn.Linear and once with SparseLinear(s, b).  The
cross-patch layer (196 tokens) is not b x b prunable for b >= 8 (DESIGN R10).

    python tools/act_memory.py [--batch 32] [--out profiles/act_memory.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2311_16883_b200 import SparseLinear  # noqa: E402
from paper_2311_16883_b200 import metrics  # noqa: E402


class Block(torch.nn.Module):
    def __init__(self, dim, hidden, lin):
        super().__init__()
        self.fc1, self.fc2 = lin(dim, hidden), lin(hidden, dim)

    def forward(self, x):
        return x + self.fc2(torch.nn.functional.gelu(self.fc1(x)))


def saved_bytes(model, x):
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    y = model(x)
    torch.cuda.synchronize()
    held = torch.cuda.memory_allocated() - base - y.numel() * y.element_size()
    y.sum().backward()
    return held


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "act_memory.json"))
    a = ap.parse_args()
    dev = torch.device("cuda")
    dim, hidden, depth, tokens = 384, 1536, 12, 196
    M = a.batch * tokens
    x = torch.randn(M, dim, device=dev, requires_grad=True)
    dense = torch.nn.Sequential(*[Block(dim, hidden, lambda i, o: torch.nn.Linear(i, o, device=dev))
                                  for _ in range(depth)])
    d_bytes = saved_bytes(dense, x)
    rows = []
    for s, b in [(0.6, 16), (0.6, 32), (0.7, 16), (0.7, 32), (0.8, 16), (0.8, 32), (0.5, 32), (0.9, 64)]:
        if M % b:
            continue
        sparse = torch.nn.Sequential(*[Block(dim, hidden, lambda i, o: SparseLinear(i, o, s, b, device=dev))
                                       for _ in range(depth)])
        s_bytes = saved_bytes(sparse, x)
        k1 = round((1 - s) * (M // b) * (dim // b))
        k2 = round((1 - s) * (M // b) * (hidden // b))
        predicted = depth * (metrics.act_bytes_saved(M, dim, b, k1, 4) + metrics.act_bytes_saved(M, hidden, b, k2, 4))
        rows.append({"sparsity": s, "block": b, "saved_MiB_dense": d_bytes / 2**20, "saved_MiB_sparse": s_bytes / 2**20,
                     "delta_MiB": (s_bytes - d_bytes) / 2**20, "delta_pct": 100.0 * (s_bytes - d_bytes) / d_bytes,
                     "predicted_delta_MiB": -predicted / 2**20})
        del sparse
        torch.cuda.empty_cache()
    out = {"model": "ResMLP-S12 MLP stack (12 x fc1 384->1536, GELU, fc2 1536->384, residual)",
           "batch": a.batch, "tokens": tokens, "rows": rows,
           "note": "fc1 and fc2 inputs pruned b x b (the cross-patch layer is not b x b prunable at 196 tokens); "
                   "paper tab:memory_saved uses 1 x b blocks on all 36 linear layers at batch 32"}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    for r in rows:
        print(f"s={r['sparsity']:.1f} b={r['block']:2d}: dense {r['saved_MiB_dense']:.1f} MiB -> sparse "
              f"{r['saved_MiB_sparse']:.1f} MiB  delta {r['delta_MiB']:+.1f} MiB ({r['delta_pct']:+.1f}%), "
              f"closed form {r['predicted_delta_MiB']:+.1f} MiB")


if __name__ == "__main__":
    main()
