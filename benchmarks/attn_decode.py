"""Paged decode attention microbenchmark (the SURVEY §8d headline measurement).

Llama-3-8B attention shape (32 q heads, 8 kv heads, head_dim 128), private KV
per sequence behind randomly permuted block tables, so algorithmic bytes =
unique HBM bytes = B * ctx * 8 * 128 * 2 (K+V) * 2 B per layer launch. The
cache spans many layers' worth of blocks (> L2) and successive launches walk
different layers, so nothing is L2-resident. Prints one JSON line per config.
"""

from __future__ import annotations

import json
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2510_14126_b200 import ops  # noqa: E402


def run(B: int, ctx: int, layers: int = 8, iters: int = 20, hkv: int = 8, group: int = 4) -> dict:
    dev = torch.device("cuda")
    hq = hkv * group
    nb_seq = (ctx + 15) // 16
    nb = B * nb_seq + 16
    cache = torch.empty(layers, 2, nb, hkv, 16, 128, dtype=torch.bfloat16, device=dev)
    cache.normal_()
    perm = torch.randperm(nb, generator=torch.Generator().manual_seed(0))[: B * nb_seq]
    table = perm.view(B, nb_seq).to(torch.int32).to(dev)
    row = torch.arange(B, dtype=torch.int32, device=dev)
    pre = torch.zeros(B, dtype=torch.int32, device=dev)
    kvl = torch.full((B,), ctx, dtype=torch.int32, device=dev)
    q = torch.randn(B, hq, 128, device=dev).to(torch.bfloat16)
    ms_ = ops.decode_splits(0, ctx)
    o_part = torch.empty(B * ms_ * hq * 128, device=dev)
    lse = torch.empty(B * ms_ * hq, device=dev)
    out = torch.empty(B, hq, 128, dtype=torch.bfloat16, device=dev)
    kvmap = ops.kv_map(cache.view(-1, 128))
    plane = nb * hkv * 16

    def launch(layer):
        ops.paged_decode_attn(kvmap, q, table, row, pre, kvl, B, hkv, group, 2 * layer * plane,
                              (2 * layer + 1) * plane, 1 / math.sqrt(128), o_part, lse, ms_, out)

    for i in range(3):
        launch(i % layers)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(iters):
        launch(i % layers)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    nbytes = B * ctx * hkv * 128 * 2 * 2 + 2 * B * hq * 128 * 2
    return {"B": B, "ctx": ctx, "ms": ms, "GBps": nbytes / ms / 1e6, "bytes": nbytes}


if __name__ == "__main__":
    peak = 6537.3
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                     "MEASURED_PEAKS.json")
    if os.path.exists(p):
        peak = json.load(open(p))["hbm_gbs"]
    for B, ctx in [(64, 1300), (128, 1300), (256, 1300), (32, 8900), (256, 8900), (8, 1300)]:
        r = run(B, ctx, layers=8 if ctx < 4000 else 2)
        r["frac_of_measured_hbm"] = r["GBps"] / peak
        print(json.dumps(r), flush=True)
