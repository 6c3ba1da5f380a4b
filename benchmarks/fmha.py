"""tcgen05 flash-attention microbenchmark (prefill and shared-prefix cascade shapes).

Llama-3-8B heads (32 q / 8 kv, head_dim 128). Reports TFLOP/s of useful work
(4 * rows * keys * 128 per kv head, causal keys counted once).
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

HKV, GROUP = 8, 4
HQ = HKV * GROUP


def _cache(nb):
    c = torch.zeros(1, 2, nb, HKV, 16, 128, dtype=torch.bfloat16, device="cuda")
    c.normal_()
    return c


def _time(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def prefill(prefix: int, prompts: list[int]) -> dict:
    dev = torch.device("cuda")
    npb = (prefix + 15) // 16
    nbs = [npb + (p + 15) // 16 for p in prompts]
    nb = npb + sum(nbs) + 16
    cache = _cache(nb)
    rows = len(prompts)
    table = torch.zeros(rows, max(nbs), dtype=torch.int32)
    nxt = npb
    for i, p in enumerate(prompts):
        npr = (p + 15) // 16
        table[i, :npb] = torch.arange(npb)
        table[i, npb:npb + npr] = torch.arange(nxt, nxt + npr)
        nxt += npr
    table = table.to(dev)
    T = sum(prompts)
    q = torch.randn(T, HQ, 128, device=dev).to(torch.bfloat16)
    out = torch.empty_like(q)
    qs = np.concatenate([[0], np.cumsum(prompts)[:-1]])
    d = lambda a: torch.as_tensor(np.asarray(a, np.int32), device=dev)
    args = (table, d(range(rows)), d([prefix] * rows), d([prefix + p for p in prompts]), d(qs),
            d(prompts), rows, max(prompts), HKV, GROUP, 0, nb * HKV * 16, 1 / math.sqrt(128))
    kvmap = ops.kv_map(cache.view(-1, 128))
    qmap = ops.QMap(q, HQ, GROUP)
    ms = _time(lambda: ops.fmha_prefill(kvmap, qmap, out, *args))
    ms_mma = _time(lambda: ops.paged_prefill_attn(kvmap, q, out, *args))
    keys = sum(p * prefix + p * (p + 1) / 2 for p in prompts)
    flops = 4.0 * keys * 128 * HQ
    return {"kind": "prefill", "prefix": prefix, "prompts": len(prompts), "tokens": T,
            "ms": ms, "tflops": flops / ms / 1e9, "mma_sync_ms": ms_mma}


def cascade(prefix: int, n_calls: int, groups: int = 2, pslots: int | None = None) -> dict:
    dev = torch.device("cuda")
    npb = (prefix + 15) // 16
    nb = groups * npb + 16
    cache = _cache(nb)
    table = torch.zeros(groups, npb, dtype=torch.int32)
    for g in range(groups):
        table[g] = torch.arange(g * npb, (g + 1) * npb)
    table = table.to(dev)
    B = groups * n_calls
    q = torch.randn(B, HQ, 128, device=dev).to(torch.bfloat16)
    pslots = pslots or (npb + 15) // 16
    o_part = torch.empty(B * (pslots + 1) * HQ * 128, device=dev)
    lse = torch.empty(B * (pslots + 1) * HQ, device=dev)
    d = lambda a: torch.as_tensor(np.asarray(a, np.int32), device=dev)
    kvmap = ops.kv_map(cache.view(-1, 128))
    qmap = ops.QMap(q, HQ, GROUP)
    lib = ops.lib()
    grow, gpl, gfi, gco = d(range(groups)), d([prefix] * groups), d(
        [g * n_calls for g in range(groups)]), d([n_calls] * groups)

    def run():
        ops._check(lib.cortex_fmha_cascade_tc(
            kvmap.ptr, qmap.ptr, table.data_ptr(), table.stride(0), grow.data_ptr(),
            gpl.data_ptr(), gfi.data_ptr(), gco.data_ptr(), groups, n_calls, pslots, HKV, GROUP,
            0, nb * HKV * 16, 1 / math.sqrt(128), o_part.data_ptr(), lse.data_ptr(), pslots + 1,
            torch.cuda.current_stream().cuda_stream), "cascade")

    ms = _time(run)
    flops = 4.0 * B * HQ * prefix * 128
    return {"kind": "cascade", "prefix": prefix, "calls": B, "slots": pslots, "ms": ms,
            "tflops": flops / ms / 1e9}


if __name__ == "__main__":
    # both tcgen05 kernels: two Q tiles per CTA (default) and one
    for q2 in (1, 0, -1):
        ops.fmha_set_2q(q2)
        for r in (prefill(1000, [200] * 2), prefill(1000, [200] * 8), prefill(0, [1000]),
                  prefill(0, [8192]), cascade(1000, 115), cascade(8192, 128)):
            r["q_tiles_per_cta"] = {1: 2, 0: 1, -1: "auto"}[q2]
            print(json.dumps(r), flush=True)
    ops.fmha_set_2q(1)
    if "--slots" in sys.argv:  # the bench's cascade shapes: prefix slots x kernel
        for prefix, n in ((1000, 108), (8192, 128)):
            for sl in (1, 2, 3, 4, 6, 8):
                for q2 in (0, 1):
                    ops.fmha_set_2q(q2)
                    r = cascade(prefix, n, pslots=sl)
                    r["q_tiles_per_cta"] = 2 if q2 else 1
                    print(json.dumps(r), flush=True)
        ops.fmha_set_2q(1)
