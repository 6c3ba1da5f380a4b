"""tcgen05 GEMM microbenchmark on the decoder's projection shapes (Llama-3-8B).

For each (M, N, K): our kernel vs torch.matmul (cuBLAS, for context only),
TFLOP/s and weight-streaming GB/s. Weights for successive launches rotate over
enough copies to exceed L2, as in a real decode step.
"""

from __future__ import annotations

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2510_14126_b200 import ops  # noqa: E402

SHAPES = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (28672, 4096), "down": (4096, 14336),
          "lm_head": (128256, 4096)}


def bench(M: int, name: str, iters: int = 20, residual: bool = False) -> dict:
    dev = torch.device("cuda")
    N, K = SHAPES[name]
    copies = max(2, int(300e6 // (N * K * 2)) + 1)
    ws = [torch.randn(N, K, device=dev).to(torch.bfloat16) * 0.05 for _ in range(copies)]
    maps = [ops.weight_map(w) for w in ws]
    x = torch.randn(max(M, 32), K, device=dev).to(torch.bfloat16)
    xm = ops.act_map(x)
    am = name == "lm_head"  # the product's lm_head: greedy-argmax partials, no logits
    out = (torch.empty(M, N // 128, device=dev, dtype=torch.int64) if am else
           torch.empty(M, N, device=dev, dtype=torch.float32 if residual else torch.bfloat16))
    res = torch.randn(M, N, device=dev) if residual else None
    gw = ops.GemmWorkspace(dev)
    for i in range(3):
        ops.gemm(maps[i % copies], xm, M, out, gw, residual=res, argmax=am)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(iters):
        ops.gemm(maps[i % copies], xm, M, out, gw, residual=res, argmax=am)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    # cuBLAS reference point
    e0.record()
    for i in range(iters):
        torch.matmul(x[:M], ws[i % copies].T)
    e1.record()
    torch.cuda.synchronize()
    ms_cublas = e0.elapsed_time(e1) / iters
    flops = 2.0 * M * N * K
    return {"M": M, "name": name, "residual": residual, "ms": ms, "tflops": flops / ms / 1e9,
            "weight_GBps": N * K * 2 / ms / 1e6, "cublas_ms": ms_cublas,
            "cublas_tflops": flops / ms_cublas / 1e9, "splits": ops.gemm_splits(M, N, K),
            "path": ops.gemm_path(M, N, K), "tile2": ops.lib().cortex_gemm2_tile(M, N, K)}


if __name__ == "__main__":
    if os.environ.get("GEMM_MODE"):  # 1: 1-SM, 2: 2-SM whole tiles, 3: cluster split-K
        ops.gemm_set_mode(int(os.environ["GEMM_MODE"]))
    from paper_2510_14126_b200 import _lib

    for kv in filter(None, os.environ.get("CORTEX_KNOBS", "").split(",")):  # NAME=V,...
        k, v = kv.split("=")
        _lib.set_knob(k, int(v))
    Ms = [int(a) for a in sys.argv[1:]] or [32, 128, 256, 700, 2048, 4096]
    for M in Ms:
        for name in (os.environ.get("GEMM_SHAPES") or ",".join(SHAPES)).split(","):
            print(json.dumps(bench(M, name, residual=name in ("o", "down"))), flush=True)
