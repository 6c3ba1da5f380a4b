"""Cluster split-K GEMM (gemm_splitk.cu) vs the 2-SM whole-tile kernel at decode M: time
per launch for each forced (token tiles mt, split count ks) with <= 74 pairs, and the
automatic plan.  python benchmarks/gemm_sk_sweep.py [M ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from gemm import SHAPES, bench  # noqa: E402
from paper_2510_14126_b200 import _lib, ops  # noqa: E402

for M in [int(a) for a in sys.argv[1:]] or [200, 256]:
    for name in ("qkv", "o", "down"):
        N, K = SHAPES[name]
        row = {"M": M, "name": name}
        ops.gemm_set_mode(1)
        row["1sm"] = round(bench(M, name, residual=name != "qkv")["ms"] * 1e3, 1)
        ops.gemm_set_mode(2)
        row["2sm"] = round(bench(M, name, residual=name != "qkv")["ms"] * 1e3, 1)
        ops.gemm_set_mode(3)
        ks, tn, mt, _ = ops.splitk_plan(M, N, K)
        row["auto"] = f"mt{mt}ks{ks}tn{tn}"
        row["auto_us"] = round(bench(M, name, residual=name != "qkv")["ms"] * 1e3, 1)
        for m in (1, 2, 3):
            for k in (2, 3, 4):
                if (N // 256) * m * k > 74:
                    continue
                _lib.set_knob("SK_KS", k)
                _lib.set_knob("SK_MT", m)
                if ops.splitk_plan(M, N, K)[0] == k:
                    row[f"mt{m}ks{k}"] = round(bench(M, name, residual=name != "qkv")["ms"] * 1e3, 1)
        _lib.set_knob("SK_KS", -1)
        _lib.set_knob("SK_MT", -1)
        ops.gemm_set_mode(0)
        print(json.dumps(row), flush=True)
