"""End-to-end logits error at the Llama-3-8B shape, 1 and 2 layers: the GPU path against
the CPU oracle that rounds to bf16 at the GPU's storage points (oracle/decoder_ref.py)
AND against the exact (no rounding, fp32) decoder on the same weights, with that
oracle's own distance to the exact decoder for scale. One 1000-token prefix, a
200-token prompt, 8 teacher-forced decode steps.  Usage (GPU box): python tools/diag_8b_e2e.py"""

from __future__ import annotations

import dataclasses
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle.decoder_ref import RefDecoder  # noqa: E402
from paper_2510_14126_b200.config import LLAMA3_8B  # noqa: E402
from paper_2510_14126_b200.model import DecodeTok, GpuWorker, PrefillSeq, StepPlan  # noqa: E402


def rel(a, b):
    a, b = a.double().cpu().reshape(-1), b.double().cpu().reshape(-1)
    return float((a - b).norm() / b.norm())


for L in (1, 2):
    cfg = dataclasses.replace(LLAMA3_8B, name=f"8b-{L}L", n_layers=L)
    P, p, nb = 1000, 200, 200
    w = GpuWorker(cfg, "cuda", n_blocks=nb, n_rows=8, row_cols=nb, max_tokens=2048, max_out=16,
                  hist_cols=64, max_seq_tokens=1400)
    w.full_logits = True
    npb = (P + 15) // 16
    w.table[0, :npb] = torch.arange(npb, dtype=torch.int32)
    w.table[1, :npb] = torch.arange(npb, dtype=torch.int32)
    w.table[1, npb:npb + 20] = torch.arange(npb, npb + 20, dtype=torch.int32)
    g = np.random.default_rng(0)
    pre = g.integers(0, cfg.vocab, P).astype(np.int32)
    prm = g.integers(0, cfg.vocab, p).astype(np.int32)
    w.forward(StepPlan(prefill=[PrefillSeq(0, 0, P, pre, out_row=0)]))
    w.forward(StepPlan(prefill=[PrefillSeq(1, P, P + p, prm, out_row=1)]))
    gl = [w.logits[0].cpu().clone()]
    toks = [int(w.slot_tok[1])]
    for k in range(8):
        w.forward(StepPlan(decode=[DecodeTok(1, P, P + p + k + 1, hist_pos=k + 1, prefix_key=0)]))
        gl.append(w.logits[0].cpu().clone())
        toks.append(int(w.slot_tok[1]))
    torch.cuda.synchronize()
    ws = w.oracle_weights()
    res = {}
    for name, exact in (("bf16-oracle", False), ("exact", True)):
        dec = RefDecoder(cfg.to_ref(), ws, max_pos=1400, exact=exact)
        s = dec.new_seq()
        s.extend(pre, "none")
        out = [s.extend(prm)]
        for t in toks[:-1]:
            out.append(s.extend([t]))
        res[name] = out
    for k in range(len(gl)):
        print(f"L={L} pos {k}: gpu vs bf16-oracle {rel(gl[k], res['bf16-oracle'][k]):.2e}  "
              f"gpu vs exact {rel(gl[k], res['exact'][k]):.2e}  bf16-oracle vs exact "
              f"{rel(res['bf16-oracle'][k], res['exact'][k]):.2e}", flush=True)
    del w
    torch.cuda.empty_cache()
