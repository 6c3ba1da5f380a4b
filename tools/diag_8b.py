"""Numerics diagnosis at the Llama-3-8B shape (one layer): where does the GPU step depart
from the CPU fp32 oracle? Runs one prefill (1000-token prefix, then a 200-token prompt
behind it, then 4 decode steps) through GpuWorker with n_layers = 1 and compares each
stage against a float64 recomputation from the GPU's OWN inputs of that stage:
  qkv+rope (q vs the GEMM of the host-recomputed attn_norm output), attention (GPU attn vs
  exact softmax attention over the GPU's q and cached K/V), the MLP / residual (final x).
Usage (GPU box): python tools/diag_8b.py
"""

from __future__ import annotations

import dataclasses
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2510_14126_b200.config import BLOCK_TOKENS, HEAD_DIM, LLAMA3_8B  # noqa: E402
from paper_2510_14126_b200.model import GpuWorker, PrefillSeq, StepPlan, DecodeTok  # noqa: E402
from paper_2510_14126_b200.engine import EngineSlice, TokenSource  # noqa: E402
from paper_2510_14126_b200 import ops  # noqa: E402


def rel(a, b):
    a, b = a.double().cpu(), b.double().cpu()
    return float((a - b).norm() / b.norm())


def main():
    from paper_2510_14126_b200 import _lib

    for a in sys.argv[1:]:  # --knob NAME=VALUE (cortex_dev.h knobs)
        if "=" in a:
            k, v = a.split("=")
            _lib.set_knob(k, int(v))
    cfg = dataclasses.replace(LLAMA3_8B, name="8b-1L", n_layers=1)
    dev = torch.device("cuda")
    P, p = 1000, 200
    nb = 200
    w = GpuWorker(cfg, dev, n_blocks=nb, n_rows=8, row_cols=nb, max_tokens=2048, max_out=16,
                  hist_cols=64, max_seq_tokens=1400)
    w.full_logits = True
    # row 0 = prefix (blocks 0..62), row 1 = call (prefix blocks then private blocks)
    npb = (P + 15) // 16
    w.table[0, :npb] = torch.arange(npb, dtype=torch.int32)
    w.table[1, :npb] = torch.arange(npb, dtype=torch.int32)
    w.table[1, npb:npb + 20] = torch.arange(npb, npb + 20, dtype=torch.int32)
    g = np.random.default_rng(0)
    pre = g.integers(0, cfg.vocab, P).astype(np.int32)
    prm = g.integers(0, cfg.vocab, p).astype(np.int32)
    wt = {k: v.float().cpu() for k, v in w.oracle_weights().items()}
    hq, hkv = cfg.n_heads, cfg.n_kv_heads

    def rms(h, wn):
        return h * torch.rsqrt((h * h).mean(-1, keepdim=True) + cfg.eps) * wn

    def host_layer_check(tokens, positions, kv_positions, label):
        """Recompute layer 0 from the embedding for `tokens` and compare q / attn / x."""
        emb = wt["embed"][torch.as_tensor(tokens, dtype=torch.long)].double()
        xn = rms(emb, wt["layers.0.attn_norm"].double()).to(torch.bfloat16).double()
        qkv = (xn @ wt["layers.0.wqkv"].double().T).to(torch.bfloat16).double()
        n = len(tokens)
        q = qkv[:, :hq * 128].reshape(n, hq, 128)
        cos = w.cos[positions].double().cpu()
        sin = w.sin[positions].double().cpu()

        def rope(x):
            x0, x1 = x[..., :64], x[..., 64:]
            c, s = cos[:, None, :], sin[:, None, :]
            return torch.cat([x0 * c - x1 * s, x1 * c + x0 * s], -1).to(torch.bfloat16).double()

        qh = rope(q)
        qg = w.q[:n].reshape(n, hq, 128).double().cpu()
        print(f"[{label}] q (GEMM + rope) rel err vs host: {rel(qg, qh):.2e}")
        # attention over the GPU's own q and cached K / V
        kk, vv = [], []
        for j in kv_positions:
            if j < P:
                blk, off = int(w.table[1, j // 16]), j % 16
            else:
                blk, off = int(w.table[1, npb + (j - P) // 16]), (j - P) % 16
            kk.append(w.cache[0, 0, blk, :, off].double().cpu())
            vv.append(w.cache[0, 1, blk, :, off].double().cpu())
        K = torch.stack(kk)  # [S, hkv, 128]
        V = torch.stack(vv)
        grp = hq // hkv
        Kr = K.repeat_interleave(grp, 1)
        Vr = V.repeat_interleave(grp, 1)
        s = torch.einsum("thd,shd->hts", qg, Kr) / math.sqrt(128)
        kpos = torch.as_tensor(kv_positions)
        mask = kpos[None, :] > torch.as_tensor(positions)[:, None]
        s = s.masked_fill(mask[None], float("-inf"))
        a = torch.einsum("hts,shd->thd", torch.softmax(s, -1), Vr)
        ag = w.attn[:n].reshape(n, hq, 128).double().cpu()
        print(f"[{label}] attention rel err vs exact (GPU q/K/V): {rel(ag, a):.2e}; vs bf16-rounded "
              f"exact {rel(ag, a.to(torch.bfloat16).double()):.2e}")
        # o-proj + residual, MLP on the GPU's own attn: final x
        h = emb + ag.reshape(n, -1) @ wt["layers.0.wo"].double().T
        xn2 = rms(h, wt["layers.0.mlp_norm"].double()).to(torch.bfloat16).double()
        gu = xn2 @ wt["layers.0.wgu"].double().T
        gg, uu = gu[:, :cfg.ffn], gu[:, cfg.ffn:]
        act = (gg / (1 + torch.exp(-gg)) * uu).to(torch.bfloat16).double()
        actg = w.act[:n].double().cpu()
        print(f"[{label}] swiglu act rel err: {rel(actg, act):.2e}")
        x = h + actg @ wt["layers.0.wd"].double().T
        xg = w.x[:n].double().cpu()
        print(f"[{label}] final residual rel err: {rel(xg, x):.2e}")
        xf = rms(xg, wt["final_norm"].double()).to(torch.bfloat16).double()
        lg = xf[-1:] @ wt["lm_head"].double().T
        print(f"[{label}] logits (from GPU x) rel err: {rel(w.logits[w.n_out - 1:w.n_out], lg):.2e}")

    torch.cuda.synchronize()
    w.forward(StepPlan(prefill=[PrefillSeq(0, 0, P, pre, out_row=0)]))
    torch.cuda.synchronize()
    host_layer_check(pre, list(range(P)), list(range(P)), "prefix prefill M=1000")
    w.forward(StepPlan(prefill=[PrefillSeq(1, P, P + p, prm, out_row=1)]))
    torch.cuda.synchronize()
    host_layer_check(prm, list(range(P, P + p)), list(range(P + p)), "prompt prefill M=200")
    toks = [int(w.slot_tok[1])]
    for k in range(4):
        kv = P + p + k + 1
        w.forward(StepPlan(decode=[DecodeTok(1, P, kv, hist_pos=k + 1, prefix_key=0)]))
        torch.cuda.synchronize()
        host_layer_check(toks[-1:], [kv - 1], list(range(kv)), f"decode step {k}")
        toks.append(int(w.slot_tok[1]))


if __name__ == "__main__":
    main()
