"""CPU baseline of the stage-engine hot path (the oracle port, timed on host cores).

ORACLE — used only by bench.py's cpu_baseline leg / `--impl reference` and by
tests; never by the product path.

The reference (stagesim) has no model arithmetic at all: its engine's "decode"
is t(b) = t0(1 + alpha(b-1)) (stagesim/engines.py:55-57). The CPU figure the
north star asks for is therefore the builder's CPU fp32 restatement of the same
decoder (oracle/decoder_ref.py semantics) on all host cores, on a bounded sample
of the benchmark workload:

  * one prompt prefill of p tokens after a resident P-token prefix, and
  * one batched greedy decode step of B sequences at context ctx,

both through all n_layers of the model shape (one random layer's weights reused
for every layer — identical FLOPs and bytes, bounded memory), plus the lm_head.
Workflows/s follows from the trace's mean per-workflow work (calls per
workflow x (p prefill tokens + o decode tokens)).
"""

from __future__ import annotations

import math
import os
import time

import torch


def _layer(d, hq, hkv, ffn, g):
    s = 0.02
    return {
        "wqkv": torch.randn((hq + 2 * hkv) * 128, d, generator=g) * s,
        "wo": torch.randn(d, hq * 128, generator=g) * s,
        "wgu": torch.randn(2 * ffn, d, generator=g) * s,
        "wd": torch.randn(d, ffn, generator=g) * s,
        "n1": torch.ones(d),
        "n2": torch.ones(d),
    }


def _rms(h, w, eps=1e-5):
    return h * torch.rsqrt((h * h).mean(-1, keepdim=True) + eps) * w


@torch.no_grad()
def _forward(L, n_layers, h, k_ctx, v_ctx, hq, hkv, ffn, causal_q):
    """h [B, T, d]; k_ctx/v_ctx [B, S, hkv, 128] context KV (reused for every layer)."""
    B, T, d = h.shape
    group = hq // hkv
    for _ in range(n_layers):
        x = _rms(h, L["n1"])
        qkv = x @ L["wqkv"].T
        q = qkv[..., : hq * 128].reshape(B, T, hq, 128)
        k = qkv[..., hq * 128:(hq + hkv) * 128].reshape(B, T, hkv, 128)
        v = qkv[..., (hq + hkv) * 128:].reshape(B, T, hkv, 128)
        kk = torch.cat([k_ctx, k], 1).repeat_interleave(group, 2)
        vv = torch.cat([v_ctx, v], 1).repeat_interleave(group, 2)
        s = torch.einsum("bthd,bshd->bhts", q, kk) / math.sqrt(128)
        if causal_q and T > 1:
            S = kk.shape[1]
            mask = torch.arange(S)[None, :] > (S - T + torch.arange(T))[:, None]
            s = s.masked_fill(mask, float("-inf"))
        a = torch.einsum("bhts,bshd->bthd", torch.softmax(s, -1), vv).reshape(B, T, hq * 128)
        h = h + a @ L["wo"].T
        x = _rms(h, L["n2"])
        gu = x @ L["wgu"].T
        act = torch.nn.functional.silu(gu[..., :ffn]) * gu[..., ffn:]
        h = h + act @ L["wd"].T
    return h


def measure(cfg, prefix: int = 1000, prompt: int = 200, out_tokens: int = 100, batch: int = 16,
            calls_per_workflow: float = 131 / 64, threads: int | None = None,
            seed: int = 0) -> dict:
    """Time the bounded sample; returns a dict with workflows/s, decode tok/s, sample text."""
    threads = threads or os.cpu_count() or 1
    torch.set_num_threads(threads)
    g = torch.Generator().manual_seed(seed)
    d, hq, hkv, ffn = cfg.d_model, cfg.n_heads, cfg.n_kv_heads, cfg.ffn
    L = _layer(d, hq, hkv, ffn, g)
    lm = torch.randn(cfg.vocab, d, generator=g) * 0.02
    # prompt prefill after the prefix
    h = torch.randn(1, prompt, d, generator=g)
    kc = torch.randn(1, prefix, hkv, 128, generator=g)
    t0 = time.perf_counter()
    hp = _forward(L, cfg.n_layers, h, kc, kc, hq, hkv, ffn, causal_q=True)
    _ = _rms(hp[:, -1], torch.ones(d)) @ lm.T
    t_prefill = time.perf_counter() - t0
    # one batched decode step at ctx = prefix + prompt + out/2
    ctx = prefix + prompt + out_tokens // 2
    h = torch.randn(batch, 1, d, generator=g)
    kc = torch.randn(batch, ctx, hkv, 128, generator=g)
    t0 = time.perf_counter()
    hd = _forward(L, cfg.n_layers, h, kc, kc, hq, hkv, ffn, causal_q=False)
    logits = _rms(hd[:, 0], torch.ones(d)) @ lm.T
    _ = logits.argmax(-1)
    t_decode = time.perf_counter() - t0
    per_call = t_prefill + out_tokens * t_decode / batch
    per_wf = calls_per_workflow * per_call
    return {
        "workflows_per_s": 1.0 / per_wf,
        "decode_tok_s": batch / t_decode,
        "prefill_tok_s": prompt / t_prefill,
        "cores": threads,
        "t_prefill_s": t_prefill,
        "t_decode_step_s": t_decode,
        "sample": (f"{cfg.name} fp32 on {threads} threads: 1 prefill of {prompt} tokens after a "
                   f"{prefix}-token prefix + 1 decode step of batch {batch} at ctx {ctx}, all "
                   f"{cfg.n_layers} layers (one layer's weights reused) + lm_head; workflows/s = "
                   f"1 / ({calls_per_workflow:.3f} calls x (prefill + {out_tokens} tokens x "
                   f"step/{batch}))"),
    }
