"""TP = 2 sharding (tp.py) checked on CPU in fp32: the two ranks' shards of one
decoder layer, each computing attention on its own heads and the MLP on its own
ffn slice, sum (after the O / down projections) to the unsharded layer."""

from __future__ import annotations

import pytest
import torch

from oracle.decoder_ref import attention_ref, rmsnorm_ref, rope_ref, rope_tables
from paper_2510_14126_b200.config import HEAD_DIM, LLAMA3_8B, TINY, TINY_TP
from paper_2510_14126_b200.tp import shard_config, shard_weights


def _weights(cfg, seed=0):
    g = torch.Generator().manual_seed(seed)
    d = cfg.d_model
    r = lambda *s: torch.randn(*s, generator=g) * 0.05  # noqa: E731
    return {"embed": r(cfg.vocab, d), "layers.0.attn_norm": 1 + r(d), "layers.0.mlp_norm": 1 + r(d),
            "layers.0.wqkv": r(cfg.qkv_dim, d), "layers.0.wo": r(d, cfg.n_heads * HEAD_DIM),
            "layers.0.wgu": r(2 * cfg.ffn, d), "layers.0.wd": r(d, cfg.ffn),
            "final_norm": 1 + r(d), "lm_head": r(cfg.vocab, d)}


def _attn(cfg, w, h, pos, cos, sin):
    """Attention contribution of layer 0 (O projection output, before the residual add)."""
    n = h.shape[0]
    hq, hkv = cfg.n_heads, cfg.n_kv_heads
    xn = rmsnorm_ref(h, w["layers.0.attn_norm"], cfg.eps)
    qkv = xn @ w["layers.0.wqkv"].T
    q = rope_ref(qkv[:, :hq * HEAD_DIM].reshape(n, hq, HEAD_DIM), cos, sin)
    k = rope_ref(qkv[:, hq * HEAD_DIM:(hq + hkv) * HEAD_DIM].reshape(n, hkv, HEAD_DIM), cos, sin)
    v = qkv[:, (hq + hkv) * HEAD_DIM:].reshape(n, hkv, HEAD_DIM)
    a = attention_ref(q, k, v, pos, pos).reshape(n, hq * HEAD_DIM)
    return a @ w["layers.0.wo"].T


def test_shard_config():
    s = shard_config(LLAMA3_8B, 2)
    assert (s.n_heads, s.n_kv_heads, s.ffn, s.group) == (16, 4, 7168, 4)
    assert s.d_model == LLAMA3_8B.d_model and s.vocab == LLAMA3_8B.vocab
    assert shard_config(TINY_TP, 2).n_kv_heads == 1
    assert shard_config(TINY, 1) is TINY
    with pytest.raises(ValueError):
        shard_config(TINY, 2)  # one kv head cannot be split


def test_shards_sum_to_the_full_layer():
    cfg = TINY_TP
    w = _weights(cfg)
    n = 12
    g = torch.Generator().manual_seed(1)
    h = torch.randn(n, cfg.d_model, generator=g)
    pos = torch.arange(n)
    cos, sin = rope_tables(64, cfg.rope_theta)
    cos, sin = cos[pos], sin[pos]
    full_attn = _attn(cfg, w, h, pos, cos, sin)
    sc = shard_config(cfg, 2)
    parts = [shard_weights(w, cfg, r, 2) for r in (0, 1)]
    for pw in parts:
        assert pw["layers.0.wqkv"].shape == (sc.qkv_dim, cfg.d_model)
        assert pw["layers.0.wo"].shape == (cfg.d_model, sc.n_heads * HEAD_DIM)
        assert pw["layers.0.wgu"].shape == (2 * sc.ffn, cfg.d_model)
        assert pw["layers.0.wd"].shape == (cfg.d_model, sc.ffn)
        assert pw["lm_head"] is w["lm_head"]  # replicated
    # attention: per-rank heads, partial O projections sum to the full one
    attn_parts = [_attn(sc, pw, h, pos, cos, sin) for pw in parts]
    torch.testing.assert_close(attn_parts[0] + attn_parts[1], full_attn, rtol=1e-5, atol=1e-5)
    # MLP on the all-reduced residual: partial down projections sum to the full one
    h2 = h + full_attn
    xn2 = rmsnorm_ref(h2, w["layers.0.mlp_norm"], cfg.eps)

    def mlp(c, ww):
        gu = xn2 @ ww["layers.0.wgu"].T
        gg, u = gu[:, :c.ffn], gu[:, c.ffn:]
        return (gg / (1 + torch.exp(-gg)) * u) @ ww["layers.0.wd"].T

    torch.testing.assert_close(mlp(sc, parts[0]) + mlp(sc, parts[1]), mlp(cfg, w), rtol=1e-5,
                               atol=1e-5)
