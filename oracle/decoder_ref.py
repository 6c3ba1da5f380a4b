"""CPU fp32 oracle of the stage engine's decoder forward (test infrastructure only).

ORACLE — imported only by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline leg, as the checker. Never part of the product path.

The reference has no model: its engine is a token-count state machine with a
closed-form step time (stagesim/engines.py:55-57) and its SPEC excludes GPU
kernels. Attention, logits and greedy tokens are therefore
"parity unpinned" by the reference; this module is the builder-written
restatement the north star asks for (BASELINE.json north_star: "attention and
logits must match within 2e-3 relative error in bf16 ... with greedy tokens
identical"), and DESIGN.md §5 records that status.

Model: Llama-style decoder (RMSNorm, RoPE rotate-half, GQA, SwiGLU, untied
lm_head). Arithmetic is fp32; every tensor the GPU path stores in bf16 is
rounded to bf16 at the same point here, so GPU and oracle differ only by fp32
summation order:
  h0 = E[tok]                                   (residual stream h is fp32)
  per layer: xn = bf16(h * rsqrt(mean(h^2) + eps) * w_attn)
             qkv = bf16(xn Wqkv^T);  q,k = bf16(rope(q,k));  K/V cache bf16
             a = bf16(softmax(q k^T / sqrt(128)) v)        (causal, fp32)
             h = a Wo^T + h
             xn = bf16(rmsnorm(h) * w_mlp);  gu = xn Wgu^T (fp32)
             act = bf16(silu(g) * u);  h = act Wd^T + h
  logits = fp32(bf16(rmsnorm(h) * w_final) Wlm^T);  token = first argmax
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

HEAD_DIM = 128


def bf16(x: torch.Tensor) -> torch.Tensor:
    return x.to(torch.bfloat16).to(torch.float32)


def rope_tables(max_pos: int, theta: float) -> tuple[torch.Tensor, torch.Tensor]:
    """cos/sin [max_pos, 64] fp32: angle = pos * theta^(-2i/128), computed in float64."""
    inv = theta ** (-np.arange(0, HEAD_DIM, 2, dtype=np.float64) / HEAD_DIM)
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
    return (torch.from_numpy(np.cos(ang).astype(np.float32)),
            torch.from_numpy(np.sin(ang).astype(np.float32)))


def no_round(x: torch.Tensor) -> torch.Tensor:
    """No rounding (the fp32 path stores fp32)."""
    return x


def rmsnorm_ref(h: torch.Tensor, w: torch.Tensor, eps: float, rnd=bf16) -> torch.Tensor:
    rstd = torch.rsqrt((h * h).mean(dim=-1, keepdim=True) + eps)
    return rnd(h * rstd * w)


def rope_ref(x: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor, rnd=bf16) -> torch.Tensor:
    """x [T, H, 128] fp32 (bf16 values); cos/sin [T, 64]."""
    x0, x1 = x[..., :64], x[..., 64:]
    c, s = cos[:, None, :], sin[:, None, :]
    return rnd(torch.cat([x0 * c - x1 * s, x1 * c + x0 * s], dim=-1))


def attention_ref(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, q_pos: torch.Tensor,
                  k_pos: torch.Tensor, rnd=bf16) -> torch.Tensor:
    """Causal GQA attention in fp32. q [T, Hq, D], k/v [S, Hkv, D]; returns bf16-rounded [T, Hq, D]."""
    hq, hkv = q.shape[1], k.shape[1]
    group = hq // hkv
    kk = k.repeat_interleave(group, dim=1)  # [S, Hq, D]
    vv = v.repeat_interleave(group, dim=1)
    s = torch.einsum("thd,shd->hts", q, kk) / math.sqrt(q.shape[-1])
    mask = k_pos[None, :] > q_pos[:, None]  # [T, S]
    s = s.masked_fill(mask[None], float("-inf"))
    p = torch.softmax(s, dim=-1)
    return rnd(torch.einsum("hts,shd->thd", p, vv))


@dataclass(frozen=True)
class RefConfig:
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    ffn: int
    vocab: int
    rope_theta: float
    eps: float = 1e-5


class RefDecoder:
    """Weights as fp32 copies of the engine's tensors (exact). `exact=True`: no bf16
    rounding anywhere (the oracle of the fp32 path, csrc/fp32.cu)."""

    def __init__(self, cfg: RefConfig, weights: dict[str, torch.Tensor], max_pos: int,
                 exact: bool = False) -> None:
        self.cfg = cfg
        self.rnd = no_round if exact else bf16
        self.w = {k: v.detach().to("cpu", torch.float32) for k, v in weights.items()}
        self.cos, self.sin = rope_tables(max_pos, cfg.rope_theta)

    def new_seq(self) -> "RefSeq":
        return RefSeq(self)


class RefSeq:
    """One logical sequence: per-layer K/V (bf16 values) and the positions held."""

    def __init__(self, model: RefDecoder) -> None:
        self.m = model
        c = model.cfg
        self.k = [torch.zeros(0, c.n_kv_heads, HEAD_DIM) for _ in range(c.n_layers)]
        self.v = [torch.zeros(0, c.n_kv_heads, HEAD_DIM) for _ in range(c.n_layers)]
        self.length = 0

    def fork(self) -> "RefSeq":
        s = RefSeq(self.m)
        s.k = [t.clone() for t in self.k]
        s.v = [t.clone() for t in self.v]
        s.length = self.length
        return s

    @torch.no_grad()
    def extend(self, tokens, want_logits: str = "last") -> torch.Tensor | None:
        """Append tokens at positions length.., return fp32 logits ('last', 'all' or 'none')."""
        m, c, w = self.m, self.m.cfg, self.m.w
        toks = torch.as_tensor(list(tokens), dtype=torch.long)
        n = toks.numel()
        pos = torch.arange(self.length, self.length + n)
        cos, sin = m.cos[pos], m.sin[pos]
        rnd = m.rnd
        h = w["embed"][toks]
        hq, hkv = c.n_heads, c.n_kv_heads
        for li in range(c.n_layers):
            p = f"layers.{li}."
            xn = rmsnorm_ref(h, w[p + "attn_norm"], c.eps, rnd)
            qkv = rnd(xn @ w[p + "wqkv"].T)
            q = qkv[:, : hq * HEAD_DIM].reshape(n, hq, HEAD_DIM)
            k = qkv[:, hq * HEAD_DIM:(hq + hkv) * HEAD_DIM].reshape(n, hkv, HEAD_DIM)
            v = qkv[:, (hq + hkv) * HEAD_DIM:].reshape(n, hkv, HEAD_DIM)
            q = rope_ref(q, cos, sin, rnd)
            k = rope_ref(k, cos, sin, rnd)
            self.k[li] = torch.cat([self.k[li], k])
            self.v[li] = torch.cat([self.v[li], v])
            kpos = torch.arange(self.k[li].shape[0])
            a = attention_ref(q, self.k[li], self.v[li], pos, kpos, rnd).reshape(n, hq * HEAD_DIM)
            h = a @ w[p + "wo"].T + h
            xn = rmsnorm_ref(h, w[p + "mlp_norm"], c.eps, rnd)
            gu = xn @ w[p + "wgu"].T  # fp32: SwiGLU is fused into the GEMM epilogue
            g, u = gu[:, : c.ffn], gu[:, c.ffn:]
            act = rnd(g / (1.0 + torch.exp(-g)) * u)
            h = act @ w[p + "wd"].T + h
        self.length += n
        if want_logits == "none":
            return None
        hs = h if want_logits == "all" else h[-1:]
        xn = rmsnorm_ref(hs, w["final_norm"], c.eps, rnd)
        return xn @ w["lm_head"].T


def greedy(logits: torch.Tensor) -> int:
    """First index of the maximum (the GPU argmax's tie rule)."""
    row = logits.reshape(-1)
    mx = row.max()
    return int(torch.nonzero(row == mx)[0, 0])


def top2_margin(logits: torch.Tensor) -> float:
    v = torch.topk(logits.reshape(-1), 2).values
    return float(v[0] - v[1])
