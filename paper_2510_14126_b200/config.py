"""Model shapes and engine sizing for the stage engines."""

from __future__ import annotations

from dataclasses import dataclass

HEAD_DIM = 128
BLOCK_TOKENS = 16


@dataclass(frozen=True)
class ModelConfig:
    """A Llama-style decoder: RMSNorm, RoPE, GQA, SwiGLU, untied lm_head."""

    name: str
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    ffn: int
    vocab: int
    rope_theta: float
    eps: float = 1e-5

    @property
    def group(self) -> int:
        return self.n_heads // self.n_kv_heads

    @property
    def qkv_dim(self) -> int:
        return (self.n_heads + 2 * self.n_kv_heads) * HEAD_DIM

    @property
    def kv_bytes_per_token(self) -> int:
        """K + V bytes of one token over all layers (bf16)."""
        return self.n_layers * 2 * self.n_kv_heads * HEAD_DIM * 2

    @property
    def kv_bytes_per_block(self) -> int:
        return self.kv_bytes_per_token * BLOCK_TOKENS

    def n_params(self) -> int:
        d, L = self.d_model, self.n_layers
        per_layer = self.qkv_dim * d + d * self.n_heads * HEAD_DIM + 2 * self.ffn * d + d * self.ffn + 2 * d
        return L * per_layer + 2 * self.vocab * d + d

    def weight_bytes(self) -> int:
        return 2 * self.n_params()

    def to_ref(self):
        """The same shape as the oracle's RefConfig (tests only)."""
        from oracle.decoder_ref import RefConfig

        return RefConfig(self.n_layers, self.d_model, self.n_heads, self.n_kv_heads, self.ffn,
                         self.vocab, self.rope_theta, self.eps)


# BASELINE config 1: "tiny random-init decoder (4L, d=256)". Head dim stays 128 so the
# 8B kernels' head_dim specialisation is the one exercised; 2 q heads share 1 kv head.
TINY = ModelConfig("tiny-4L-d256", n_layers=4, d_model=256, n_heads=2, n_kv_heads=1, ffn=768,
                   vocab=1024, rope_theta=10000.0)

# Tiny shape that splits two ways (BASELINE config 5 is tensor-parallel = 2): 4 q heads
# over 2 kv heads, so each TP rank keeps one whole GQA group of head_dim 128.
TINY_TP = ModelConfig("tiny-tp-4L-d256", n_layers=4, d_model=256, n_heads=4, n_kv_heads=2,
                      ffn=768, vocab=1024, rope_theta=10000.0)

# BASELINE configs 2-5: Llama-3-8B shape (random init).
LLAMA3_8B = ModelConfig("llama3-8b", n_layers=32, d_model=4096, n_heads=32, n_kv_heads=8,
                        ffn=14336, vocab=128256, rope_theta=500000.0)

MODELS = {m.name: m for m in (TINY, TINY_TP, LLAMA3_8B)}
