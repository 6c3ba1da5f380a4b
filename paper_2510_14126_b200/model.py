"""Decoder forward of a stage engine on one B200.

`GpuWorker` owns everything device-resident on one GPU: the random-init bf16
weights (one model serves every stage), the paged KV arena
(cache, block table, per-row generated-token state) shared by the engines placed
on this GPU (each engine owns disjoint block ids and table rows), and the
activation buffers. `forward(plan)` runs one batched step over a mix of decode
tokens (one per call, attention via the split-K decode kernel) and prefill
tokens (prompts / stage prefixes, causal paged prefill kernel): one weight
stream per step, every projection a tcgen05 GEMM.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, ops
from .config import BLOCK_TOKENS, HEAD_DIM, ModelConfig

BF16 = torch.bfloat16


def rope_tables(max_pos: int, theta: float) -> tuple[np.ndarray, np.ndarray]:
    """cos/sin [max_pos, 64] fp32, angle = pos * theta^(-2i/128) evaluated in float64."""
    inv = theta ** (-np.arange(0, HEAD_DIM, 2, dtype=np.float64) / HEAD_DIM)
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)


def init_weights(cfg: ModelConfig, device, seed: int = 0, std: float = 0.02) -> dict:
    """Random-init weights, N(0, std^2) projections, norms 1 + N(0, 0.1^2)."""
    g = torch.Generator(device=device).manual_seed(seed)

    def rnd(*shape, s=std):
        return (torch.randn(*shape, generator=g, device=device) * s).to(BF16)

    def norm(d):
        return (1.0 + 0.1 * torch.randn(d, generator=g, device=device)).to(BF16)

    d = cfg.d_model
    w = {"embed": rnd(cfg.vocab, d, s=1.0)}
    for i in range(cfg.n_layers):
        p = f"layers.{i}."
        w[p + "attn_norm"] = norm(d)
        w[p + "wqkv"] = rnd(cfg.qkv_dim, d)
        w[p + "wo"] = rnd(d, cfg.n_heads * HEAD_DIM)
        w[p + "mlp_norm"] = norm(d)
        w[p + "wgu"] = rnd(2 * cfg.ffn, d)
        w[p + "wd"] = rnd(d, cfg.ffn)
    w["final_norm"] = norm(d)
    w["lm_head"] = rnd(cfg.vocab, d)
    return w


def init_weights_f32(cfg: ModelConfig, device, seed: int = 0, std: float = 0.02) -> dict:
    """fp32 random-init weights for the fp32 path (config 1's exact-arithmetic check):
    same distributions as init_weights, no bf16 rounding, canonical gate/up layout."""
    g = torch.Generator(device=device).manual_seed(seed)

    def rnd(*shape, s=std):
        return torch.randn(*shape, generator=g, device=device) * s

    def norm(d):
        return 1.0 + 0.1 * torch.randn(d, generator=g, device=device)

    d = cfg.d_model
    w = {"embed": rnd(cfg.vocab, d, s=1.0)}
    for i in range(cfg.n_layers):
        p = f"layers.{i}."
        w[p + "attn_norm"] = norm(d)
        w[p + "wqkv"] = rnd(cfg.qkv_dim, d)
        w[p + "wo"] = rnd(d, cfg.n_heads * HEAD_DIM)
        w[p + "mlp_norm"] = norm(d)
        w[p + "wgu"] = rnd(2 * cfg.ffn, d)
        w[p + "wd"] = rnd(d, cfg.ffn)
    w["final_norm"] = norm(d)
    w["lm_head"] = rnd(cfg.vocab, d)
    return w


@dataclass
class PrefillSeq:
    """New tokens of one sequence: positions [kv_len - n, kv_len) of table row `row`."""

    row: int
    prefix_len: int  # tokens of the row's prefix segment (0 when prefilling a prefix row)
    kv_len: int      # total tokens of the sequence after this step
    tokens: np.ndarray
    out_row: int = -1   # table row receiving the greedy token of the last position (-1: none)
    hist_pos: int = 0


@dataclass
class DecodeTok:
    """One decode token of row `row` at position kv_len - 1 (input = slot_tok[row])."""

    row: int
    prefix_len: int
    kv_len: int
    hist_pos: int
    prefix_key: int = -1  # identity of the shared prefix segment (unique-bytes accounting)


class KernelProfile:
    """CUDA-event timing of selected kernel classes inside forward() (bench only).

    Each record: (class, start event, end event, algorithmic bytes, flops)."""

    def __init__(self, classes, every: int = 1, isolate: bool = False) -> None:
        self.classes = set(classes)
        self.recs: list = []
        self.every = every  # time the kernels of one step in `every` (event overhead)
        # isolate: the sampled steps run their attention passes one after another on the
        # main stream (no side-stream overlap), so each class's events bracket that class
        # alone - per-class rooflines, not the schedule's overlap
        self.isolate = isolate

    def sampled(self, step: int) -> bool:
        return step % self.every == 0

    def open(self, cls):
        if cls not in self.classes:
            return None
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    def close(self, cls, e0, nbytes: float, flops: float) -> None:
        if e0 is None:
            return
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record()
        self.recs.append((cls, e0, e1, nbytes, flops))

    def summary(self) -> dict:
        torch.cuda.synchronize()
        out: dict = {}
        for cls, e0, e1, b, f in self.recs:
            d = out.setdefault(cls, {"launches": 0, "ms": 0.0, "bytes": 0.0, "flops": 0.0})
            d["launches"] += 1
            d["ms"] += e0.elapsed_time(e1)
            d["bytes"] += b
            d["flops"] += f
        return out


def token_slot(prefix_len: int, pos: int) -> tuple[int, int]:
    """(block column, offset) of logical position `pos` in a row with a prefix segment."""
    if pos < prefix_len:
        return pos // BLOCK_TOKENS, pos % BLOCK_TOKENS
    npb = (prefix_len + BLOCK_TOKENS - 1) // BLOCK_TOKENS
    j = pos - prefix_len
    return npb + j // BLOCK_TOKENS, j % BLOCK_TOKENS


@dataclass
class StepPlan:
    decode: list[DecodeTok] = field(default_factory=list)
    prefill: list[PrefillSeq] = field(default_factory=list)

    @property
    def n_tokens(self) -> int:
        return len(self.decode) + sum(len(p.tokens) for p in self.prefill)


class GpuWorker:
    """Weights + KV arena + activation buffers of one GPU."""

    def __init__(self, cfg: ModelConfig, device, n_blocks: int, n_rows: int, row_cols: int,
                 max_tokens: int = 4096, max_out: int = 512, hist_cols: int = 1024,
                 max_seq_tokens: int = 16384, weights: dict | None = None, seed: int = 0,
                 tp=None, precision: str = "bf16") -> None:
        # tp: a tp.TpComm when this worker is one rank of a TP = 2 replica. `cfg` is the
        # full model; the worker holds its rank's shard (tp.py) and self.cfg is the shard.
        # precision "f32": every tensor and every kernel fp32 (csrc/fp32.cu) — the tiny
        # config-1 model's exact-arithmetic path ("1e-5 in fp32, greedy tokens identical").
        if precision not in ("bf16", "f32"):
            raise ValueError(f"precision {precision!r}")
        self.f32 = precision == "f32"
        if self.f32:
            if tp is not None:
                raise ValueError("the fp32 path has no tensor parallelism")
            self._init_f32(cfg, device, n_blocks, n_rows, row_cols, max_tokens, max_out,
                           hist_cols, max_seq_tokens, weights, seed)
            return
        self.full_cfg = cfg
        self.tp = tp
        if tp is not None:
            from .tp import shard_config, shard_weights

            if tp.max_tokens < max_tokens or tp.d != cfg.d_model:
                raise ValueError("TpComm buffer smaller than the worker's step")
            full = weights if weights is not None else init_weights(cfg, device, seed)
            weights = shard_weights(full, cfg, tp.rank, tp.size)
            cfg = shard_config(cfg, tp.size)
        self.cfg = cfg
        self.device = torch.device(device)
        self.n_blocks = n_blocks
        self.max_tokens = max_tokens
        self.max_out = max_out
        self.max_seq_tokens = max_seq_tokens
        dev = self.device
        self.w = weights if weights is not None else init_weights(cfg, dev, seed)
        # gate/up rows interleaved in blocks of 64 so the gate_up GEMM's epilogue applies
        # SwiGLU in place (the canonical layout stays available via oracle_weights())
        for i in range(cfg.n_layers):
            k = f"layers.{i}.wgu"
            self.w[k] = ops.interleave_gate_up(self.w[k])
        self.wmap = {k: ops.weight_map(v) for k, v in self.w.items() if v.dim() == 2 and k != "embed"}
        cos, sin = rope_tables(max_seq_tokens + 1, cfg.rope_theta)
        self.cos = torch.from_numpy(cos).to(dev)
        self.sin = torch.from_numpy(sin).to(dev)
        # paged KV arena
        # zero-filled once: masked slots of partial blocks are multiplied by p = 0, so the
        # cache must never hold NaN/Inf bit patterns (stale values are finite)
        self.cache = torch.zeros(cfg.n_layers, 2, n_blocks, cfg.n_kv_heads, BLOCK_TOKENS, HEAD_DIM,
                                 dtype=BF16, device=dev)
        self.kvmap = ops.kv_map(self.cache.view(-1, HEAD_DIM))
        self.table = torch.zeros(n_rows, row_cols, dtype=torch.int32, device=dev)
        self.slot_tok = torch.zeros(n_rows, dtype=torch.int32, device=dev)
        self.hist = torch.zeros(n_rows, hist_cols, dtype=torch.int32, device=dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        # activations
        d, T = cfg.d_model, max_tokens
        self.x = torch.zeros(T, d, dtype=torch.float32, device=dev)  # fp32 residual stream
        self.xn = torch.zeros(T, d, dtype=BF16, device=dev)
        self.qkv = torch.zeros(T, cfg.qkv_dim, dtype=BF16, device=dev)
        self.q = torch.zeros(T, cfg.n_heads * HEAD_DIM, dtype=BF16, device=dev)
        self.attn = torch.zeros(T, cfg.n_heads * HEAD_DIM, dtype=BF16, device=dev)
        self.act = torch.zeros(T, cfg.ffn, dtype=BF16, device=dev)
        self.xn_out = torch.zeros(max_out, d, dtype=BF16, device=dev)
        self.logits = torch.zeros(max_out, cfg.vocab, dtype=torch.float32, device=dev)
        # greedy tokens straight from the lm_head GEMM's epilogue: (max, index) per
        # 128-vocab chunk, reduced per row; the full fp32 logits are written only when
        # `full_logits` is set (parity checks) or an on_forward hook may read them
        self.lm_part = torch.zeros(max_out, cfg.vocab // 128, dtype=torch.int64, device=dev)
        self.full_logits = False
        # RoPE + paged KV append in the QKV GEMM's epilogue (False: separate kernel; A/B),
        # its per-token operands computed once per step
        self.fuse_qkv_rope = True
        self.tok_dst = torch.zeros(T, dtype=torch.int32, device=dev)
        self.tok_cs = torch.zeros(T, 128, dtype=torch.float32, device=dev)
        self.out_tok = torch.zeros(max_out, dtype=torch.int32, device=dev)
        self.xn_map = ops.act_map(self.xn)
        self.attn_map = ops.act_map(self.attn)
        self.act_map = ops.act_map(self.act)
        self.xn_out_map = ops.act_map(self.xn_out)
        self.gemm_ws = ops.GemmWorkspace(dev)
        self.max_splits = ops.decode_splits(0, max_seq_tokens) + 1
        self.o_part = torch.empty(max_out * self.max_splits * cfg.n_heads * HEAD_DIM,
                                  dtype=torch.float32, device=dev)
        self.lse_part = torch.empty(max_out * self.max_splits * cfg.n_heads, dtype=torch.float32,
                                    device=dev)
        # metadata staging (one H2D copy per step)
        self._meta_cap = 16 * (T + max_out) + 64
        self._ring = 8  # pinned staging buffers, reused only after their copy ran
        self.meta_dev_small = torch.zeros(4 * 4096, dtype=torch.int32, device=dev)
        self.h2d_bytes = 0
        self.meta_host = [torch.zeros(self._meta_cap, dtype=torch.int32, pin_memory=True)
                          for _ in range(self._ring)]
        self.meta_evt = [None] * self._ring
        self._meta_i = 0
        # allocator / table-copy requests come in bursts (an admit is 2 uploads): their own
        # deeper ring, so a burst never waits for the GPU to drain the previous step
        self._ring_small = 64
        self.meta_host_small = [torch.zeros(4 * 1024, dtype=torch.int32, pin_memory=True)
                                for _ in range(self._ring_small)]
        self.meta_evt_small = [None] * self._ring_small
        self._meta_i_small = 0
        self.meta_dev = torch.zeros(self._meta_cap, dtype=torch.int32, device=dev)
        self.scale = 1.0 / math.sqrt(HEAD_DIM)
        self.launches = 0  # kernels of this library launched since construction
        self.steps = 0
        self.on_forward = None  # optional hook(plan, n_out) for parity checking
        self.check_finite = os.environ.get("CORTEX_CHECK_FINITE") == "1"  # debug only
        # TP: optional host hook at every exchange point (device sync + a host barrier) so
        # that two ranks sharing one GPU never have a kernel waiting on the other rank
        self.tp_sync = None
        self.prof: KernelProfile | None = None  # optional per-kernel-class CUDA-event timing
        self.cascade = True  # shared-prefix decode attention (prefix KV read once per step)
        # tcgen05 flash attention for prefill + the cascade pass (CORTEX_TC_ATTN=0: mma.sync)
        self.tc_attention = os.environ.get("CORTEX_TC_ATTN", "1") != "0"
        self.qmap = ops.QMap(self.q, cfg.n_heads, cfg.group)
        self.overlap_cascade = True
        # prefix slots of the cascade pass: 0 = by prefix length (below), or a fixed count
        self.cascade_slots = int(os.environ.get("CORTEX_CASCADE_SLOTS", "0"))
        # balanced decode plan (equal tile ranges per CTA) instead of per-call 512-token
        # splits; measured slower on config-2 contexts (benchmarks/attn_step.py), so opt-in
        self.flat_decode = os.environ.get("CORTEX_FLAT_DECODE", "0") == "1"
        # the side stream (cascade pass + prompt prefill, concurrent with the context
        # splits) at high priority: its big tensor-core CTAs are dispatched ahead of the
        # splits' as SMs free up instead of waiting for the split grid to drain
        # (benchmarks/replay_ab.py prio: 12.22 vs 12.56 ms per config-2 step)
        self.side = torch.cuda.Stream(device=dev, priority=-1)
        # the prompt prefill on a second high-priority side stream, beside the cascade pass
        # (benchmarks/attn_step.py --layer-only: 88.9 vs 92.0 us per config-2 layer)
        self.side2 = torch.cuda.Stream(device=dev, priority=-1)
        self._ev_join2 = torch.cuda.Event()
        self._ev_fork = torch.cuda.Event()
        self._ev_join = torch.cuda.Event()
        # layer loop launched from native code (csrc/step.cu, one ctypes call per step)
        # instead of ~10 ctypes calls per layer; the Python loop stays for TP, the
        # per-class profile window and the non-default A/B paths
        self.native_layers = True
        self._native = None
        self._step_desc = _lib.StepDesc()

    def _init_f32(self, cfg, device, n_blocks, n_rows, row_cols, max_tokens, max_out, hist_cols,
                  max_seq_tokens, weights, seed) -> None:
        self.full_cfg = self.cfg = cfg
        self.tp = None
        self.device = dev = torch.device(device)
        self.n_blocks, self.max_tokens, self.max_out = n_blocks, max_tokens, max_out
        self.max_seq_tokens = max_seq_tokens
        self.w = weights if weights is not None else init_weights_f32(cfg, dev, seed)
        cos, sin = rope_tables(max_seq_tokens + 1, cfg.rope_theta)
        self.cos = torch.from_numpy(cos).to(dev)
        self.sin = torch.from_numpy(sin).to(dev)
        f32 = torch.float32
        self.cache = torch.zeros(cfg.n_layers, 2, n_blocks, cfg.n_kv_heads, BLOCK_TOKENS, HEAD_DIM,
                                 dtype=f32, device=dev)
        self.table = torch.zeros(n_rows, row_cols, dtype=torch.int32, device=dev)
        self.slot_tok = torch.zeros(n_rows, dtype=torch.int32, device=dev)
        self.hist = torch.zeros(n_rows, hist_cols, dtype=torch.int32, device=dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        d, T = cfg.d_model, max_tokens
        self.x = torch.zeros(T, d, dtype=f32, device=dev)
        self.xn = torch.zeros(T, d, dtype=f32, device=dev)
        self.qkv = torch.zeros(T, cfg.qkv_dim, dtype=f32, device=dev)
        self.q = torch.zeros(T, cfg.n_heads * HEAD_DIM, dtype=f32, device=dev)
        self.attn = torch.zeros(T, cfg.n_heads * HEAD_DIM, dtype=f32, device=dev)
        self.act = torch.zeros(T, cfg.ffn, dtype=f32, device=dev)
        self.xn_out = torch.zeros(max_out, d, dtype=f32, device=dev)
        self.logits = torch.zeros(max_out, cfg.vocab, dtype=f32, device=dev)
        self.out_tok = torch.zeros(max_out, dtype=torch.int32, device=dev)
        self._meta_cap = 16 * (T + max_out) + 64
        self._ring = 8
        self.meta_host = [torch.zeros(self._meta_cap, dtype=torch.int32, pin_memory=True)
                          for _ in range(self._ring)]
        self.meta_evt = [None] * self._ring
        self._meta_i = 0
        self.meta_dev = torch.zeros(self._meta_cap, dtype=torch.int32, device=dev)
        self.h2d_bytes = 0
        self.scale = 1.0 / math.sqrt(HEAD_DIM)
        self.launches = 0
        self.steps = 0
        self.on_forward = None
        self.check_finite = False
        self.tp_sync = None
        self.prof = None

    # ------------------------------------------------------------------ helpers

    def oracle_weights(self) -> dict:
        """The weights in the canonical layout (gate rows then up rows) — for the checker."""
        if self.f32:
            return dict(self.w)
        out = dict(self.w)
        for i in range(self.cfg.n_layers):
            k = f"layers.{i}.wgu"
            out[k] = ops.deinterleave_gate_up(self.w[k])
        return out

    def _native_desc(self):
        """cortex_decoder_t of this worker (built once; keeps its pointer arrays alive)."""
        if self._native is None:
            cfg, wm, w = self.cfg, self.wmap, self.w
            L = cfg.n_layers
            arr = lambda vals: (ctypes.c_void_p * L)(*vals)
            keep = {
                "wqkv": arr([wm[f"layers.{i}.wqkv"].ptr for i in range(L)]),
                "wo": arr([wm[f"layers.{i}.wo"].ptr for i in range(L)]),
                "wgu": arr([wm[f"layers.{i}.wgu"].ptr for i in range(L)]),
                "wd": arr([wm[f"layers.{i}.wd"].ptr for i in range(L)]),
                "n1": arr([w[f"layers.{i}.attn_norm"].data_ptr() for i in range(L)]),
                "n2": arr([w[f"layers.{i}.mlp_norm"].data_ptr() for i in range(L)]),
            }
            ws = self.gemm_ws
            d = _lib.DecoderDesc(
                L, cfg.d_model, cfg.n_heads, cfg.n_kv_heads, cfg.ffn, cfg.eps, self.scale,
                ctypes.cast(keep["wqkv"], ctypes.c_void_p), ctypes.cast(keep["wo"], ctypes.c_void_p),
                ctypes.cast(keep["wgu"], ctypes.c_void_p), ctypes.cast(keep["wd"], ctypes.c_void_p),
                ctypes.cast(keep["n1"], ctypes.c_void_p), ctypes.cast(keep["n2"], ctypes.c_void_p),
                self.xn_map.ptr, self.attn_map.ptr, self.act_map.ptr, self.kvmap.ptr,
                self.qmap.ptr, self.x.data_ptr(), self.xn.data_ptr(), self.q.data_ptr(),
                self.attn.data_ptr(), self.act.data_ptr(), self.cache.data_ptr(),
                self.layer_rows(1)[0] // 2, self.table.data_ptr(), self.table.stride(0),
                self.tok_dst.data_ptr(), self.tok_cs.data_ptr(), ws.ws.data_ptr(),
                ws.ws.numel() * 4, ws.counters.data_ptr(), ws.counters.numel())
            self._native = (d, keep)
        return self._native[0]

    def layer_rows(self, layer: int) -> tuple[int, int]:
        per_plane = self.n_blocks * self.cfg.n_kv_heads * BLOCK_TOKENS
        return (2 * layer) * per_plane, (2 * layer + 1) * per_plane

    def _upload(self, arrays: list[np.ndarray], dev_buf: torch.Tensor | None = None,
                small: bool = False) -> list[torch.Tensor]:
        """Stage int32 arrays through a pinned ring into `dev_buf` (one async H2D copy).
        A device buffer may be rewritten by the next upload: stream order guarantees
        the kernels that read it ran first."""
        dev_buf = self.meta_dev if dev_buf is None else dev_buf
        sizes = [a.size for a in arrays]
        total = sum(sizes)
        hosts, evts = ((self.meta_host_small, self.meta_evt_small) if small
                       else (self.meta_host, self.meta_evt))
        if total > min(hosts[0].numel(), dev_buf.numel()):
            raise ValueError("step metadata exceeds staging capacity")
        if small:
            i = self._meta_i_small
            self._meta_i_small = (i + 1) % self._ring_small
        else:
            i = self._meta_i
            self._meta_i = (i + 1) % self._ring
        if evts[i] is not None:
            evts[i].synchronize()
        buf = hosts[i]
        host = buf.numpy()
        off = 0
        offs = []
        for a in arrays:
            host[off:off + a.size] = a
            offs.append(off)
            off += a.size
        dev_buf[:total].copy_(buf[:total], non_blocking=True)
        evt = torch.cuda.Event()
        evt.record()
        evts[i] = evt
        self.h2d_bytes += 4 * total
        return [dev_buf[o:o + n] for o, n in zip(offs, sizes)]

    def upload_small(self, arrays: list[np.ndarray]) -> list[torch.Tensor]:
        """Staging for allocator / table requests (separate device buffer and ring)."""
        return self._upload(arrays, self.meta_dev_small, small=True)

    # Block-pool requests travel in the kernel parameters (host arrays, the _h exports):
    # no staging copy, so an admit adds no copy-engine round trip to the step.

    def alloc_blocks(self, pool, reqs: list[tuple[int, int, int]]) -> None:
        """Allocate from `pool` (an EngineSlice): reqs = (table row, first col, blocks)."""
        ops.kv_alloc_h(pool.bitmap, pool.n_blocks, pool.block_base, [r[2] for r in reqs],
                       [r[0] for r in reqs], [r[1] for r in reqs], self.table, self.status)
        self.launches += (len(reqs) + 255) // 256

    def free_blocks(self, pool, reqs: list[tuple[int, int, int]]) -> None:
        ops.kv_free_h(pool.bitmap, pool.n_blocks, pool.block_base, self.table,
                      [r[0] for r in reqs], [r[1] for r in reqs], [r[2] for r in reqs],
                      self.status)
        self.launches += (len(reqs) + 255) // 256

    def copy_prefix_row(self, src_row: int, dst_row: int, n_blocks: int) -> None:
        ops.table_copy_h(self.table, [src_row], [dst_row], [0], [n_blocks])
        self.launches += 1

    def copy_first_token(self, src_row: int, dst_row: int) -> None:
        """Empty-prompt call on a resident prefix: its first token is the prefix's."""
        self.slot_tok[dst_row] = self.slot_tok[src_row]
        self.hist[dst_row, 0] = self.slot_tok[src_row]

    def forward_prefill_chunk(self, seq: PrefillSeq) -> int:
        return self.forward(StepPlan(prefill=[seq]))

    def forward_decode(self, toks: list[DecodeTok]) -> int:
        return self.forward(StepPlan(decode=toks))

    # ------------------------------------------------------------------ forward

    @torch.no_grad()
    def forward(self, plan: StepPlan) -> int:
        """Run one batched step; returns the number of greedy tokens produced."""
        for _ in self.forward_steps(plan):
            if self.tp_sync is not None:  # functional TP runs with both ranks on one GPU
                self.tp_sync()
        if self.check_finite:
            self._check_finite(plan)
        return self.n_out

    def _check_finite(self, plan: StepPlan) -> None:
        """Debug mode (CORTEX_CHECK_FINITE=1): synchronise after every step and fail with
        the step's plan when an output row's logits are not all finite."""
        bad = (~torch.isfinite(self.logits[: self.n_out])).any(dim=1).nonzero().flatten()
        if bad.numel() == 0:
            return
        rows = bad.tolist()[:8]
        lines = [f"non-finite logits in {bad.numel()} of {self.n_out} output rows {rows}"]
        for r in rows:
            if r < len(plan.decode):
                d = plan.decode[r]
                lines.append(f"  decode row {r}: table row {d.row} prefix {d.prefix_len} "
                             f"kv_len {d.kv_len} hist_pos {d.hist_pos} prefix_key "
                             f"{d.prefix_key}")
            else:
                lines.append(f"  prefill output row {r}")
        lines.append(f"  decode {len(plan.decode)}, prefill "
                     f"{[(s.row, s.prefix_len, s.kv_len, len(s.tokens)) for s in plan.prefill]}")
        raise FloatingPointError("\n".join(lines))

    @torch.no_grad()
    def forward_steps(self, plan: StepPlan):
        """forward() as a generator that yields at every TP exchange point (after the
        partial-output GEMM and its signal were enqueued, before the reduce that reads
        the peer's partial); a TP = 1 worker never yields. The result is left in
        self.n_out."""
        cfg = self.cfg
        n_dec = len(plan.decode)
        T = plan.n_tokens
        self.n_out = 0
        if T == 0:
            return
        if T > self.max_tokens:
            raise ValueError(f"step of {T} tokens exceeds max_tokens={self.max_tokens}")
        if self.f32:
            self._forward_f32(plan)
            return
        i32 = np.int32
        pos = np.empty(T, i32)
        app_col = np.empty(T, i32)
        app_off = np.empty(T, i32)
        app_row = np.empty(T, i32)
        tok_ids = np.zeros(T, i32)
        dec_row = np.empty(n_dec, i32)
        dec_prefix = np.empty(n_dec, i32)
        dec_kvlen = np.empty(n_dec, i32)
        out_rows, out_slot, out_hist = [], [], []
        # shared-prefix (cascade) groups: calls on the same resident prefix made contiguous
        groups = []
        if n_dec and self.cascade and all(d.prefix_key >= 0 for d in plan.decode if d.prefix_len):
            plan.decode.sort(key=lambda d: d.prefix_key if d.prefix_len else -1)
            for i, d in enumerate(plan.decode):
                if not d.prefix_len:
                    continue
                if groups and groups[-1][0] == d.prefix_key:
                    groups[-1][3] += 1
                else:
                    groups.append([d.prefix_key, d.prefix_len, i, 1])
        for i, d in enumerate(plan.decode):
            p = d.kv_len - 1
            c, o = token_slot(d.prefix_len, p)
            pos[i], app_row[i], app_col[i], app_off[i] = p, d.row, c, o
            dec_row[i], dec_prefix[i], dec_kvlen[i] = d.row, d.prefix_len, d.kv_len
            out_rows.append(i)
            out_slot.append(d.row)
            out_hist.append(d.hist_pos)
        n_pf = len(plan.prefill)
        pf_row = np.empty(n_pf, i32)
        pf_prefix = np.empty(n_pf, i32)
        pf_kvlen = np.empty(n_pf, i32)
        pf_qstart = np.empty(n_pf, i32)
        pf_qlen = np.empty(n_pf, i32)
        t = n_dec
        max_qlen = 0
        for j, s in enumerate(plan.prefill):
            n = len(s.tokens)
            p0 = s.kv_len - n
            ps = np.arange(p0, s.kv_len, dtype=np.int64)
            pos[t:t + n] = ps
            app_row[t:t + n] = s.row
            if s.prefix_len == 0:
                app_col[t:t + n] = ps // BLOCK_TOKENS
                app_off[t:t + n] = ps % BLOCK_TOKENS
            else:
                npb = (s.prefix_len + BLOCK_TOKENS - 1) // BLOCK_TOKENS
                jj = ps - s.prefix_len
                if (jj < 0).any():
                    raise ValueError("prefill of a private segment cannot write prefix positions")
                app_col[t:t + n] = npb + jj // BLOCK_TOKENS
                app_off[t:t + n] = jj % BLOCK_TOKENS
            tok_ids[t:t + n] = s.tokens
            pf_row[j], pf_prefix[j], pf_kvlen[j], pf_qstart[j], pf_qlen[j] = (
                s.row, s.prefix_len, s.kv_len, t, n)
            max_qlen = max(max_qlen, n)
            if s.out_row >= 0:
                out_rows.append(t + n - 1)
                out_slot.append(s.out_row)
                out_hist.append(s.hist_pos)
            t += n
        n_out = len(out_rows)
        if n_out > self.max_out:
            raise ValueError("too many output rows in one step")
        garr = np.asarray(groups, i32).reshape(-1, 4).T.copy() if groups else np.zeros((4, 0), i32)
        pslots = 0
        if n_dec and groups:
            # prefix partial slots (each a run of key tiles of the cascade pass): 2 up to
            # 2K-token prefixes, 4 beyond (benchmarks/fmha.py --slots, per layer: P = 1000
            # 2 slots 15.7 us (1 slot 22.0, 4 slots 17.8); P = 8192 4 slots 52.2 us with two
            # Q tiles per CTA (2 slots 64.7, 8 slots 60.6))
            npb_max = int(((garr[1] + BLOCK_TOKENS - 1) // BLOCK_TOKENS).max())
            want = self.cascade_slots or min(4, max(2, -(-npb_max // 128)))
            pslots = min(want, (npb_max + 15) // 16)
        fplan = None
        if n_dec and self.flat_decode:
            fplan = ops.decode_flat_plan(dec_prefix, dec_kvlen, cfg.n_kv_heads, bool(groups),
                                        self.max_splits - pslots)
        tstart = fplan[0] if fplan is not None else np.zeros(0, i32)
        (d_pos, d_arow, d_acol, d_aoff, d_tok, d_drow, d_dpre, d_dkv, d_prow, d_ppre, d_pkv,
         d_pqs, d_pql, d_orow, d_oslot, d_ohist, d_grow, d_gplen, d_gfirst, d_gcount,
         d_tstart) = self._upload([
            pos, app_row, app_col, app_off, tok_ids, dec_row, dec_prefix, dec_kvlen, pf_row,
            pf_prefix, pf_kvlen, pf_qstart, pf_qlen, np.asarray(out_rows, i32),
            np.asarray(out_slot, i32), np.asarray(out_hist, i32), garr[0], garr[1], garr[2],
            garr[3], tstart])
        max_splits = 1
        dec_groups = None
        flat = (d_tstart, fplan[1], fplan[2]) if fplan is not None else None
        if n_dec:
            if fplan is not None:
                max_splits = pslots + fplan[3]
            elif groups:  # private tokens only: splits of a prefix-less sequence
                max_splits = pslots + max(ops.decode_splits(0, int(b - a))
                                          for a, b in zip(dec_prefix, dec_kvlen))
            else:
                max_splits = max(ops.decode_splits(int(a), int(b))
                                 for a, b in zip(dec_prefix, dec_kvlen))
            if groups:
                dec_groups = (d_grow, d_gplen, d_gfirst, d_gcount, len(groups), int(garr[3].max()),
                              pslots)
            if max_splits > self.max_splits:
                raise ValueError("decode context exceeds max_seq_tokens")
        w, wm = self.w, self.wmap
        x, xn, ws = self.x, self.xn, self.gemm_ws
        hq, hkv = cfg.n_heads, cfg.n_kv_heads
        nl = 0
        if n_dec:
            ops.embed(w["embed"], self.slot_tok, n_dec, x, index=d_drow)
            nl += 1
        if T > n_dec:
            ops.embed(w["embed"], d_tok[n_dec:], T - n_dec, x[n_dec:])
            nl += 1
        o_part = self.o_part[: max(n_dec, 1) * max_splits * hq * HEAD_DIM]
        lse_part = self.lse_part[: max(n_dec, 1) * max_splits * hq]
        prof = self.prof if self.prof is not None and self.prof.sampled(self.steps) else None
        tok_kv_bytes = hkv * HEAD_DIM * 2 * 2  # K + V of one token in one layer
        if prof is not None:
            uniq = sum(d.kv_len - d.prefix_len for d in plan.decode)
            uniq += sum({(d.prefix_key if d.prefix_key >= 0 else ("row", d.row)): d.prefix_len
                         for d in plan.decode}.values())
            dec_bytes = uniq * tok_kv_bytes + n_dec * hq * HEAD_DIM * 2 * 2
            # the per-call context splits alone (private KV, HBM-bound kernel)
            ctx_bytes = (sum(d.kv_len - d.prefix_len for d in plan.decode) * tok_kv_bytes
                         + n_dec * hq * HEAD_DIM * 2 * 2)
            ctx_flops = 4.0 * hq * HEAD_DIM * sum(d.kv_len - d.prefix_len for d in plan.decode)
            dec_flops = 4.0 * hq * HEAD_DIM * float(dec_kvlen.sum())
            pf_keys = sum(int(q) * (int(k) - int(q)) + int(q) * (int(q) + 1) // 2
                          for q, k in zip(pf_qlen, pf_kvlen))
            pf_bytes = float(pf_kvlen.sum()) * tok_kv_bytes + 2 * 2 * (T - n_dec) * hq * HEAD_DIM
            pf_flops = 4.0 * hq * HEAD_DIM * pf_keys

        def gemm(name, xmap, M, out, residual=None, swiglu=False, argmax=False):
            e0 = prof.open("gemm") if prof is not None else None
            ops.gemm(wm[name], xmap, M, out, ws, residual=residual, swiglu=swiglu, argmax=argmax)
            if e0 is not None:
                N, K = wm[name].rows, wm[name].cols
                ob = out.element_size() * (2 if residual is not None else 1)
                n_out = out.shape[1]
                prof.close("gemm", e0, 2.0 * N * K + 2.0 * M * K + ob * M * n_out,
                           2.0 * M * N * K)

        tp = self.tp
        if self.fuse_qkv_rope:
            ops.rope_token_prep(self.table, d_pos, d_arow, d_acol, d_aoff, self.cos, self.sin, T,
                                hkv, self.tok_dst, self.tok_cs)
            nl += 1
        native = (self.native_layers and tp is None and prof is None and self.fuse_qkv_rope
                  and self.tc_attention and flat is None)
        if native:
            sd = self._step_desc
            ptr = lambda t: t.data_ptr() if t is not None and t.numel() else None
            sd.n_tok, sd.n_dec, sd.n_pf, sd.max_qlen, sd.max_splits = (T, n_dec, n_pf, max_qlen,
                                                                       max_splits)
            sd.layer_begin, sd.layer_end = 0, cfg.n_layers
            sd.dec_row, sd.dec_prefix, sd.dec_kvlen = ptr(d_drow), ptr(d_dpre), ptr(d_dkv)
            sd.pf_row, sd.pf_prefix, sd.pf_kvlen = ptr(d_prow), ptr(d_ppre), ptr(d_pkv)
            sd.pf_qstart, sd.pf_qlen = ptr(d_pqs), ptr(d_pql)
            if dec_groups is not None:
                sd.grp_row, sd.grp_plen, sd.grp_first, sd.grp_count = (
                    ptr(t) for t in dec_groups[:4])
                sd.n_groups, sd.max_group_count, sd.prefix_slots = dec_groups[4:]
            else:
                sd.grp_row = sd.grp_plen = sd.grp_first = sd.grp_count = None
                sd.n_groups = sd.max_group_count = sd.prefix_slots = 0
            sd.o_part, sd.lse_part = o_part.data_ptr(), lse_part.data_ptr()
            sd.stream = torch.cuda.current_stream().cuda_stream
            sd.side_stream = self.side.cuda_stream if self.overlap_cascade else None
            sd.side_stream2 = (self.side2.cuda_stream if self.overlap_cascade and self.side2
                               is not None else None)
            ops._check(ops.lib().cortex_decoder_layers(ctypes.byref(self._native_desc()),
                                                       ctypes.byref(sd)),
                       "cortex_decoder_layers")
            # launches, counted as the Python loop counts them
            nl += cfg.n_layers * (6 + (2 if n_dec else 0) + (1 if n_pf else 0))
        for li in range(0 if not native else cfg.n_layers, cfg.n_layers):
            p = f"layers.{li}."
            k0, v0 = self.layer_rows(li)
            if tp is None or li == 0:  # TP: fused into the previous layer's down exchange
                ops.rmsnorm(x, w[p + "attn_norm"], T, xn, cfg.eps)
                nl += 1
            # QKV GEMM with RoPE + the paged KV append in its epilogue (the qkv activation
            # is never written)
            if self.fuse_qkv_rope:
                e0 = prof.open("gemm") if prof is not None else None
                ops.gemm_qkv_rope(wm[p + "wqkv"], self.xn_map, T, ws, self.q, self.cache, k0, v0,
                                  self.tok_dst, self.tok_cs, hq, hkv)
                if e0 is not None:
                    N, K = wm[p + "wqkv"].rows, wm[p + "wqkv"].cols
                    prof.close("gemm", e0, 2.0 * N * K + 2.0 * T * K + 2.0 * T * N,
                               2.0 * T * N * K)
                nl += 1
            else:
                gemm(p + "wqkv", self.xn_map, T, self.qkv)
                ops.rope_kv_append(self.qkv, self.q, self.cache, k0, v0, self.table, d_pos,
                                   d_arow, d_acol, d_aoff, self.cos, self.sin, T, hq, hkv)
                nl += 2
            def prefill_attn(stream=None):
                if self.tc_attention:
                    ops.fmha_prefill(self.kvmap, self.qmap, self.attn, self.table, d_prow, d_ppre,
                                     d_pkv, d_pqs, d_pql, n_pf, max_qlen, hkv, cfg.group, k0, v0,
                                     self.scale, stream=stream)
                else:
                    ops.paged_prefill_attn(self.kvmap, self.q, self.attn, self.table, d_prow,
                                           d_ppre, d_pkv, d_pqs, d_pql, n_pf, max_qlen, hkv,
                                           cfg.group, k0, v0, self.scale, stream=stream)

            pf_done = False
            if n_dec:
                e0 = prof.open("attn_decode") if prof is not None else None
                dargs = (self.kvmap, self.q, self.table, d_drow, d_dpre, d_dkv, n_dec, hkv,
                         cfg.group, k0, v0, self.scale, o_part, lse_part, max_splits, self.attn)
                qmap = self.qmap if self.tc_attention else None
                isolate = prof is not None and prof.isolate
                if dec_groups is not None and qmap is not None and isolate:
                    # profiled in isolation: cascade pass, context splits (timed alone),
                    # combine; the prompt prefill follows as its own class
                    ops.paged_decode_attn(*dargs, groups=dec_groups, qmap=qmap, parts=1)
                    e2 = prof.open("attn_decode_ctx")
                    ops.paged_decode_attn(*dargs, groups=dec_groups, qmap=qmap, parts=2,
                                          flat=flat)
                    if e2 is not None:
                        prof.close("attn_decode_ctx", e2, ctx_bytes, ctx_flops)
                    ops.paged_decode_attn(*dargs, groups=dec_groups, qmap=qmap, parts=4,
                                          flat=flat)
                elif dec_groups is not None and qmap is not None and self.overlap_cascade:
                    # tensor-core passes - the shared-prefix (cascade) pass on a side stream,
                    # the prompt prefill on a second one - concurrent with the per-call
                    # context splits (HBM) on the main stream; join before the LSE combine
                    main = torch.cuda.current_stream()
                    self._ev_fork.record(main)
                    self.side.wait_event(self._ev_fork)
                    two = self.side2 is not None and n_pf > 0
                    if two:
                        self.side2.wait_event(self._ev_fork)

                    def ctx_splits():
                        e2 = prof.open("attn_decode_ctx") if prof is not None else None
                        ops.paged_decode_attn(*dargs, groups=dec_groups, qmap=qmap, parts=2,
                                              flat=flat)
                        if e2 is not None:
                            prof.close("attn_decode_ctx", e2, ctx_bytes, ctx_flops)

                    ops.paged_decode_attn(*dargs, groups=dec_groups, qmap=qmap, parts=1,
                                          stream=self.side)
                    if n_pf:
                        prefill_attn(self.side2 if two else self.side)
                        pf_done = True
                        nl += 1
                    ctx_splits()
                    self._ev_join.record(self.side)
                    main.wait_event(self._ev_join)
                    if two:
                        self._ev_join2.record(self.side2)
                        main.wait_event(self._ev_join2)
                    ops.paged_decode_attn(*dargs, groups=dec_groups, qmap=qmap, parts=4,
                                          flat=flat)
                else:
                    ops.paged_decode_attn(*dargs, groups=dec_groups, qmap=qmap, flat=flat)
                if e0 is not None:
                    prof.close("attn_decode", e0, dec_bytes + (pf_bytes if pf_done else 0.0),
                               dec_flops + (pf_flops if pf_done else 0.0))
                nl += 2
            if n_pf and not pf_done:
                e0 = prof.open("attn_prefill") if prof is not None else None
                prefill_attn()
                if e0 is not None:
                    prof.close("attn_prefill", e0, pf_bytes, pf_flops)
                nl += 1
            if tp is None:
                gemm(p + "wo", self.attn_map, T, x, residual=x)
                ops.rmsnorm(x, w[p + "mlp_norm"], T, xn, cfg.eps)
                nl += 2
            else:  # partial O -> [peer exchange + residual + mlp_norm] (csrc/tp.cu)
                gemm(p + "wo", self.attn_map, T, tp.out())
                tp.signal()
                yield li
                tp.reduce(x, T, w[p + "mlp_norm"], cfg.eps, xn)
                nl += 3
            gemm(p + "wgu", self.xn_map, T, self.act, swiglu=True)  # SwiGLU in the epilogue
            nl += 1
            if tp is None:
                gemm(p + "wd", self.act_map, T, x, residual=x)
                nl += 1
            else:  # partial down -> [exchange + residual + next layer's attn_norm]
                gemm(p + "wd", self.act_map, T, tp.out())
                tp.signal()
                yield li
                nxt = f"layers.{li + 1}.attn_norm"
                tp.reduce(x, T, w.get(nxt), cfg.eps, xn if nxt in w else None)
                nl += 3
        if n_out:
            ops.rmsnorm(x, w["final_norm"], n_out, self.xn_out, cfg.eps, rows=d_orow)
            if self.full_logits or self.on_forward is not None or cfg.vocab % 128:
                gemm("lm_head", self.xn_out_map, n_out, self.logits)
                ops.argmax(self.logits, n_out, cfg.vocab, out_tok=self.out_tok, slot=d_oslot,
                           slot_tok=self.slot_tok, hist=self.hist, hist_pos=d_ohist)
            else:  # argmax fused into the lm_head epilogue: no logits round trip
                gemm("lm_head", self.xn_out_map, n_out, self.lm_part, argmax=True)
                ops.argmax_partials(self.lm_part, n_out, out_tok=self.out_tok, slot=d_oslot,
                                    slot_tok=self.slot_tok, hist=self.hist, hist_pos=d_ohist)
            nl += 3
        self.launches += nl
        self.steps += 1
        self.n_out = n_out
        if self.on_forward is not None:
            self.on_forward(plan, n_out)

    def _forward_f32(self, plan: StepPlan) -> None:
        """The fp32 step (csrc/fp32.cu): same plan semantics as the bf16 forward — decode
        tokens first (input = slot_tok[row]), then prefill tokens — every tensor fp32."""
        cfg, w = self.cfg, self.w
        i32 = np.int32
        n_dec, T = len(plan.decode), plan.n_tokens
        pos, row, col, off, pre = (np.empty(T, i32) for _ in range(5))
        tok_ids = np.zeros(T, i32)
        out_rows, out_slot, out_hist = [], [], []
        for i, d in enumerate(plan.decode):
            p = d.kv_len - 1
            c, o = token_slot(d.prefix_len, p)
            pos[i], row[i], col[i], off[i], pre[i] = p, d.row, c, o, d.prefix_len
            out_rows.append(i)
            out_slot.append(d.row)
            out_hist.append(d.hist_pos)
        t = n_dec
        for s in plan.prefill:
            n = len(s.tokens)
            for j, p in enumerate(range(s.kv_len - n, s.kv_len)):
                if s.prefix_len and p < s.prefix_len:
                    raise ValueError("prefill of a private segment cannot write prefix positions")
                c, o = token_slot(s.prefix_len, p)
                pos[t + j], row[t + j], col[t + j], off[t + j] = p, s.row, c, o
            pre[t:t + n] = s.prefix_len
            tok_ids[t:t + n] = s.tokens
            if s.out_row >= 0:
                out_rows.append(t + n - 1)
                out_slot.append(s.out_row)
                out_hist.append(s.hist_pos)
            t += n
        n_out = len(out_rows)
        if n_out > self.max_out:
            raise ValueError("too many output rows in one step")
        (d_pos, d_row, d_col, d_off, d_pre, d_tok, d_orow, d_oslot, d_ohist) = self._upload([
            pos, row, col, off, pre, tok_ids, np.asarray(out_rows, i32), np.asarray(out_slot, i32),
            np.asarray(out_hist, i32)])
        x, xn, hq, hkv = self.x, self.xn, cfg.n_heads, cfg.n_kv_heads
        nl = 0
        if n_dec:
            ops.f32_embed(w["embed"], self.slot_tok, n_dec, x, index=d_row)
            nl += 1
        if T > n_dec:
            ops.f32_embed(w["embed"], d_tok[n_dec:], T - n_dec, x[n_dec:])
            nl += 1
        plane = self.n_blocks * hkv * BLOCK_TOKENS
        for li in range(cfg.n_layers):
            p = f"layers.{li}."
            k0, v0 = 2 * li * plane, (2 * li + 1) * plane
            ops.f32_rmsnorm(x, w[p + "attn_norm"], T, xn, cfg.eps)
            ops.f32_gemm(xn, T, w[p + "wqkv"], self.qkv)
            ops.f32_rope_kv_append(self.qkv, self.q, self.cache, k0, v0, self.table, d_pos, d_row,
                                   d_col, d_off, self.cos, self.sin, T, hq, hkv)
            ops.f32_attention(self.q, self.cache, k0, v0, self.table, d_row, d_pre, d_pos, T, hq,
                              hkv, self.scale, self.attn)
            ops.f32_gemm(self.attn, T, w[p + "wo"], x, residual=x)
            ops.f32_rmsnorm(x, w[p + "mlp_norm"], T, xn, cfg.eps)
            ops.f32_gemm(xn, T, w[p + "wgu"], self.act, swiglu=True)
            ops.f32_gemm(self.act, T, w[p + "wd"], x, residual=x)
            nl += 8
        if n_out:
            ops.f32_rmsnorm(x, w["final_norm"], n_out, self.xn_out, cfg.eps, rows=d_orow)
            ops.f32_gemm(self.xn_out, n_out, w["lm_head"], self.logits)
            ops.argmax(self.logits, n_out, cfg.vocab, out_tok=self.out_tok, slot=d_oslot,
                       slot_tok=self.slot_tok, hist=self.hist, hist_pos=d_ohist)
            nl += 3
        self.launches += nl
        self.steps += 1
        self.n_out = n_out
        if self.on_forward is not None:
            self.on_forward(plan, n_out)
