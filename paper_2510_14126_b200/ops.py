"""Thin torch-facing wrappers over the C ABI (device pointers + the current stream).

Each wrapper checks the status code and raises KernelError on failure. Tensors
must already live on the GPU with the dtype/layout documented per op; nothing
here copies or allocates behind the caller's back (outputs are passed in).
"""

from __future__ import annotations

import ctypes

import numpy as np

import torch

from . import _lib
from .errors import KernelError

_L = None


def lib():
    global _L
    if _L is None:
        _L = _lib.load()
    return _L


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _check(rc: int, what: str) -> None:
    if rc != 0:
        raise KernelError(f"{what} failed: {_lib.STATUS_NAMES.get(rc, rc)} ({rc})")


class TensorMap:
    """A 128-byte CUtensorMap over a 2-D bf16 row-major tensor, box (box_rows, 64)."""

    __slots__ = ("buf", "tensor", "rows", "cols", "box_rows")

    def __init__(self, t: torch.Tensor, box_rows: int, rows: int | None = None) -> None:
        if t.dtype != torch.bfloat16 or t.dim() != 2 or t.stride(1) != 1:
            raise ValueError("TensorMap needs a 2-D row-major bf16 tensor")
        self.tensor = t  # keep the storage alive
        self.rows = int(rows if rows is not None else t.shape[0])
        self.cols = int(t.shape[1])
        self.box_rows = box_rows
        self.buf = ctypes.create_string_buffer(128)
        _check(
            lib().cortex_tmap_encode_2d_bf16(
                ctypes.addressof(self.buf), t.data_ptr(), self.rows, self.cols,
                t.stride(0) * 2, box_rows, 64,
            ),
            "cortex_tmap_encode_2d_bf16",
        )

    @property
    def ptr(self) -> int:
        return ctypes.addressof(self.buf)


def weight_map(w: torch.Tensor) -> TensorMap:
    return TensorMap(w, 128)


_ACT_BOX = None


def act_map(x: torch.Tensor) -> TensorMap:
    """Activation (token) operand of the GEMMs: boxes of the rows the build expects."""
    global _ACT_BOX
    if _ACT_BOX is None:
        _ACT_BOX = int(lib().cortex_act_box_rows())
    return TensorMap(x, _ACT_BOX)


def kv_map(cache2d: torch.Tensor) -> TensorMap:
    return TensorMap(cache2d, 16)


class GemmWorkspace:
    """Split-K scratch (fp32 partials + per-tile arrival counters, kept zeroed)."""

    def __init__(self, device, max_floats: int = 16 << 20, n_counters: int = 1 << 16) -> None:
        self.ws = torch.empty(max_floats, dtype=torch.float32, device=device)
        self.counters = torch.zeros(n_counters, dtype=torch.int32, device=device)


def interleave_gate_up(w: torch.Tensor) -> torch.Tensor:
    """[gate rows; up rows] (2F x d) -> blocks of 64 gate rows then the matching 64 up rows."""
    f2, d = w.shape
    f = f2 // 2
    return torch.stack([w[:f].view(f // 64, 64, d), w[f:].view(f // 64, 64, d)], dim=1).reshape(f2, d)


def deinterleave_gate_up(w: torch.Tensor) -> torch.Tensor:
    f2, d = w.shape
    v = w.view(f2 // 128, 2, 64, d)
    return torch.cat([v[:, 0].reshape(f2 // 2, d), v[:, 1].reshape(f2 // 2, d)])


def gemm_splits(M: int, N: int, K: int) -> int:
    return int(lib().cortex_gemm_splits(M, N, K))


def gemm_path(M: int, N: int, K: int) -> int:
    return int(lib().cortex_gemm_path(M, N, K))


def gemm_set_mode(mode: int) -> int:
    """Test hook: 0 auto, 1 force 1-SM, 2 force 2-SM, 3 prefer cluster split-K."""
    return _lib.set_knob("GEMM_MODE", mode)


def fmha_set_2q(on: int) -> int:
    """1: two Q tiles per CTA in the tcgen05 attention (default), 0: one, -1: chosen per
    launch by wave count (the isolated-kernel optimum; in the step, where these passes
    share the GPU with the context splits, two tiles measured faster)."""
    return _lib.set_knob("FMHA_2Q", on)


def gemm_set_stream_k(force: int) -> int:
    """-1 automatic, 0 whole tiles, 1 stream-K (2-SM kernel scheduling)."""
    return _lib.set_knob("GEMM_STREAM_K", force)


def splitk_plan(M: int, N: int, K: int) -> tuple[int, int, int, int]:
    """(splits, token tile, token tiles, weight sub-tiles) of the cluster split-K kernel."""
    tn, mt, nw = ctypes.c_int32(0), ctypes.c_int32(0), ctypes.c_int32(0)
    ks = int(lib().cortex_gemm_splitk_plan(M, N, K, ctypes.byref(tn), ctypes.byref(mt),
                                           ctypes.byref(nw)))
    return ks, tn.value, mt.value, nw.value


def gemm(wmap: TensorMap, xmap: TensorMap, M: int, out: torch.Tensor, ws: GemmWorkspace,
         residual: torch.Tensor | None = None, swiglu: bool = False, argmax: bool = False,
         stream=None) -> torch.Tensor:
    """out[:M] = X[:M] @ W^T (+ residual). out is bf16 or fp32 [>=M, N] row-major.
    swiglu: W rows interleaved (64 gate, 64 up, ...) and out = silu(g) * u, bf16 [>=M, N/2].
    argmax: out is the greedy-token partials, int64 [>=M, N/128] (float2 (max, index) per
    128-column chunk, reduced by argmax_partials); no logits are written."""
    N, K = wmap.rows, wmap.cols
    if xmap.cols != K or M > xmap.rows:
        raise ValueError("gemm shape mismatch")
    if argmax:
        if out.dtype != torch.int64 or out.shape[1] != N // 128 or residual is not None:
            raise ValueError("argmax gemm writes int64 [M, N/128] partials without residual")
        out_f32 = 3
    elif swiglu:
        if out.dtype != torch.bfloat16 or out.shape[1] != N // 2 or residual is not None:
            raise ValueError("swiglu gemm writes bf16 [M, N/2] without residual")
        out_f32 = 2
    else:
        out_f32 = 1 if out.dtype == torch.float32 else 0
    ldr = residual.stride(0) if residual is not None else 0
    _check(
        lib().cortex_gemm_bf16(
            wmap.ptr, xmap.ptr, M, N, K, out.data_ptr(), out.stride(0), out_f32, _ptr(residual),
            ldr, ws.ws.data_ptr(), ws.ws.numel() * 4, ws.counters.data_ptr(),
            ws.counters.numel(), _stream(stream),
        ),
        "cortex_gemm_bf16",
    )
    return out


def rope_token_prep(table, tok_pos, tok_row, tok_col, tok_off, cos_tab, sin_tab, n_tok, hkv,
                    tok_dst, tok_cs, stream=None) -> None:
    """Per-step operands of gemm_qkv_rope: K/V row within a plane, cos | sin per token."""
    _check(lib().cortex_rope_token_prep(
        table.data_ptr(), table.stride(0), tok_pos.data_ptr(), tok_row.data_ptr(),
        tok_col.data_ptr(), tok_off.data_ptr(), cos_tab.data_ptr(), sin_tab.data_ptr(), n_tok,
        hkv, tok_dst.data_ptr(), tok_cs.data_ptr(), _stream(stream)), "cortex_rope_token_prep")


def gemm_qkv_rope(wmap: TensorMap, xmap: TensorMap, M: int, ws: GemmWorkspace, q_out, cache,
                  k_row0, v_row0, tok_dst, tok_cs, hq: int, hkv: int, stream=None) -> None:
    """QKV projection with RoPE + paged KV append in the epilogue (rope_kv_append fused);
    tok_dst / tok_cs from rope_token_prep."""
    N, K = wmap.rows, wmap.cols
    if xmap.cols != K or M > xmap.rows or N != (hq + 2 * hkv) * 128:
        raise ValueError("qkv gemm shape mismatch")
    e = _lib.RopeEpilogue(q_out.data_ptr(), cache.data_ptr(), k_row0, v_row0, tok_dst.data_ptr(),
                          tok_cs.data_ptr(), hq, hkv)
    _check(lib().cortex_gemm_qkv_rope(wmap.ptr, xmap.ptr, M, N, K, ctypes.byref(e),
                                      ws.ws.data_ptr(), ws.ws.numel() * 4,
                                      ws.counters.data_ptr(), ws.counters.numel(),
                                      _stream(stream)), "cortex_gemm_qkv_rope")


def embed(emb: torch.Tensor, tokens: torch.Tensor, n_tok: int, out: torch.Tensor,
          index: torch.Tensor | None = None, stream=None) -> None:
    _check(lib().cortex_embed(emb.data_ptr(), tokens.data_ptr(), _ptr(index), n_tok,
                              emb.shape[1], out.data_ptr(), _stream(stream)), "cortex_embed")


def rmsnorm(x: torch.Tensor, w: torch.Tensor, n_rows: int, y: torch.Tensor, eps: float,
            rows: torch.Tensor | None = None, stream=None) -> None:
    _check(lib().cortex_rmsnorm(x.data_ptr(), _ptr(rows), n_rows, w.data_ptr(), x.shape[1],
                                eps, y.data_ptr(), _stream(stream)), "cortex_rmsnorm")


def rope_kv_append(qkv, q_out, cache, k_row0, v_row0, table, tok_pos, tok_row, tok_col, tok_off,
                   cos_tab, sin_tab, n_tok, hq, hkv, stream=None) -> None:
    _check(
        lib().cortex_rope_kv_append(
            qkv.data_ptr(), q_out.data_ptr(), cache.data_ptr(), k_row0, v_row0, table.data_ptr(),
            table.stride(0), tok_pos.data_ptr(), tok_row.data_ptr(), tok_col.data_ptr(),
            tok_off.data_ptr(), cos_tab.data_ptr(), sin_tab.data_ptr(), n_tok, hq, hkv,
            _stream(stream),
        ),
        "cortex_rope_kv_append",
    )


def argmax(logits: torch.Tensor, n_rows: int, vocab: int, out_tok: torch.Tensor | None = None,
           slot: torch.Tensor | None = None, slot_tok: torch.Tensor | None = None,
           hist: torch.Tensor | None = None, hist_pos: torch.Tensor | None = None,
           stream=None) -> None:
    _check(
        lib().cortex_argmax(
            logits.data_ptr(), logits.stride(0), n_rows, vocab, _ptr(out_tok), _ptr(slot),
            _ptr(slot_tok), _ptr(hist), hist.stride(0) if hist is not None else 0, _ptr(hist_pos),
            _stream(stream),
        ),
        "cortex_argmax",
    )


def argmax_partials(part: torch.Tensor, n_rows: int, out_tok=None, slot=None, slot_tok=None,
                    hist=None, hist_pos=None, stream=None) -> None:
    """Greedy token per row from gemm(..., argmax=True) partials (same rule as argmax)."""
    _check(
        lib().cortex_argmax_partials(
            part.data_ptr(), part.shape[1], n_rows, _ptr(out_tok), _ptr(slot), _ptr(slot_tok),
            _ptr(hist), hist.stride(0) if hist is not None else 0, _ptr(hist_pos),
            _stream(stream)),
        "cortex_argmax_partials",
    )


def decode_splits(prefix_len: int, kv_len: int) -> int:
    return int(lib().cortex_decode_splits(prefix_len, kv_len))


class QMap:
    """3-D TMA descriptor over q [n_tok, hq, 128] for the tensor-core attention kernels."""

    __slots__ = ("buf", "tensor")

    def __init__(self, q: torch.Tensor, hq: int, group: int) -> None:
        if q.dtype != torch.bfloat16 or not q.is_contiguous():
            raise ValueError("QMap needs a contiguous bf16 tensor")
        self.tensor = q
        self.buf = ctypes.create_string_buffer(128)
        n_tok = q.numel() // (hq * 128)
        _check(lib().cortex_tmap_encode_q(ctypes.addressof(self.buf), q.data_ptr(), n_tok, hq,
                                          group), "cortex_tmap_encode_q")

    @property
    def ptr(self) -> int:
        return ctypes.addressof(self.buf)


def paged_decode_attn(kvmap: TensorMap, q, table, seq_row, seq_prefix, seq_kvlen, n_seqs,
                      n_kv_heads, group, k_row0, v_row0, scale, o_part, lse_part, max_splits, out,
                      groups=None, qmap: QMap | None = None, parts: int = 7,
                      stream=None, flat=None) -> None:
    """groups: None, or (grp_row, grp_plen, grp_first, grp_count, n_groups, max_count,
    prefix_slots) for shared-prefix (cascade) attention; qmap selects the tcgen05 cascade;
    parts: 1 cascade pass | 2 context splits | 4 combine; flat: None (fixed per-call
    splits) or (seq_tile_start, total_tiles, tiles_per_chunk) from decode_flat_plan."""
    if groups is None:
        g = (None, None, None, None, 0, 0, 0)
    else:
        g = (_ptr(groups[0]), _ptr(groups[1]), _ptr(groups[2]), _ptr(groups[3])) + tuple(groups[4:])
    f = (None, 0, 0) if flat is None else (_ptr(flat[0]), int(flat[1]), int(flat[2]))
    _check(
        lib().cortex_paged_decode_attn(
            kvmap.ptr, q.data_ptr(), table.data_ptr(), table.stride(0), seq_row.data_ptr(),
            seq_prefix.data_ptr(), seq_kvlen.data_ptr(), *f, n_seqs, n_kv_heads, group, k_row0,
            v_row0, scale, o_part.data_ptr(), lse_part.data_ptr(), max_splits, out.data_ptr(),
            *g, qmap.ptr if qmap is not None else None, parts, _stream(stream),
        ),
        "cortex_paged_decode_attn",
    )


FLAT_MAX_W = 48  # kFlatMaxW in attention.cu


def decode_flat_plan(seq_prefix, seq_kvlen, n_kv_heads: int, cascade: bool, max_pieces: int,
                     W: int | None = None):
    """Host half of the balanced decode plan (numpy int arrays in): (per-call flat tile
    starts, total tiles, tiles per chunk, most slots a call's pieces need), or None when
    the calls would need more than `max_pieces` slots each even at the widest chunk."""
    prefix = np.asarray(seq_prefix, np.int64)
    kvlen = np.asarray(seq_kvlen, np.int64)
    if len(prefix) == 0:
        return None
    npb = (prefix + 15) // 16
    n = (kvlen - prefix + 15) // 16 + (0 if cascade else npb)
    start = np.zeros_like(n)
    np.cumsum(n[:-1], out=start[1:])
    total = int(n.sum())
    if W is None:
        W = int(lib().cortex_decode_tiles_per_chunk(total, n_kv_heads))
    pieces = int(((start + n - 1) // W - start // W + 1).max())
    if pieces > max_pieces:  # widen the chunks: a call spans <= ceil(n / W) + 1 of them
        W = min(FLAT_MAX_W, max(W, -(-int(n.max()) // max(max_pieces - 1, 1))))
        pieces = int(((start + n - 1) // W - start // W + 1).max())
        if pieces > max_pieces:
            return None
    return start.astype(np.int32), total, W, pieces


def fmha_prefill(kvmap: TensorMap, qmap: QMap, out, table, seq_row, seq_prefix, seq_kvlen,
                 seq_qstart, seq_qlen, n_seqs, max_qlen, n_kv_heads, group, k_row0, v_row0,
                 scale, stream=None) -> None:
    _check(
        lib().cortex_fmha_prefill_tc(
            kvmap.ptr, qmap.ptr, out.data_ptr(), table.data_ptr(), table.stride(0),
            seq_row.data_ptr(), seq_prefix.data_ptr(), seq_kvlen.data_ptr(),
            seq_qstart.data_ptr(), seq_qlen.data_ptr(), n_seqs, max_qlen, n_kv_heads, group,
            k_row0, v_row0, scale, _stream(stream),
        ),
        "cortex_fmha_prefill_tc",
    )


def paged_prefill_attn(kvmap: TensorMap, q, out, table, seq_row, seq_prefix, seq_kvlen,
                       seq_qstart, seq_qlen, n_seqs, max_qlen, n_kv_heads, group, k_row0, v_row0,
                       scale, stream=None) -> None:
    _check(
        lib().cortex_paged_prefill_attn(
            kvmap.ptr, q.data_ptr(), out.data_ptr(), table.data_ptr(), table.stride(0),
            seq_row.data_ptr(), seq_prefix.data_ptr(), seq_kvlen.data_ptr(),
            seq_qstart.data_ptr(), seq_qlen.data_ptr(), n_seqs, max_qlen, n_kv_heads, group,
            k_row0, v_row0, scale, _stream(stream),
        ),
        "cortex_paged_prefill_attn",
    )


def kv_alloc(bitmap, nblocks, id_base, counts, rows, cols, n_req, table, status,
             stream=None) -> None:
    _check(
        lib().cortex_kv_alloc(bitmap.data_ptr(), nblocks, id_base, counts.data_ptr(),
                              rows.data_ptr(), cols.data_ptr(), n_req, table.data_ptr(),
                              table.stride(0), status.data_ptr(), _stream(stream)),
        "cortex_kv_alloc",
    )


def kv_free(bitmap, nblocks, id_base, table, rows, cols, counts, n_req, status,
            stream=None) -> None:
    _check(
        lib().cortex_kv_free(bitmap.data_ptr(), nblocks, id_base, table.data_ptr(),
                             table.stride(0), rows.data_ptr(), cols.data_ptr(), counts.data_ptr(),
                             n_req, status.data_ptr(), _stream(stream)),
        "cortex_kv_free",
    )


def table_copy(table, src_rows, dst_rows, dst_cols, counts, n, stream=None) -> None:
    _check(
        lib().cortex_table_copy(table.data_ptr(), table.stride(0), src_rows.data_ptr(),
                                dst_rows.data_ptr(), dst_cols.data_ptr(), counts.data_ptr(), n,
                                _stream(stream)),
        "cortex_table_copy",
    )


def kv_count_free(bitmap, nblocks, out_free, stream=None) -> None:
    _check(lib().cortex_kv_count_free(bitmap.data_ptr(), nblocks, out_free.data_ptr(),
                                      _stream(stream)), "cortex_kv_count_free")


def _hptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _i32(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.int32))


def kv_alloc_h(bitmap, nblocks, id_base, counts, rows, cols, table, status, stream=None) -> None:
    """kv_alloc with the request arrays in host memory (passed in the kernel parameters)."""
    c, r, k = _i32(counts), _i32(rows), _i32(cols)
    _check(lib().cortex_kv_alloc_h(bitmap.data_ptr(), nblocks, id_base, _hptr(c), _hptr(r),
                                   _hptr(k), len(c), table.data_ptr(), table.stride(0),
                                   status.data_ptr(), _stream(stream)), "cortex_kv_alloc_h")


def kv_free_h(bitmap, nblocks, id_base, table, rows, cols, counts, status, stream=None) -> None:
    r, k, c = _i32(rows), _i32(cols), _i32(counts)
    _check(lib().cortex_kv_free_h(bitmap.data_ptr(), nblocks, id_base, table.data_ptr(),
                                  table.stride(0), _hptr(r), _hptr(k), _hptr(c), len(r),
                                  status.data_ptr(), _stream(stream)), "cortex_kv_free_h")


def table_copy_h(table, src_rows, dst_rows, dst_cols, counts, stream=None) -> None:
    s, d, k, c = _i32(src_rows), _i32(dst_rows), _i32(dst_cols), _i32(counts)
    _check(lib().cortex_table_copy_h(table.data_ptr(), table.stride(0), _hptr(s), _hptr(d),
                                     _hptr(k), _hptr(c), len(s), _stream(stream)),
           "cortex_table_copy_h")


# ---------------------------------------------------------------- fp32 path (config 1)

def f32_gemm(x: torch.Tensor, M: int, w: torch.Tensor, out: torch.Tensor,
             residual: torch.Tensor | None = None, swiglu: bool = False, stream=None) -> None:
    """out[:M] = x[:M] @ w^T (+ residual); swiglu: w = [gate; up] (2F x K), out [M, F]."""
    N = w.shape[0] // 2 if swiglu else w.shape[0]
    K = w.shape[1]
    mode = 2 if swiglu else (1 if residual is not None else 0)
    _check(lib().cortex_f32_gemm(x.data_ptr(), x.stride(0), w.data_ptr(), M, N, K,
                                 out.data_ptr(), out.stride(0), _ptr(residual),
                                 residual.stride(0) if residual is not None else 0, mode,
                                 _stream(stream)), "cortex_f32_gemm")


def f32_embed(emb, tokens, n_tok, out, index=None, stream=None) -> None:
    _check(lib().cortex_f32_embed(emb.data_ptr(), tokens.data_ptr(), _ptr(index), n_tok,
                                  emb.shape[1], out.data_ptr(), _stream(stream)),
           "cortex_f32_embed")


def f32_rmsnorm(x, w, n_rows, y, eps, rows=None, stream=None) -> None:
    _check(lib().cortex_f32_rmsnorm(x.data_ptr(), _ptr(rows), n_rows, w.data_ptr(), x.shape[1],
                                    eps, y.data_ptr(), _stream(stream)), "cortex_f32_rmsnorm")


def f32_rope_kv_append(qkv, q_out, cache, k_row0, v_row0, table, tok_pos, tok_row, tok_col,
                       tok_off, cos_tab, sin_tab, n_tok, hq, hkv, stream=None) -> None:
    _check(lib().cortex_f32_rope_kv_append(
        qkv.data_ptr(), q_out.data_ptr(), cache.data_ptr(), k_row0, v_row0, table.data_ptr(),
        table.stride(0), tok_pos.data_ptr(), tok_row.data_ptr(), tok_col.data_ptr(),
        tok_off.data_ptr(), cos_tab.data_ptr(), sin_tab.data_ptr(), n_tok, hq, hkv,
        _stream(stream)), "cortex_f32_rope_kv_append")


def f32_attention(q, cache, k_row0, v_row0, table, tok_row, tok_prefix, tok_pos, n_tok, hq, hkv,
                  scale, out, stream=None) -> None:
    _check(lib().cortex_f32_attention(
        q.data_ptr(), cache.data_ptr(), k_row0, v_row0, table.data_ptr(), table.stride(0),
        tok_row.data_ptr(), tok_prefix.data_ptr(), tok_pos.data_ptr(), n_tok, hq, hkv, scale,
        out.data_ptr(), _stream(stream)), "cortex_f32_attention")
