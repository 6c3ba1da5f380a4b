"""ctypes binding of libcortex_b200.so (the C ABI in include/cortex_b200.h).

There is no fallback: if the library is missing or cannot be loaded the import
of any op fails with an ImportError naming the build command.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import c_float, c_int32, c_int64, c_uint64, c_void_p
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libcortex_b200.so"

P = c_void_p
I32 = c_int32
I64 = c_int64
U64 = c_uint64
F32 = c_float

# name -> argtypes (every export returns int32 status)
SIGNATURES: dict[str, list] = {
    "cortex_abi_version": [],
    "cortex_kv_alloc": [P, I32, I32, P, P, P, I32, P, I32, P, P],
    "cortex_kv_free": [P, I32, I32, P, I32, P, P, P, I32, P, P],
    "cortex_table_copy": [P, I32, P, P, P, P, I32, P],
    "cortex_kv_count_free": [P, I32, P, P],
    "cortex_kv_alloc_h": [P, I32, I32, P, P, P, I32, P, I32, P, P],
    "cortex_kv_free_h": [P, I32, I32, P, I32, P, P, P, I32, P, P],
    "cortex_table_copy_h": [P, I32, P, P, P, P, I32, P],
    "cortex_tmap_encode_2d_bf16": [P, P, U64, U64, U64, ctypes.c_uint32, ctypes.c_uint32],
    "cortex_gemm_bf16": [P, P, I32, I32, I32, P, I32, I32, P, I32, P, U64, P, I32, P],
    "cortex_gemm_qkv_rope": [P, P, I32, I32, I32, P, P, U64, P, I32, P],
    "cortex_rope_token_prep": [P, I32, P, P, P, P, P, P, I32, I32, P, P, P],
    "cortex_embed": [P, P, P, I32, I32, P, P],
    "cortex_rmsnorm": [P, P, I32, P, I32, F32, P, P],
    "cortex_rope_kv_append": [P, P, P, I64, I64, P, I32, P, P, P, P, P, P, I32, I32, I32, P],
    "cortex_argmax": [P, I64, I32, I32, P, P, P, P, I32, P, P],
    "cortex_argmax_partials": [P, I32, I32, P, P, P, P, I32, P, P],
    "cortex_f32_gemm": [P, I32, P, I32, I32, I32, P, I32, P, I32, I32, P],
    "cortex_f32_embed": [P, P, P, I32, I32, P, P],
    "cortex_f32_rmsnorm": [P, P, I32, P, I32, F32, P, P],
    "cortex_f32_rope_kv_append": [P, P, P, I64, I64, P, I32, P, P, P, P, P, P, I32, I32, I32, P],
    "cortex_f32_attention": [P, P, I64, I64, P, I32, P, P, P, I32, I32, I32, F32, P, P],
    "cortex_decode_splits": [I32, I32],
    "cortex_paged_decode_attn": [P, P, P, I32, P, P, P, P, I32, I32, I32, I32, I32, I64, I64,
                                 F32, P, P, I32, P, P, P, P, P, I32, I32, I32, P, I32, P],
    "cortex_tmap_encode_q": [P, P, U64, I32, I32],
    "cortex_fmha_prefill_tc": [P, P, P, P, I32, P, P, P, P, P, I32, I32, I32, I32, I64, I64, F32,
                               P],
    "cortex_fmha_cascade_tc": [P, P, P, I32, P, P, P, P, I32, I32, I32, I32, I32, I64, I64, F32,
                               P, P, I32, P],
    "cortex_decoder_layers": [P, P],
    "cortex_sym_alloc": [U64, P],
    "cortex_sym_free": [P],
    "cortex_ipc_get_handle": [P, P],
    "cortex_ipc_open_handle": [P, P],
    "cortex_ipc_close": [P],
    "cortex_tp_flag_bytes": [],
    "cortex_tp_signal": [P, ctypes.c_uint32, P],
    "cortex_tp_allreduce_rmsnorm": [P, P, P, I32, I32, P, F32, P, P, ctypes.c_uint32, P, P],
}

# The private tuning / test interface (csrc/cortex_dev.h): not part of the boundary.
DEV_SIGNATURES: dict[str, list] = {
    "cortex_dev_set_knob": [I32, I32],
    "cortex_dev_get_knob": [I32],
    "cortex_dev_last_cuda_error": [],
    "cortex_gemm_splits": [I32, I32, I32],
    "cortex_gemm_path": [I32, I32, I32],
    "cortex_gemm2_tile": [I32, I32, I32],
    "cortex_gemm_splitk_plan": [I32, I32, I32, P, P, P],
    "cortex_decode_tiles_per_chunk": [I32, I32],
    "cortex_act_box_rows": [],
    "cortex_paged_prefill_attn": [P, P, P, P, I32, P, P, P, P, P, I32, I32, I32, I32, I64, I64,
                                  F32, P],
}

# knob ids (csrc/cortex_dev.h, enum CortexKnob)
KNOBS = {name: i for i, name in enumerate(
    ["PDL", "GEMM_MODE", "GEMM_STREAM_K", "GEMM_TN", "GEMM_L2PF", "SK_KS", "SK_MT", "SK_NW",
     "SK_ISSUE", "FMHA_2Q", "FMHA_PLO", "GEMM_TILE_OVH"])}

class RopeEpilogue(ctypes.Structure):
    """cortex_rope_epilogue_t (include/cortex_b200.h)."""

    _fields_ = [("q_out", P), ("cache", P), ("k_row0", I64), ("v_row0", I64), ("tok_dst", P),
                ("tok_cs", P), ("hq", I32), ("hkv", I32)]


class DecoderDesc(ctypes.Structure):
    """cortex_decoder_t (include/cortex_b200.h)."""

    _fields_ = [("n_layers", I32), ("d_model", I32), ("hq", I32), ("hkv", I32), ("ffn", I32),
                ("eps", F32), ("softmax_scale", F32),
                ("tmap_wqkv", P), ("tmap_wo", P), ("tmap_wgu", P), ("tmap_wd", P),
                ("attn_norm", P), ("mlp_norm", P),
                ("tmap_xn", P), ("tmap_attn", P), ("tmap_act", P), ("tmap_kv", P),
                ("tmap_q", P),
                ("x", P), ("xn", P), ("q", P), ("attn", P), ("act", P), ("cache", P),
                ("plane_rows", I64), ("table", P), ("table_stride", I32),
                ("tok_dst", P), ("tok_cs", P),
                ("workspace", P), ("workspace_bytes", U64), ("counters", P), ("n_counters", I32)]


class StepDesc(ctypes.Structure):
    """cortex_step_t (include/cortex_b200.h)."""

    _fields_ = [("n_tok", I32), ("n_dec", I32), ("n_pf", I32), ("max_qlen", I32),
                ("max_splits", I32), ("layer_begin", I32), ("layer_end", I32),
                ("dec_row", P), ("dec_prefix", P), ("dec_kvlen", P),
                ("pf_row", P), ("pf_prefix", P), ("pf_kvlen", P), ("pf_qstart", P),
                ("pf_qlen", P),
                ("grp_row", P), ("grp_plen", P), ("grp_first", P), ("grp_count", P),
                ("n_groups", I32), ("max_group_count", I32), ("prefix_slots", I32),
                ("o_part", P), ("lse_part", P), ("stream", P), ("side_stream", P),
                ("side_stream2", P)]


STATUS_NAMES = {0: "ok", -1: "bad argument", -2: "CUDA error", -3: "out of KV blocks",
                -4: "unsupported",
                -5: "cross-GPU wait timed out"}

_LIB: ctypes.CDLL | None = None


def load() -> ctypes.CDLL:
    """Load the library (once) and declare every export's signature."""
    global _LIB
    if _LIB is None:
        # CORTEX_LIB: an alternative build of the same library (tuning variants)
        path = Path(os.environ.get("CORTEX_LIB") or str(LIB_PATH))
        if not path.exists():
            raise ImportError(
                f"{path} is missing; build it with `python -m paper_2510_14126_b200.build` "
                "(there is no CPU fallback)"
            )
        lib = ctypes.CDLL(str(path))
        for name, argtypes in {**SIGNATURES, **DEV_SIGNATURES}.items():
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = c_int32
        _LIB = lib
    return _LIB


def exported_symbols() -> list[str]:
    return list(SIGNATURES)


def set_knob(name: str, value: int) -> int:
    """Tuning / test hook (csrc/cortex_dev.h); returns the previous value."""
    lib = load()
    k = KNOBS[name]
    prev = lib.cortex_dev_get_knob(k)
    rc = lib.cortex_dev_set_knob(k, int(value))
    if rc != 0:
        raise ValueError(f"knob {name} = {value} rejected ({rc})")
    return prev
