"""Tensor parallelism (TP = 2) inside one engine replica (BASELINE config 5).

The reference engine has no model (stagesim/engines.py:101-246), so TP has no
reference counterpart beyond config 5's "tensor-parallel=2 per replica". The
split is Megatron-style over the two GPUs of a replica:

  * attention: rank r owns q heads [r*Hq/2, (r+1)*Hq/2) and the kv heads they
    read (GQA groups stay whole), i.e. its slice of wqkv rows, its half of the
    KV cache (every block id exists on both ranks, each holding its kv heads),
    and the matching wo columns;
  * MLP: rank r owns ffn rows [r*F/2, (r+1)*F/2) of gate and up and the matching
    wd columns;
  * embedding, norms and lm_head are replicated.

The O and down projections therefore produce fp32 partial sums. Each is followed
by ONE kernel (csrc/tp.cu) that reads the peer's partial straight from the peer's
HBM over NVLink, adds both partials to the residual stream in a fixed order and
writes the next RMSNorm's output: all-reduce + residual + norm in one pass,
no NCCL call on the data path. Both ranks hold bit-identical residual streams,
so their logits and greedy tokens are identical.

`TpComm` owns a rank's symmetric exchange buffer; peers are connected either
in-process (`connect_local`, two workers on one GPU — the single-GPU parity test
drives them in lockstep, see `lockstep`) or across processes by CUDA IPC
(`connect_ipc`, handles exchanged over the process group).
"""

from __future__ import annotations

import ctypes
from dataclasses import replace

import torch

from . import ops
from .config import HEAD_DIM, ModelConfig

FLAG_BYTES = 256


def shard_config(cfg: ModelConfig, tp: int) -> ModelConfig:
    """The per-rank shape of a TP-`tp` replica (heads and ffn divided)."""
    if tp == 1:
        return cfg
    if cfg.n_kv_heads % tp or cfg.n_heads % tp or cfg.ffn % (64 * tp):
        raise ValueError(f"{cfg.name} cannot be split {tp} ways")
    return replace(cfg, name=f"{cfg.name}/tp{tp}", n_heads=cfg.n_heads // tp,
                   n_kv_heads=cfg.n_kv_heads // tp, ffn=cfg.ffn // tp)


def shard_weights(w: dict, cfg: ModelConfig, rank: int, tp: int) -> dict:
    """Rank `rank`'s slices of the canonical (gate rows then up rows) weights."""
    if tp == 1:
        return dict(w)
    hq, hkv, f = cfg.n_heads // tp, cfg.n_kv_heads // tp, cfg.ffn // tp
    qd, kd = cfg.n_heads * HEAD_DIM, cfg.n_kv_heads * HEAD_DIM
    out = {}
    for k, v in w.items():
        if k.endswith(".wqkv"):
            q = v[rank * hq * HEAD_DIM:(rank + 1) * hq * HEAD_DIM]
            kk = v[qd + rank * hkv * HEAD_DIM:qd + (rank + 1) * hkv * HEAD_DIM]
            vv = v[qd + kd + rank * hkv * HEAD_DIM:qd + kd + (rank + 1) * hkv * HEAD_DIM]
            out[k] = torch.cat([q, kk, vv]).contiguous()
        elif k.endswith(".wo"):
            out[k] = v[:, rank * hq * HEAD_DIM:(rank + 1) * hq * HEAD_DIM].contiguous()
        elif k.endswith(".wgu"):
            out[k] = torch.cat([v[rank * f:(rank + 1) * f],
                                v[cfg.ffn + rank * f:cfg.ffn + (rank + 1) * f]]).contiguous()
        elif k.endswith(".wd"):
            out[k] = v[:, rank * f:(rank + 1) * f].contiguous()
        else:
            out[k] = v
    return out


class _CudaArray:
    """__cuda_array_interface__ over a raw device pointer (a torch view, no copy)."""

    def __init__(self, ptr: int, n: int, typestr: str = "<f4") -> None:
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                         "data": (ptr, False), "version": 3}


class TpComm:
    """One rank's side of a TP = 2 replica: the symmetric partial-output buffer,
    the peer's mapping of it, and the exchange epoch."""

    def __init__(self, device, rank: int, size: int, max_tokens: int, d: int) -> None:
        if size != 2 or rank not in (0, 1):
            raise ValueError("TpComm supports tensor-parallel size 2")
        self.device = torch.device(device)
        self.rank, self.size = rank, size
        self.max_tokens, self.d = max_tokens, d
        self.part_bytes = max_tokens * d * 4
        L = ops.lib()
        if int(L.cortex_tp_flag_bytes()) != FLAG_BYTES:
            raise RuntimeError("library / host disagree on the TP flag area")
        p = ctypes.c_void_p()
        ops._check(L.cortex_sym_alloc(FLAG_BYTES + 2 * self.part_bytes, ctypes.byref(p)),
                   "cortex_sym_alloc")
        self.base = int(p.value)
        self.y = [torch.as_tensor(_CudaArray(self._part(self.base, par), max_tokens * d),
                                  device=self.device).view(max_tokens, d) for par in (0, 1)]
        self.peer_base: int | None = None
        self._ipc = False
        self.epoch = 0
        self.status = torch.zeros(1, dtype=torch.int32, device=self.device)

    def _part(self, base: int, parity: int) -> int:
        return base + FLAG_BYTES + parity * self.part_bytes

    # ---- connection ----

    @staticmethod
    def connect_local(a: "TpComm", b: "TpComm") -> None:
        """Both ranks in this process (single-GPU parity runs)."""
        a.peer_base, b.peer_base = b.base, a.base

    def connect_ipc(self, group=None) -> None:
        """Exchange CUDA IPC handles with the peer over the process group (collective)."""
        import torch.distributed as dist

        h = ctypes.create_string_buffer(64)
        ops._check(ops.lib().cortex_ipc_get_handle(ctypes.c_void_p(self.base), h),
                   "cortex_ipc_get_handle")
        allh = [None] * dist.get_world_size(group)
        dist.all_gather_object(allh, (self.rank, h.raw), group=group)
        peer = [raw for r, raw in allh if r != self.rank]
        if len(peer) != 1:
            raise RuntimeError("TP group must hold exactly two ranks")
        p = ctypes.c_void_p()
        ops._check(ops.lib().cortex_ipc_open_handle(ctypes.create_string_buffer(peer[0], 64),
                                                    ctypes.byref(p)), "cortex_ipc_open_handle")
        self.peer_base = int(p.value)
        self._ipc = True

    def close(self) -> None:
        if self._ipc and self.peer_base:
            ops.lib().cortex_ipc_close(ctypes.c_void_p(self.peer_base))
        self.peer_base = None
        if self.base:
            torch.cuda.synchronize(self.device)
            self.y = []
            ops.lib().cortex_sym_free(ctypes.c_void_p(self.base))
            self.base = 0

    # ---- one exchange: out() -> GEMM -> signal() -> (yield) -> reduce() ----

    def out(self) -> torch.Tensor:
        """The partial-output buffer the next GEMM writes (parity of the next epoch)."""
        return self.y[(self.epoch + 1) & 1]

    def signal(self, stream=None) -> None:
        if self.peer_base is None:
            raise RuntimeError("TpComm is not connected to its peer")
        self.epoch += 1
        ops._check(ops.lib().cortex_tp_signal(ctypes.c_void_p(self.peer_base),
                                              ctypes.c_uint32(self.epoch & 0xFFFFFFFF),
                                              ops._stream(stream)), "cortex_tp_signal")

    def reduce(self, x: torch.Tensor, n_rows: int, norm_w: torch.Tensor | None, eps: float,
               out: torch.Tensor | None, stream=None) -> None:
        """x[:n] += partial(rank 0) + partial(rank 1); out[:n] = rmsnorm(x) * norm_w."""
        par = self.epoch & 1
        mine, peer = self._part(self.base, par), self._part(self.peer_base, par)
        y0, y1 = (mine, peer) if self.rank == 0 else (peer, mine)
        ops._check(ops.lib().cortex_tp_allreduce_rmsnorm(
            ctypes.c_void_p(y0), ctypes.c_void_p(y1), x.data_ptr(), n_rows, self.d,
            ops._ptr(norm_w), eps, ops._ptr(out), ctypes.c_void_p(self.base),
            ctypes.c_uint32(self.epoch & 0xFFFFFFFF), self.status.data_ptr(),
            ops._stream(stream)), "cortex_tp_allreduce_rmsnorm")


def lockstep(gens) -> None:
    """Drive the forward generators of the ranks of one replica that share a GPU
    and a stream: each rank runs up to its next exchange point (GEMM + signal
    enqueued) before any rank enqueues the reduce that reads it, so every wait is
    satisfied by stream order and no kernel ever spins on another."""
    live = list(gens)
    while live:
        nxt = []
        for g in live:
            try:
                next(g)
                nxt.append(g)
            except StopIteration:
                pass
        live = nxt
