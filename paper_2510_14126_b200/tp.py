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
import os
import pickle
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


# ---------------------------------------------------------------------------- replica host side
#
# One process per GPU: the replica's rank 0 (the LEADER) runs the runtime - scheduling,
# admission, routing, workflows - exactly as a TP = 1 engine; rank 1 (the FOLLOWER) holds
# the other half of the weights and KV heads and only replays the leader's device calls
# (block allocation / free / table copies and every forward), in the same order, so its
# block pool, tables and kernels mirror the leader's. The calls cross in a shared-memory
# byte ring (both ranks of a replica live on one node), one message per forward.


class ByteRing:
    """Single-producer / single-consumer ring of length-prefixed byte messages in a
    memory-mapped /dev/shm file. The producer writes the payload, then publishes it
    by advancing the tail (x86 store order keeps them in that order)."""

    HDR = 128  # bytes: head (consumer) at 0, tail (producer) at 64

    def __init__(self, path: str, create: bool, cap: int = 1 << 24) -> None:
        import numpy as np

        self.path, self.owner, self.cap = path, create, cap
        if create:
            with open(path, "wb") as f:
                f.truncate(self.HDR + cap)
        self.mm = np.memmap(path, dtype=np.uint8, mode="r+", shape=(self.HDR + cap,))
        self.ctl = self.mm[:self.HDR].view(np.int64)
        self.data = self.mm[self.HDR:]

    def _write(self, pos: int, b) -> None:
        import numpy as np

        arr = np.frombuffer(b, dtype=np.uint8)
        i = pos % self.cap
        k = min(len(arr), self.cap - i)
        self.data[i:i + k] = arr[:k]
        if k < len(arr):
            self.data[:len(arr) - k] = arr[k:]

    def _read(self, pos: int, n: int) -> bytes:
        i = pos % self.cap
        k = min(n, self.cap - i)
        if k == n:
            return self.data[i:i + n].tobytes()
        return self.data[i:i + k].tobytes() + self.data[:n - k].tobytes()

    def send(self, payload: bytes, timeout: float = 60.0) -> None:
        import struct
        import time

        n = 8 + len(payload)
        if n > self.cap:
            raise ValueError("message larger than the ring")
        tail = int(self.ctl[8])
        t_end = time.perf_counter() + timeout
        while tail + n - int(self.ctl[0]) > self.cap:
            if time.perf_counter() > t_end:
                raise TimeoutError("TP follower stopped draining its ring")
            time.sleep(0)
        self._write(tail, struct.pack("<q", len(payload)))
        self._write(tail + 8, payload)
        self.ctl[8] = tail + n

    def recv(self) -> bytes | None:
        import struct

        head = int(self.ctl[0])
        if int(self.ctl[8]) == head:
            return None
        (m,) = struct.unpack("<q", self._read(head, 8))
        out = self._read(head + 8, m)
        self.ctl[0] = head + 8 + m
        return out

    def close(self) -> None:
        self.mm = self.ctl = self.data = None
        if self.owner:
            try:
                os.unlink(self.path)
            except FileNotFoundError:
                pass


class TpLeader:
    """Stands in for the leader's GpuWorker: every device-mutating call is applied
    locally and recorded for the follower; a forward flushes the record first, so the
    follower launches the same step while the leader does."""

    def __init__(self, worker, ring: ByteRing) -> None:
        object.__setattr__(self, "_w", worker)
        object.__setattr__(self, "_ring", ring)
        object.__setattr__(self, "_out", [])

    def __getattr__(self, name):
        return getattr(self._w, name)

    def __setattr__(self, name, value) -> None:
        setattr(self._w, name, value)

    def _rec(self, *op) -> None:
        self._out.append(op)

    def flush(self) -> None:
        if self._out:
            self._ring.send(pickle.dumps(self._out, protocol=5))
            self._out.clear()

    def alloc_blocks(self, pool, reqs) -> None:
        self._rec("alloc_blocks", (pool.block_base, pool.n_blocks), list(reqs))
        self._w.alloc_blocks(pool, reqs)

    def free_blocks(self, pool, reqs) -> None:
        self._rec("free_blocks", (pool.block_base, pool.n_blocks), list(reqs))
        self._w.free_blocks(pool, reqs)

    def copy_prefix_row(self, src_row: int, dst_row: int, n_blocks: int) -> None:
        self._rec("copy_prefix_row", src_row, dst_row, n_blocks)
        self._w.copy_prefix_row(src_row, dst_row, n_blocks)

    def copy_first_token(self, src_row: int, dst_row: int) -> None:
        self._rec("copy_first_token", src_row, dst_row)
        self._w.copy_first_token(src_row, dst_row)

    def forward(self, plan) -> int:
        self._rec("forward", plan)
        self.flush()  # pickled before forward() reorders the plan
        return self._w.forward(plan)

    def forward_prefill_chunk(self, seq) -> int:
        from .model import StepPlan

        return self.forward(StepPlan(prefill=[seq]))

    def forward_decode(self, toks) -> int:
        from .model import StepPlan

        return self.forward(StepPlan(decode=toks))

    def collective(self, kind: str, *args) -> None:
        """Tell the follower to join the next process-group collective (bench plumbing)."""
        self._rec("collective", kind, args)
        self.flush()

    def stop(self) -> None:
        self._rec("stop")
        self.flush()


class _Pool:
    """The follower's copy of one engine's block pool (bitmap starts all free)."""

    def __init__(self, worker, block_base: int, n_blocks: int) -> None:
        import numpy as np

        self.block_base, self.n_blocks = block_base, n_blocks
        nwords = (n_blocks + 31) // 32
        words = np.zeros(nwords, dtype=np.uint64)
        full, rem = divmod(n_blocks, 32)
        words[:full] = 0xFFFFFFFF
        if rem:
            words[full] = (1 << rem) - 1
        self.bitmap = torch.from_numpy(words.astype(np.uint32).view(np.int32)).to(worker.device)


class TpFollower:
    """Replays the leader's device calls on this rank's shard until "stop"."""

    def __init__(self, worker, ring: ByteRing, on_collective=None) -> None:
        self.w, self.ring = worker, ring
        self.pools: dict[int, _Pool] = {}
        self.on_collective = on_collective  # fn(kind, args) joining the leader's collective
        self.forwards = 0

    def _pool(self, key) -> _Pool:
        base, n = key
        p = self.pools.get(base)
        if p is None:
            p = self.pools[base] = _Pool(self.w, base, n)
        return p

    def apply(self, ops_list) -> bool:
        """Apply one message; False once the leader said stop."""
        w = self.w
        for op in ops_list:
            name = op[0]
            if name == "forward":
                w.forward(op[1])
                self.forwards += 1
            elif name in ("alloc_blocks", "free_blocks"):
                getattr(w, name)(self._pool(op[1]), op[2])
            elif name in ("copy_prefix_row", "copy_first_token"):
                getattr(w, name)(*op[1:])
            elif name == "collective":
                if op[1] == "arm":  # a new topology arm: fresh engine slices (bitmaps all free)
                    self.pools.clear()
                if self.on_collective is None:
                    raise RuntimeError("leader issued a collective the follower cannot join")
                self.on_collective(op[1], op[2])
            elif name == "stop":
                return False
            else:
                raise ValueError(f"unknown TP op {name!r}")
        return True

    def serve(self, idle_sleep: float = 0.0) -> None:
        import time

        while True:
            msg = self.ring.recv()
            if msg is None:
                time.sleep(idle_sleep)
                continue
            if not self.apply(pickle.loads(msg)):
                return


def open_replica_ring(dist, replica: int, tp_rank: int, cap: int = 1 << 24) -> ByteRing:
    """Create (leader) / attach (follower) the replica's call ring in /dev/shm.
    Collective over the default process group (a name broadcast and two barriers)."""
    obj = [f"{os.getpid()}_{os.environ.get('MASTER_PORT', '0')}"]
    dist.broadcast_object_list(obj, src=0)
    shm = "/dev/shm" if os.path.isdir("/dev/shm") else "/tmp"
    path = os.path.join(shm, f"cortex_tp_{obj[0]}_{replica}")
    ring = ByteRing(path, create=True, cap=cap) if tp_rank == 0 else None
    dist.barrier()
    if ring is None:
        ring = ByteRing(path, create=False, cap=cap)
    dist.barrier()
    return ring
