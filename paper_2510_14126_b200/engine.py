"""`GpuEngineState`: the reference engine interface backed by a B200.

Drop-in for `stagesim.engines.EngineState` (/root/reference/pkg/src/stagesim/
engines.py:101-246): same constructor, attributes, methods, return values and
errors, so the reference `Simulator` (simulation.py:363-369 is the factory seam)
and scheduling policies (scheduling.py:129-165) drive it unchanged.

Two halves:
  * host accounting — a line-for-line restatement of the reference's token
    bookkeeping (kv_used float, kv_reserved int, resident prefixes, batch,
    decode_epoch). Scheduling decisions read only these, so dispatch order,
    routing and eviction are bit-identical to the CPU engine by construction;
  * the GPU mirror — every state transition also enqueues the matching device
    work on the engine's GPU: block allocation from the engine's bitmap pool
    (prefix blocks on a cold admit, prompt blocks, one block per 16 generated
    tokens), prefix and prompt prefill, batched greedy decode up to the tokens
    the reference has emitted (floor of tokens_emitted), and block release on
    completion / eviction.

Block-allocation order (the contract oracle/engine_ref.py restates): per admit,
[prefix blocks if cold, then ceil(p/16) prompt blocks]; per decode step, one
block for each call whose next token starts a block, in batch order; frees on
complete_call (the call's private blocks) and evict_idle_prefix (the prefix).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import ops
from .config import BLOCK_TOKENS
from .errors import AdmitWithoutCapacity, InternalInvariantViolation, PrefixInUse
from .model import DecodeTok, GpuWorker, PrefillSeq
from .tokens import prefix_tokens, prompt_tokens

PREFILL = "prefill"
DECODE = "decode"


def _blocks(n: int) -> int:
    return (n + BLOCK_TOKENS - 1) // BLOCK_TOKENS


@dataclass(frozen=True)
class EngineParams:
    """Mirror of stagesim.engines.EngineParams (engines.py:35-57)."""

    kv_capacity_tokens: int
    prefill_rate: float
    base_token_time: float
    batch_slope: float
    max_batch: int

    def __post_init__(self) -> None:
        if self.kv_capacity_tokens <= 0:
            raise ValueError("kv_capacity_tokens must be positive")
        if self.prefill_rate <= 0:
            raise ValueError("prefill_rate must be positive")
        if self.base_token_time <= 0:
            raise ValueError("base_token_time must be positive")
        if self.batch_slope < 0:
            raise ValueError("batch_slope must be >= 0")
        if self.max_batch < 1:
            raise ValueError("max_batch must be >= 1")

    def token_time(self, batch_size: int) -> float:
        return self.base_token_time * (1.0 + self.batch_slope * (batch_size - 1))


@dataclass
class PendingCall:
    """Mirror of stagesim.engines.PendingCall (engines.py:70-78)."""

    request_id: int
    stage_id: str
    enqueue_time: float
    prompt_tokens: int = 0
    target_output_tokens: int = 0


@dataclass
class InFlightCall:
    """Mirror of stagesim.engines.InFlightCall (engines.py:81-92) + its GPU slot."""

    request_id: int
    stage_id: str
    prompt_tokens: int
    target_output_tokens: int
    tokens_emitted: float = 0.0
    phase: str = PREFILL
    # GPU mirror (not part of the reference record)
    slot: int = field(default=-1, repr=False, compare=False)
    prefix_len: int = field(default=0, repr=False, compare=False)  # P of the row's prefix segment
    n_prompt: int = field(default=0, repr=False, compare=False)    # prompt tokens on the GPU
    have: int = field(default=0, repr=False, compare=False)        # greedy tokens materialised
    priv_blocks: int = field(default=0, repr=False, compare=False)
    visit: int = field(default=0, repr=False, compare=False)

    @property
    def remaining_tokens(self) -> float:
        return self.target_output_tokens - self.tokens_emitted


@dataclass
class ResidentPrefix:
    """Mirror of stagesim.engines.ResidentPrefix (engines.py:95-98) + its block row."""

    tokens: int
    last_used: float
    row: int = field(default=-1, repr=False, compare=False)
    n_blocks: int = field(default=0, repr=False, compare=False)


class TokenSource:
    """Synthetic token ids shared by every engine of a run (visit counts are global)."""

    def __init__(self, seed: int, vocab: int) -> None:
        self.seed = seed
        self.vocab = vocab
        self.visits: dict[tuple[int, str], int] = {}

    def prompt(self, rid: int, sid: str, n: int) -> tuple[int, np.ndarray]:
        visit = self.visits.get((rid, sid), 0)
        self.visits[(rid, sid)] = visit + 1
        return visit, prompt_tokens(self.seed, rid, sid, visit, n, self.vocab)

    def prefix(self, sid: str, n: int) -> np.ndarray:
        return prefix_tokens(self.seed, sid, n, self.vocab)


@dataclass
class EngineSlice:
    """The part of a GpuWorker an engine owns: block ids and table rows."""

    worker: GpuWorker
    block_base: int
    n_blocks: int
    slot_rows: list[int]
    prefix_rows: list[int]
    tokens: TokenSource
    bitmap: torch.Tensor = None  # int32 words, bit = 1 -> free

    def __post_init__(self) -> None:
        if self.bitmap is None:
            nwords = (self.n_blocks + 31) // 32
            words = np.zeros(nwords, dtype=np.uint64)
            full, rem = divmod(self.n_blocks, 32)
            words[:full] = 0xFFFFFFFF
            if rem:
                words[full] = (1 << rem) - 1
            self.bitmap = torch.from_numpy(words.astype(np.uint32).view(np.int32)).to(
                self.worker.device)


class EngineObserver:
    """Hooks for parity checking (no-ops by default)."""

    def on_alloc(self, engine, requests):  # requests: [(row, col, count)]
        pass

    def on_free(self, engine, requests):
        pass

    def on_complete(self, engine, call):
        pass


class GpuEngineState:
    """One engine: resident prefixes, an active batch, KV accounting — on a B200."""

    def __init__(self, engine_id: int, params, home_pool: str, gpu: EngineSlice | None = None,
                 observer: EngineObserver | None = None) -> None:
        # --- reference state (engines.py:104-114) ---
        self.engine_id = engine_id
        self.params = params
        self.home_pool = home_pool
        self.lent_to: str | None = None
        self.resident: dict[str, ResidentPrefix] = {}
        self.batch: list[InFlightCall] = []
        self.kv_used = 0.0
        self.kv_reserved = 0
        self.decode_epoch = 0
        self.last_advance = 0.0
        # --- GPU mirror ---
        if gpu is None:
            raise InternalInvariantViolation("GpuEngineState needs an EngineSlice (no CPU fallback)")
        self.gpu = gpu
        self.worker = gpu.worker
        self.obs = observer or EngineObserver()
        self._free_slots = list(gpu.slot_rows)
        self._free_prefix_rows = list(gpu.prefix_rows)
        if len(self._free_slots) < params.max_batch:
            raise InternalInvariantViolation("engine slice has fewer slot rows than max_batch")
        self.decode_steps = 0
        self.decode_tokens = 0
        self.prefill_tokens = 0
        self.blocks_in_use = 0
        self.peak_blocks = 0
        self.closed = False  # set by close() (retired: the device slice was returned)

    # ------------------------------------------------------------------ views

    @property
    def serving_pool(self) -> str:
        return self.lent_to if self.lent_to is not None else self.home_pool

    def resident_prefix_tokens(self) -> int:
        return sum(p.tokens for p in self.resident.values())

    def decode_batch_size(self) -> int:
        return sum(1 for c in self.batch if c.phase == DECODE)

    def free_kv(self) -> int:
        return self.params.kv_capacity_tokens - self.kv_reserved

    def kv_demand(self, call, prefix_tokens: int) -> int:
        demand = call.prompt_tokens + call.target_output_tokens
        if call.stage_id not in self.resident:
            demand += prefix_tokens
        return demand

    def can_admit(self, call, prefix_tokens: int) -> bool:
        if len(self.batch) >= self.params.max_batch:
            return False
        return self.kv_reserved + self.kv_demand(call, prefix_tokens) <= self.params.kv_capacity_tokens

    def active_stage_calls(self, stage_id: str) -> int:
        return sum(1 for c in self.batch if c.stage_id == stage_id)

    def evictable_prefixes(self, keep_stage: str) -> list[tuple[float, str, int]]:
        out = [
            (p.last_used, sid, p.tokens)
            for sid, p in self.resident.items()
            if sid != keep_stage and self.active_stage_calls(sid) == 0
        ]
        out.sort()
        return out

    def recomputed_kv_used(self) -> float:
        return self.resident_prefix_tokens() + sum(
            c.prompt_tokens + c.tokens_emitted for c in self.batch
        )

    def recomputed_kv_reserved(self) -> int:
        return self.resident_prefix_tokens() + sum(
            c.prompt_tokens + c.target_output_tokens for c in self.batch
        )

    # ------------------------------------------------------------------ transitions

    def admit(self, call, prefix_tokens: int, now: float):
        """Admit a call; returns (in-flight record, prefill-done time) — engines.py:142-166."""
        if not self.can_admit(call, prefix_tokens):
            raise AdmitWithoutCapacity(
                f"engine {self.engine_id} cannot admit request {call.request_id} stage {call.stage_id}"
            )
        cold_tokens = 0
        cold = call.stage_id not in self.resident
        if not cold:
            self.resident[call.stage_id].last_used = now
        else:
            cold_tokens = prefix_tokens
            self.resident[call.stage_id] = ResidentPrefix(prefix_tokens, now)
            self.kv_used += prefix_tokens
            self.kv_reserved += prefix_tokens
        inflight = InFlightCall(
            request_id=call.request_id,
            stage_id=call.stage_id,
            prompt_tokens=call.prompt_tokens,
            target_output_tokens=call.target_output_tokens,
        )
        self.batch.append(inflight)
        self.kv_used += call.prompt_tokens
        self.kv_reserved += call.prompt_tokens + call.target_output_tokens
        prefill_done = now + (call.prompt_tokens + cold_tokens) / self.params.prefill_rate
        self._gpu_admit(inflight, self.resident[call.stage_id], cold)
        return inflight, prefill_done

    def prefill_finished(self, call: InFlightCall) -> None:
        call.phase = DECODE
        self.decode_epoch += 1

    def advance_decode(self, to_time: float) -> None:
        """engines.py:172-194, then decode on the GPU up to floor(tokens_emitted)."""
        dt = to_time - self.last_advance
        if dt < 0:
            raise ValueError("advance_decode must not move backwards")
        self.last_advance = to_time
        if dt == 0.0:
            return
        b = self.decode_batch_size()
        if b == 0:
            return
        per_call = dt / self.params.token_time(b)
        for call in self.batch:
            if call.phase != DECODE:
                continue
            emitted = min(per_call, call.remaining_tokens)
            call.tokens_emitted += emitted
            self.kv_used += emitted
        self._gpu_catch_up({id(c): min(c.target_output_tokens, max(1, math.floor(c.tokens_emitted)))
                            for c in self.batch if c.phase == DECODE})

    def next_completion(self, now: float):
        decoding = [c for c in self.batch if c.phase == DECODE]
        if not decoding:
            return None
        call = min(decoding, key=lambda c: (c.remaining_tokens, c.request_id))
        t = now + call.remaining_tokens * self.params.token_time(len(decoding))
        return call, t

    def complete_call(self, call: InFlightCall) -> None:
        """engines.py:206-214; the GPU finishes the call's tokens and frees its blocks."""
        snap = call.target_output_tokens - call.tokens_emitted
        call.tokens_emitted = float(call.target_output_tokens)
        self.kv_used += snap
        self.kv_used -= call.prompt_tokens + call.target_output_tokens
        self.kv_reserved -= call.prompt_tokens + call.target_output_tokens
        self._gpu_catch_up({id(call): max(1, call.target_output_tokens)})
        self.obs.on_complete(self, call)
        self.batch.remove(call)
        self.decode_epoch += 1
        self._gpu_release(call)

    def evict_idle_prefix(self, stage_id: str) -> None:
        if self.active_stage_calls(stage_id):
            raise PrefixInUse(f"stage '{stage_id}' has active calls on engine {self.engine_id}")
        prefix = self.resident.pop(stage_id, None)
        if prefix is not None:
            self.kv_used -= prefix.tokens
            self.kv_reserved -= prefix.tokens
            if prefix.n_blocks:
                self._free([(prefix.row, 0, prefix.n_blocks)])
            if prefix.row >= 0:
                self._free_prefix_rows.append(prefix.row)

    def close(self) -> None:
        """Retire hook: return every device block of this engine to its pool.

        The reference retires an idle engine on autoscale scale-in by moving it to
        `Simulator.retired_engines` (simulation.py:800-809) and has no hook for it;
        the retired object's host accounting stays readable (the final report walks
        retired engines, simulation.py:863), so only the device half is released:
        the resident prefixes' blocks (and any in-flight call's private blocks)
        go back to the bitmap, after which the slice can host a new engine.
        Any later transition on this engine raises InternalInvariantViolation.
        """
        if self.closed:
            return
        for call in self.batch:
            if call.priv_blocks:
                self._free([(call.slot, _blocks(call.prefix_len), call.priv_blocks)])
                call.priv_blocks = 0
        for p in self.resident.values():
            if p.n_blocks:
                self._free([(p.row, 0, p.n_blocks)])
                p.n_blocks = 0
        if self.blocks_in_use:
            raise InternalInvariantViolation(
                f"engine {self.engine_id}: {self.blocks_in_use} blocks unaccounted at close")
        self.closed = True

    # ------------------------------------------------------------------ GPU mirror

    def _alloc(self, reqs: list[tuple[int, int, int]]) -> None:
        """reqs: (table row, first column, blocks) served in order, lowest free block first."""
        reqs = [r for r in reqs if r[2] > 0]
        if not reqs:
            return
        self.worker.alloc_blocks(self.gpu, reqs)
        self.blocks_in_use += sum(r[2] for r in reqs)
        self.peak_blocks = max(self.peak_blocks, self.blocks_in_use)
        self.obs.on_alloc(self, reqs)

    def _free(self, reqs: list[tuple[int, int, int]]) -> None:
        reqs = [r for r in reqs if r[2] > 0]
        if not reqs:
            return
        self.worker.free_blocks(self.gpu, reqs)
        self.blocks_in_use -= sum(r[2] for r in reqs)
        self.obs.on_free(self, reqs)

    def _prefill(self, seqs: list[PrefillSeq]) -> None:
        """Run prefill sequences, chunked to the worker's token budget."""
        w = self.worker
        for s in seqs:
            n = len(s.tokens)
            start = 0
            while start < n:
                m = min(n - start, w.max_tokens)
                last = start + m == n
                kv_len = s.kv_len - n + start + m
                w.forward_prefill_chunk(PrefillSeq(s.row, s.prefix_len, kv_len,
                                                   s.tokens[start:start + m],
                                                   s.out_row if last else -1, s.hist_pos))
                start += m
            self.prefill_tokens += n

    def _check_open(self) -> None:
        if self.closed:
            raise InternalInvariantViolation(f"engine {self.engine_id} was retired (closed)")

    def _gpu_admit(self, call: InFlightCall, prefix: ResidentPrefix, cold: bool) -> None:
        self._check_open()
        w = self.worker
        P = prefix.tokens
        npb = _blocks(P)
        if cold and P > 0:
            if not self._free_prefix_rows:
                raise InternalInvariantViolation(f"engine {self.engine_id}: no free prefix row")
            prefix.row = self._free_prefix_rows.pop(0)
            prefix.n_blocks = npb
        if not self._free_slots:
            raise InternalInvariantViolation(f"engine {self.engine_id}: no free slot")
        call.slot = self._free_slots.pop(0)
        call.prefix_len = P
        call.visit, toks = self.gpu.tokens.prompt(call.request_id, call.stage_id, call.prompt_tokens)
        if call.prompt_tokens == 0 and P == 0:
            toks = np.zeros(1, np.int32)  # no context at all: a single BOS token (id 0)
        call.n_prompt = len(toks)
        call.priv_blocks = _blocks(call.n_prompt)
        reqs = []
        if cold and npb:
            reqs.append((prefix.row, 0, npb))
        reqs.append((call.slot, npb, call.priv_blocks))
        self._alloc(reqs)
        if cold and npb:
            self._prefill([PrefillSeq(prefix.row, 0, P, self.gpu.tokens.prefix(call.stage_id, P),
                                      out_row=prefix.row, hist_pos=0)])
        if npb:
            w.copy_prefix_row(prefix.row, call.slot, npb)
        if call.n_prompt:
            self._prefill([PrefillSeq(call.slot, P, P + call.n_prompt, toks, out_row=call.slot,
                                      hist_pos=0)])
        else:  # warm/cold prefix, empty prompt: first token is the prefix's greedy token
            w.copy_first_token(prefix.row, call.slot)
        call.have = 1

    def _gpu_catch_up(self, targets: dict[int, int]) -> None:
        """Batched greedy decode steps until each call has its target token count."""
        if self.closed and any(c.have < targets.get(id(c), 0) for c in self.batch):
            self._check_open()
        while True:
            step = [c for c in self.batch if id(c) in targets and c.have < targets[id(c)]]
            if not step:
                return
            allocs = []
            toks = []
            for c in step:
                j = c.n_prompt + c.have - 1  # private index of the token fed this step
                if j % BLOCK_TOKENS == 0:
                    allocs.append((c.slot, _blocks(c.prefix_len) + j // BLOCK_TOKENS, 1))
                    c.priv_blocks += 1
                kv_len = c.prefix_len + j + 1
                pre = self.resident.get(c.stage_id)
                toks.append(DecodeTok(c.slot, c.prefix_len, kv_len, hist_pos=c.have,
                                      prefix_key=pre.row if pre is not None else -1))
            self._alloc(allocs)
            self.worker.forward_decode(toks)
            for c in step:
                c.have += 1
            self.decode_steps += 1
            self.decode_tokens += len(step)

    def _gpu_release(self, call: InFlightCall) -> None:
        self._free([(call.slot, _blocks(call.prefix_len), call.priv_blocks)])
        call.priv_blocks = 0
        self._free_slots.append(call.slot)
        self._free_slots.sort()

    # ------------------------------------------------------------------ inspection

    def slot_row_ids(self, call: InFlightCall) -> np.ndarray:
        """Block ids of a call's row: prefix blocks then private blocks."""
        return self.read_row(call.slot, _blocks(call.prefix_len) + call.priv_blocks)

    def read_status(self) -> int:
        return int(self.worker.status[0])

    def read_row(self, row: int, n: int) -> np.ndarray:
        return self.worker.table[row, :n].cpu().numpy()

    def read_tokens(self, call: InFlightCall, n: int | None = None) -> np.ndarray:
        n = call.have if n is None else n
        return self.worker.hist[call.slot, :n].cpu().numpy()


def make_slices(worker: GpuWorker, n_engines: int, blocks_per_engine: int, max_batch: int,
                tokens: TokenSource, n_prefix_rows: int = 4) -> list[EngineSlice]:
    """Partition a worker's KV arena: engine e owns block ids
    [e*blocks_per_engine, (e+1)*blocks_per_engine) and its own table rows."""
    rows_per = max_batch + n_prefix_rows
    if n_engines * blocks_per_engine > worker.n_blocks or n_engines * rows_per > worker.table.shape[0]:
        raise InternalInvariantViolation("worker arena too small for the requested engines")
    out = []
    for e in range(n_engines):
        r0 = e * rows_per
        out.append(EngineSlice(worker, e * blocks_per_engine, blocks_per_engine,
                               list(range(r0, r0 + max_batch)),
                               list(range(r0 + max_batch, r0 + rows_per)), tokens))
    return out


def blocks_for(params, n_prefix_rows: int = 4) -> int:
    """Block-pool size that can never run out after a successful token admission:
    ceil(capacity/16) + per-call rounding (max_batch) + per-prefix rounding + BOS slack."""
    return _blocks(params.kv_capacity_tokens) + 2 * params.max_batch + n_prefix_rows
