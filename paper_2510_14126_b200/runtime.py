"""Wall-clock stage-pool runtime (throughput mode).

Replaces the reference's virtual-clock event loop (stagesim/simulation.py:816-837)
with a real continuous-batching loop over GPU engines, while keeping its
semantics where they are not about time:

  * topology: one engine pool per LLM stage ("isolated", workloads.py:167-181) or a
    single pool serving both stages ("shared", :182-195); the SQL executor stays
    on host cores as wall-clock timers;
  * per-workflow outcomes, prompt/output lengths and executor service times come
    from the reference's counter streams (workflow.py mirror), so they are
    bit-identical to the reference for any timing;
  * admission is the reference's token reservation (engines.py:137-140) and
    routing its warm-prefix / least-kv_used / lowest-id rule with LRU eviction
    (scheduling.py:129-165); dispatch within a pool is FCFS (policy "fcfs",
    simulation.py:636-637) with no overtaking (:656-670).

Each loop iteration is one fused GPU step for all engines sharing the GPU: every
decoding call advances one token, and pending prompt / stage-prefix prefill is
packed into the same forward up to a token budget (chunked prefill). Output
length is forced to the call's target (EOS ignored), so the host never waits on
generated tokens except to hand a finished call's SQL to the executor.
"""

from __future__ import annotations

import heapq
import time
from collections import deque
from dataclasses import dataclass, field

import numpy as np
import torch

from .config import BLOCK_TOKENS, ModelConfig
from .engine import (
    DECODE,
    PREFILL,
    EngineParams,
    GpuEngineState,
    InFlightCall,
    PendingCall,
    TokenSource,
    _blocks,
    make_slices,
)
from .errors import InternalInvariantViolation
from .model import DecodeTok, GpuWorker, PrefillSeq, StepPlan
from .placement import ROLE_BOTH, ROLE_FIXER, ROLE_GENERATOR
from .workflow import EXECUTOR, FIXER, GENERATOR, Nl2Sql, Workflow


@dataclass
class _PendingPrefill:
    seq: PrefillSeq          # full sequence (all tokens)
    call: InFlightCall | None
    done: int = 0


class WallClockEngine(GpuEngineState):
    """GpuEngineState whose device work is batched by the runtime instead of run eagerly."""

    def __init__(self, *a, **kw) -> None:
        super().__init__(*a, **kw)
        self.pending: deque[_PendingPrefill] = deque()
        self.cold_admits = 0  # stage-prefix prefills (an admit that found no resident prefix)

    def _gpu_admit(self, call: InFlightCall, prefix, cold: bool) -> None:
        w = self.worker
        P = prefix.tokens
        npb = _blocks(P)
        if cold and P > 0:
            if not self._free_prefix_rows:
                raise InternalInvariantViolation(f"engine {self.engine_id}: no free prefix row")
            prefix.row = self._free_prefix_rows.pop(0)
            prefix.n_blocks = npb
            self.cold_admits += 1
        call.slot = self._free_slots.pop(0)
        call.prefix_len = P
        call.visit, toks = self.gpu.tokens.prompt(call.request_id, call.stage_id, call.prompt_tokens)
        if call.prompt_tokens == 0:
            raise InternalInvariantViolation("wall-clock engine needs a non-empty prompt")
        call.n_prompt = len(toks)
        call.priv_blocks = _blocks(call.n_prompt)
        reqs = []
        if cold and npb:
            reqs.append((prefix.row, 0, npb))
        reqs.append((call.slot, npb, call.priv_blocks))
        self._alloc(reqs)
        if cold and npb:
            self.pending.append(_PendingPrefill(
                PrefillSeq(prefix.row, 0, P, self.gpu.tokens.prefix(call.stage_id, P)), None))
        if npb:
            w.copy_prefix_row(prefix.row, call.slot, npb)
        self.pending.append(_PendingPrefill(
            PrefillSeq(call.slot, P, P + call.n_prompt, toks, out_row=call.slot, hist_pos=0), call))
        call.have = 0

    # ---- step assembly (called by the runtime) ----

    def take_prefill(self, budget: int, out: list, started: list) -> int:
        """Move up to `budget` prefill tokens (FIFO, chunked) into `out`."""
        used = 0
        while self.pending and used < budget:
            item = self.pending[0]
            s = item.seq
            n = len(s.tokens)
            m = min(n - item.done, budget - used)
            last = item.done + m == n
            kv_len = s.kv_len - n + item.done + m
            out.append(PrefillSeq(s.row, s.prefix_len, kv_len, s.tokens[item.done:item.done + m],
                                  s.out_row if last else -1, s.hist_pos))
            item.done += m
            used += m
            self.prefill_tokens += m
            if last:
                self.pending.popleft()
                if item.call is not None:
                    started.append((self, item.call))
            else:
                break
        return used

    def plan_decode(self, toks: list, calls: list) -> None:
        allocs = []
        for c in self.batch:
            if c.phase != DECODE or c.have >= c.target_output_tokens:
                continue
            j = c.n_prompt + c.have - 1
            if j % BLOCK_TOKENS == 0:
                allocs.append((c.slot, _blocks(c.prefix_len) + j // BLOCK_TOKENS, 1))
                c.priv_blocks += 1
            pre = self.resident.get(c.stage_id)
            toks.append(DecodeTok(c.slot, c.prefix_len, c.prefix_len + j + 1, hist_pos=c.have,
                                  prefix_key=pre.row if pre is not None else -1))
            calls.append((self, c))
        self._alloc(allocs)

    def emit(self, call: InFlightCall) -> None:
        """One generated token became resident (reference: kv_used += emitted)."""
        call.have += 1
        call.tokens_emitted += 1.0
        self.kv_used += 1.0

    def finish(self, call: InFlightCall) -> None:
        """Release a call whose tokens are complete (engines.py:206-214)."""
        call.tokens_emitted = float(call.target_output_tokens)
        self.kv_used -= call.prompt_tokens + call.target_output_tokens
        self.kv_reserved -= call.prompt_tokens + call.target_output_tokens
        self.batch.remove(call)
        self.decode_epoch += 1
        self._gpu_release(call)


@dataclass
class RunStats:
    steps: int = 0
    completed: int = 0
    failed: int = 0
    decode_tokens: int = 0
    prefill_tokens: int = 0
    calls: int = 0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    handoffs: int = 0
    latencies: list = field(default_factory=list)


class _Done:
    """Completion marker for host-only workers (CPU tests)."""

    @staticmethod
    def query() -> bool:
        return True


class PoolRuntime:
    """Closed-loop NL2SQL serving on one GPU (all engines share its weights).

    `role` selects the stage pools this GPU serves: "both" (the 1-GPU baseline:
    generator and fixer engines side by side, partitioned HBM) or one side of a
    disjoint generator/fixer pair (placement.py), with `channel` the pair's
    shared-memory handoff rings."""

    def __init__(self, worker: GpuWorker, spec: Nl2Sql, params: EngineParams, *,
                 mode: str = "isolated", engines_per_pool: tuple[int, int] = (1, 1),
                 concurrency: int = 256, n_workflows: int | None = None, seed: int = 0,
                 rid_offset: int = 0, rid_stride: int = 1, prefill_budget: int | None = None,
                 n_prefix_rows: int = 4, role: str = ROLE_BOTH, channel=None) -> None:
        self.worker = worker
        self.role = role
        self.channel = channel
        if role != ROLE_BOTH and (mode != "isolated" or channel is None):
            raise ValueError("disjoint placement needs isolated pools and a pair channel")
        self.remote = 0  # workflows of this pair currently owned by the peer rank
        self.spec = spec
        self.params = params
        self.seed = seed
        self.concurrency = concurrency
        self.n_workflows = n_workflows
        self.rid_offset = rid_offset
        self.rid_stride = rid_stride
        self.prefill_budget = prefill_budget or max(256, worker.max_tokens - params.max_batch * 2)
        tokens = TokenSource(seed, worker.cfg.vocab)
        if role == ROLE_GENERATOR:
            pools = [(f"pool:{GENERATOR}", (GENERATOR,), engines_per_pool[0])]
        elif role == ROLE_FIXER:
            pools = [(f"pool:{FIXER}", (FIXER,), engines_per_pool[1])]
        elif mode == "isolated":
            pools = [(f"pool:{GENERATOR}", (GENERATOR,), engines_per_pool[0]),
                     (f"pool:{FIXER}", (FIXER,), engines_per_pool[1])]
        elif mode == "shared":
            pools = [("pool:llm", (GENERATOR, FIXER), sum(engines_per_pool))]
        else:
            raise ValueError(mode)
        n_eng = sum(p[2] for p in pools)
        bpe = worker.n_blocks // n_eng
        slices = make_slices(worker, n_eng, bpe, params.max_batch, tokens, n_prefix_rows)
        self.engines: list[WallClockEngine] = []
        self.pool_engines: dict[str, list[WallClockEngine]] = {}
        self.stage_pool: dict[str, str] = {}
        eid = 0
        for pool_id, stages, n in pools:
            self.pool_engines[pool_id] = []
            for sid in stages:
                self.stage_pool[sid] = pool_id
            for _ in range(n):
                e = WallClockEngine(eid, params, pool_id, slices[eid])
                self.engines.append(e)
                self.pool_engines[pool_id].append(e)
                eid += 1
        self.queues: dict[str, deque] = {p: deque() for p in self.pool_engines}
        self.workflows: dict[int, Workflow] = {}
        self.timers: list = []  # (ready_time, seq, rid)
        self.waiting_d2h: deque = deque()  # (event, rid)
        self._tseq = 0
        self._next_rid_i = 0
        self.stats = RunStats()
        self.t0 = time.perf_counter()
        self._cuda = torch.device(worker.device).type == "cuda"
        self.result_host = torch.zeros(max(64, 2 * concurrency), worker.hist.shape[1],
                                       dtype=torch.int32, pin_memory=self._cuda)
        self._res_i = 0
        self.on_result = None  # optional hook(call, tokens) when a call's SQL reaches the host
        self.finished: list[Workflow] = []

    # ------------------------------------------------------------------ workflows

    def now(self) -> float:
        return time.perf_counter() - self.t0

    def _start_workflow(self) -> bool:
        if self.role == ROLE_FIXER:
            return False  # workflows of a pair start on its generator rank
        if self.n_workflows is not None and self._next_rid_i >= self.n_workflows:
            return False
        rid = self.rid_offset + self._next_rid_i * self.rid_stride
        self._next_rid_i += 1
        wf = Workflow(rid, self.spec, self.seed, arrival=self.now())
        self.workflows[rid] = wf
        self._enter(wf)
        return True

    def _enter(self, wf: Workflow) -> None:
        if wf.stage != EXECUTOR and wf.stage not in self.stage_pool:
            if self.role != ROLE_GENERATOR or wf.stage != FIXER:
                raise InternalInvariantViolation(f"no pool serves stage {wf.stage} on this rank")
            # the fixer pool lives on the peer rank: hand the workflow across (metadata only)
            self.channel.to_fixer.push(wf.rid, self.t0 + wf.arrival)
            del self.workflows[wf.rid]
            self.remote += 1
            self.stats.handoffs += 1
            return
        r = wf.enter()
        if wf.stage == EXECUTOR:
            self._tseq += 1
            heapq.heappush(self.timers, (self.now() + r, self._tseq, wf.rid))
        else:
            p, o = r
            call = PendingCall(wf.rid, wf.stage, self.now(), p, o)
            self.queues[self.stage_pool[wf.stage]].append(call)

    def _after_stage(self, wf: Workflow) -> None:
        nxt = wf.finish()
        if nxt is None:
            wf.done_time = self.now()
            if wf.terminal == "Success":
                self.stats.completed += 1
            else:
                self.stats.failed += 1
            self.stats.latencies.append(wf.done_time - wf.arrival)
            self.finished.append(wf)
            del self.workflows[wf.rid]
            if self.role == ROLE_FIXER:
                self.channel.to_generator.push(wf.rid, self.t0 + wf.done_time)
            else:
                self._start_workflow()
        else:
            self._enter(wf)

    # ------------------------------------------------------------------ dispatch

    def _route(self, call: PendingCall, P: int, engines):
        admissible = [e for e in engines if e.can_admit(call, P)]
        if admissible:
            return min(admissible, key=lambda e: (call.stage_id not in e.resident, e.kv_used,
                                                  e.engine_id)), []
        ordered = sorted(engines, key=lambda e: (call.stage_id not in e.resident, e.kv_used,
                                                 e.engine_id))
        for e in ordered:
            if len(e.batch) >= e.params.max_batch:
                continue
            needed = e.kv_demand(call, P) - e.free_kv()
            if needed <= 0:
                return e, []
            ev, freed = [], 0
            for _, sid, tok in e.evictable_prefixes(call.stage_id):
                ev.append(sid)
                freed += tok
                if freed >= needed:
                    return e, ev
        return None, []

    def _dispatch(self) -> None:
        for pool_id, q in self.queues.items():
            engines = self.pool_engines[pool_id]
            while q:
                call = q[0]
                P = self.spec.prefix(call.stage_id)
                e, evictions = self._route(call, P, engines)
                if e is None:
                    break
                for sid in evictions:
                    e.evict_idle_prefix(sid)
                e.admit(call, P, self.now())
                q.popleft()
                self.stats.calls += 1

    # ------------------------------------------------------------------ step

    def _poll_peer(self) -> None:
        if self.role == ROLE_GENERATOR:
            for _rid, _t in self.channel.to_generator.pop_all():  # finished on the fixer rank
                self.remote -= 1
                if len(self.workflows) + self.remote < self.concurrency:
                    self._start_workflow()
        elif self.role == ROLE_FIXER:
            for rid, t in self.channel.to_fixer.pop_all():
                wf = Workflow(rid, self.spec, self.seed, arrival=t - self.t0)
                wf.replay_to(FIXER)
                self.workflows[rid] = wf
                self._enter(wf)

    def step(self) -> None:
        w = self.worker
        if self.channel is not None:
            self._poll_peer()
        now = self.now()
        while self.timers and self.timers[0][0] <= now:  # executor visits finishing
            _, _, rid = heapq.heappop(self.timers)
            self._after_stage(self.workflows[rid])
        while self.waiting_d2h and self.waiting_d2h[0][0].query():  # SQL text reached the host
            _, call, idx, n = self.waiting_d2h.popleft()
            if self.on_result is not None:
                self.on_result(call, self.result_host[idx, :n].numpy().copy())
            self._after_stage(self.workflows[call.request_id])
        self._dispatch()
        toks, dcalls = [], []
        for e in self.engines:
            e.plan_decode(toks, dcalls)
        pre, started = [], []
        budget = min(self.prefill_budget, w.max_tokens - len(toks))
        for e in self.engines:
            if budget <= 0:
                break
            budget -= e.take_prefill(budget, pre, started)
        if not toks and not pre:
            if self.timers or self.waiting_d2h:
                time.sleep(0.0005)
            return
        w.forward(StepPlan(decode=toks, prefill=pre))
        self.stats.steps += 1
        self.stats.decode_tokens += len(toks)
        self.stats.prefill_tokens += sum(len(s.tokens) for s in pre)
        done = []
        for e, c in dcalls:
            e.emit(c)
            if c.have >= c.target_output_tokens:
                done.append((e, c))
        for e, c in started:  # prompt prefill complete -> first token exists
            c.phase = DECODE
            e.decode_epoch += 1
            e.emit(c)
            if c.have >= c.target_output_tokens:
                done.append((e, c))
        for e, c in done:
            self._complete(e, c)

    def _complete(self, e: WallClockEngine, c: InFlightCall) -> None:
        """Copy the call's generated tokens (its SQL) to the host, then release it."""
        w = self.worker
        n = max(1, c.target_output_tokens)
        i = self._res_i
        self._res_i = (i + 1) % self.result_host.shape[0]
        self.result_host[i, :n].copy_(w.hist[c.slot, :n], non_blocking=True)
        if self._cuda:
            ev = torch.cuda.Event()
            ev.record()
        else:
            ev = _Done
        self.stats.d2h_bytes += 4 * n
        e.finish(c)
        self.waiting_d2h.append((ev, c, i, n))

    # ------------------------------------------------------------------ driving

    def fill(self) -> None:
        while len(self.workflows) + self.remote < self.concurrency and self._start_workflow():
            pass

    def run_steps(self, k: int) -> None:
        for _ in range(k):
            self.step()

    def run_until(self, n_completed: int, max_seconds: float = 600.0) -> None:
        t_end = time.perf_counter() + max_seconds
        while self.stats.completed + self.stats.failed < n_completed:
            if not self.workflows and not self.remote and self.role != ROLE_FIXER:
                break
            self.step()
            if time.perf_counter() > t_end:
                raise InternalInvariantViolation("runtime did not finish in time")

    def blocks_in_use(self) -> dict[int, int]:
        return {e.engine_id: e.blocks_in_use for e in self.engines}
