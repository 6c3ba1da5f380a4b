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
from .cluster import (
    CMD_ADMIT,
    CMD_EVICT,
    EVT_DONE,
    STAGE_CODE,
    STAGE_OF,
    EngineSpec,
    ReplicaLink,
    plan_engines,
    pool_stages,
)
from .engine import ResidentPrefix
from .errors import InternalInvariantViolation, PrefixInUse
from .model import DecodeTok, GpuWorker, PrefillSeq, StepPlan
from .workflow import EXECUTOR, Nl2Sql, Workflow


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
    handoffs: int = 0  # calls admitted on an engine of another replica
    latencies: list = field(default_factory=list)


class _Done:
    """Completion marker for host-only workers (CPU tests)."""

    @staticmethod
    def query() -> bool:
        return True


class ReplicaExecutor:
    """The engines one replica (one GPU, or the leader of a TP pair) hosts, and its step.

    `admit` / `evict` apply the scheduler's decisions to a local engine (whose own
    accounting is the reference's, engine.py); `step_gpu` runs ONE fused forward for
    every engine on the GPU: each decoding call advances one token and pending prompt /
    stage-prefix prefill is packed in up to a token budget (chunked prefill). A call
    whose tokens are complete is released on the spot (its KV blocks return to the
    pool) and its generated tokens (the SQL) are copied to pinned host memory; the call
    is reported done once that copy has landed (`poll_done`)."""

    def __init__(self, worker, params: EngineParams, specs: list[EngineSpec], *, seed: int = 0,
                 prefill_budget: int | None = None, n_prefix_rows: int = 4,
                 result_rows: int = 512, stats: RunStats | None = None) -> None:
        self.worker = worker
        self.params = params
        self.prefill_budget = prefill_budget or max(256, worker.max_tokens - params.max_batch * 2)
        self.tokens = TokenSource(seed, worker.cfg.vocab)
        n_eng = len(specs)
        bpe = worker.n_blocks // max(n_eng, 1)
        slices = make_slices(worker, n_eng, bpe, params.max_batch, self.tokens, n_prefix_rows)
        self.engines: list[WallClockEngine] = []
        self.by_id: dict[int, WallClockEngine] = {}
        for sp, sl in zip(specs, slices):
            e = WallClockEngine(sp.engine_id, params, sp.pool, sl)
            self.engines.append(e)
            self.by_id[sp.engine_id] = e
        self.stats = stats if stats is not None else RunStats()
        self._cuda = torch.device(worker.device).type == "cuda"
        self.result_host = torch.zeros(max(64, result_rows), worker.hist.shape[1],
                                       dtype=torch.int32, pin_memory=self._cuda)
        self._res_i = 0
        self.waiting_d2h: deque = deque()  # (event, engine, call, result row, n tokens)
        self.on_result = None  # optional hook(call, tokens) when a call's SQL reaches the host
        self._status_host = torch.zeros(2, dtype=torch.int32, pin_memory=self._cuda)
        self._status_evt = None

    # ---- scheduler decisions
    def admit(self, eid: int, call: PendingCall, P: int, visit: int, now: float) -> None:
        # the workflow's visit index of this stage keys the prompt's token stream
        # (tokens.py), wherever the call's earlier visits ran
        self.tokens.visits[(call.request_id, call.stage_id)] = visit
        self.by_id[eid].admit(call, P, now)

    def evict(self, eid: int, sid: str) -> None:
        self.by_id[eid].evict_idle_prefix(sid)

    # ---- the step
    def poll_done(self) -> list[tuple[WallClockEngine, InFlightCall]]:
        """Calls whose SQL reached the host since the last poll (in completion order)."""
        out = []
        while self.waiting_d2h and self.waiting_d2h[0][0].query():
            _, e, call, idx, n = self.waiting_d2h.popleft()
            if self.on_result is not None:
                self.on_result(call, self.result_host[idx, :n].numpy().copy())
            out.append((e, call))
        return out

    def idle(self) -> bool:
        return not any(e.batch or e.pending for e in self.engines)

    def step_gpu(self) -> bool:
        """One fused forward; False when there was nothing to run."""
        w = self.worker
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
            return False
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
        self._poll_status()
        return True

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
        self.waiting_d2h.append((ev, e, c, i, n))

    # ---- device status
    def check_status(self) -> None:
        """Raise InternalInvariantViolation when a kernel reported an error.

        The device status word (allocator out-of-blocks / double free, a TP exchange
        that timed out) is written by the kernels and never read on the hot path; a
        non-zero value means the block tables or the residual stream can no longer be
        trusted. Synchronous read: call it outside timed regions (the runtime's
        run_steps/run_until do at their end); `step_gpu` polls it asynchronously every
        STATUS_EVERY steps."""
        w = self.worker
        for name, t in (("worker", getattr(w, "status", None)),
                        ("tp", getattr(getattr(w, "tp", None), "status", None))):
            if isinstance(t, torch.Tensor) and int(t.reshape(-1)[0]) != 0:
                raise InternalInvariantViolation(
                    f"device status of the {name} is {int(t.reshape(-1)[0])} (kernel error)")

    STATUS_EVERY = 64

    def _poll_status(self) -> None:
        """Asynchronous status check: copy the status words to pinned memory every
        STATUS_EVERY steps and inspect the previous copy once its event completed."""
        if not self._cuda:
            return
        if self._status_evt is not None and self._status_evt.query():
            if int(self._status_host[0]) or int(self._status_host[1]):
                self.check_status()
                raise InternalInvariantViolation(
                    f"device status {self._status_host.tolist()} (kernel error)")
            self._status_evt = None
        if self._status_evt is None and self.stats.steps % self.STATUS_EVERY == 0:
            self._status_host[0:1].copy_(self.worker.status.reshape(-1)[:1], non_blocking=True)
            tp = getattr(self.worker, "tp", None)
            if tp is not None and getattr(tp, "status", None) is not None:
                self._status_host[1:2].copy_(tp.status.reshape(-1)[:1], non_blocking=True)
            self._status_evt = torch.cuda.Event()
            self._status_evt.record()


class RemoteEngine:
    """The scheduler's view of an engine hosted by another replica.

    Keeps the reference's admission accounting (engines.py:129-140, 142-166, 206-226)
    for the decisions the scheduler takes itself: `kv_reserved`, the resident prefixes
    and the batch change only through the commands it sends (admit / evict) and the
    done events it receives, so they never under-count the engine's own state (a call
    is released on the engine before its done event arrives): an admission the
    scheduler grants always succeeds on the engine. `kv_used` (routing's tie-break,
    scheduling.py:134-140) adds the generated tokens the replica republishes every step."""

    def __init__(self, spec: EngineSpec, params: EngineParams, link: ReplicaLink, row: int) -> None:
        self.engine_id = spec.engine_id
        self.params = params
        self.home_pool = spec.pool
        self.link = link
        self.row = row
        self.resident: dict[str, ResidentPrefix] = {}
        self.batch: list[PendingCall] = []
        self.kv_reserved = 0
        self._kv_base = 0.0

    @property
    def kv_used(self) -> float:
        return self._kv_base + float(self.link.stat_f[self.row, 0])

    @property
    def blocks_in_use(self) -> int:
        return int(self.link.stat[self.row, 1])

    def resident_prefix_tokens(self) -> int:
        return sum(p.tokens for p in self.resident.values())

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
        out = [(p.last_used, sid, p.tokens) for sid, p in self.resident.items()
               if sid != keep_stage and self.active_stage_calls(sid) == 0]
        out.sort()
        return out

    def submit_admit(self, call: PendingCall, P: int, visit: int, now: float) -> None:
        if not self.can_admit(call, P):
            raise InternalInvariantViolation(f"engine {self.engine_id}: admit without capacity")
        if call.stage_id in self.resident:
            self.resident[call.stage_id].last_used = now
        else:
            self.resident[call.stage_id] = ResidentPrefix(P, now)
            self._kv_base += P
            self.kv_reserved += P
        self.batch.append(call)
        self._kv_base += call.prompt_tokens
        self.kv_reserved += call.prompt_tokens + call.target_output_tokens
        self.link.cmd.push(CMD_ADMIT, self.engine_id, call.request_id, STAGE_CODE[call.stage_id],
                           visit, call.prompt_tokens, call.target_output_tokens, P)

    def submit_evict(self, sid: str) -> None:
        if self.active_stage_calls(sid):
            raise PrefixInUse(f"stage '{sid}' has active calls on engine {self.engine_id}")
        prefix = self.resident.pop(sid, None)
        if prefix is not None:
            self._kv_base -= prefix.tokens
            self.kv_reserved -= prefix.tokens
            self.link.cmd.push(CMD_EVICT, self.engine_id, STAGE_CODE[sid])

    def on_done(self, rid: int, sid: str) -> None:
        for i, c in enumerate(self.batch):
            if c.request_id == rid and c.stage_id == sid:
                del self.batch[i]
                self._kv_base -= c.prompt_tokens
                self.kv_reserved -= c.prompt_tokens + c.target_output_tokens
                return
        raise InternalInvariantViolation(f"engine {self.engine_id}: done for unknown call {rid}")


class PoolRuntime:
    """Closed-loop NL2SQL serving over stage pools (the scheduler, on replica 0).

    Holds the workflow state machine, the executor (SQL) visits as host timers, one
    FCFS queue per pool, and routes every call over ALL engines of its pool with the
    reference rule (warm prefix first, then least kv_used, then lowest engine id, with
    LRU eviction of idle prefixes as the fallback, scheduling.py:129-165). Engines are
    local (`ReplicaExecutor` of this process, driven by `step`) or remote (`RemoteEngine`
    over a `ReplicaLink` to the replica that hosts them, driven by its `ReplicaServer`).

    Single process (the 1-GPU baseline): every engine local, `mode` isolated (one
    generator + one fixer pool) or shared (one pool serving both stages)."""

    def __init__(self, worker: GpuWorker, spec: Nl2Sql, params: EngineParams, *,
                 mode: str = "isolated", engines_per_pool: tuple[int, int] = (1, 1),
                 concurrency: int = 256, n_workflows: int | None = None, seed: int = 0,
                 rid_offset: int = 0, rid_stride: int = 1, prefill_budget: int | None = None,
                 n_prefix_rows: int = 4, engines: list[EngineSpec] | None = None,
                 links: dict[int, ReplicaLink] | None = None,
                 remote_params: EngineParams | None = None) -> None:
        self.worker = worker
        self.spec = spec
        self.params = params
        self.seed = seed
        self.mode = mode
        self.concurrency = concurrency
        self.n_workflows = n_workflows
        self.rid_offset = rid_offset
        self.rid_stride = rid_stride
        specs = engines if engines is not None else plan_engines(mode, 1,
                                                                 engines_per_pool=engines_per_pool)
        self.stats = RunStats()
        local = [s for s in specs if s.replica == 0]
        self.executor = ReplicaExecutor(worker, params, local, seed=seed,
                                        prefill_budget=prefill_budget,
                                        n_prefix_rows=n_prefix_rows,
                                        result_rows=2 * concurrency, stats=self.stats)
        self.links = links or {}
        rows: dict[int, int] = {}
        self.handles: dict[int, object] = {}
        for s in specs:
            if s.replica == 0:
                self.handles[s.engine_id] = self.executor.by_id[s.engine_id]
            else:
                if s.replica not in self.links:
                    raise ValueError(f"engine {s.engine_id} on replica {s.replica} needs a link")
                r = rows.get(s.replica, 0)
                rows[s.replica] = r + 1
                self.handles[s.engine_id] = RemoteEngine(s, remote_params or params,
                                                         self.links[s.replica], r)
        self.stage_pool: dict[str, str] = {}
        self.pool_engines: dict[str, list] = {}
        for pool_id, stages in pool_stages(mode).items():
            self.pool_engines[pool_id] = [self.handles[s.engine_id] for s in specs
                                          if s.pool == pool_id]
            if not self.pool_engines[pool_id]:
                raise ValueError(f"pool {pool_id} has no engine")
            for sid in stages:
                self.stage_pool[sid] = pool_id
        self.engines = self.executor.engines  # the local engines
        self.queues: dict[str, deque] = {p: deque() for p in self.pool_engines}
        self.workflows: dict[int, Workflow] = {}
        self.timers: list = []  # (ready_time, seq, rid)
        self._tseq = 0
        self._next_rid_i = 0
        self.t0 = time.perf_counter()
        self.finished: list[Workflow] = []

    # ------------------------------------------------------------------ views
    @property
    def on_result(self):
        return self.executor.on_result

    @on_result.setter
    def on_result(self, fn) -> None:
        self.executor.on_result = fn

    @property
    def all_engines(self) -> list:
        return [self.handles[k] for k in sorted(self.handles)]

    def blocks_in_use(self) -> dict[int, int]:
        return {eid: h.blocks_in_use for eid, h in sorted(self.handles.items())}

    def now(self) -> float:
        return time.perf_counter() - self.t0

    # ------------------------------------------------------------------ workflows
    def _start_workflow(self) -> bool:
        if self.n_workflows is not None and self._next_rid_i >= self.n_workflows:
            return False
        rid = self.rid_offset + self._next_rid_i * self.rid_stride
        self._next_rid_i += 1
        wf = Workflow(rid, self.spec, self.seed, arrival=self.now())
        self.workflows[rid] = wf
        self._enter(wf)
        return True

    def _enter(self, wf: Workflow) -> None:
        r = wf.enter()
        if wf.stage == EXECUTOR:
            self._tseq += 1
            heapq.heappush(self.timers, (self.now() + r, self._tseq, wf.rid))
        else:
            if wf.stage not in self.stage_pool:
                raise InternalInvariantViolation(f"no pool serves stage {wf.stage}")
            p, o = r
            call = PendingCall(wf.rid, wf.stage, self.now(), p, o)
            self.queues[self.stage_pool[wf.stage]].append((call, wf.visits[wf.stage] - 1))

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
            self._start_workflow()
        else:
            self._enter(wf)

    # ------------------------------------------------------------------ dispatch
    @staticmethod
    def _route(call: PendingCall, P: int, engines):
        """scheduling.py:129-165: warm-first, least kv_used, lowest id; LRU eviction."""
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
                call, visit = q[0]
                P = self.spec.prefix(call.stage_id)
                e, evictions = self._route(call, P, engines)
                if e is None:
                    break
                now = self.now()
                if isinstance(e, RemoteEngine):
                    for sid in evictions:
                        e.submit_evict(sid)
                    e.submit_admit(call, P, visit, now)
                    self.stats.handoffs += 1
                else:
                    for sid in evictions:
                        self.executor.evict(e.engine_id, sid)
                    self.executor.admit(e.engine_id, call, P, visit, now)
                q.popleft()
                self.stats.calls += 1

    # ------------------------------------------------------------------ step
    def _poll_links(self) -> None:
        for link in self.links.values():
            for rec in link.evt.pop_all():
                if rec[0] != EVT_DONE:
                    raise InternalInvariantViolation(f"unknown replica event {rec}")
                _, eid, rid, code = rec[:4]
                self.handles[eid].on_done(rid, STAGE_OF[code])
                self._after_stage(self.workflows[rid])

    def step(self) -> None:
        """One scheduling round + one fused forward of this replica's engines."""
        self._poll_links()
        now = self.now()
        while self.timers and self.timers[0][0] <= now:  # executor visits finishing
            _, _, rid = heapq.heappop(self.timers)
            self._after_stage(self.workflows[rid])
        for _e, call in self.executor.poll_done():  # SQL text reached the host
            self._after_stage(self.workflows[call.request_id])
        self._dispatch()
        if not self.executor.step_gpu():
            if self.timers or self.executor.waiting_d2h or self.links:
                time.sleep(0.0002)

    # ------------------------------------------------------------------ driving
    def fill(self) -> None:
        while len(self.workflows) < self.concurrency and self._start_workflow():
            pass

    def check_status(self) -> None:
        self.executor.check_status()

    def run_steps(self, k: int) -> None:
        for _ in range(k):
            self.step()
        self.check_status()

    def run_until(self, n_completed: int, max_seconds: float = 600.0) -> None:
        t_end = time.perf_counter() + max_seconds
        while self.stats.completed + self.stats.failed < n_completed:
            if not self.workflows:
                break
            self.step()
            if time.perf_counter() > t_end:
                raise InternalInvariantViolation("runtime did not finish in time")
        self.check_status()


class ReplicaServer:
    """Replica r != 0: applies the scheduler's commands to its engines, runs its GPU
    steps, reports calls done and republishes its engines' status every step."""

    def __init__(self, executor: ReplicaExecutor, link: ReplicaLink) -> None:
        self.executor = executor
        self.link = link
        self.t0 = time.perf_counter()
        self.stats = executor.stats
        self._row = {e.engine_id: i for i, e in enumerate(executor.engines)}

    @property
    def worker(self):
        return self.executor.worker

    @property
    def engines(self):
        return self.executor.engines

    def step(self) -> None:
        ex, link = self.executor, self.link
        now = time.perf_counter() - self.t0
        for rec in link.cmd.pop_all():
            if rec[0] == CMD_ADMIT:
                _, eid, rid, code, visit, p, o, P = rec
                ex.admit(eid, PendingCall(rid, STAGE_OF[code], now, p, o), P, visit, now)
            elif rec[0] == CMD_EVICT:
                ex.evict(rec[1], STAGE_OF[rec[2]])
            else:
                raise InternalInvariantViolation(f"unknown scheduler command {rec}")
        ran = ex.step_gpu()
        for e, call in ex.poll_done():
            link.evt.push(EVT_DONE, e.engine_id, call.request_id, STAGE_CODE[call.stage_id])
        for e in ex.engines:
            i = self._row[e.engine_id]
            link.stat_f[i, 0] = sum(c.tokens_emitted for c in e.batch)
            link.stat[i, 1] = e.blocks_in_use
            link.stat[i, 2] = len(e.batch)
        if not ran:
            time.sleep(0.0002)

    def serve_while(self, phase: int) -> None:
        while self.link.phase == phase:
            self.step()

    def check_status(self) -> None:
        self.executor.check_status()
