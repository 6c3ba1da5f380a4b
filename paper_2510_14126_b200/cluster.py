"""Stage pools across GPUs: engine placement and the scheduler <-> replica links.

The reference lays out one engine pool per LLM stage ("isolated",
stagesim/workloads.py:167-181) or one pool serving both LLM stages ("shared",
:182-195), each pool holding `engines_per_stage` / `total_engines` independent
engines, and routes every call over ALL engines of its pool
(stagesim/scheduling.py:129-165, called from simulation.py:655-714). Here an engine
is placed on a *replica*: one process driving one GPU (or the leader of a TP = 2
GPU pair). With N replicas:

  * N = 1: both engines of the 1-GPU baseline share the GPU (isolated: one
    generator + one fixer engine; shared: two engines of one pool);
  * N >= 2, isolated: the generator pool holds one engine on each of replicas
    [0, g) and the fixer pool one engine on each of [g, N) (disjoint device sets,
    any split g : N - g, e.g. config 5's generator 2 / fixer 6 GPUs);
  * N >= 2, shared: one pool of N engines, one per replica (config 3's baseline).

Replica 0 also runs the scheduler (workflow state machine, executor timers, pool
queues, the reference routing rule over every engine of a pool). It reaches the
engines of other replicas through a `ReplicaLink`: a shared-memory segment per
replica (all replicas live on one node) with a command ring (admit / evict,
scheduler -> replica), an event ring (call done, replica -> scheduler) and a
per-engine status row the replica republishes every step (tokens emitted by its
in-flight calls, KV blocks in use). Stage handoff is host metadata only: no KV or
activations move between GPUs, so there is no data-path
collective.

The rings are single-producer / single-consumer int64 arrays in a memory-mapped
/dev/shm file: the producer writes a record, then publishes it by bumping the
tail, which x86's store ordering makes visible in that order.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

from .workflow import FIXER, GENERATOR

POOL_GENERATOR = f"pool:{GENERATOR}"
POOL_FIXER = f"pool:{FIXER}"
POOL_SHARED = "pool:llm"
STAGE_CODE = {GENERATOR: 0, FIXER: 1}
STAGE_OF = {v: k for k, v in STAGE_CODE.items()}

_SHM_DIR = "/dev/shm" if os.path.isdir("/dev/shm") else "/tmp"


@dataclass(frozen=True)
class EngineSpec:
    """One engine of a pool: its id (pool order = routing tie-break order, as the
    reference numbers engines in pool order, simulation.py:390-395) and its replica."""

    engine_id: int
    pool: str
    replica: int


def pool_stages(mode: str) -> dict[str, tuple[str, ...]]:
    if mode == "isolated":
        return {POOL_GENERATOR: (GENERATOR,), POOL_FIXER: (FIXER,)}
    if mode == "shared":
        return {POOL_SHARED: (GENERATOR, FIXER)}
    raise ValueError(f"unknown topology mode {mode!r}")


def parse_split(text: str | None, n: int) -> tuple[int, int] | None:
    """'g:f' -> (g, f) with g + f == n (None: the even split)."""
    if not text:
        return None
    g, f = (int(x) for x in text.split(":"))
    if g < 1 or f < 1 or g + f != n:
        raise ValueError(f"split {text!r} must be g:f with g, f >= 1 and g + f = {n}")
    return g, f


def plan_engines(mode: str, n_replicas: int, split: tuple[int, int] | None = None,
                 engines_per_pool: tuple[int, int] = (1, 1)) -> list[EngineSpec]:
    """Engine placement (module docstring). `engines_per_pool` applies at N = 1 only
    (engines sharing the one GPU); `split` = (generator replicas, fixer replicas)."""
    if n_replicas < 1:
        raise ValueError("need at least one replica")
    if n_replicas == 1:
        if mode == "isolated":
            g, f = engines_per_pool
            return ([EngineSpec(i, POOL_GENERATOR, 0) for i in range(g)]
                    + [EngineSpec(g + i, POOL_FIXER, 0) for i in range(f)])
        pool_stages(mode)
        n = sum(engines_per_pool)
        return [EngineSpec(i, POOL_SHARED, 0) for i in range(n)]
    if mode == "isolated":
        g, f = split if split is not None else (max(1, n_replicas // 2),
                                                n_replicas - max(1, n_replicas // 2))
        if g + f != n_replicas or g < 1 or f < 1:
            raise ValueError("isolated placement needs a g:f split with g, f >= 1")
        return ([EngineSpec(r, POOL_GENERATOR, r) for r in range(g)]
                + [EngineSpec(r, POOL_FIXER, r) for r in range(g, n_replicas)])
    pool_stages(mode)
    if split is not None:
        raise ValueError("a generator:fixer split needs isolated pools")
    return [EngineSpec(r, POOL_SHARED, r) for r in range(n_replicas)]


# ----------------------------------------------------------------------------- links

REC = 8          # int64 words per record
_HDR = 16        # ring header words (head and tail on separate cache lines)
_CTRL = 16       # control words
_STAT = 4        # status words per engine: emitted (f64 bits), blocks, n_batch, seq

CMD_ADMIT, CMD_EVICT = 1, 2
EVT_DONE = 1


class Ring:
    """SPSC ring of REC-word int64 records."""

    def __init__(self, words: np.ndarray, base: int, cap: int) -> None:
        self.w = words
        self.head_i = base
        self.tail_i = base + 8
        self.rec0 = base + _HDR
        self.cap = cap

    @staticmethod
    def words(cap: int) -> int:
        return _HDR + REC * cap

    def push(self, *vals: int) -> None:
        tail = int(self.w[self.tail_i])
        if tail - int(self.w[self.head_i]) >= self.cap:
            raise RuntimeError("replica link ring full (closed-loop bound violated)")
        j = self.rec0 + REC * (tail % self.cap)
        self.w[j:j + len(vals)] = vals
        self.w[self.tail_i] = tail + 1  # publish after the record

    def pop_all(self) -> list[tuple[int, ...]]:
        head = int(self.w[self.head_i])
        tail = int(self.w[self.tail_i])
        out = []
        for i in range(head, tail):
            j = self.rec0 + REC * (i % self.cap)
            out.append(tuple(int(x) for x in self.w[j:j + REC]))
        if tail != head:
            self.w[self.head_i] = tail
        return out


class ReplicaLink:
    """Shared segment between the scheduler (replica 0) and replica r.

    cmd: scheduler -> replica   (CMD_ADMIT eid rid stage visit p o P | CMD_EVICT eid stage)
    evt: replica -> scheduler   (EVT_DONE eid rid stage)
    stat[e]: per engine of the replica, republished every step
    ctrl[0]: phase word (written by the scheduler)"""

    def __init__(self, name: str, create: bool, cap: int, n_engines: int) -> None:
        self.n_engines = n_engines
        nwords = _CTRL + 2 * Ring.words(cap) + _STAT * n_engines
        self.path = os.path.join(_SHM_DIR, name)
        self.owner = create
        if create:  # (a stale file of a crashed run with the same name is overwritten)
            with open(self.path, "wb") as f:
                f.truncate(8 * nwords)
        self.words = np.memmap(self.path, dtype=np.int64, mode="r+", shape=(nwords,))
        self.cmd = Ring(self.words, _CTRL, cap)
        self.evt = Ring(self.words, _CTRL + Ring.words(cap), cap)
        s0 = _CTRL + 2 * Ring.words(cap)
        self.stat = self.words[s0:s0 + _STAT * n_engines].reshape(n_engines, _STAT)
        self.stat_f = self.stat.view(np.float64)

    @property
    def phase(self) -> int:
        return int(self.words[0])

    @phase.setter
    def phase(self, v: int) -> None:
        self.words[0] = v

    def close(self) -> None:
        self.cmd = self.evt = None
        self.stat = self.stat_f = None
        self.words = None
        if self.owner:
            try:
                os.unlink(self.path)
            except FileNotFoundError:
                pass


def link_name(tag: str, replica: int) -> str:
    return f"cortex_{tag}_r{replica}"


def open_links(dist, replica: int, n_replicas: int, engines: list[EngineSpec], cap: int,
               member: bool = True):
    """Collective over the default process group. Replica 0 creates one link per other
    replica; a barrier orders creation before attachment. Returns {replica: link} on
    replica 0, the replica's own link elsewhere (None for non-members: TP followers)."""
    obj = [f"{os.getpid()}_{os.environ.get('MASTER_PORT', '0')}"]
    dist.broadcast_object_list(obj, src=0)
    tag = obj[0]
    per = {r: sum(1 for e in engines if e.replica == r) for r in range(n_replicas)}
    out = None
    if replica == 0 and member:
        out = {r: ReplicaLink(link_name(tag, r), True, cap, per[r]) for r in range(1, n_replicas)}
    dist.barrier()
    if replica != 0 and member:
        out = ReplicaLink(link_name(tag, replica), False, cap, per[replica])
    dist.barrier()
    return out
