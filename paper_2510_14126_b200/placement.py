"""Disjoint device placement of the two stage pools across ranks.

The reference's isolated topology gives each LLM stage its own engine pool
(stagesim/workloads.py:167-181); its multi-GPU configurations put the
generator pool and the fixer pool on disjoint GPU sets (configs 3-4: 4 + 4).
Here, with N = 2k ranks (one process per GPU), ranks [0, k) each run a
generator engine and ranks [k, 2k) a fixer engine. Generator rank p and fixer
rank p + k form a PAIR that shares one closed loop of workflows:

  * the generator rank starts workflows, runs the generator call and the first
    executor visit (host timer); when that visit's outcome routes to the fixer
    (stagesim/simulation.py:521-534 enters the next stage), the request id and
    arrival time cross to the fixer rank through a shared-memory ring;
  * the fixer rank rebuilds the workflow from its id - every draw is a counter
    stream keyed by (rid, stage, visit), so the state at that point is a pure
    function of the rid - runs fixer/executor visits until the workflow ends,
    and sends a completion notice back so the generator rank can start the
    next workflow (closed loop, concurrency per pair).

No KV or activations move between GPUs: a stage handoff is host metadata only
(engines.py:206-214 releases the generated KV at completion),
so there is no data-path collective. The rings are single-producer /
single-consumer int64 arrays in a memory-mapped /dev/shm file (both ranks of a pair live
on one node); the producer writes a record, then publishes it by bumping the
tail, which x86's store ordering makes visible in that order.
"""

from __future__ import annotations

import os
import struct
import numpy as np

ROLE_BOTH = "both"
ROLE_GENERATOR = "generator"
ROLE_FIXER = "fixer"

_HDR = 16  # int64 words per ring header (head and tail on separate cache lines)
_CTRL = 8  # int64 words of control (phase word)
_SHM_DIR = "/dev/shm" if os.path.isdir("/dev/shm") else "/tmp"


def role_of(rank: int, world: int) -> tuple[str, int, int]:
    """(role, pair index, peer rank) for `rank` under disjoint placement.

    world == 1 (or odd) -> both pools on each rank (replicas)."""
    if world < 2 or world % 2:
        return ROLE_BOTH, rank, -1
    k = world // 2
    if rank < k:
        return ROLE_GENERATOR, rank, rank + k
    return ROLE_FIXER, rank - k, rank - k


def _f2i(x: float) -> int:
    return struct.unpack("<q", struct.pack("<d", x))[0]


def _i2f(x: int) -> float:
    return struct.unpack("<d", struct.pack("<q", int(x)))[0]


class Ring:
    """SPSC ring of (rid, time) records over an int64 view."""

    def __init__(self, words: np.ndarray, hdr: int, rec: int, cap: int) -> None:
        self.w = words
        self.head_i = hdr       # consumer index
        self.tail_i = hdr + 8   # producer index
        self.rec = rec
        self.cap = cap

    def push(self, rid: int, t: float) -> None:
        tail = int(self.w[self.tail_i])
        if tail - int(self.w[self.head_i]) >= self.cap:
            raise RuntimeError("placement ring full (closed loop bound violated)")
        j = self.rec + 2 * (tail % self.cap)
        self.w[j] = rid
        self.w[j + 1] = _f2i(t)
        self.w[self.tail_i] = tail + 1  # publish after the record

    def pop_all(self) -> list[tuple[int, float]]:
        head = int(self.w[self.head_i])
        tail = int(self.w[self.tail_i])
        out = []
        for i in range(head, tail):
            j = self.rec + 2 * (i % self.cap)
            out.append((int(self.w[j]), _i2f(self.w[j + 1])))
        if tail != head:
            self.w[self.head_i] = tail
        return out


class PairChannel:
    """The shared segment of one generator/fixer pair: two rings + a phase word.

    `to_fixer` carries handoffs (rid, arrival), `to_generator` completion notices
    (rid, finish time); `phase` lets the generator rank drive its fixer through
    the warmup / timed / done phases of a benchmark."""

    def __init__(self, name: str, create: bool, cap: int) -> None:
        words = _CTRL + 2 * (_HDR + 2 * cap)
        self.path = os.path.join(_SHM_DIR, name)
        self.owner = create
        if create:  # (a stale file of a crashed run with the same name is overwritten)
            with open(self.path, "wb") as f:
                f.truncate(8 * words)
        self.words = np.memmap(self.path, dtype=np.int64, mode="r+", shape=(words,))
        base = _CTRL
        self.to_fixer = Ring(self.words, base, base + _HDR, cap)
        base += _HDR + 2 * cap
        self.to_generator = Ring(self.words, base, base + _HDR, cap)

    @property
    def phase(self) -> int:
        return int(self.words[0])

    @phase.setter
    def phase(self, v: int) -> None:
        self.words[0] = v

    def close(self) -> None:
        del self.to_fixer, self.to_generator
        self.words = None
        if self.owner:
            try:
                os.unlink(self.path)
            except FileNotFoundError:
                pass


def channel_name(tag: str, pair: int) -> str:
    return f"cortex_{tag}_{pair}"


def open_pair_channel(dist, rank: int, world: int, cap: int, tag: str | None = None,
                      member: bool = True):
    """Create (generator side) / attach (fixer side) this rank's pair channel.

    rank / world index the engine replicas (= processes unless replicas are TP
    groups). Collective over the default process group: the generator ranks create
    their segments, a barrier orders creation before attachment. member=False (a TP
    follower rank) joins the collectives without opening a channel."""
    role, pair, _ = role_of(rank, world)
    if role == ROLE_BOTH:
        return None
    if tag is None:
        obj = [f"{os.getpid()}_{os.environ.get('MASTER_PORT', '0')}"]
        dist.broadcast_object_list(obj, src=0)
        tag = obj[0]
    ch = PairChannel(channel_name(tag, pair), create=True, cap=cap) \
        if role == ROLE_GENERATOR and member else None
    dist.barrier()
    if ch is None and member:
        ch = PairChannel(channel_name(tag, pair), create=False, cap=cap)
    dist.barrier()
    return ch
