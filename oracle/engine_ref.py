"""CPU oracle of the engine's block-level behaviour (test infrastructure only).

ORACLE — imported only by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline leg, as the checker. Never part of the product path.

Replays the reference engine's call stream (the golden
tests/golden/config1/engine_calls.jsonl, recorded from the reference
`Simulator` driving the reference `EngineState`, stagesim/engines.py:142-226)
through the block contract of DESIGN.md §3 and returns, for every completed
call, the block ids its row must hold (prefix blocks, then private blocks):

  admit(call, P)      -> alloc [ceil(P/16) if the stage was not resident and P>0,
                                ceil(p'/16)]  (p' = p, or 1 BOS token if p = P = 0)
  advance_decode(t)   -> catch-up: target(c) = min(o, max(1, floor(tokens_emitted)))
                         for decode-phase calls; step s feeds each call still short
                         of its target (batch order); a call whose fed token has
                         private index j = p' + have - 1 with j % 16 == 0 gets one
                         block, requests in batch order, one allocation per step
  complete_call(c)    -> catch-up to max(1, o), then free the private blocks
  evict_idle_prefix   -> free the stage's prefix blocks
  retire (scale-in)   -> free every resident prefix (the engine is idle); a
                         later engine on the recycled slice starts from an
                         all-free pool (simulation.py:800-809)
"""

from __future__ import annotations

import json
import math
from pathlib import Path

from .alloc_ref import BlockPoolRef

BLOCK = 16


def nblocks(n: int) -> int:
    return (n + BLOCK - 1) // BLOCK


class EngineBlocksRef:
    def __init__(self, n_blocks: int, id_base: int) -> None:
        self.pool = BlockPoolRef(n_blocks, id_base)
        self.prefix: dict[str, list[int]] = {}
        self.calls: dict[int, dict] = {}
        self.completed: list[dict] = []
        self.alloc_log: list[list[int]] = []

    def admit(self, rid: int, sid: str, P: int, p: int, o: int) -> None:
        cold = sid not in self.prefix
        n_prompt = p if (p > 0 or P > 0) else 1
        counts = []
        if cold and P > 0:
            counts.append(nblocks(P))
        counts.append(nblocks(n_prompt))
        ids = self.pool.alloc(counts)
        self.alloc_log.append(counts)
        if cold:
            self.prefix[sid] = ids[0] if P > 0 else []
        self.calls[rid] = {"rid": rid, "sid": sid, "P": P, "n_prompt": n_prompt, "o": o,
                           "have": 1, "priv": list(ids[-1]), "prefix_ids": list(self.prefix[sid])}

    def catch_up(self, order: list[int], targets: dict[int, int]) -> None:
        while True:
            step = [rid for rid in order if rid in targets and self.calls[rid]["have"] < targets[rid]]
            if not step:
                return
            need = []
            for rid in step:
                c = self.calls[rid]
                j = c["n_prompt"] + c["have"] - 1
                if j % BLOCK == 0:
                    need.append(rid)
            if need:
                got = self.pool.alloc([1] * len(need))
                self.alloc_log.append([1] * len(need))
                for rid, ids in zip(need, got):
                    self.calls[rid]["priv"].extend(ids)
            for rid in step:
                self.calls[rid]["have"] += 1

    def complete(self, rid: int, order: list[int]) -> dict:
        c = self.calls[rid]
        self.catch_up(order, {rid: max(1, c["o"])})
        done = dict(c)
        done["row"] = c["prefix_ids"] + c["priv"]
        self.completed.append(done)
        self.pool.free(c["priv"])
        del self.calls[rid]
        return done

    def retire(self) -> None:
        assert not self.calls, "only idle engines retire (simulation.py:802-806)"
        for sid in sorted(self.prefix):
            self.evict(sid)

    def evict(self, sid: str) -> None:
        ids = self.prefix.pop(sid, None)
        if ids:
            self.pool.free(ids)


def replay_blocks(records, engine_blocks: dict[int, tuple[int, int]]) -> dict[int, EngineBlocksRef]:
    """Run the block contract over an engine-call stream.

    records: iterable of dicts as written by tests/golden/make_golden.py.
    engine_blocks: engine id -> (n_blocks, id_base).
    """
    engines: dict[int, EngineBlocksRef] = {}
    for rec in records:
        eid = rec["eng"]
        if rec["op"] == "create":
            continue
        if eid not in engines:
            engines[eid] = EngineBlocksRef(*engine_blocks[eid])
        e = engines[eid]
        op = rec["op"]
        if op == "admit":
            call, P, _now = rec["args"]
            e.admit(call["request_id"], call["stage_id"], P, call["prompt_tokens"],
                    call["target_output_tokens"])
        elif op == "advance_decode":
            batch = rec["state"]["batch"]
            order = [b[0] for b in batch]
            targets = {b[0]: min(b[3], max(1, math.floor(b[4]))) for b in batch if b[5] == "decode"}
            e.catch_up(order, targets)
        elif op == "complete_call":
            rid = rec["args"][0]
            # order = batch before removal: the state after the op lacks rid, so rebuild
            order = [b[0] for b in rec["state"]["batch"]] + [rid]
            e.complete(rid, order)
        elif op == "evict_idle_prefix":
            e.evict(rec["args"][0])
        elif op == "retire":
            e.retire()
    return engines


def load_records(path: str | Path) -> list[dict]:
    with open(path) as f:
        return [json.loads(line) for line in f]
