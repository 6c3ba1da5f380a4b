"""Replay utilities shared by the CPU and GPU parity tests.

`replay_calls` drives engines with a recorded reference call stream (the golden
engine_calls.jsonl / engine_scenarios.json, produced by the reference itself)
and asserts after every call that the engine's observable state, return values
and errors equal the reference's, bit for bit.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from paper_2510_14126_b200.engine import (
    EngineObserver,
    EngineParams,
    EngineSlice,
    GpuEngineState,
    PendingCall,
    TokenSource,
    blocks_for,
    make_slices,
)

GOLDEN = Path(__file__).resolve().parent / "golden"
CONFIG1_PARAMS = EngineParams(16384, 5000.0, 0.02, 0.1, 8)
CONFIG1_POOLS = {0: "pool:sql_generator", 1: "pool:sql_fixer"}
# tests/golden/evict: AC-2's tight shared topology (make_golden.EVICT)
EVICT_PARAMS = EngineParams(3200, 2000.0, 0.02, 0.1, 12)
EVICT_POOLS = {0: "pool:llm", 1: "pool:llm"}


def engine_state(e) -> dict:
    return {
        "kv_used": e.kv_used,
        "kv_reserved": e.kv_reserved,
        "decode_epoch": e.decode_epoch,
        "last_advance": e.last_advance,
        "resident": {sid: [p.tokens, p.last_used] for sid, p in sorted(e.resident.items())},
        "batch": [[c.request_id, c.stage_id, c.prompt_tokens, c.target_output_tokens,
                   c.tokens_emitted, c.phase] for c in e.batch],
    }


def load_jsonl(path) -> list[dict]:
    with open(path) as f:
        return [json.loads(line) for line in f]


def find_call(engine, rid):
    for c in engine.batch:
        if c.request_id == rid:
            return c
    raise AssertionError(f"request {rid} not in engine {engine.engine_id}")


def _pending(d: dict, t: float) -> PendingCall:
    return PendingCall(d["request_id"], d["stage_id"], t, d["prompt_tokens"],
                       d["target_output_tokens"])


def replay_calls(records: list[dict], engines: dict, factory=None, params=None) -> int:
    """Drive engines with a reference call stream; returns the number of state checks.

    With `factory` (integration.gpu_engine_factory), "create" records build the
    engine and "retire" records close it and recycle its slice (the elastic run).
    """
    checks = 0
    for i, rec in enumerate(records):
        op, args = rec["op"], rec["args"]
        if op == "create":
            engines[rec["eng"]] = factory(rec["eng"], params, args[0])
            engines[rec["eng"]].last_advance = args[1]  # simulation.py:365
            continue
        if op == "retire":
            factory.release(engines[rec["eng"]])
            continue
        e = engines[rec["eng"]]
        if op == "can_admit":
            got = e.can_admit(_pending(args[0], 0.0), args[1])
            assert got == rec["ret"], (i, rec)
            continue
        if op == "admit":
            _, done = e.admit(_pending(args[0], args[2]), args[1], args[2])
            assert done == rec["ret"], (i, done, rec["ret"])
        elif op == "prefill_finished":
            e.prefill_finished(find_call(e, args[0]))
        elif op == "advance_decode":
            e.advance_decode(args[0])
        elif op == "next_completion":
            r = e.next_completion(args[0])
            got = None if r is None else [r[0].request_id, r[1]]
            assert got == rec["ret"], (i, got, rec["ret"])
            continue
        elif op == "complete_call":
            e.complete_call(find_call(e, args[0]))
        elif op == "evict_idle_prefix":
            e.evict_idle_prefix(args[0])
        else:
            raise AssertionError(op)
        assert engine_state(e) == rec["state"], (i, op)
        checks += 1
    return checks


class RecordingObserver(EngineObserver):
    """Collects per-call block rows and generated tokens at completion."""

    def __init__(self, read_device: bool) -> None:
        self.read_device = read_device
        self.completed: dict[int, list[dict]] = {}
        self.allocs: dict[int, list[list[int]]] = {}

    def on_alloc(self, engine, requests):
        self.allocs.setdefault(engine.engine_id, []).append([r[2] for r in requests])

    def on_complete(self, engine, call):
        rec = {"rid": call.request_id, "sid": call.stage_id, "visit": call.visit,
               "P": call.prefix_len, "p": call.prompt_tokens, "o": call.target_output_tokens,
               "slot": call.slot, "have": call.have}
        if self.read_device:
            rec["row"] = engine.slot_row_ids(call).tolist()
            rec["tokens"] = engine.read_tokens(call, max(1, call.target_output_tokens)).tolist()
        self.completed.setdefault(engine.engine_id, []).append(rec)


class FakeWorker:
    """Host-only stand-in for GpuWorker (CPU tests of the host logic): records the
    device requests the engine issues instead of running them."""

    def __init__(self, n_blocks: int, n_rows: int) -> None:
        self.device = "cpu"
        self.n_blocks = n_blocks
        self.max_tokens = 1 << 30
        self.table = np.zeros((n_rows, 1), np.int32)
        self.log: list[tuple] = []

    def alloc_blocks(self, pool, reqs):
        self.log.append(("alloc", pool.block_base, [tuple(r) for r in reqs]))

    def free_blocks(self, pool, reqs):
        self.log.append(("free", pool.block_base, [tuple(r) for r in reqs]))

    def forward_prefill_chunk(self, seq):
        self.log.append(("prefill", seq.row, seq.prefix_len, seq.kv_len, len(seq.tokens)))

    def forward_decode(self, toks):
        self.log.append(("decode", [(t.row, t.kv_len, t.hist_pos) for t in toks]))

    def copy_prefix_row(self, src, dst, n):
        self.log.append(("copy", src, dst, n))

    def copy_first_token(self, src, dst):
        self.log.append(("first", src, dst))


class HostWorker(FakeWorker):
    """FakeWorker that PoolRuntime can drive: a step is recorded, not computed."""

    def __init__(self, n_blocks: int, n_rows: int, vocab: int = 1024, hist_cols: int = 160,
                 max_tokens: int = 4096) -> None:
        import types

        import torch

        super().__init__(n_blocks, n_rows)
        self.cfg = types.SimpleNamespace(vocab=vocab)
        self.max_tokens = max_tokens
        self.hist = torch.zeros(n_rows, hist_cols, dtype=torch.int32)
        self.steps = 0

    def forward(self, plan) -> int:
        self.steps += 1
        return len(plan.decode) + sum(len(s.tokens) for s in plan.prefill)


def golden_engines(worker, params, pools: dict, observer=None, seed: int = 0,
                   vocab: int = 1024):
    """Engines 0..n-1 on consecutive slices of `worker` (block ids [e*bpe, (e+1)*bpe))."""
    bpe = blocks_for(params)
    tokens = TokenSource(seed, vocab)
    slices = make_slices(worker, len(pools), bpe, params.max_batch, tokens)
    engines = {i: GpuEngineState(i, params, pools[i], slices[i], observer) for i in pools}
    return engines, bpe


def config1_engines(worker, observer=None, seed: int = 0, vocab: int = 1024):
    return golden_engines(worker, CONFIG1_PARAMS, CONFIG1_POOLS, observer, seed, vocab)
