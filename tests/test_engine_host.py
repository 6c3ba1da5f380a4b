"""CPU tests of the engine boundary's host half against the reference's goldens.

The GPU work is replaced by a recording FakeWorker (a test double, not a
fallback: the product constructor refuses to run without a device slice). These
tests pin that `GpuEngineState` is a drop-in for the reference `EngineState`:
same return values, same errors, same state after every call of the reference's
own call stream, bit for bit — and that the device requests it issues follow the
block contract restated by oracle/engine_ref.py.
"""

from __future__ import annotations

import json

import pytest

from harness import (
    CONFIG1_PARAMS,
    EVICT_PARAMS,
    EVICT_POOLS,
    GOLDEN,
    FakeWorker,
    RecordingObserver,
    config1_engines,
    engine_state,
    find_call,
    golden_engines,
    load_jsonl,
    replay_calls,
)
from oracle.engine_ref import replay_blocks
from paper_2510_14126_b200.engine import (
    EngineParams,
    GpuEngineState,
    PendingCall,
    TokenSource,
    blocks_for,
    make_slices,
)
from paper_2510_14126_b200.errors import AdmitWithoutCapacity, PrefixInUse


def _scenario_engine(params: dict):
    p = EngineParams(**params)
    worker = FakeWorker(blocks_for(p) * 2, 64)
    sl = make_slices(worker, 1, blocks_for(p), p.max_batch, TokenSource(0, 1024))[0]
    return GpuEngineState(0, p, "pool:x", sl), worker


SCENARIOS = json.loads((GOLDEN / "engine_scenarios.json").read_text())


@pytest.mark.parametrize("name", sorted(SCENARIOS))
def test_engine_scenarios_match_reference(name):
    sc = SCENARIOS[name]
    eng, _ = _scenario_engine(sc["params"])
    for step in sc["steps"]:
        op = step["op"]
        kind = op[0]
        ret = None
        if kind in ("kv_demand", "can_admit"):
            c = PendingCall(op[1][0], op[1][1], 0.0, op[1][2], op[1][3])
            ret = getattr(eng, kind)(c, op[2])
        elif kind == "admit":
            c = PendingCall(op[1][0], op[1][1], op[3], op[1][2], op[1][3])
            _, ret = eng.admit(c, op[2], op[3])
        elif kind == "admit_expect_error":
            c = PendingCall(op[1][0], op[1][1], op[3], op[1][2], op[1][3])
            try:
                eng.admit(c, op[2], op[3])
                ret = "no-error"
            except AdmitWithoutCapacity:
                ret = "AdmitWithoutCapacity"
        elif kind == "prefill_finished":
            eng.prefill_finished(find_call(eng, op[1]))
        elif kind == "complete_call":
            eng.complete_call(find_call(eng, op[1]))
        elif kind == "advance_decode":
            eng.advance_decode(op[1])
        elif kind == "advance_expect_error":
            try:
                eng.advance_decode(op[1])
                ret = "no-error"
            except ValueError:
                ret = "ValueError"
        elif kind == "next_completion":
            r = eng.next_completion(op[1])
            ret = None if r is None else [r[0].request_id, r[1]]
        elif kind == "evictable_prefixes":
            ret = [list(x) for x in eng.evictable_prefixes(op[1])]
        elif kind == "evict_idle_prefix":
            eng.evict_idle_prefix(op[1])
        elif kind == "evict_expect_error":
            try:
                eng.evict_idle_prefix(op[1])
                ret = "no-error"
            except PrefixInUse:
                ret = "PrefixInUse"
        assert ret == step["ret"], (name, op)
        assert engine_state(eng) == step["state"], (name, op)
        assert eng.free_kv() == step["free_kv"]
        assert eng.decode_batch_size() == step["decode_batch_size"]
        assert eng.resident_prefix_tokens() == step["resident_prefix_tokens"]
        assert eng.recomputed_kv_used() == step["recomputed_kv_used"]
        assert eng.recomputed_kv_reserved() == step["recomputed_kv_reserved"]


def test_config1_call_stream_matches_reference():
    """The reference Simulator's 2071 engine calls (config 1, seed 0), replayed."""
    records = load_jsonl(GOLDEN / "config1" / "engine_calls.jsonl")
    worker = FakeWorker(10 * blocks_for(CONFIG1_PARAMS), 64)
    obs = RecordingObserver(read_device=False)
    engines, bpe = config1_engines(worker, obs)
    checks = replay_calls(records, engines)
    assert checks > 1000
    # the allocation request stream equals the oracle's block contract
    ref = replay_blocks(records, {0: (bpe, 0), 1: (bpe, bpe)})
    for eid in (0, 1):
        assert obs.allocs[eid] == ref[eid].alloc_log, eid
        assert [c["rid"] for c in obs.completed[eid]] == [c["rid"] for c in ref[eid].completed]
    # every call's materialised tokens reached its target
    for eid in (0, 1):
        for c in obs.completed[eid]:
            assert c["have"] == max(1, c["o"])


def test_evict_call_stream_matches_reference():
    """AC-2's tight shared topology (tests/golden/evict): the reference routes with
    eviction (scheduling.py:143-165), so its stream holds evict_idle_prefix calls
    (engines.py:219-226); replayed bit for bit, the prefix frees follow the contract."""
    records = load_jsonl(GOLDEN / "evict" / "engine_calls.jsonl")
    n_ev = sum(1 for r in records if r["op"] == "evict_idle_prefix")
    assert n_ev >= 10
    worker = FakeWorker(4 * blocks_for(EVICT_PARAMS), 64)
    obs = RecordingObserver(read_device=False)
    engines, bpe = golden_engines(worker, EVICT_PARAMS, EVICT_POOLS, obs)
    checks = replay_calls(records, engines)
    assert checks > 2000
    ref = replay_blocks(records, {0: (bpe, 0), 1: (bpe, bpe)})
    for eid in (0, 1):
        assert obs.allocs[eid] == ref[eid].alloc_log, eid
        assert [c["rid"] for c in obs.completed[eid]] == [c["rid"] for c in ref[eid].completed]
    # every eviction freed exactly the evicted stage's prefix blocks (row, col 0, ceil(P/16))
    prefix_frees = [e for e in worker.log if e[0] == "free" and e[2][0][1] == 0]
    assert len(prefix_frees) == n_ev
    assert all(e[2][0][2] == 63 for e in prefix_frees)  # P = 1000 -> 63 blocks


def test_no_cpu_fallback():
    from paper_2510_14126_b200.errors import InternalInvariantViolation

    with pytest.raises(InternalInvariantViolation):
        GpuEngineState(0, CONFIG1_PARAMS, "pool:x", None)


def test_decode_requests_respect_block_boundaries():
    """One block per 16 private tokens, allocated when the fed token starts a block."""
    p = EngineParams(4096, 1000.0, 0.01, 0.0, 4)
    eng, worker = _scenario_engine(p.__dict__)
    call = PendingCall(0, "gen", 0.0, 20, 40)
    fl, _ = eng.admit(call, 40, 0.0)  # prefix 40 -> 3 blocks; prompt 20 -> 2 blocks
    eng.prefill_finished(fl)
    eng.advance_decode(1.0)  # 100 tokens' worth -> capped at target 40
    allocs = [e for e in worker.log if e[0] == "alloc"]
    assert allocs[0][2] == [(4, 0, 3), (0, 3, 2)]
    # fed tokens have private index 20..58 (have 1..39); blocks start at 32 and 48
    assert [a[2] for a in allocs[1:]] == [[(0, 5, 1)], [(0, 6, 1)]]
    decodes = [e for e in worker.log if e[0] == "decode"]
    assert len(decodes) == 39
    assert decodes[0][1] == [(0, 61, 1)]
    eng.complete_call(fl)
    frees = [e for e in worker.log if e[0] == "free"]
    assert frees[-1][2] == [(0, 3, 4)]
