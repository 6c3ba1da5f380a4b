"""CPU tests of elastic pools: borrowing and autoscale.

The golden run (tests/golden/elastic, made by the reference itself) has the
reference's borrowing (stagesim/simulation.py:715-763) and autoscale
(:765-809) on: a fixer engine is lent to the generator pool and serves 19
generator calls (the generator prefix is planted on it cold), engines are
created on scale-out and retired on scale-in (one of them holding a borrowed
prefix). Here the device half is a recording FakeWorker (test double); the
GPU version of these checks is tests/test_parity_gpu.py::test_elastic_*.
"""

from __future__ import annotations

import filecmp
import json
import sys
from pathlib import Path

import numpy as np
import pytest

from harness import CONFIG1_PARAMS, GOLDEN, FakeWorker, RecordingObserver, load_jsonl, replay_calls
from oracle.engine_ref import replay_blocks
from paper_2510_14126_b200.engine import blocks_for
from paper_2510_14126_b200.integration import gpu_engine_factory, gpu_simulator

ELASTIC = GOLDEN / "elastic"


class FakeArena(FakeWorker):
    """FakeWorker with the arena shape gpu_engine_factory carves."""

    def __init__(self, n_engines: int, params=CONFIG1_PARAMS) -> None:
        import types

        bpe = blocks_for(params)
        super().__init__(n_engines * bpe, n_engines * (params.max_batch + 4))
        self.table = np.zeros((self.table.shape[0], bpe), np.int32)
        self.cfg = types.SimpleNamespace(vocab=1024)


def _stagesim() -> bool:
    root = Path(__file__).resolve().parents[1]
    for cand in (root / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (cand / "stagesim").exists() and str(cand) not in sys.path:
            sys.path.insert(0, str(cand))
    try:
        import stagesim  # noqa: F401

        return True
    except ImportError:
        return False


def test_elastic_golden_exercises_borrow_and_autoscale():
    audit = json.loads((ELASTIC / "audit.json").read_text())
    assert len(audit["borrows"]) == 3 and len(audit["returns"]) == 3
    llm = [e for e in audit["scale_events"] if "executor" not in e[1]]
    assert sum(e[2] > 0 for e in llm) == 2 and sum(e[2] < 0 for e in llm) == 4
    records = load_jsonl(ELASTIC / "engine_calls.jsonl")
    home = {r["eng"]: r["args"][0] for r in records if r["op"] == "create"}
    borrowed = [r for r in records if r["op"] == "admit"
                and "pool:" + r["args"][0]["stage_id"] != home[r["eng"]]]
    assert len(borrowed) == 19  # generator calls served by a lent fixer engine


def test_elastic_call_stream_matches_reference():
    """Engines created / retired as the reference did; state bit-exact after every call,
    device requests equal the block oracle's, slices recycled with empty pools."""
    records = load_jsonl(ELASTIC / "engine_calls.jsonl")
    worker = FakeArena(6)
    obs = RecordingObserver(read_device=False)
    factory = gpu_engine_factory(worker, CONFIG1_PARAMS, seed=0, observer=obs)
    engines: dict = {}
    checks = replay_calls(records, engines, factory=factory, params=CONFIG1_PARAMS)
    assert checks > 2000
    assert sorted(engines) == [0, 1, 2, 3, 4, 5]
    # scale-out after a retirement reused the retired engine's slice
    bases = {eid: factory.assigned[eid][0] for eid in engines}
    assert bases[4] == bases[3] and bases[5] == bases[1]
    ref = replay_blocks(records, {eid: (factory.assigned[eid][1], 0) for eid in engines})
    for eid, e in engines.items():
        assert obs.allocs.get(eid, []) == ref[eid].alloc_log, eid
        assert [c["rid"] for c in obs.completed.get(eid, [])] == \
            [c["rid"] for c in ref[eid].completed]
        assert e.blocks_in_use == sum(len(v) for v in ref[eid].prefix.values())
        if e.closed:
            assert e.blocks_in_use == 0 and ref[eid].pool.n_free() == ref[eid].pool.nblocks
    retired = {r["eng"] for r in records if r["op"] == "retire"}
    assert {eid for eid, e in engines.items() if e.closed} == retired


def test_reference_simulator_elastic_host(tmp_path):
    """The reference Simulator with borrowing + autoscale drives GpuEngineState
    (device half recorded): its four outputs and audit equal the golden byte for byte."""
    if not _stagesim():
        pytest.skip("reference package not importable")
    sys.path.insert(0, str(GOLDEN))
    from make_golden import ELASTIC as CFG
    from make_golden import CappedSimulator, elastic_config
    from stagesim.reporting import write_run_outputs

    worker = FakeArena(6)
    factory = gpu_engine_factory(worker, CONFIG1_PARAMS, seed=0)
    sim_cls = gpu_simulator(type("Cap", (CappedSimulator,), {"cap": CFG["cap"]}), factory)
    sim = sim_cls(elastic_config())
    result = sim.run()
    write_run_outputs(result, tmp_path)
    for name in ("dispatch.csv", "requests.csv", "kv_usage.csv", "summary.json"):
        assert filecmp.cmp(tmp_path / name, ELASTIC / name, shallow=False), name
    a = sim.audit
    audit = json.loads((ELASTIC / "audit.json").read_text())
    assert [list(x) for x in a.borrows] == audit["borrows"]
    assert [list(x) for x in a.scale_events] == audit["scale_events"]
    assert all(e.closed for e in sim.retired_engines.values())
    # kv_blocks.csv: the reference's kv_usage rows + a block count per sample
    sim.write_kv_blocks(tmp_path / "kv_blocks.csv")
    rows = (tmp_path / "kv_blocks.csv").read_text().splitlines()
    ref_rows = (ELASTIC / "kv_usage.csv").read_text().splitlines()
    assert len(rows) == len(ref_rows)
    for r, q in zip(rows[1:], ref_rows[1:]):
        head, nb = r.rsplit(",", 1)
        assert head == q
        kv_used = float(q.split(",")[3])
        # the blocks cover the materialised tokens (floor of each call's emitted count)
        assert int(nb) * 16 >= kv_used - CONFIG1_PARAMS.max_batch


def test_reference_simulator_evict_host(tmp_path):
    """AC-2's tight shared topology (tests/golden/evict): the reference Simulator's own
    routing evicts idle prefixes on GpuEngineState engines (device half recorded); its
    outputs equal the golden byte for byte and every eviction frees the prefix blocks."""
    if not _stagesim():
        pytest.skip("reference package not importable")
    sys.path.insert(0, str(GOLDEN))
    from make_golden import EVICT, CappedSimulator, evict_config
    from stagesim.reporting import write_run_outputs

    from harness import EVICT_PARAMS

    worker = FakeArena(2, EVICT_PARAMS)
    factory = gpu_engine_factory(worker, EVICT_PARAMS, seed=0)
    sim = gpu_simulator(type("Cap", (CappedSimulator,), {"cap": EVICT["cap"]}), factory)(
        evict_config())
    result = sim.run()
    write_run_outputs(result, tmp_path)
    for name in ("dispatch.csv", "requests.csv", "kv_usage.csv", "summary.json"):
        assert filecmp.cmp(tmp_path / name, GOLDEN / "evict" / name, shallow=False), name
    prefix_frees = [e for e in worker.log if e[0] == "free" and e[2][0][1] == 0]
    assert len(prefix_frees) == 12
