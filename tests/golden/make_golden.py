"""Generate the golden fixtures of tests/golden/ by running the REFERENCE itself.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The outputs are committed; nothing on the GPU box reads /root/reference.

Fixtures
  config1/{dispatch,requests,kv_usage}.csv + summary.json
      stagesim's own byte-stable outputs (stagesim/reporting.py:38-98) for
      BASELINE config 1: NL2SQL preset, retry budget 5, isolated 1+1 engines,
      default engine params (stagesim/workloads.py:33-39), Poisson rate 1.0,
      seed 0, arrivals capped at 64 workflows, slack policy.
  config1/engine_calls.jsonl
      every engine-facing call the reference Simulator made in that run
      (admit / prefill_finished / advance_decode / next_completion /
      complete_call / evict_idle_prefix / can_admit) with arguments, return
      value and the engine's observable state afterwards.
  engine_scenarios.json
      scripted EngineState call sequences (the situations of
      pkg/tests/test_engines.py: demand, reservation, prefill time, decode
      progress, completion, eviction, LRU order, errors) with the reference's
      results after every call.
  elastic/{dispatch,requests,kv_usage}.csv + summary.json + engine_calls.jsonl
      + audit.json
      the same NL2SQL trace with the reference's elastic policies on: borrowing
      (simulation.py:715-763) and autoscale (:765-809) over isolated 1+3
      engines, Poisson rate 2.0, 96 workflows (ELASTIC below). The call stream
      adds "create" (autoscale scale-out / start-up) and "retire" (scale-in)
      records; audit.json holds the reference's borrow / return / scale events.
  evict/{dispatch,requests,kv_usage}.csv + summary.json + engine_calls.jsonl
      AC-2's tight shared topology (EVICT below): two shared engines of 3200
      tokens each, so routing evicts idle stage prefixes (route_call_with_eviction,
      scheduling.py:143-165 -> evict_idle_prefix, engines.py:219-226).
  trace_seed0_{n}_pf{p}.json
      per-workflow stage/retry outcomes (prompt/output tokens per LLM visit,
      terminal, retries) for n workflows, computed by the reference Simulator.
"""

from __future__ import annotations

import json
import shutil
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF_SRC = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF_SRC))

import stagesim as ss  # noqa: E402
from stagesim import simulation as sim_mod  # noqa: E402
from stagesim.engines import DECODE, EngineParams, EngineState, PendingCall  # noqa: E402
from stagesim.reporting import write_run_outputs  # noqa: E402
from stagesim.workloads import (  # noqa: E402
    FIXER,
    GENERATOR,
    Nl2SqlParams,
    TopologyPreset,
    build_nl2sql,
    build_topology,
)


def engine_state(e: EngineState) -> dict:
    return {
        "kv_used": e.kv_used,
        "kv_reserved": e.kv_reserved,
        "decode_epoch": e.decode_epoch,
        "last_advance": e.last_advance,
        "resident": {sid: [p.tokens, p.last_used] for sid, p in sorted(e.resident.items())},
        "batch": [[c.request_id, c.stage_id, c.prompt_tokens, c.target_output_tokens,
                   c.tokens_emitted, c.phase] for c in e.batch],
    }


def call_dict(c) -> dict:
    return {"request_id": c.request_id, "stage_id": c.stage_id,
            "prompt_tokens": c.prompt_tokens, "target_output_tokens": c.target_output_tokens}


class RecordingEngine(EngineState):
    """Reference EngineState that logs its engine-facing calls (harness only)."""

    log: list = []

    def _rec(self, op, args, ret):
        RecordingEngine.log.append({"eng": self.engine_id, "op": op, "args": args, "ret": ret,
                                    "state": engine_state(self)})

    def can_admit(self, call, prefix_tokens):
        r = super().can_admit(call, prefix_tokens)
        RecordingEngine.log.append({"eng": self.engine_id, "op": "can_admit",
                                    "args": [call_dict(call), prefix_tokens], "ret": r})
        return r

    def admit(self, call, prefix_tokens, now):
        inflight, done = super().admit(call, prefix_tokens, now)
        self._rec("admit", [call_dict(call), prefix_tokens, now], done)
        return inflight, done

    def prefill_finished(self, call):
        super().prefill_finished(call)
        self._rec("prefill_finished", [call.request_id], None)

    def advance_decode(self, to_time):
        super().advance_decode(to_time)
        self._rec("advance_decode", [to_time], None)

    def next_completion(self, now):
        r = super().next_completion(now)
        RecordingEngine.log.append({"eng": self.engine_id, "op": "next_completion", "args": [now],
                                    "ret": None if r is None else [r[0].request_id, r[1]]})
        return r

    def complete_call(self, call):
        super().complete_call(call)
        self._rec("complete_call", [call.request_id], None)

    def evict_idle_prefix(self, stage_id):
        super().evict_idle_prefix(stage_id)
        self._rec("evict_idle_prefix", [stage_id], None)


class CappedSimulator(ss.Simulator):
    """Reference Simulator with the arrival stream cut after `cap` workflows
    (the reference is Poisson-until-duration only, simulation.py:503-506)."""

    cap = 64
    engine_cls = EngineState

    def _schedule(self, time, kind, **refs):
        if kind == sim_mod.EVENT_ARRIVAL and self._next_rid >= self.cap:
            return
        super()._schedule(time, kind, **refs)

    def _add_engine(self, pool_id, params):
        engine = self.engine_cls(self._next_engine_id, params, pool_id)
        engine.last_advance = self.clock
        self.engines[engine.engine_id] = engine
        self._kv_integral[engine.engine_id] = 0.0
        self._next_engine_id += 1
        return engine


def config1(seed: int = 0, p_fail: float = 0.5, budget: int = 5, duration: float = 100000.0,
            engines=(1, 1), params: EngineParams | None = None, mode: str = "isolated"):
    params = params or EngineParams(16384, 5000.0, 0.02, 0.1, 8)
    vw = ss.validate_workflow(build_nl2sql(Nl2SqlParams(
        p_fail=p_fail, p_syntax_err=p_fail / 2, p_empty_result=p_fail / 2, retry_budget=budget)))
    if mode == "isolated":
        preset = TopologyPreset(mode="isolated",
                                engines_per_stage={GENERATOR: engines[0], FIXER: engines[1]},
                                engine_params=params)
    else:
        preset = TopologyPreset(mode="shared", total_engines=sum(engines), engine_params=params)
    return ss.SimConfig(workflow=vw, topology=build_topology(preset, vw),
                        policy=ss.PolicyConfig(kind="slack"), arrival_rate=1.0,
                        duration=duration, warmup=0.0, seed=seed)


def gen_config1() -> None:
    out = HERE / "config1"
    if out.exists():
        shutil.rmtree(out)
    RecordingEngine.log = []
    sim = CappedSimulator(config1())
    sim.cap = 64
    # engines were built in __init__ with the default class; rebuild recording ones
    sim2_cls = type("Rec", (CappedSimulator,), {"engine_cls": RecordingEngine, "cap": 64})
    sim = sim2_cls(config1())
    result = sim.run()
    write_run_outputs(result, out)
    with (out / "engine_calls.jsonl").open("w") as f:
        for rec in RecordingEngine.log:
            f.write(json.dumps(rec, sort_keys=True) + "\n")
    print("config1:", result.report.summary_line(), "calls:", len(RecordingEngine.log))


ELASTIC = {"engines": (1, 3), "rate": 2.0, "cap": 96, "duration": 150.0,
           "borrow": {"enabled": True, "util_low": 0.5, "util_high": 0.6},
           "autoscale": {"enabled": True, "check_interval": 1.0, "cooldown": 8.0,
                         "min_engines": 1, "max_engines": 4}}


def elastic_config():
    """Config-1 trace with borrowing + autoscale on (the ELASTIC parameters)."""
    import dataclasses

    from stagesim.scheduling import AutoscaleConfig, BorrowConfig

    cfg = config1(engines=ELASTIC["engines"], duration=ELASTIC["duration"])
    pol = ss.PolicyConfig(kind="slack", borrow=BorrowConfig(**ELASTIC["borrow"]),
                          autoscale=AutoscaleConfig(**ELASTIC["autoscale"]))
    return dataclasses.replace(cfg, policy=pol, arrival_rate=ELASTIC["rate"])


class ElasticRecordingSimulator(CappedSimulator):
    """Logs engine creation and retirement into RecordingEngine.log."""

    engine_cls = RecordingEngine
    cap = ELASTIC["cap"]

    def _add_engine(self, pool_id, params):
        engine = super()._add_engine(pool_id, params)
        RecordingEngine.log.append({"eng": engine.engine_id, "op": "create",
                                    "args": [pool_id, engine.last_advance],
                                    "ret": None})
        return engine

    def _apply_scale(self, pool, decision):
        before = set(self.retired_engines)
        super()._apply_scale(pool, decision)
        for eid in sorted(set(self.retired_engines) - before):
            RecordingEngine.log.append({"eng": eid, "op": "retire", "args": [], "ret": None})


def gen_elastic() -> None:
    out = HERE / "elastic"
    if out.exists():
        shutil.rmtree(out)
    RecordingEngine.log = []
    sim = ElasticRecordingSimulator(elastic_config())
    result = sim.run()
    write_run_outputs(result, out)
    with (out / "engine_calls.jsonl").open("w") as f:
        for rec in RecordingEngine.log:
            f.write(json.dumps(rec, sort_keys=True) + "\n")
    a = sim.audit
    audit = {"borrows": [list(x) for x in a.borrows], "returns": [list(x) for x in a.returns],
             "scale_events": [list(x) for x in a.scale_events]}
    (out / "audit.json").write_text(json.dumps(audit, sort_keys=True) + "\n")
    print("elastic:", result.report.summary_line(), "calls:", len(RecordingEngine.log),
          "borrows:", len(a.borrows), "scale events:", len(a.scale_events))


EVICT = {"engines": (1, 1), "rate": 2.1, "cap": 96, "seed": 2,
         "params": (3200, 2000.0, 0.02, 0.1, 12)}


def evict_config():
    """AC-2's tight shared topology (pkg/tests/test_acceptance.py:79-99: capacity 3200 =
    2P + room for ~4 calls, max_batch 12, prefill 2000 tok/s, rate 2.1) over 2 shared
    engines: an engine holding the other stage's idle prefix must evict it
    (scheduling.py:143-165 -> engines.py:219-226) before it can admit."""
    import dataclasses

    cfg = config1(seed=EVICT["seed"], engines=EVICT["engines"], mode="shared",
                  params=EngineParams(*EVICT["params"]))
    return dataclasses.replace(cfg, arrival_rate=EVICT["rate"])


def gen_evict() -> None:
    out = HERE / "evict"
    if out.exists():
        shutil.rmtree(out)
    RecordingEngine.log = []
    cls = type("Rec", (CappedSimulator,), {"engine_cls": RecordingEngine, "cap": EVICT["cap"]})
    sim = cls(evict_config())
    result = sim.run()
    write_run_outputs(result, out)
    with (out / "engine_calls.jsonl").open("w") as f:
        for rec in RecordingEngine.log:
            f.write(json.dumps(rec, sort_keys=True) + "\n")
    n_ev = sum(1 for r in RecordingEngine.log if r["op"] == "evict_idle_prefix")
    print("evict:", result.report.summary_line(), "calls:", len(RecordingEngine.log),
          "evictions:", n_ev)


def gen_traces() -> None:
    for n, pf in ((64, 0.5), (1024, 0.5), (1024, 0.6)):
        cls = type("Cap", (CappedSimulator,), {"cap": n})
        sim = cls(config1(p_fail=pf, engines=(4, 4),
                          params=EngineParams(10**9, 1e9, 1e-6, 0.0, 10**6)))
        res = sim.run()
        wfs = []
        for rid in sorted(sim.requests):
            req = sim.requests[rid]
            wfs.append({"rid": rid, "terminal": req.terminal,
                        "retries": req.state.retries_used,
                        "stages": [h[0] for h in req.state.stage_history],
                        "labels": [h[3] for h in req.state.stage_history]})
        # the LLM-call token draws, in dispatch order per request
        calls = {}
        for d in res.traces.dispatches:
            calls.setdefault(d.request_id, []).append(d.stage_id)
        (HERE / f"trace_seed0_{n}_pf{int(pf * 10)}.json").write_text(
            json.dumps({"n": n, "p_fail": pf, "seed": 0, "budget": 5, "workflows": wfs},
                       sort_keys=True) + "\n")
        succ = sum(1 for w in wfs if w["terminal"] == "Success")
        print(f"trace n={n} pf={pf}: success={succ} failure={n - succ}")


def gen_engine_scenarios() -> None:
    def params(**kw):
        base = dict(kv_capacity_tokens=16384, prefill_rate=5000.0, base_token_time=0.02,
                    batch_slope=0.1, max_batch=8)
        base.update(kw)
        return base

    # each scenario: engine params + ops; op = [method, args...]; calls are [rid, sid, p, o]
    scenarios = {
        "demand_warm_cold": (params(), [
            ["kv_demand", [1, "gen", 100, 50], 1000],
            ["admit", [0, "gen", 0, 0], 1000, 0.0],
            ["kv_demand", [1, "gen", 100, 50], 1000],
            ["kv_demand", [2, "other", 100, 50], 1000]]),
        "capacity_bound": (params(kv_capacity_tokens=4096), [
            ["admit", [0, "other", 0, 0], 4000, 0.0],
            ["prefill_finished", 0],
            ["complete_call", 0],
            ["can_admit", [1, "gen", 100, 50], 0],
            ["can_admit", [1, "other", 50, 46], 4000],
            ["can_admit", [1, "other", 50, 47], 4000]]),
        "batch_bound": (params(max_batch=2), [
            ["admit", [0, "g", 1, 1], 0, 0.0],
            ["admit", [1, "g", 1, 1], 0, 0.0],
            ["can_admit", [2, "g", 1, 1], 0]]),
        "reservation": (params(kv_capacity_tokens=100), [
            ["admit", [0, "g", 10, 50], 0, 0.0],
            ["can_admit", [1, "g", 10, 50], 0],
            ["admit_expect_error", [1, "g", 200, 200], 0, 0.0]]),
        "prefill_times": (params(prefill_rate=1000.0), [
            ["admit", [0, "gen", 200, 0], 800, 0.0],
            ["admit", [1, "gen", 200, 0], 800, 5.0],
            ["admit", [2, "gen", 0, 0], 800, 3.0]]),
        "decode_progress": (params(base_token_time=0.05, batch_slope=0.2), [
            ["admit", [0, "g", 0, 100], 0, 0.0], ["prefill_finished", 0],
            ["advance_decode", 2.5], ["next_completion", 2.5], ["advance_decode", 5.0],
            ["complete_call", 0],
            ["admit", [1, "g", 0, 100], 0, 5.0], ["prefill_finished", 1],
            ["admit", [2, "g", 0, 100], 0, 5.0], ["prefill_finished", 2],
            ["advance_decode", 8.0], ["next_completion", 8.0], ["advance_decode", 11.0],
            ["complete_call", 1], ["next_completion", 11.0], ["complete_call", 2]]),
        "fractional_segments": (params(), [
            ["admit", [0, "g", 37, 151], 100, 0.0], ["prefill_finished", 0],
            ["admit", [1, "g", 5, 60], 100, 0.05], ["prefill_finished", 1],
            *[["advance_decode", 0.05 + 0.0137 * (i + 1)] for i in range(40)],
            ["next_completion", 0.05 + 0.0137 * 40]]),
        "prefill_not_decoding": (params(), [
            ["admit", [0, "g", 10, 20], 0, 0.0], ["advance_decode", 1.0],
            ["prefill_finished", 0], ["advance_decode", 1.1], ["advance_decode", 1.1]]),
        "eviction_lru": (params(), [
            ["admit", [0, "a", 0, 0], 10, 1.0], ["complete_call", 0],
            ["admit", [1, "b", 0, 0], 20, 2.0], ["complete_call", 1],
            ["admit", [2, "c", 0, 0], 30, 3.0], ["complete_call", 2],
            ["admit", [3, "a", 0, 0], 10, 4.0], ["complete_call", 3],
            ["evictable_prefixes", "z"], ["evictable_prefixes", "b"],
            ["admit", [4, "b", 3, 3], 20, 5.0],
            ["evict_expect_error", "b"],
            ["evict_idle_prefix", "c"], ["evict_idle_prefix", "c"],
            ["evictable_prefixes", "z"]]),
        "backwards_advance": (params(), [
            ["advance_decode", 2.0], ["advance_expect_error", 1.0]]),
    }
    out = {}
    for name, (prm, ops) in scenarios.items():
        eng = EngineState(0, EngineParams(**prm), "pool:x")
        inflight = {}
        steps = []
        for op in ops:
            kind = op[0]
            ret = None
            if kind in ("kv_demand", "can_admit"):
                c = PendingCall(op[1][0], op[1][1], 0.0, op[1][2], op[1][3])
                ret = getattr(eng, kind)(c, op[2])
            elif kind == "admit":
                c = PendingCall(op[1][0], op[1][1], op[3], op[1][2], op[1][3])
                fl, ret = eng.admit(c, op[2], op[3])
                inflight[fl.request_id] = fl
            elif kind == "admit_expect_error":
                c = PendingCall(op[1][0], op[1][1], op[3], op[1][2], op[1][3])
                try:
                    eng.admit(c, op[2], op[3])
                    ret = "no-error"
                except ss.AdmitWithoutCapacity:
                    ret = "AdmitWithoutCapacity"
            elif kind == "prefill_finished":
                eng.prefill_finished(inflight[op[1]])
            elif kind == "complete_call":
                eng.complete_call(inflight[op[1]])
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
                except ss.PrefixInUse:
                    ret = "PrefixInUse"
            else:
                raise ValueError(kind)
            steps.append({"op": op, "ret": ret, "state": engine_state(eng),
                          "free_kv": eng.free_kv(), "decode_batch_size": eng.decode_batch_size(),
                          "resident_prefix_tokens": eng.resident_prefix_tokens(),
                          "recomputed_kv_used": eng.recomputed_kv_used(),
                          "recomputed_kv_reserved": eng.recomputed_kv_reserved()})
        out[name] = {"params": prm, "steps": steps}
    (HERE / "engine_scenarios.json").write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
    print("scenarios:", len(out))


if __name__ == "__main__":
    gen_engine_scenarios()
    gen_config1()
    gen_elastic()
    gen_evict()
    gen_traces()
