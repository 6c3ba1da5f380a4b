"""The runtime's workflow mirror reproduces the reference's per-workflow outcomes.

Goldens are the reference Simulator's own results (tests/golden/make_golden.py):
64 and 1024 workflows at p_fail 0.5 and 1024 at p_fail 0.6, seed 0, budget 5.
"""

from __future__ import annotations

import json

import pytest

from harness import GOLDEN
from paper_2510_14126_b200.workflow import EXECUTOR, Nl2Sql, Workflow, stream_uniform


def walk(rid: int, spec: Nl2Sql, seed: int = 0) -> Workflow:
    wf = Workflow(rid, spec, seed)
    while True:
        wf.enter()
        if wf.finish() is None:
            return wf


@pytest.mark.parametrize("name,pf", [("trace_seed0_64_pf5.json", 0.5),
                                     ("trace_seed0_1024_pf5.json", 0.5),
                                     ("trace_seed0_1024_pf6.json", 0.6)])
def test_outcomes_match_reference(name, pf):
    gold = json.loads((GOLDEN / name).read_text())
    spec = Nl2Sql(p_fail=pf, p_syntax_err=pf / 2, p_empty_result=pf / 2, retry_budget=5)
    for w in gold["workflows"]:
        wf = walk(w["rid"], spec)
        assert wf.terminal == w["terminal"], w["rid"]
        assert wf.retries == w["retries"], w["rid"]
        assert [h[0] for h in wf.history] == w["stages"], w["rid"]
        assert [h[1] for h in wf.history] == w["labels"], w["rid"]


def test_config1_token_draws_match_reference_dispatches():
    """Prompt/output lengths equal the reference's sums for config 1."""
    spec = Nl2Sql(retry_budget=5)
    sums = {"sql_generator": [0, 0, 0], "sql_fixer": [0, 0, 0]}
    for rid in range(64):
        wf = Workflow(rid, spec, 0)
        while True:
            r = wf.enter()
            if wf.stage != EXECUTOR:
                s = sums[wf.stage]
                s[0] += 1
                s[1] += r[0]
                s[2] += r[1]
            if wf.finish() is None:
                break
    assert sums["sql_generator"] == [64, 13103, 6513]
    assert sums["sql_fixer"] == [67, 13370, 6565]


def test_stream_uniform_range_and_determinism():
    u = [stream_uniform(0, "arrivals", i) for i in range(1000)]
    assert all(0.0 < x <= 1.0 for x in u)
    assert u == [stream_uniform(0, "arrivals", i) for i in range(1000)]
