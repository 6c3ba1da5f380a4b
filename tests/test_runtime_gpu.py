"""Wall-clock pool runtime on the B200 (throughput mode), tiny decoder.

64 NL2SQL workflows (seed 0, budget 5) through isolated generator/fixer engines
sharing one GPU, closed loop of 16. Checked: per-workflow outcomes, retries and
stage sequences equal the reference's own trace (timing-independent by the
reference's design), every generated SQL equals the CPU oracle decoder's greedy
continuation (teacher forced, near-ties excepted), and the block pools return to
exactly the resident prefixes at the end.
"""

from __future__ import annotations

import json

import numpy as np
import pytest
import torch

from harness import GOLDEN
from oracle.decoder_ref import RefDecoder, greedy, top2_margin
from paper_2510_14126_b200.config import TINY
from paper_2510_14126_b200.engine import EngineParams, blocks_for
from paper_2510_14126_b200.model import GpuWorker
from paper_2510_14126_b200.runtime import PoolRuntime
from paper_2510_14126_b200.tokens import prefix_tokens, prompt_tokens
from paper_2510_14126_b200.workflow import Nl2Sql, Uniform

pytestmark = pytest.mark.gpu


def _runtime(cuda, concurrency=16, n=64, mode="isolated"):
    spec = Nl2Sql(retry_budget=5, executor_service_time=Uniform(0.001, 0.004))
    params = EngineParams(1000 + concurrency * 450, 5000.0, 0.02, 0.1, concurrency)
    bpe = blocks_for(params)
    worker = GpuWorker(TINY, cuda, n_blocks=2 * bpe, n_rows=2 * (concurrency + 4), row_cols=100,
                       max_tokens=1024, max_out=2 * concurrency + 16, hist_cols=160,
                       max_seq_tokens=1500)
    return PoolRuntime(worker, spec, params, mode=mode, concurrency=concurrency, n_workflows=n,
                       prefill_budget=700)


@pytest.mark.parametrize("mode", ["isolated", "shared"])
def test_runtime_outcomes_and_tokens(cuda, mode):
    rt = _runtime(cuda, mode=mode)
    results = []
    rt.on_result = lambda call, toks: results.append((call.request_id, call.stage_id, call.visit,
                                                     call.prompt_tokens, toks))
    rt.fill()
    rt.run_until(64, max_seconds=300)
    torch.cuda.synchronize()
    assert int(rt.worker.status[0]) == 0
    gold = json.loads((GOLDEN / "trace_seed0_64_pf5.json").read_text())
    got = {wf.rid: wf for wf in rt.finished}
    assert len(got) == 64
    for w in gold["workflows"]:
        wf = got[w["rid"]]
        assert wf.terminal == w["terminal"]
        assert wf.retries == w["retries"]
        assert [h[0] for h in wf.history] == w["stages"]
    assert rt.stats.completed == 62 and rt.stats.failed == 2
    assert len(results) == 131
    # pools hold only resident prefixes
    for e in rt.engines:
        assert not e.batch
        assert e.blocks_in_use == sum(p.n_blocks for p in e.resident.values())
    # every 8th SQL against the oracle decoder
    dec = RefDecoder(TINY.to_ref(), rt.worker.oracle_weights(), max_pos=2048)
    pre = {}
    mism = n_tok = 0
    for rid, sid, visit, p, toks in results[::8]:
        if sid not in pre:
            s0 = dec.new_seq()
            s0.extend(prefix_tokens(0, sid, 1000, TINY.vocab), "none")
            pre[sid] = s0
        seq = pre[sid].fork()
        logits = seq.extend(prompt_tokens(0, rid, sid, visit, p, TINY.vocab))
        for k, t in enumerate(toks):
            if k:
                logits = seq.extend([int(toks[k - 1])])
            n_tok += 1
            if greedy(logits) != int(t):
                mism += 1
                assert top2_margin(logits) < 2e-2
    assert n_tok > 1000
    assert mism <= max(3, n_tok // 500)


def test_runtime_long_prefix_config4(cuda):
    """BASELINE config 4's shape on the tiny decoder: 8K-token schema prefixes and 512-token
    outputs, so private contexts pass one 512-token decode split (a short 2nd split) and the
    8K prefix is chunk-prefilled and reused across retries. Outcomes equal the reference
    trace; SQL of a first call and a retry match the CPU oracle; logits stay finite."""
    from paper_2510_14126_b200.workflow import Constant

    n, conc, P = 8, 8, 8192
    spec = Nl2Sql(retry_budget=5, generator_prefix_tokens=P, fixer_prefix_tokens=P,
                  output_tokens=Constant(512), executor_service_time=Uniform(0.001, 0.004))
    max_seq = P + 300 + 512
    params = EngineParams(P + conc * 812, 5000.0, 0.02, 0.1, conc)
    bpe = blocks_for(params)
    worker = GpuWorker(TINY, cuda, n_blocks=2 * bpe, n_rows=2 * (conc + 4),
                       row_cols=(max_seq + 15) // 16 + 2, max_tokens=2048, max_out=2 * conc + 16,
                       hist_cols=520, max_seq_tokens=max_seq + 16)
    rt = PoolRuntime(worker, spec, params, mode="isolated", concurrency=conc, n_workflows=n,
                     prefill_budget=1500)
    results = []
    rt.on_result = lambda call, toks: results.append((call.request_id, call.stage_id, call.visit,
                                                     call.prompt_tokens, toks))
    finite = []
    worker.on_forward = lambda plan, n_out: finite.append(
        bool(torch.isfinite(worker.logits[:n_out]).all()))
    rt.fill()
    rt.run_until(n, max_seconds=600)
    torch.cuda.synchronize()
    assert int(worker.status[0]) == 0
    assert all(finite)
    gold = {w["rid"]: w for w in json.loads((GOLDEN / "trace_seed0_64_pf5.json").read_text())
            ["workflows"]}
    got = {wf.rid: wf for wf in rt.finished}
    assert sorted(got) == list(range(n))
    for rid, wf in got.items():
        assert wf.terminal == gold[rid]["terminal"]
        assert [h[0] for h in wf.history] == gold[rid]["stages"]
    assert all(len(t) == 512 for *_, t in results)
    dec = RefDecoder(TINY.to_ref(), worker.oracle_weights(), max_pos=max_seq + 16)
    picks = [results[0]] + [r for r in results if r[1] != results[0][1]][:1]
    mism = n_tok = 0
    for rid, sid, visit, p, toks in picks:
        seq = dec.new_seq()
        seq.extend(prefix_tokens(0, sid, P, TINY.vocab), "none")
        logits = seq.extend(prompt_tokens(0, rid, sid, visit, p, TINY.vocab))
        for k, t in enumerate(toks):
            if k:
                logits = seq.extend([int(toks[k - 1])])
            n_tok += 1
            if greedy(logits) != int(t):
                mism += 1
                assert top2_margin(logits) < 2e-2, (rid, sid, k)
    assert n_tok == 1024 and mism <= 3
