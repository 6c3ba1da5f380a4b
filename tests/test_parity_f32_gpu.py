"""Config-1 parity in fp32 (BASELINE configs[0]; the north star's "1e-5 in fp32, greedy
tokens identical"), on a B200.

The reference Simulator's config-1 engine call stream (tests/golden/config1: NL2SQL,
budget 5, isolated 1 + 1 engines, seed 0, 64 workflows, 131 LLM calls) drives two
GpuEngineState engines whose worker runs the fp32 path (csrc/fp32.cu: fp32 weights,
residual stream, activations, paged KV cache and logits). Checked:
  * engine state bit-exact with the reference after every call, block tables equal the
    CPU block oracle's;
  * every completed call's generated tokens are IDENTICAL to the CPU fp32 decoder
    oracle's own free-running greedy continuation (oracle/decoder_ref.py, exact mode:
    no rounding anywhere), and every position's logits are within 1e-5 relative
    (Frobenius) of the oracle's.
"""

from __future__ import annotations

import pytest
import torch

from harness import (
    CONFIG1_PARAMS,
    GOLDEN,
    RecordingObserver,
    config1_engines,
    load_jsonl,
    replay_calls,
)
from oracle.decoder_ref import RefDecoder, greedy
from oracle.engine_ref import replay_blocks
from paper_2510_14126_b200.config import TINY
from paper_2510_14126_b200.engine import blocks_for
from paper_2510_14126_b200.model import GpuWorker
from paper_2510_14126_b200.tokens import prefix_tokens, prompt_tokens

pytestmark = pytest.mark.gpu

F32_TOL = 1e-5


def test_config1_fp32_free_running_identity(cuda):
    records = load_jsonl(GOLDEN / "config1" / "engine_calls.jsonl")
    bpe = blocks_for(CONFIG1_PARAMS)
    worker = GpuWorker(TINY, cuda, n_blocks=2 * bpe, n_rows=24, row_cols=bpe, max_tokens=2048,
                       max_out=64, hist_cols=512, max_seq_tokens=16384 + 64, precision="f32")
    logits = {}

    def capture(plan, n_out):
        rows = [(d.row, d.hist_pos) for d in plan.decode]
        rows += [(s.out_row, s.hist_pos) for s in plan.prefill if s.out_row >= 0]
        lg = worker.logits[:len(rows)].detach().cpu()
        for i, key in enumerate(rows):
            logits[key] = lg[i].clone()

    worker.on_forward = capture

    class Obs(RecordingObserver):
        def on_complete(self, engine, call):
            super().on_complete(engine, call)
            n = max(1, call.target_output_tokens)
            self.completed[engine.engine_id][-1]["logits"] = [logits.pop((call.slot, k))
                                                              for k in range(n)]

    obs = Obs(read_device=True)
    engines, bpe = config1_engines(worker, obs, vocab=TINY.vocab)
    replay_calls(records, engines)
    torch.cuda.synchronize()
    assert int(worker.status[0]) == 0
    ref = replay_blocks(records, {0: (bpe, 0), 1: (bpe, bpe)})
    for eid in (0, 1):
        assert [g["row"] for g in obs.completed[eid]] == [e["row"] for e in ref[eid].completed]

    dec = RefDecoder(TINY.to_ref(), worker.oracle_weights(), max_pos=16384 + 64, exact=True)
    prefixes = {}
    n_tok = n_calls = 0
    worst = 0.0
    for eid in (0, 1):
        for c in obs.completed[eid]:
            sid, P, p = c["sid"], c["P"], c["p"]
            if (sid, P) not in prefixes:
                s0 = dec.new_seq()
                lg = s0.extend(prefix_tokens(0, sid, P, TINY.vocab)) if P else None
                prefixes[(sid, P)] = (s0, lg)
            s0, plg = prefixes[(sid, P)]
            seq = s0.fork()
            lg = seq.extend(prompt_tokens(0, c["rid"], sid, c["visit"], p, TINY.vocab)) if p \
                else plg
            want = []
            for k in range(len(c["tokens"])):
                if k:
                    lg = seq.extend([want[-1]])  # free running: the oracle's own tokens
                want.append(greedy(lg))
                r = lg.reshape(-1)
                err = float((c["logits"][k] - r).norm() / r.norm())
                worst = max(worst, err)
            assert c["tokens"] == want, (eid, c["rid"], sid)
            n_tok += len(want)
            n_calls += 1
    print(f"\nconfig1 fp32: {n_calls} calls, {n_tok} tokens identical (free running), worst "
          f"position logit rel err {worst:.2e}")
    assert n_calls == 131 and n_tok > 10000
    assert worst < F32_TOL
