"""The native layer loop (csrc/step.cu, cortex_decoder_layers) against the Python loop of
GpuWorker.forward: the same launches with the same arguments, so every step's residual
stream, q / attention activations, KV cache and greedy tokens must be bit-identical.
Steps cover the engine's mixes (stagesim/engines.py:142-194): a cold stage-prefix
prefill, prompt prefills behind the resident prefix, decode steps with the shared-prefix
(cascade) groups and the side-stream overlap, decode + prefill in one step, and a
prefix-less call decoding beside the grouped ones."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2510_14126_b200.config import ModelConfig
from paper_2510_14126_b200.model import DecodeTok, GpuWorker, PrefillSeq, StepPlan

pytestmark = pytest.mark.gpu

CFG = ModelConfig("mid-3L", n_layers=3, d_model=512, n_heads=8, n_kv_heads=2, ffn=1024,
                  vocab=2048, rope_theta=500000.0)
P, PROMPT = 200, 40


def _plans(rng):
    pre = rng.integers(0, CFG.vocab, P).astype(np.int32)
    prompts = [rng.integers(0, CFG.vocab, PROMPT).astype(np.int32) for _ in range(4)]
    solo = rng.integers(0, CFG.vocab, 37).astype(np.int32)
    plans = [StepPlan(prefill=[PrefillSeq(0, 0, P, pre)])]
    plans.append(StepPlan(prefill=[PrefillSeq(r, P, P + PROMPT, prompts[r - 1], out_row=r)
                                   for r in (1, 2, 3)] + [PrefillSeq(5, 0, 37, solo, out_row=5)]))
    for k in range(4):
        dec = [DecodeTok(r, P, P + PROMPT + k + 1, hist_pos=k + 1, prefix_key=0) for r in (1, 2, 3)]
        dec.append(DecodeTok(5, 0, 37 + k + 1, hist_pos=k + 1))
        pf = []
        if k == 1:  # a fourth prompt joins mid-stream: decode + prefill in one step
            pf = [PrefillSeq(4, P, P + PROMPT, prompts[3], out_row=4)]
        if k >= 2:
            dec.append(DecodeTok(4, P, P + PROMPT + k - 1, hist_pos=k - 1, prefix_key=0))
        plans.append(StepPlan(decode=dec, prefill=pf))
    return plans


def _run(cuda, native: bool, overlap: bool, two_side: bool = True):
    torch.manual_seed(0)
    w = GpuWorker(CFG, cuda, n_blocks=64, n_rows=8, row_cols=32, max_tokens=512, max_out=16,
                  hist_cols=16, max_seq_tokens=512, seed=3)
    w.native_layers = native
    w.overlap_cascade = overlap
    if not two_side:
        w.side2 = None
    npb = (P + 15) // 16
    tab = torch.zeros(8, 32, dtype=torch.int32)
    tab[0, :npb] = torch.arange(npb)
    nxt = npb
    for r in (1, 2, 3, 4):
        tab[r, :npb] = torch.arange(npb)
        tab[r, npb:npb + 4] = torch.arange(nxt, nxt + 4)
        nxt += 4
    tab[5, :4] = torch.arange(nxt, nxt + 4)
    w.table.copy_(tab.to(cuda))
    snaps = []
    for plan in _plans(np.random.default_rng(7)):
        w.forward(plan)
        torch.cuda.synchronize()
        T = plan.n_tokens
        snaps.append((w.x[:T].clone(), w.q[:T].clone(), w.attn[:T].clone(),
                      w.out_tok[:w.n_out].clone(), w.slot_tok.clone()))
    assert int(w.status[0]) == 0
    return snaps, w.cache.clone(), w.launches


@pytest.mark.parametrize("overlap", [True, False])
def test_native_layers_bit_identical(cuda, overlap):
    got, cache_n, launches_n = _run(cuda, True, overlap)
    want, cache_p, launches_p = _run(cuda, False, overlap)
    assert launches_n == launches_p
    for i, (g, w) in enumerate(zip(got, want)):
        for name, a, b in zip(("x", "q", "attn", "out_tok", "slot_tok"), g, w):
            assert torch.equal(a, b), (i, name)
    assert torch.equal(cache_n, cache_p)
    assert torch.isfinite(got[-1][0]).all()


def test_stream_schedules_bit_identical(cuda):
    """The attention passes' stream placement (two side streams, one, or all on the main
    stream) changes only the overlap, never a value."""
    ref, cache_ref, _ = _run(cuda, True, True)
    for overlap, two in ((True, False), (False, True)):
        got, cache, _ = _run(cuda, True, overlap, two)
        for i, (g, w) in enumerate(zip(got, ref)):
            for name, a, b in zip(("x", "q", "attn", "out_tok", "slot_tok"), g, w):
                assert torch.equal(a, b), (overlap, two, i, name)
        assert torch.equal(cache, cache_ref)
