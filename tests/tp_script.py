"""A scripted sequence of decoder steps for the TP = 2 tests (shared by the
in-process and the two-process variants).

Two table rows with randomly permuted private blocks: row 0 prefills 200 tokens,
then decodes while row 1 prefills 150 tokens in the same step (mixed
prefill + decode), then both rows decode. Every step's logits are kept.
"""

from __future__ import annotations

import numpy as np
import torch

from paper_2510_14126_b200.model import DecodeTok, GpuWorker, PrefillSeq, StepPlan

N_BLOCKS, ROWS, COLS = 64, 2, 32
MAX_TOKENS, MAX_OUT, HIST, MAX_SEQ = 512, 8, 64, 1024
LENS = (200, 150)
DECODE_STEPS = 14


def prompts(vocab: int) -> list[np.ndarray]:
    rng = np.random.default_rng(11)
    return [rng.integers(0, vocab, n).astype(np.int32) for n in LENS]


def make_worker(cfg, device, weights, tp=None) -> GpuWorker:
    w = GpuWorker(cfg, device, N_BLOCKS, ROWS, COLS, max_tokens=MAX_TOKENS, max_out=MAX_OUT,
                  hist_cols=HIST, max_seq_tokens=MAX_SEQ, weights=weights, tp=tp)
    w.full_logits = True  # the tests compare every step's logits
    perm = torch.randperm(N_BLOCKS, generator=torch.Generator().manual_seed(5)).to(torch.int32)
    w.table.copy_(perm.view(ROWS, COLS).to(w.device))
    return w


def plans(vocab: int) -> list[StepPlan]:
    """Fresh plan objects (forward() reorders a plan's decode list in place)."""
    p0, p1 = prompts(vocab)
    out = [StepPlan(prefill=[PrefillSeq(0, 0, len(p0), p0, out_row=0, hist_pos=0)])]
    out.append(StepPlan(decode=[DecodeTok(0, 0, len(p0) + 1, hist_pos=1)],
                        prefill=[PrefillSeq(1, 0, len(p1), p1, out_row=1, hist_pos=0)]))
    for k in range(DECODE_STEPS):
        out.append(StepPlan(decode=[DecodeTok(0, 0, len(p0) + 2 + k, hist_pos=2 + k),
                                    DecodeTok(1, 0, len(p1) + 1 + k, hist_pos=1 + k)]))
    return out


def run_lockstep(workers, vocab: int, between=None) -> list[list[torch.Tensor]]:
    """Run the script on the ranks of one replica; returns per-rank lists of step logits.
    `between` (optional) is called at every exchange point of every rank."""
    from paper_2510_14126_b200.tp import lockstep

    logs = [[] for _ in workers]
    for step in range(len(plans(vocab))):
        gens = [w.forward_steps(plans(vocab)[step]) for w in workers]
        if between is None:
            lockstep(gens)
        else:
            for g in gens:  # one rank per process: sync at every exchange point
                for _ in g:
                    between()
        for i, w in enumerate(workers):
            logs[i].append(w.logits[:w.n_out].clone())
    return logs
