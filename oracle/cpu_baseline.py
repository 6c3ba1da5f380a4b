"""CPU baseline of the stage-engine hot path, timed on the host cores.

ORACLE — used only by bench.py's cpu_baseline leg / `--impl reference` and by tests;
never by the product path.

Two parts, both on the box the GPU numbers come from:

1. The reference's own CPU path (`control_path`): the unmodified reference `stagesim`
   (installed in baseline/_ref) runs its `Simulator` over the same seeded NL2SQL trace
   (seed 0, retry budget 5, the bench workload's prefix / prompt / output draws),
   single-threaded as it is by design (simulation.py:816-837): isolated
   1 + 1 engines with the bench's engine constants, 512 workflows. Its wall time per
   workflow is the reference's per-workflow scheduling / accounting cost. The reference
   has no model arithmetic (its decode is t(b) = t0(1 + alpha(b-1)), engines.py:55-57).

2. The model arithmetic the GPU engine performs, as the builder's CPU fp32 restatement
   of the same decoder (oracle/decoder_ref.py semantics) on ALL host threads:
     * a prompt prefill of 200 tokens attending a 1000-token resident prefix, and
     * DECODE_STEPS (20) batched greedy decode steps of 16 calls at context ~1250,
   through all n_layers layers, each layer with its OWN weights (32 distinct fp32
   weight sets: the full 30 GB of the 8B shape is streamed per decode step; layer i's
   tensors are element permutations of one random draw, so setup costs a copy, not
   7.5 G random draws), plus the final norm, lm_head and argmax.

Workflows/s = 1 / (control cost per workflow + model cost per workflow), the model cost
being the trace's own mean over its first 1024 workflows of
    sum over the workflow's LLM calls of [p x t_prefill_per_token + o x t_step / 16]
with p, o the calls' prompt / output draws (workflow.py, the reference's counter
streams). This is a CPU engine at batch 16; the sample string states it.
"""

from __future__ import annotations

import math
import os
import platform
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
PROMPT, PREFIX, BATCH, DECODE_STEPS = 200, 1000, 16, 20


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def _rms(h, w, eps=1e-5):
    return h * torch.rsqrt((h * h).mean(-1, keepdim=True) + eps) * w


def _layers(cfg, seed: int) -> list[dict]:
    """n_layers distinct fp32 weight sets (layer i = a fixed element permutation of one
    N(0, 0.02^2) draw, rolled by i: distinct memory, identical statistics)."""
    g = torch.Generator().manual_seed(seed)
    d, hq, hkv, ffn = cfg.d_model, cfg.n_heads, cfg.n_kv_heads, cfg.ffn
    shapes = {"wqkv": ((hq + 2 * hkv) * 128, d), "wo": (d, hq * 128), "wgu": (2 * ffn, d),
              "wd": (d, ffn)}
    base = {k: torch.randn(*s, generator=g) * 0.02 for k, s in shapes.items()}
    out = []
    for i in range(cfg.n_layers):
        L = {k: torch.roll(v.reshape(-1), 7919 * i).reshape(v.shape) for k, v in base.items()}
        L["n1"] = torch.ones(d)
        L["n2"] = torch.ones(d)
        out.append(L)
    return out


@torch.no_grad()
def _forward(layers, h, k_ctx, v_ctx, hq, hkv, ffn, causal_q):
    """h [B, T, d]; k_ctx / v_ctx [B, S, hkv, 128] context KV per layer (same tensor reused
    per layer: the attention bytes are small next to the weights)."""
    B, T, d = h.shape
    group = hq // hkv
    for L in layers:
        x = _rms(h, L["n1"])
        qkv = x @ L["wqkv"].T
        q = qkv[..., : hq * 128].reshape(B, T, hq, 128)
        k = qkv[..., hq * 128:(hq + hkv) * 128].reshape(B, T, hkv, 128)
        v = qkv[..., (hq + hkv) * 128:].reshape(B, T, hkv, 128)
        kk = torch.cat([k_ctx, k], 1).repeat_interleave(group, 2)
        vv = torch.cat([v_ctx, v], 1).repeat_interleave(group, 2)
        s = torch.einsum("bthd,bshd->bhts", q, kk) / math.sqrt(128)
        if causal_q and T > 1:
            S = kk.shape[1]
            mask = torch.arange(S)[None, :] > (S - T + torch.arange(T))[:, None]
            s = s.masked_fill(mask, float("-inf"))
        a = torch.einsum("bhts,bshd->bthd", torch.softmax(s, -1), vv).reshape(B, T, hq * 128)
        h = h + a @ L["wo"].T
        x = _rms(h, L["n2"])
        gu = x @ L["wgu"].T
        act = torch.nn.functional.silu(gu[..., :ffn]) * gu[..., ffn:]
        h = h + act @ L["wd"].T
    return h


def _stagesim():
    base = ROOT / "baseline" / "_ref"
    for p in sorted(base.rglob("stagesim/__init__.py")) if base.exists() else []:
        if str(p.parent.parent) not in sys.path:
            sys.path.insert(0, str(p.parent.parent))
        break
    import stagesim

    return stagesim


def control_path_seconds_per_workflow(spec, max_batch: int = 256, n_workflows: int = 512,
                                      seed: int = 0) -> tuple[float, str]:
    """Wall time per workflow of the reference Simulator on the seeded trace (1 thread)."""
    import dataclasses

    ss = _stagesim()
    from stagesim import simulation as sim_mod
    from stagesim.dists import Distribution
    from stagesim.engines import EngineParams as REngineParams
    from stagesim.workloads import FIXER, GENERATOR, Nl2SqlParams, TopologyPreset, \
        build_nl2sql, build_topology

    class Capped(ss.Simulator):
        def _schedule(self, time_, kind, **refs):
            if kind == sim_mod.EVENT_ARRIVAL and self._next_rid >= n_workflows:
                return
            super()._schedule(time_, kind, **refs)

    P = max(spec.generator_prefix_tokens, spec.fixer_prefix_tokens)
    p_hi = int(spec.prompt_tokens.high)
    o_hi = int(getattr(spec.output_tokens, "high", getattr(spec.output_tokens, "value", 0)))
    nl = Nl2SqlParams(p_fail=spec.p_fail, p_syntax_err=spec.p_syntax_err,
                      p_empty_result=spec.p_empty_result, retry_budget=spec.retry_budget)
    fields = {f.name for f in dataclasses.fields(nl)}
    extra = {}
    if "generator_prefix_tokens" in fields:
        extra["generator_prefix_tokens"] = spec.generator_prefix_tokens
        extra["fixer_prefix_tokens"] = spec.fixer_prefix_tokens
    if "output_tokens" in fields and not hasattr(spec.output_tokens, "high"):
        extra["output_tokens"] = Distribution.constant(spec.output_tokens.value)
    nl = dataclasses.replace(nl, **extra)
    vw = ss.validate_workflow(build_nl2sql(nl))
    params = REngineParams(P + max_batch * (p_hi + o_hi), 5000.0, 0.02, 0.1, max_batch)
    preset = TopologyPreset(mode="isolated", engines_per_stage={GENERATOR: 1, FIXER: 1},
                            engine_params=params)
    cfg = ss.SimConfig(workflow=vw, topology=build_topology(preset, vw),
                       policy=ss.PolicyConfig(kind="slack"), arrival_rate=16.0,
                       duration=1e9, warmup=0.0, seed=seed)
    sim = Capped(cfg)
    t0 = time.perf_counter()
    sim.run()
    dt = time.perf_counter() - t0
    return dt / n_workflows, (f"reference stagesim Simulator.run, {n_workflows} workflows of the "
                              f"seed-{seed} trace, isolated 1+1 engines, max_batch {max_batch}, "
                              f"1 thread: {dt:.2f} s")


def trace_calls(spec, n: int = 1024, seed: int = 0) -> tuple[float, float, float]:
    """Mean LLM calls, prompt tokens and output tokens per workflow of the seeded trace."""
    from paper_2510_14126_b200.workflow import EXECUTOR, Workflow

    calls = p_sum = o_sum = 0
    for rid in range(n):
        wf = Workflow(rid, spec, seed)
        while True:
            r = wf.enter()
            if wf.stage != EXECUTOR:
                calls += 1
                p_sum += r[0]
                o_sum += r[1]
            if wf.finish() is None:
                break
    return calls / n, p_sum / n, o_sum / n


def measure(cfg, spec=None, threads: int | None = None, seed: int = 0) -> dict:
    """Time the sample; returns workflows/s, decode tok/s, cores, kind, sample, cpu model."""
    if spec is None:
        from paper_2510_14126_b200.workflow import Nl2Sql

        spec = Nl2Sql(retry_budget=5)
    threads = threads or os.cpu_count() or 1
    torch.set_num_threads(threads)
    try:
        ctl_s, ctl_note = control_path_seconds_per_workflow(spec, seed=seed)
    except ImportError as e:  # the reference is installed by __graft_entry__.build()
        raise RuntimeError("reference stagesim not installed in baseline/_ref") from e
    g = torch.Generator().manual_seed(seed + 1)
    d, hq, hkv, ffn = cfg.d_model, cfg.n_heads, cfg.n_kv_heads, cfg.ffn
    layers = _layers(cfg, seed)
    lm = torch.randn(cfg.vocab, d, generator=g) * 0.02
    # prompt prefill behind the resident prefix
    h = torch.randn(1, PROMPT, d, generator=g)
    kc = torch.randn(1, PREFIX, hkv, 128, generator=g)
    t0 = time.perf_counter()
    hp = _forward(layers, h, kc, kc, hq, hkv, ffn, causal_q=True)
    _ = (_rms(hp[:, -1], torch.ones(d)) @ lm.T).argmax(-1)
    t_prefill = time.perf_counter() - t0
    # DECODE_STEPS batched decode steps, context growing by one token per step
    ctx = PREFIX + PROMPT + 50
    kc = torch.randn(BATCH, ctx + DECODE_STEPS, hkv, 128, generator=g)
    h = torch.randn(BATCH, 1, d, generator=g)
    t0 = time.perf_counter()
    for s in range(DECODE_STEPS):
        k = kc[:, :ctx + s]
        hd = _forward(layers, h, k, k, hq, hkv, ffn, causal_q=False)
        tok = (_rms(hd[:, 0], torch.ones(d)) @ lm.T).argmax(-1)
        h = hd + 1e-3 * tok.to(hd.dtype)[:, None, None]  # next step depends on this one
    t_step = (time.perf_counter() - t0) / DECODE_STEPS
    calls, p_mean, o_mean = trace_calls(spec, seed=seed)
    model_s = p_mean * t_prefill / PROMPT + o_mean * t_step / BATCH
    per_wf = ctl_s + model_s
    return {
        "workflows_per_s": 1.0 / per_wf,
        "decode_tok_s": BATCH / t_step,
        "prefill_tok_s": PROMPT / t_prefill,
        "cores": threads,
        "kind": "port",
        "cpu_model": cpu_model(),
        "t_prefill_s": t_prefill,
        "t_decode_step_s": t_step,
        "control_path": {"seconds_per_workflow": ctl_s, "workflows_per_s": 1.0 / ctl_s,
                         "sample": ctl_note},
        "sample": (f"{cfg.name} fp32 on {threads} threads: 1 prefill of {PROMPT} tokens after a "
                   f"{PREFIX}-token prefix + {DECODE_STEPS} decode steps of batch {BATCH} at ctx "
                   f"{ctx}+, all {cfg.n_layers} layers with their own weights + lm_head; "
                   f"workflows/s = 1 / (reference control path {ctl_s * 1e3:.2f} ms + trace mean "
                   f"{calls:.3f} calls: {p_mean:.1f} prompt tok x prefill/tok + {o_mean:.1f} "
                   f"output tok x step/{BATCH}) per workflow"),
    }
