"""A/B of kernel variants on a FIXED recorded step mix (config 2, N = 1).

Runs the bench's closed loop to steady state, records the next `--record` steps' plans
(the exact decode / prefill mix the timed window sees), then replays that plan list
through the worker under each variant, interleaved over `--rounds` rounds, timing every
replay with CUDA events. The mix is identical across variants, so differences are the
kernels' alone (the KV values replayed are stale, the work is the same).

    python benchmarks/replay_ab.py [--record 60] [--rounds 3] [--variants base,plo0,...]
Variants: base | plo0 (P as bf16 only) | norope (unfused RoPE / KV append) |
          logits (full lm_head logits + argmax) | pdl0 (no programmatic dependent launch) |
          fmha1q / fmha2q / fmhaauto (tcgen05 attention with one / two Q tiles per CTA, or
          chosen per launch by wave count) |
          python (layer loop in Python, not csrc/step.cu) | serial (attention passes on one
          stream) | slots1 / slots4 (cascade prefix slots) | prio / prio0 / priomax (side stream priority -1 / 0 / highest) |
          oneside (prompt prefill on the cascade's side stream, not a second one)
"""

from __future__ import annotations

import argparse
import copy
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2510_14126_b200 import _lib  # noqa: E402
from paper_2510_14126_b200.runtime import PoolRuntime  # noqa: E402

VARIANTS = {
    "base": ({}, {}),
    "plo0": ({"FMHA_PLO": 0}, {}),
    "norope": ({}, {"fuse_qkv_rope": False}),
    "logits": ({}, {"full_logits": True}),
    "pdl0": ({"PDL": 0}, {}),
    "fmha1q": ({"FMHA_2Q": 0}, {}),
    "fmha2q": ({"FMHA_2Q": 1}, {}),
    "fmhaauto": ({"FMHA_2Q": -1}, {}),
    "python": ({}, {"native_layers": False}),
    "serial": ({}, {"overlap_cascade": False}),
    "slots1": ({}, {"cascade_slots": 1}),
    "slots3": ({}, {"cascade_slots": 3}),
    "ovh0": ({"GEMM_TILE_OVH": 0}, {}),    # 2-SM tile planner's per-tile overhead (32)
    "ovh16": ({"GEMM_TILE_OVH": 16}, {}),
    "ovh64": ({"GEMM_TILE_OVH": 64}, {}),
    "ovh96": ({"GEMM_TILE_OVH": 96}, {}),
    "ovh128": ({"GEMM_TILE_OVH": 128}, {}),
    "ovh192": ({"GEMM_TILE_OVH": 192}, {}),
    "ovh256": ({"GEMM_TILE_OVH": 256}, {}),
    "l2pf8": ({"GEMM_L2PF": 8}, {}),       # weight K blocks prefetched to L2 pre-PDL-wait
    "l2pf32": ({"GEMM_L2PF": 32}, {}),
    "skiss1": ({"SK_ISSUE": 1}, {}),       # split-K TMA issuing threads (2)
    "skiss4": ({"SK_ISSUE": 4}, {}),
    "slots4": ({}, {"cascade_slots": 4}),
    # side stream (cascade + prompt prefill) at high priority: its CTAs are dispatched
    # ahead of the context splits' as SMs free up
    "prio": ({}, {"side": lambda: torch.cuda.Stream(priority=-1)}),
    "prio0": ({}, {"side": lambda: torch.cuda.Stream(priority=0)}),
    "priomax": ({}, {"side": lambda: torch.cuda.Stream(priority=-100)}),
    "oneside": ({}, {"side2": None}),
    "cascade_lo": ({}, {"side": lambda: torch.cuda.Stream(priority=0)}),  # prefill high only
    "casc_top": ({}, {"side": lambda: torch.cuda.Stream(priority=-3)}),  # cascade above prefill
    "pf_top": ({}, {"side2": lambda: torch.cuda.Stream(priority=-3)}),   # prefill above cascade  # prompt prefill behind the cascade on one side stream
}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--record", type=int, default=60)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--workload", default="config2")
    ap.add_argument("--variants", default="base,plo0,norope,logits")
    ap.add_argument("--kernels", action="store_true",
                    help="also print per-kernel device time per step (PDL off), for all "
                         "recorded steps and for the decode-only ones")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    spec, _ = bench.workload(args.workload)
    params = bench.engine_params(spec, 256, 1)
    w = bench.build_worker("llama3-8b", spec, [[params, params]], torch.device("cuda", 0))
    rt = PoolRuntime(w, spec, params, concurrency=256, prefill_budget=4096 - 512)
    rt.fill()
    while rt.stats.completed + rt.stats.failed < 256:
        rt.step()
    rt.run_steps(20)
    plans = []
    inner = w.forward

    def rec(plan):
        plans.append(copy.deepcopy(plan))
        return inner(plan)

    w.forward = rec
    rt.run_steps(args.record)
    w.forward = inner
    torch.cuda.synchronize()
    toks = sum(p.n_tokens for p in plans)
    dec = sum(len(p.decode) for p in plans)
    names = args.variants.split(",")
    res = {n: [] for n in names}
    for _ in range(args.rounds):
        for n in names:
            knobs, attrs = VARIANTS[n]
            prev_k = {k: _lib.set_knob(k, v) for k, v in knobs.items()}
            prev_a = {k: getattr(w, k) for k in attrs}
            for k, v in attrs.items():
                setattr(w, k, v() if callable(v) else v)
            for p in plans[:3]:  # warm the variant
                w.forward(copy.deepcopy(p))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for p in plans:
                w.forward(copy.deepcopy(p))
            e1.record()
            torch.cuda.synchronize()
            res[n].append(e0.elapsed_time(e1) / len(plans))
            for k, v in prev_k.items():
                _lib.set_knob(k, v)
            for k, v in prev_a.items():
                setattr(w, k, v)
    out = {"steps": len(plans), "tokens_per_step": toks / len(plans),
           "decode_per_step": dec / len(plans),
           "ms_per_step": {n: sorted(v) for n, v in res.items()},
           "best_ms_per_step": {n: min(v) for n, v in res.items()}}
    print(json.dumps(out), flush=True)
    if args.kernels:
        dec_only = [p for p in plans if not p.prefill]
        for label, sel in (("all steps", plans), ("decode-only steps", dec_only)):
            if not sel:
                continue
            rows = kernel_table(w, sel)
            tot = sum(r[2] for r in rows)
            print(f"per-step kernel time, {label} ({len(sel)} steps, PDL off): {tot:.3f} ms "
                  f"(tokens/step {sum(p.n_tokens for p in sel) / len(sel):.0f})")
            for name, n, ms in rows[:24]:
                print(f"  {name[:64]:64s} {n:7.1f} launches {ms:8.3f} ms {100 * ms / tot:5.1f}%")


def kernel_table(w, plans, n_rep: int = 2) -> list:
    """Per-kernel device time (CUPTI) of replaying `plans` with PDL off (so a kernel's
    duration is its own execution, not its early launch waiting on the predecessor)."""
    from collections import defaultdict

    prev = _lib.set_knob("PDL", 0)
    try:
        for p in plans[:3]:
            w.forward(copy.deepcopy(p))
        torch.cuda.synchronize()
        acts = [torch.profiler.ProfilerActivity.CUDA]
        with torch.profiler.profile(activities=acts) as prof:
            for _ in range(n_rep):
                for p in plans:
                    w.forward(copy.deepcopy(p))
            torch.cuda.synchronize()
    finally:
        _lib.set_knob("PDL", prev)
    per = defaultdict(lambda: [0, 0.0])
    for ev in prof.events():
        if ev.device_type != torch.autograd.DeviceType.CUDA:
            continue
        name = ev.name.replace("void ", "").replace("(anonymous namespace)::", "").split("(")[0]
        per[name][0] += 1
        per[name][1] += (ev.time_range.end - ev.time_range.start) / 1e3
    steps = n_rep * len(plans)
    return sorted(((k, n / steps, ms / steps) for k, (n, ms) in per.items()), key=lambda r: -r[2])


if __name__ == "__main__":
    main()

