"""Live kernel timeline of config-2 steps (torch.profiler / CUPTI, real clocks, warm caches).

Complements the ncu launch list (serialised, cold-cache): per kernel name the
count and total busy time inside `--steps` runtime steps, the GPU-busy union of
all kernel intervals (streams overlap: decode splits || cascade / prefill
attention), and the idle time between kernels — launch gaps a CUDA graph or
programmatic dependent launch could recover.

    python benchmarks/step_trace.py [--steps 20] [--json out.json]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from collections import defaultdict

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=400)
    ap.add_argument("--workload", default="config2")
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    from paper_2510_14126_b200.runtime import PoolRuntime

    spec, _ = bench.workload(args.workload)
    params = bench.engine_params(spec, 256, 1)
    worker = bench.build_worker("llama3-8b", spec, [[params, params]], torch.device("cuda", 0))
    rt = PoolRuntime(worker, spec, params, concurrency=256, prefill_budget=4096 - 512)
    rt.fill()
    while rt.stats.completed + rt.stats.failed < 256:  # the bench's ramp
        rt.step()
    rt.run_steps(args.warmup)
    torch.cuda.synchronize()
    # tokens per step (decode + prefill) and the GEMM M it implies
    sizes = []
    inner = rt.worker.forward

    step_ev = []

    def fwd(plan):
        sizes.append((len(plan.decode), plan.n_tokens - len(plan.decode)))
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        n = inner(plan)
        b.record()
        step_ev.append((a, b))
        return n

    rt.worker.forward = fwd
    acts = [torch.profiler.ProfilerActivity.CUDA]
    with torch.profiler.profile(activities=acts) as prof:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        rt.run_steps(args.steps)
        e1.record()
        torch.cuda.synchronize()
    span_ms = e0.elapsed_time(e1)
    ivs = []
    per = defaultdict(lambda: [0, 0.0])
    for ev in prof.events():
        if ev.device_type != torch.autograd.DeviceType.CUDA:
            continue
        name = ev.name
        if name.startswith("Memcpy") or name.startswith("Memset"):
            cls = name.split()[0]
        else:
            cls = name.replace("void ", "").replace("(anonymous namespace)::", "").split("(")[0]
        t0 = ev.time_range.start
        t1 = ev.time_range.end
        ivs.append((t0, t1))
        per[cls][0] += 1
        per[cls][1] += (t1 - t0) / 1e3
    # gaps on the GPU timeline (all streams merged): idle time before each kernel class
    evs = sorted((ev.time_range.start, ev.time_range.end,
                  ev.name.replace("void ", "").replace("(anonymous namespace)::", "").split("(")[0]
                  .split("<")[0])
                 for ev in prof.events() if ev.device_type == torch.autograd.DeviceType.CUDA)
    gaps = defaultdict(lambda: [0, 0.0])
    end = evs[0][1]
    prev = evs[0][2]
    for a, b, nm in evs[1:]:
        if a > end:
            key = f"{prev} -> {nm}"
            gaps[key][0] += 1
            gaps[key][1] += (a - end) / 1e3
        if b > end:
            end, prev = b, nm
    print("largest idle gap classes (count, total ms):")
    for k, (n, ms) in sorted(gaps.items(), key=lambda kv: -kv[1][1])[:14]:
        print(f"  {k[:90]:90s} {n:6d} {ms:8.3f} ms  avg {1e3 * ms / n:6.2f} us")
    ivs.sort()
    busy = 0.0
    cur0, cur1 = ivs[0]
    for a, b in ivs[1:]:
        if a > cur1:
            busy += cur1 - cur0
            cur0, cur1 = a, b
        else:
            cur1 = max(cur1, b)
    busy += cur1 - cur0
    busy_ms = busy / 1e3
    total_ms = (ivs[-1][1] - ivs[0][0]) / 1e3
    rows = sorted(per.items(), key=lambda kv: -kv[1][1])
    import numpy as np

    tt = np.array([a + b for a, b in sizes])
    print(f"tokens/step: mean {tt.mean():.0f} min {tt.min()} max {tt.max()}; decode mean "
          f"{np.mean([a for a, _ in sizes]):.0f}; steps with prefill "
          f"{sum(1 for _, b in sizes if b)}/{len(sizes)}; T = {tt.tolist()}")
    st = [a.elapsed_time(b) for a, b in step_ev]
    print("per-step forward ms by T:", sorted(zip(tt.tolist(), [round(x, 3) for x in st])))
    out = {"steps": args.steps, "tokens_per_step": tt.tolist(), "forward_ms": st, "event_span_ms": span_ms, "kernel_span_ms": total_ms,
           "gpu_busy_ms": busy_ms, "idle_ms": total_ms - busy_ms,
           "per_step_ms": span_ms / args.steps,
           "kernels": [{"name": k, "launches": n, "ms": ms, "ms_per_step": ms / args.steps,
                        "share_of_busy": ms / busy_ms} for k, (n, ms) in rows]}
    print(f"span {span_ms:.2f} ms for {args.steps} steps ({span_ms / args.steps:.3f} ms/step); "
          f"GPU busy {busy_ms:.2f} ms, idle {total_ms - busy_ms:.2f} ms")
    for k, (n, ms) in rows[:30]:
        print(f"{k[:60]:60s} {n:6d} {ms:9.3f} ms  {ms / args.steps:7.3f} ms/step  "
              f"{ms / busy_ms:6.3f}")
    if args.json:
        with open(args.json, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
