"""Is a config-2 step GPU-bound or host-bound?

Runs the bench runtime and splits the host wall time of each step into: time the
host spent blocked on a staging-ring slot, time inside GpuWorker.forward (Python +
launches; a launch also waits here when the GPU's launch queue is full, so with the GPU
behind, forward's time is the GPU's pace, not host work), and scheduler time (dispatch,
planning, completions). Then forward's host cost alone: 40 steps each started on a
drained GPU, with the layer loop in Python and in native code (csrc/step.cu).
"""

from __future__ import annotations

import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main(steps: int = 300) -> None:
    torch.cuda.set_device(0)
    from paper_2510_14126_b200.runtime import PoolRuntime

    spec, _ = bench.workload("config2")
    params = bench.engine_params(spec, 256, 1)
    worker = bench.build_worker("llama3-8b", spec, [[params, params]], torch.device("cuda", 0))
    rt = PoolRuntime(worker, spec, params, concurrency=256, prefill_budget=4096 - 512)
    cfg = worker.full_cfg
    w = rt.worker
    rt.fill()
    rt.run_steps(150)
    torch.cuda.synchronize()
    acc = {"blocked": 0.0, "forward": 0.0}
    evt_lists = [w.meta_evt, w.meta_evt_small]

    class TimedEvent:
        def __init__(self, e):
            self.e = e

        def synchronize(self):
            t = time.perf_counter()
            self.e.synchronize()
            acc["blocked"] += time.perf_counter() - t

        def query(self):
            return self.e.query()

    orig_fwd = w.forward

    def fwd(plan):
        t = time.perf_counter()
        r = orig_fwd(plan)
        acc["forward"] += time.perf_counter() - t
        return r

    w.forward = fwd
    t0 = time.perf_counter()
    for _ in range(steps):
        for evts in evt_lists:
            for i, e in enumerate(evts):
                if e is not None and not isinstance(e, TimedEvent):
                    evts[i] = TimedEvent(e)
        rt.step()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    out = {"steps": steps, "wall_ms_per_step": 1e3 * wall / steps,
           "blocked_ms_per_step": 1e3 * acc["blocked"] / steps,
           "forward_ms_per_step (incl. blocked)": 1e3 * acc["forward"] / steps,
           "scheduler_ms_per_step": 1e3 * (wall - acc["forward"]) / steps}
    # host submission cost alone: the GPU drained before every step, so no launch can
    # wait for queue space; forward's wall time is then pure host work (per the layer loop
    # in Python vs native csrc/step.cu)
    sub = {}
    for native in (True, False):
        w.native_layers = native
        acc["forward"] = 0.0
        for _ in range(40):
            torch.cuda.synchronize()
            rt.step()
        torch.cuda.synchronize()
        sub["native" if native else "python"] = 1e3 * acc["forward"] / 40
    w.native_layers = True
    out["host_forward_ms_gpu_idle"] = sub
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
