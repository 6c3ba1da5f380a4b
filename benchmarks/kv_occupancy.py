"""The paper's key quantity on the GPU engines: KV occupancy per stage pool, stage-isolated
vs a single shared pool (BASELINE config 3 semantics at one GPU).

Same seeded NL2SQL trace, same engine count (2), same closed-loop concurrency; the
isolated topology gives each LLM stage its own engine pool (one resident prefix per
engine), the shared topology lets both engines serve both stages (both prefixes end
up resident on each engine, stagesim/workloads.py:182-195). Occupancy is measured in
allocated KV blocks (16 tokens x 128 KiB for the Llama-3-8B shape), time-weighted over
the run as in stagesim/simulation.py:445-453, plus the peak.

Prints one JSON line per topology and a comparison line.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def run(mode: str, model: str, n_workflows: int, concurrency: int, max_batch: int,
        per_pool: int) -> dict:
    from paper_2510_14126_b200.config import MODELS
    from paper_2510_14126_b200.engine import EngineParams, blocks_for
    from paper_2510_14126_b200.model import GpuWorker
    from paper_2510_14126_b200.runtime import PoolRuntime

    cfg = MODELS[model]
    spec, _ = bench.workload("config2")
    P, p_hi, o_hi = 1000, 300, 150
    # engine capacity: both stage prefixes + max_batch full calls (a shared-pool engine
    # may hold both prefixes)
    cap = 2 * P + max_batch * (p_hi + o_hi)
    params = EngineParams(cap, 5000.0, 0.02, 0.1, max_batch)
    bpe = blocks_for(params)
    n_eng = 2 * per_pool
    worker = GpuWorker(cfg, "cuda", n_blocks=n_eng * bpe, n_rows=n_eng * (max_batch + 4),
                       row_cols=(P + p_hi + o_hi + 15) // 16 + 2, max_tokens=4096,
                       max_out=n_eng * max_batch + 64, hist_cols=o_hi + 8,
                       max_seq_tokens=P + p_hi + o_hi + 16)
    rt = PoolRuntime(worker, spec, params, mode=mode, engines_per_pool=(per_pool, per_pool),
                     concurrency=concurrency, n_workflows=n_workflows, prefill_budget=3584)
    rt.fill()
    samples = []
    t0 = time.perf_counter()
    while rt.workflows:
        rt.step()
        samples.append((time.perf_counter(), {e.engine_id: e.blocks_in_use for e in rt.engines},
                        {e.engine_id: e.resident_prefix_tokens() for e in rt.engines}))
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    kv = bench._kv_stats(rt, [(s[0], s[1]) for s in samples], cfg)
    total = [sum(s[1].values()) for s in samples]
    ts = [s[0] for s in samples]
    mean_total = sum(total[i] * (ts[i + 1] - ts[i]) for i in range(len(ts) - 1)) / (ts[-1] - ts[0])
    prefix_resident = max(sum(s[2].values()) for s in samples)
    cold = sum(e.cold_admits for e in rt.engines) if hasattr(rt.engines[0], "cold_admits") else None
    return {"topology": mode, "workflows": n_workflows, "engines": n_eng,
            "max_batch": max_batch, "prefix_prefills": cold, "completed": rt.stats.completed,
            "failed": rt.stats.failed, "wall_s": wall,
            "workflows_per_s": (rt.stats.completed + rt.stats.failed) / wall,
            "pools": kv, "total_peak_blocks": max(total), "total_mean_blocks": mean_total,
            "total_peak_gib": max(total) * cfg.kv_bytes_per_block / 2 ** 30,
            "total_mean_gib": mean_total * cfg.kv_bytes_per_block / 2 ** 30,
            "peak_resident_prefix_tokens": prefix_resident}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--workflows", type=int, default=512)
    ap.add_argument("--concurrency", type=int, default=256)
    ap.add_argument("--max-batch", type=int, default=256,
                    help="per-engine batch cap; below the concurrency, shared-pool calls "
                         "spill onto engines without their prefix")
    ap.add_argument("--engines-per-pool", type=int, default=1)
    args = ap.parse_args()
    res = {}
    for mode in ("isolated", "shared"):
        res[mode] = run(mode, args.model, args.workflows, args.concurrency, args.max_batch,
                        args.engines_per_pool)
        print(json.dumps(res[mode]), flush=True)
    iso, sh = res["isolated"], res["shared"]
    print(json.dumps({
        "comparison": f"isolated vs shared (config 3 semantics, 1 GPU, "
                      f"{2 * args.engines_per_pool} engines, max_batch {args.max_batch})",
        "prefix_prefills": {"isolated": iso["prefix_prefills"], "shared": sh["prefix_prefills"]},
        "resident_prefix_tokens": {"isolated": iso["peak_resident_prefix_tokens"],
                                   "shared": sh["peak_resident_prefix_tokens"]},
        "mean_kv_gib": {"isolated": iso["total_mean_gib"], "shared": sh["total_mean_gib"]},
        "peak_kv_gib": {"isolated": iso["total_peak_gib"], "shared": sh["total_peak_gib"]},
        "workflows_per_s": {"isolated": iso["workflows_per_s"], "shared": sh["workflows_per_s"]},
    }), flush=True)
