#!/usr/bin/env python
"""Benchmark: NL2SQL workflows/s and decode tok/s of GPU stage engines (BASELINE config 2).

Workload (BASELINE.json configs[1], the metric's configuration): Llama-3-8B-shaped
random-init bf16 decoder; isolated generator and fixer engine pools (at N=1 both
engines share the GPU: separate KV block pools and table rows, one weight copy);
256 concurrent workflows in a closed loop; NL2SQL trace from the reference's
seeded streams (seed 0, retry budget 5, prefix 1000, prompt U(100,300), output
U(50,150), executor U(0.1,0.4) s on host timers).

A step = one fused GPU forward of the runtime: every decoding call emits a token
and pending prompt/prefix prefill is packed in (chunked, <= 4096 tokens/step).
`value` = successful workflows per second over the K timed steps, on the device
clock (CUDA events on the engine stream), max over ranks. Inputs: every step's
token ids and metadata are uploaded from pinned host memory and every finished
call's tokens (its SQL) are read back — those bytes are `e2e`'s h2d/d2h, and
`e2e` is the same window on the host wall clock through the runtime's public
API (PoolRuntime.step).

N>1 (torchrun): one process per GPU, each an independent replica with the same
per-GPU load, workflows interleaved by rank (weak scaling, no data-path
collective).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "NL2SQL workflows/sec & decode tok/s at 1/2/4/8 B200; KV occupancy/stage; % HBM roofline"


def _peaks() -> tuple[dict, str]:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int) -> None:
        self.index = index
        self.rows: list[list[str]] = []
        self.proc = None
        self.thread = None

    def start(self) -> None:
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return

        def reader():
            for line in self.proc.stdout:
                self.rows.append([x.strip() for x in line.split(",")])

        self.thread = threading.Thread(target=reader, daemon=True)
        self.thread.start()

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait(timeout=5)
        self.thread.join(timeout=5)
        sm = [float(r[0]) for r in self.rows if len(r) >= 6 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 6 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 6 for i in range(4)
                          if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(sm)}


def workload(name: str):
    from paper_2510_14126_b200.workflow import Constant, Nl2Sql, Uniform

    if name == "config2":
        return Nl2Sql(retry_budget=5), "config2: NL2SQL isolated gen+fixer, prefix 1000, prompt " \
            "U(100,300), output U(50,150), budget 5, seed 0"
    if name == "config4":
        return Nl2Sql(retry_budget=5, generator_prefix_tokens=8192, fixer_prefix_tokens=8192,
                      output_tokens=Constant(512)), \
            "config4: NL2SQL isolated, 8K schema prefix, 512-token outputs, budget 5, seed 0"
    if name == "config5":
        return Nl2Sql(retry_budget=5, p_fail=0.6, p_syntax_err=0.3, p_empty_result=0.3), \
            "config5: NL2SQL isolated, heavy retry (p_fail 0.6 = 0.3 syntax + 0.3 empty), " \
            "budget 5, seed 0"
    raise ValueError(name)


def build_worker(model_name: str, spec, concurrency: int, device, role: str = "both",
                 max_tokens: int = 4096, tp_comm=None):
    """The GPU worker (weights, KV arena) sized for `concurrency` calls per engine."""
    from paper_2510_14126_b200.config import MODELS
    from paper_2510_14126_b200.engine import EngineParams, blocks_for
    from paper_2510_14126_b200.model import GpuWorker

    cfg = MODELS[model_name]
    P = max(spec.generator_prefix_tokens, spec.fixer_prefix_tokens)
    p_hi = int(spec.prompt_tokens.high)
    o_hi = int(getattr(spec.output_tokens, "high", getattr(spec.output_tokens, "value", 0)))
    max_seq = P + p_hi + o_hi
    # token capacity that always admits max_batch calls (prefix counted once per engine)
    cap = P + concurrency * (p_hi + o_hi)
    params = EngineParams(cap, 5000.0, 0.02, 0.1, concurrency)
    n_eng = 2 if role == "both" else 1
    bpe = blocks_for(params)
    worker = GpuWorker(cfg, device, n_blocks=n_eng * bpe, n_rows=n_eng * (concurrency + 4),
                       row_cols=(max_seq + 15) // 16 + 2, max_tokens=max_tokens,
                       max_out=2 * concurrency + 64, hist_cols=o_hi + 8,
                       max_seq_tokens=max_seq + 16, seed=0, tp=tp_comm)
    return worker, params


def build_runtime(model_name: str, wl_name: str, concurrency: int, device, rank: int, world: int,
                  max_tokens: int = 4096, role: str = "both", channel=None, tp_comm=None,
                  tp_ring=None):
    """rank / world: replica index and count. tp_comm + tp_ring: this rank leads a TP = 2
    replica (its worker is wrapped so the follower rank mirrors every device call)."""
    from paper_2510_14126_b200.runtime import PoolRuntime
    from paper_2510_14126_b200.tp import TpLeader

    spec, desc = workload(wl_name)
    worker, params = build_worker(model_name, spec, concurrency, device, role, max_tokens,
                                  tp_comm)
    cfg = worker.full_cfg
    if tp_ring is not None:
        worker = TpLeader(worker, tp_ring)
    if role == "both":  # replicas: workflows interleaved by rank
        rid_offset, rid_stride = rank, world
    else:  # disjoint pairs: workflows interleaved by pair
        rid_offset, rid_stride = rank % (world // 2), world // 2
    rt = PoolRuntime(worker, spec, params, mode="isolated", concurrency=concurrency, seed=0,
                     rid_offset=rid_offset, rid_stride=rid_stride,
                     prefill_budget=max_tokens - 512, role=role, channel=channel)
    return rt, cfg, desc


def run_cpu_baseline(model_name: str) -> dict:
    from oracle.cpu_baseline import measure
    from paper_2510_14126_b200.config import MODELS

    return measure(MODELS[model_name])


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1500)
    ap.add_argument("--warmup", type=int, default=400)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--workload", default="config2")
    ap.add_argument("--concurrency", type=int, default=256)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-steps", type=int, default=40)
    ap.add_argument("--roofline-window", default="timed", choices=["timed", "after"],
                    help="where the dominant kernel's CUDA events are recorded: inside the "
                         "timed steps, or in --profile-steps identical steps right after them")
    ap.add_argument("--placement", default="disjoint", choices=["disjoint", "replicas"],
                    help="N>1: generator and fixer pools on disjoint GPUs (pairs), or "
                         "both pools on every GPU")
    ap.add_argument("--tp", type=int, default=1, choices=[1, 2],
                    help="tensor-parallel size of each engine replica (config 5: 2); "
                         "replicas are rank pairs (2i, 2i+1), placement applies to replicas")
    args = ap.parse_args()
    if os.environ.get("CORTEX_DUMP_AFTER"):  # debugging stuck runs: periodic stack dumps
        import faulthandler

        faulthandler.dump_traceback_later(float(os.environ["CORTEX_DUMP_AFTER"]), repeat=True)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    spec, desc = workload(args.workload)

    if args.impl == "reference":
        if rank != 0:
            return
        cb = run_cpu_baseline(args.model)
        line = {
            "metric": METRIC, "impl": "reference", "value": cb["workflows_per_s"],
            "unit": "workflows/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": desc, "model": args.model + "-shape",
                       "concurrency": args.concurrency},
            "decode_tok_s": cb["decode_tok_s"],
            "cpu_baseline": {"value": cb["workflows_per_s"], "unit": "workflows/s",
                             "cores": cb["cores"], "kind": "port", "sample": cb["sample"]},
            "e2e": {"value": cb["workflows_per_s"], "unit": "workflows/s",
                    "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)
        return

    dist = None
    # CORTEX_DIST_BACKEND=gloo: functional runs with more ranks than GPUs (ranks share a
    # device; the handoff is host-only, so no kernel waits on another rank)
    backend = os.environ.get("CORTEX_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local %= torch.cuda.device_count()
        # ranks time-sliced on a shared GPU: programmatic dependent launch off (with it,
        # 2 of 6 disjoint N = 2 runs on one GPU hung; without it 6 of 6 completed,
        # DESIGN.md §6.1); one process per GPU keeps it on
        os.environ.setdefault("CORTEX_PDL", "0")
    comm_dev = torch.device("cuda", local) if backend == "nccl" else torch.device("cpu")
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)

    from paper_2510_14126_b200.model import KernelProfile
    from paper_2510_14126_b200.placement import ROLE_BOTH, ROLE_FIXER, open_pair_channel, role_of

    # TP = 2: ranks (2i, 2i+1) form replica i; rank 2i leads (runs the runtime), 2i+1 follows
    tp = args.tp
    if world % tp:
        raise SystemExit("--tp must divide the number of ranks")
    rrank, rworld, tp_rank = rank // tp, world // tp, rank % tp
    role, pair, _ = (role_of(rrank, rworld) if args.placement == "disjoint"
                     else (ROLE_BOTH, rrank, -1))
    # per-GPU load is fixed as N grows: a disjoint pair (2 GPUs) carries 2x the workflows
    conc = args.concurrency * (2 if role != ROLE_BOTH else 1)
    channel = (open_pair_channel(dist, rrank, rworld, cap=2 * conc + 64, member=tp_rank == 0)
               if role != ROLE_BOTH else None)
    tp_comm = tp_ring = None
    if tp > 1:
        from paper_2510_14126_b200.config import MODELS
        from paper_2510_14126_b200.tp import TpComm, open_replica_ring

        groups = [dist.new_group([tp * i + j for j in range(tp)]) for i in range(rworld)]
        tp_comm = TpComm(device, tp_rank, tp, 4096, MODELS[args.model].d_model)
        tp_comm.connect_ipc(groups[rrank])
        tp_ring = open_replica_ring(dist, rrank, tp_rank)
        if os.environ.get("CORTEX_TP_HOST_SYNC") == "1":
            # functional runs with a replica's two ranks on ONE GPU (gloo): every exchange
            # waits on the host until both ranks' partials exist (no cross-rank spinning)
            def host_sync(g=groups[rrank]):
                torch.cuda.synchronize()
                dist.barrier(group=g)
            tp_sync = host_sync
        else:
            tp_sync = None
        if tp_rank:
            _follow(args, device, role, conc, tp_comm, tp_ring, dist, comm_dev, tp_sync)
            return
    rt, cfg, desc = build_runtime(args.model, args.workload, conc, device, rrank, rworld,
                                  role=role, channel=channel, tp_comm=tp_comm, tp_ring=tp_ring)
    w = rt.worker
    if tp > 1:
        w.tp_sync = tp_sync

    def coll_barrier() -> None:
        if tp_ring is not None:
            w.collective("barrier")
        dist.barrier()

    def coll_all_reduce(t, op) -> None:
        if tp_ring is not None:
            w.collective("all_reduce", t.numel(), str(t.dtype), op)
        dist.all_reduce(t, op=op)

    rt.fill()

    def run_phase(n_steps: int, phase: int) -> None:
        """The generator side (or a replica) runs n_steps; a fixer rank serves its
        pair until the generator moves the channel past `phase`."""
        if role == ROLE_FIXER:
            while channel.phase == phase:
                rt.step()
        else:
            rt.run_steps(n_steps)
            if channel is not None:
                channel.phase = phase + 1

    run_phase(max(3, args.warmup), 0)
    if dist is not None:
        coll_barrier()

    # kernel-class shares (untimed) -> the dominant kernel for the roofline
    # attn_decode_ctx (the per-call context splits alone, nested in attn_decode) is the
    # HBM-bound decode-attention kernel the north star's >= 70 % target is about
    w.prof = KernelProfile(["gemm", "attn_decode", "attn_prefill", "attn_decode_ctx"])
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    run_phase(args.profile_steps, 1)
    e1.record()
    shares = w.prof.summary()
    prof_ms = e0.elapsed_time(e1)
    w.prof = None
    dominant = max((k for k in shares if k != "attn_decode_ctx"),
                   key=lambda k: shares[k]["ms"], default="gemm")

    # ---------------- timed region ----------------
    peaks, peak_src = _peaks()
    # roofline events either inside the timed steps or in a window right after them
    # (inside the timed steps only every 8th step is instrumented: ~0.7% event overhead)
    w.prof = KernelProfile([dominant], every=8) if args.roofline_window == "timed" else None
    clocks = ClockSampler(local)
    if dist is not None:
        coll_barrier()
    torch.cuda.synchronize()
    s0 = (rt.stats.completed, rt.stats.failed, rt.stats.decode_tokens, rt.stats.prefill_tokens,
          rt.stats.steps, w.launches, w.h2d_bytes, rt.stats.d2h_bytes)
    kv0 = _kv_snapshot(rt)
    clocks.start()
    t_wall0 = time.perf_counter()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    kv_samples = []
    if role == ROLE_FIXER:
        while channel.phase == 2:
            rt.step()
            kv_samples.append(_kv_snapshot(rt))
    else:
        for _ in range(args.steps):
            rt.step()
            kv_samples.append(_kv_snapshot(rt))
        if channel is not None:
            channel.phase = 3
    ev1.record()
    torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall0
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    if dist is not None:
        t = torch.tensor([ms, t_wall * 1e3], device=comm_dev)
        coll_all_reduce(t, dist.ReduceOp.MAX)
        ms, t_wall = float(t[0]), float(t[1]) / 1e3
    s1 = (rt.stats.completed, rt.stats.failed, rt.stats.decode_tokens, rt.stats.prefill_tokens,
          rt.stats.steps, w.launches, w.h2d_bytes, rt.stats.d2h_bytes)
    d = [b - a for a, b in zip(s0, s1)]
    completed, failed, dec_tok, pf_tok, steps, launches, h2d, d2h = d
    if dist is not None:
        t = torch.tensor([completed, failed, dec_tok, pf_tok], device=comm_dev,
                         dtype=torch.float64)
        coll_all_reduce(t, dist.ReduceOp.SUM)
        completed, failed, dec_tok, pf_tok = [float(x) for x in t]
    if args.roofline_window != "timed":
        w.prof = KernelProfile([dominant])
        run_phase(args.profile_steps, 3)
    kshare = w.prof.summary().get(dominant, {"launches": 0, "ms": 0.0, "bytes": 0.0, "flops": 0.0})
    w.prof = None
    secs = ms / 1e3
    value = completed / secs
    e2e_value = completed / t_wall

    # roofline of the dominant kernel (algorithmic bytes or flops per launch / avg duration)
    if dominant == "gemm" and shares.get("gemm") and \
            shares["gemm"]["flops"] / max(shares["gemm"]["bytes"], 1) > 200:
        bound, unit, peak = "tensor", "TFLOP/s", peaks["bf16_tflops_sustained"]
        per_launch = kshare["flops"] / max(kshare["launches"], 1)
        achieved = kshare["flops"] / max(kshare["ms"] / 1e3, 1e-12) / 1e12
    else:
        bound, unit, peak = "hbm", "GB/s", peaks["hbm_gbs"]
        per_launch = kshare["bytes"] / max(kshare["launches"], 1)
        achieved = kshare["bytes"] / max(kshare["ms"] / 1e3, 1e-12) / 1e9
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):  # DRAM bytes per launch of this class from the committed ncu list
        with open(tpath) as f:
            tj = json.load(f)
        if dominant in tj.get("classes", {}):
            traffic = tj["classes"][dominant]["dram_bytes_per_launch"]
            traffic_src = tj.get("source")
    roofline = {"kernel": dominant, "bound": bound, "achieved": achieved, "peak": peak,
                "unit": unit, "frac": achieved / peak, "traffic": traffic,
                "traffic_source": traffic_src,
                "algorithmic_bytes_per_launch": kshare["bytes"] / max(kshare["launches"], 1),
                "per_launch_algorithmic": per_launch, "avg_launch_ms": kshare["ms"] / max(
                    kshare["launches"], 1), "launches": kshare["launches"],
                "peak_source": peak_src + (" sustained" if bound == "tensor" else "")}

    # every kernel class of the (untimed) profile window against both roofs; the
    # attention window covers the side-stream tensor-core passes (cascade prefix +
    # prompt prefill) overlapped with the HBM-bound per-call decode splits
    rooflines = {}
    for k, v in shares.items():
        sec = max(v["ms"], 1e-9) / 1e3
        gbs, tfs = v["bytes"] / sec / 1e9, v["flops"] / sec / 1e12
        rooflines[k] = {"ms": v["ms"], "launches": v["launches"],
                        "hbm_gbs": gbs, "hbm_frac": gbs / peaks["hbm_gbs"],
                        "tflops": tfs, "tensor_frac": tfs / peaks["bf16_tflops_sustained"],
                        "bytes_per_launch": v["bytes"] / max(v["launches"], 1),
                        "flops_per_launch": v["flops"] / max(v["launches"], 1)}

    kv = _kv_stats(rt, kv_samples, cfg)
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "workflows/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms / max(steps, 1),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic: seeded NL2SQL trace (reference counter streams), random-init weights",
        "config": {"workload": desc, "model": cfg.name + "-shape", "concurrency": args.concurrency,
                   "engines": ("isolated: 1 generator + 1 fixer engine per replica"
                               if role == ROLE_BOTH
                               else f"isolated, disjoint placement: replicas 0..{rworld // 2 - 1} "
                                    f"generator pool, {rworld // 2}..{rworld - 1} fixer pool; "
                                    f"{rworld // 2} pair(s) of {conc} workflows (host handoff)")
                   + (f"; {rworld} replica(s) of TP=2 (GPU pairs, fused NVLink all-reduce)"
                      if tp > 1 else ""),
                   "l2": "inputs larger than L2 (16 GB of weights + KV streamed every step)"},
        "decode_tok_s": dec_tok / secs,
        "prefill_tok_s": pf_tok / secs,
        "workflows_finished_per_s": (completed + failed) / secs,
        "kv_occupancy": kv,
        "kernel_shares": {k: {"ms": v["ms"], "share": v["ms"] / prof_ms, "launches": v["launches"]}
                          for k, v in shares.items()},
        "roofline": roofline,
        "rooflines_by_class": rooflines,
        "clocks": clk,
        "e2e": {"value": e2e_value, "unit": "workflows/s", "h2d_bytes_per_step": h2d / steps,
                "d2h_bytes_per_step": d2h / steps},
        "gpu_launches": launches,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = run_cpu_baseline(args.model)
        line["cpu_baseline"] = {"value": cb["workflows_per_s"], "unit": "workflows/s",
                                "cores": cb["cores"], "kind": "port", "sample": cb["sample"],
                                "decode_tok_s": cb["decode_tok_s"]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        if tp_ring is not None:
            w.stop()
        dist.barrier()
        if channel is not None:
            channel.close()
        if tp_ring is not None:
            tp_ring.close()
        dist.destroy_process_group()


def _follow(args, device, role, conc, tp_comm, tp_ring, dist, comm_dev, tp_sync=None) -> None:
    """TP follower rank: build the other half of the replica's worker and replay the
    leader's device calls until it stops; join the leader's collectives with zeros."""
    from paper_2510_14126_b200.tp import TpFollower

    spec, _ = workload(args.workload)
    worker, _ = build_worker(args.model, spec, conc, device, role, tp_comm=tp_comm)
    worker.tp_sync = tp_sync

    def on_collective(kind, a) -> None:
        if kind == "barrier":
            dist.barrier()
        elif kind == "all_reduce":
            n, dtype, op = a
            dist.all_reduce(torch.zeros(n, dtype=getattr(torch, dtype.split(".")[-1]),
                                        device=comm_dev), op=op)
        else:
            raise ValueError(kind)

    TpFollower(worker, tp_ring, on_collective=on_collective).serve()
    torch.cuda.synchronize()
    if int(tp_comm.status[0]) or int(worker.status[0]):
        raise SystemExit("TP follower: device status error")
    dist.barrier()
    tp_ring.close()
    dist.destroy_process_group()



def _kv_snapshot(rt):
    return (time.perf_counter(), {e.engine_id: e.blocks_in_use for e in rt.engines})


def _kv_stats(rt, samples, cfg) -> dict:
    """Peak and time-weighted mean KV blocks per pool (the paper's key quantity)."""
    out = {}
    pools = {p: [e.engine_id for e in es] for p, es in rt.pool_engines.items()}
    for pool, eids in pools.items():
        vals = [sum(s[1][e] for e in eids) for s in samples]
        ts = [s[0] for s in samples]
        if len(vals) < 2:
            continue
        integ = sum(vals[i] * (ts[i + 1] - ts[i]) for i in range(len(vals) - 1))
        mean = integ / (ts[-1] - ts[0])
        out[pool] = {"peak_blocks": max(vals), "mean_blocks": mean,
                     "peak_gib": max(vals) * cfg.kv_bytes_per_block / 2 ** 30,
                     "mean_gib": mean * cfg.kv_bytes_per_block / 2 ** 30}
    return out


if __name__ == "__main__":
    main()
