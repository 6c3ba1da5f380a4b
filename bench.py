#!/usr/bin/env python
"""Benchmark: NL2SQL workflows/s and decode tok/s of GPU stage engines (BASELINE configs 2-5).

Workload (BASELINE.json configs[1], the metric's configuration, at N = 1): Llama-3-8B-
shaped random-init bf16 decoder; isolated generator and fixer engine pools (at N = 1 both
engines share the GPU: separate KV block pools and table rows, one weight copy); 256
concurrent workflows per GPU in a closed loop; NL2SQL trace from the reference's seeded
streams (seed 0, retry budget 5, prefix 1000, prompt U(100,300), output U(50,150),
executor U(0.1,0.4) s on host timers). `--workload config4 / config5` select the
8K-prefix and heavy-retry traces, `--mode shared` one pool serving both stages.

A step = one scheduling round + one fused GPU forward of every engine on the GPU: each
decoding call emits a token and pending prompt / prefix prefill is packed in (chunked,
<= 4096 tokens per step). Before the timed window the closed loop is RAMPED (untimed,
`ramp_steps`) until as many workflows as the concurrency have finished and every pool
holds calls, whatever --warmup says, then --warmup steps run, then exactly --steps steps are timed.
`value` = successful workflows per second over the timed steps, on the device clock
(CUDA events on the engine stream), max over ranks. `e2e` = the same window on the host
wall clock through the runtime's public API (PoolRuntime.step), which uploads every
step's token ids / metadata from pinned host memory and reads every finished call's
generated tokens (its SQL) back to the host (h2d / d2h bytes per step).

After the timed window the other topology (shared pool when the timed one is isolated)
runs on the same GPUs for its KV occupancy (`kv_occupancy_<mode>`): the paper's key
quantity, per pool, next to the timed arm's `kv_occupancy`.

N > 1 (torchrun): one process per GPU (a replica; with --tp 2, a GPU pair led by its even
rank). The generator pool and the fixer pool sit on disjoint replica sets (--split g:f,
default even), or one shared pool spans every replica (--mode shared); replica 0 runs the
scheduler and routes every call over all engines of its pool (cluster.py). Concurrency is
256 workflows per GPU (weak scaling). No data-path collective.
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
import torch.distributed as tdist

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "NL2SQL workflows/sec & decode tok/s at 1/2/4/8 B200; KV occupancy/stage; % HBM roofline"
PHASE_WARM, PHASE_TIMED, PHASE_AFTER = 0, 1, 2


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
                 "--format=csv,noheader,nounits", "-lms", "100"],
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
    from paper_2510_14126_b200.workflow import Constant, Nl2Sql

    if name == "config2":
        return Nl2Sql(retry_budget=5), "config2: NL2SQL gen+fixer, prefix 1000, prompt " \
            "U(100,300), output U(50,150), budget 5, seed 0"
    if name == "config4":
        return Nl2Sql(retry_budget=5, generator_prefix_tokens=8192, fixer_prefix_tokens=8192,
                      output_tokens=Constant(512)), \
            "config4: NL2SQL, 8K schema prefix, 512-token outputs, budget 5, seed 0"
    if name == "config5":
        return Nl2Sql(retry_budget=5, p_fail=0.6, p_syntax_err=0.3, p_empty_result=0.3), \
            "config5: NL2SQL, heavy retry (p_fail 0.6 = 0.3 syntax + 0.3 empty), budget 5, seed 0"
    raise ValueError(name)


def _maxes(spec) -> tuple[int, int, int]:
    P = max(spec.generator_prefix_tokens, spec.fixer_prefix_tokens)
    p_hi = int(spec.prompt_tokens.high)
    o_hi = int(getattr(spec.output_tokens, "high", getattr(spec.output_tokens, "value", 0)))
    return P, p_hi, o_hi


def engine_params(spec, max_batch: int, n_prefixes: int):
    """Engine constants: a token capacity that always admits max_batch full calls (the
    resident stage prefixes counted once each), so the batch cap binds, not the KV."""
    from paper_2510_14126_b200.engine import EngineParams

    P, p_hi, o_hi = _maxes(spec)
    return EngineParams(n_prefixes * P + max_batch * (p_hi + o_hi), 5000.0, 0.02, 0.1, max_batch)


def build_worker(model_name: str, spec, params_list, device, max_tokens: int = 4096,
                 tp_comm=None):
    """The GPU worker (weights, KV arena) for the engines of one replica; the arena is
    sized for the largest engine set in `params_list` (one list per topology arm)."""
    from paper_2510_14126_b200.config import MODELS
    from paper_2510_14126_b200.engine import blocks_for
    from paper_2510_14126_b200.model import GpuWorker

    cfg = MODELS[model_name]
    P, p_hi, o_hi = _maxes(spec)
    max_seq = P + p_hi + o_hi
    n_blocks = max(sum(blocks_for(p) for p in pl) for pl in params_list)
    n_rows = max(sum(p.max_batch + 4 for p in pl) for pl in params_list)
    max_out = max(sum(p.max_batch for p in pl) for pl in params_list) + 64
    return GpuWorker(cfg, device, n_blocks=n_blocks, n_rows=n_rows,
                     row_cols=(max_seq + 15) // 16 + 2, max_tokens=max_tokens, max_out=max_out,
                     hist_cols=o_hi + 8, max_seq_tokens=max_seq + 16, seed=0, tp=tp_comm)


def run_cpu_baseline(model_name: str, spec) -> dict:
    from oracle.cpu_baseline import measure
    from paper_2510_14126_b200.config import MODELS

    return measure(MODELS[model_name], spec)


class Arm:
    """One topology on this process: the scheduler + its local engines (replica 0) or
    the replica server (others), plus the links between them."""

    def __init__(self, args, mode, spec, worker, n_rep, replica, tp_rank, dist, conc_total,
                 max_batch):
        from paper_2510_14126_b200.cluster import open_links, parse_split, plan_engines
        from paper_2510_14126_b200.runtime import PoolRuntime, ReplicaExecutor, ReplicaServer

        self.mode = mode
        split = parse_split(args.split, n_rep) if mode == "isolated" else None
        self.specs = plan_engines(mode, n_rep, split)
        mine = [s for s in self.specs if s.replica == replica]
        self.params = engine_params(spec, max_batch, 2 if mode == "shared" else 1)
        self.links = None
        if n_rep > 1:
            self.links = open_links(dist, replica, n_rep, self.specs, cap=4 * conc_total + 64,
                                    member=tp_rank == 0)
        self.rt = self.server = None
        self.stats = None
        if tp_rank != 0:
            return
        if replica == 0:
            self.rt = PoolRuntime(worker, spec, self.params, mode=mode, concurrency=conc_total,
                                  seed=0, prefill_budget=worker.max_tokens - 512,
                                  engines=self.specs, links=self.links)
            self.stats = self.rt.stats
        else:
            ex = ReplicaExecutor(worker, self.params, mine, seed=0,
                                 prefill_budget=worker.max_tokens - 512,
                                 result_rows=2 * max_batch * max(len(mine), 1))
            self.server = ReplicaServer(ex, self.links)
            self.stats = ex.stats

    def set_phase(self, phase: int) -> None:
        if self.rt is not None and self.links:
            for link in self.links.values():
                link.phase = phase

    def close(self) -> None:
        if self.links is None:
            return
        if isinstance(self.links, dict):
            for link in self.links.values():
                link.close()
        else:
            self.links.close()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1500)
    ap.add_argument("--warmup", type=int, default=400)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--workload", default="config2")
    ap.add_argument("--concurrency", type=int, default=256, help="workflows per GPU")
    ap.add_argument("--mode", default="isolated", choices=["isolated", "shared"],
                    help="stage-isolated pools (the paper's design) or one shared pool")
    ap.add_argument("--split", default=None,
                    help="N > 1 isolated: generator:fixer replicas, e.g. 2:6 (default even)")
    ap.add_argument("--no-shared-arm", action="store_true",
                    help="skip the other-topology KV-occupancy arm after the timed window")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-steps", type=int, default=40)
    ap.add_argument("--tp", type=int, default=1, choices=[1, 2],
                    help="tensor-parallel size of each engine replica (config 5: 2); replicas "
                         "are rank pairs (2i, 2i+1)")
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
        cb = run_cpu_baseline(args.model, spec)
        line = {
            "metric": METRIC, "impl": "reference", "value": cb["workflows_per_s"],
            "unit": "workflows/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": desc, "model": args.model + "-shape",
                       "concurrency": args.concurrency, "topology": args.mode},
            "decode_tok_s": cb["decode_tok_s"],
            "cpu_baseline": {"value": cb["workflows_per_s"], "unit": "workflows/s",
                             "cores": cb["cores"], "kind": cb["kind"], "sample": cb["sample"],
                             "cpu_model": cb["cpu_model"], "control_path": cb["control_path"]},
            "e2e": {"value": cb["workflows_per_s"], "unit": "workflows/s",
                    "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)
        return

    dist = None
    # one process per GPU over NCCL; with fewer GPUs than ranks (a functional check of the
    # multi-replica path on a 1-GPU box) the ranks share devices over gloo, with
    # programmatic dependent launch off (ranks time-sliced on one GPU)
    shared = world > torch.cuda.device_count()
    if shared:
        local %= torch.cuda.device_count()
        from paper_2510_14126_b200 import _lib

        _lib.set_knob("PDL", 0)
    if world > 1:
        dist = tdist
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    red_dev = torch.device("cpu") if shared else device  # where the reductions run

    from paper_2510_14126_b200.cluster import parse_split, plan_engines

    tp = args.tp
    if world % tp:
        raise SystemExit("--tp must divide the number of ranks")

    replica, n_rep, tp_rank = rank // tp, world // tp, rank % tp
    # weak scaling: 256 workflows per GPU; an engine's batch cap admits the whole closed
    # loop of its GPU at N = 1 (two engines share it) and twice that alone on a replica
    conc_total = args.concurrency * world
    max_batch = args.concurrency if n_rep == 1 else 2 * args.concurrency * tp
    other = "shared" if args.mode == "isolated" else "isolated"
    arms = [args.mode] + ([] if args.no_shared_arm else [other])

    def arm_params(mode):
        split = parse_split(args.split, n_rep) if mode == "isolated" else None
        n_mine = sum(1 for s in plan_engines(mode, n_rep, split) if s.replica == replica)
        return [engine_params(spec, max_batch, 2 if mode == "shared" else 1)] * max(n_mine, 1)

    tp_comm = tp_ring = None
    if tp > 1:
        from paper_2510_14126_b200.config import MODELS
        from paper_2510_14126_b200.tp import TpComm, open_replica_ring

        groups = [dist.new_group([tp * i + j for j in range(tp)]) for i in range(n_rep)]
        tp_comm = TpComm(device, tp_rank, tp, 4096, MODELS[args.model].d_model)
        tp_comm.connect_ipc(groups[replica])
        tp_ring = open_replica_ring(dist, replica, tp_rank)
    worker = build_worker(args.model, spec, [arm_params(m) for m in arms], device,
                          tp_comm=tp_comm)
    if tp > 1 and shared:
        # functional TP runs with a replica's two ranks on ONE GPU: every exchange point
        # waits on the host until both ranks' partials exist (no kernel spins on a rank
        # that is time-sliced out)
        def tp_sync(g=groups[replica]):
            torch.cuda.synchronize()
            dist.barrier(group=g)

        worker.tp_sync = tp_sync
    cfg = worker.full_cfg
    if tp_rank:
        _follow(worker, tp_ring, dist, red_dev, tp_comm, arms, args, spec, n_rep, replica,
                tp_rank, conc_total, max_batch)
        return
    if tp_ring is not None:
        from paper_2510_14126_b200.tp import TpLeader

        worker = TpLeader(worker, tp_ring)

    def barrier() -> None:
        if dist is None:
            return
        if tp_ring is not None:
            worker.collective("barrier")
        dist.barrier()

    def all_reduce(t, op) -> None:
        if dist is None:
            return
        if tp_ring is not None:
            worker.collective("all_reduce", t.numel(), str(t.dtype), op)
        dist.all_reduce(t, op=op)

    line = None
    for ai, mode in enumerate(arms):
        if tp_ring is not None:
            worker.collective("arm")  # the follower joins the arm's link set-up collectives
        arm = Arm(args, mode, spec, worker, n_rep, replica, tp_rank, dist, conc_total,
                  max_batch)
        res = run_arm(args, arm, worker, cfg, desc, barrier, all_reduce, red_dev, local, n_rep,
                      world, timed=ai == 0)
        arm.close()
        if ai == 0:
            line = res
        elif line is not None:
            line["kv_occupancy_" + mode] = res
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = run_cpu_baseline(args.model, spec)
        line["cpu_baseline"] = {"value": cb["workflows_per_s"], "unit": "workflows/s",
                                "cores": cb["cores"], "kind": cb["kind"],
                                "sample": cb["sample"], "cpu_model": cb["cpu_model"],
                                "control_path": cb["control_path"],
                                "decode_tok_s": cb["decode_tok_s"]}
    if rank == 0:
        if shared:
            line["config"]["functional_only"] = (
                f"{world} ranks on {torch.cuda.device_count()} GPU(s) over gloo: not a measurement")
        print(json.dumps(line), flush=True)
    if dist is not None:
        if tp_ring is not None:
            worker.stop()
        dist.barrier()
        if tp_ring is not None:
            tp_ring.close()
        dist.destroy_process_group()


def run_arm(args, arm, worker, cfg, desc, barrier, all_reduce, device, local, n_rep, world,
            timed: bool):
    """Ramp, warm up and time one topology arm. The timed arm returns the bench line
    (on replica 0); the secondary arm its KV occupancy (a window of >= 200 steps)."""
    from paper_2510_14126_b200.model import KernelProfile

    rt, srv = arm.rt, arm.server
    steps = args.steps if timed else max(args.steps, 200)

    def serve(phase):
        if srv is not None:
            srv.serve_while(phase)

    # ---- ramp (untimed) to the closed loop's steady state, whatever --warmup says: the
    # first workflow needs ~100 steps (prompt prefill + 50-150 decode steps + an executor
    # visit), so a window right after fill() would be pure decode with no completions.
    # Ramp until as many workflows as the concurrency have finished (one turnover of the
    # closed loop: the initial wave of simultaneous arrivals has drained) and every pool
    # holds calls.
    ramp_steps = 0
    prof_ms, shares = 0.0, {}
    if rt is not None:
        rt.fill()
        t_ramp = time.perf_counter() + 900.0
        target = max(1, rt.concurrency)
        while True:
            done = rt.stats.completed + rt.stats.failed
            busy = all(any(len(e.batch) for e in es) for es in rt.pool_engines.values())
            if done >= target and busy:
                break
            if time.perf_counter() > t_ramp:
                raise SystemExit("bench: closed loop did not reach steady state in 900 s")
            rt.step()
            ramp_steps += 1
        rt.run_steps(max(3, args.warmup))
        if timed:
            # kernel-class shares (untimed) -> the dominant kernel for the roofline;
            # attn_decode_ctx (the per-call context splits, nested in attn_decode) is the
            # HBM-bound decode-attention kernel of the north star's >= 70 % target
            worker.prof = KernelProfile(["gemm", "attn_decode", "attn_prefill",
                                         "attn_decode_ctx"], isolate=True)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            rt.run_steps(args.profile_steps)
            e1.record()
            shares = worker.prof.summary()
            prof_ms = e0.elapsed_time(e1)
            worker.prof = None
        arm.set_phase(PHASE_TIMED)
    else:
        serve(PHASE_WARM)
    barrier()
    dominant = max((k for k in shares if k != "attn_decode_ctx"),
                   key=lambda k: shares[k]["ms"], default="gemm")

    # ---------------- timed region ----------------
    peaks, peak_src = _peaks()
    ncu_window = timed and os.environ.get("CORTEX_NCU_TIMED") == "1"
    if rt is not None and timed:
        # the dominant kernel class timed with CUDA events inside the timed steps (every
        # 8th step instrumented, every 4th in runs under 100 steps so a 20-step window
        # still samples 5 step mixes); under the ncu capture every step,
        # so the algorithmic bytes of exactly the captured launches are known
        worker.prof = KernelProfile([dominant, "attn_decode_ctx"] if ncu_window else [dominant],
                                    every=1 if ncu_window else (4 if steps < 100 else 8))
    clocks = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    st = arm.stats
    s0 = (st.completed, st.failed, st.decode_tokens, st.prefill_tokens, st.steps,
          worker.launches, worker.h2d_bytes, st.d2h_bytes)
    kv_samples = []
    clocks.start()
    # CORTEX_NCU_TIMED=1: an NVTX range "timed" around exactly the timed steps, so an
    # `ncu --nvtx --nvtx-include timed/` launch list describes the same launches whose
    # algorithmic bytes are written to gpurun_out/ncu_window_algorithmic.json
    # (tools/ncu_traffic.py -> profiles/traffic.json -> roofline.traffic)
    if ncu_window:
        torch.cuda.nvtx.range_push("timed")
    t_wall0 = time.perf_counter()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    if rt is not None:
        for _ in range(steps):
            rt.step()
            kv_samples.append(_kv_snapshot(rt))
        arm.set_phase(PHASE_AFTER)
    else:
        serve(PHASE_TIMED)
    ev1.record()
    torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall0
    if ncu_window:
        torch.cuda.nvtx.range_pop()
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms, t_wall * 1e3], device=device)
    all_reduce(t, tdist.ReduceOp.MAX)
    ms, t_wall = float(t[0]), float(t[1]) / 1e3
    s1 = (st.completed, st.failed, st.decode_tokens, st.prefill_tokens, st.steps,
          worker.launches, worker.h2d_bytes, st.d2h_bytes)
    d = [b - a for a, b in zip(s0, s1)]
    completed, failed, dec_tok, pf_tok, _n, launches, h2d, d2h = d
    t = torch.tensor([completed, failed, dec_tok, pf_tok, launches, h2d, d2h], device=device,
                     dtype=torch.float64)
    all_reduce(t, tdist.ReduceOp.SUM)
    completed, failed, dec_tok, pf_tok, launches, h2d, d2h = [float(x) for x in t]
    kshare = {"launches": 0, "ms": 0.0, "bytes": 0.0, "flops": 0.0}
    if worker.prof is not None:
        summ = worker.prof.summary()
        kshare = summ.get(dominant, kshare)
        worker.prof = None
        if ncu_window:
            os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
            with open(os.path.join(ROOT, "gpurun_out", "ncu_window_algorithmic.json"), "w") as f:
                json.dump({k: {"launches": v["launches"], "bytes": v["bytes"],
                               "flops": v["flops"]} for k, v in summ.items()}, f)
    # a kernel-reported error voids the run: no JSON line
    (rt or srv).check_status()
    barrier()
    if rt is None:
        return None

    secs = ms / 1e3
    value = completed / secs
    kv = _kv_stats(rt, kv_samples, cfg)
    if not timed:
        kv.update(topology=arm.mode, workflows_per_s=value, ramp_steps=ramp_steps,
                  timed_steps=steps)
        return kv

    # roofline of the dominant kernel (algorithmic bytes or flops per launch / its average
    # duration); the bound follows the timed window's own arithmetic intensity against
    # the measured ridge point
    ridge = peaks["bf16_tflops_sustained"] * 1e12 / (peaks["hbm_gbs"] * 1e9)
    if dominant == "gemm" and kshare["flops"] / max(kshare["bytes"], 1) > ridge:
        bound, unit, peak = "tensor", "TFLOP/s", peaks["bf16_tflops_sustained"]
        per_launch = kshare["flops"] / max(kshare["launches"], 1)
        achieved = kshare["flops"] / max(kshare["ms"] / 1e3, 1e-12) / 1e12
        peak_note = " sustained bf16"
    else:
        bound, unit, peak = "hbm", "GB/s", peaks["hbm_gbs"]
        per_launch = kshare["bytes"] / max(kshare["launches"], 1)
        achieved = kshare["bytes"] / max(kshare["ms"] / 1e3, 1e-12) / 1e9
        peak_note = " copy bandwidth"
    traffic, traffic_src, traffic_ratio = None, None, None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):  # DRAM bytes per launch from the committed ncu launch list
        with open(tpath) as f:
            tj = json.load(f)
        # only a list captured on this bench's own timed window
        if dominant in tj.get("classes", {}) and tj.get("window") == window_tag(args):
            traffic = tj["classes"][dominant]["dram_bytes_per_launch"]
            traffic_src = tj.get("source")
            traffic_ratio = tj["classes"][dominant].get("dram_per_algorithmic_byte")
    roofline = {"kernel": dominant, "bound": bound, "achieved": achieved, "peak": peak,
                "unit": unit, "frac": achieved / peak, "traffic": traffic,
                "traffic_source": traffic_src,
                # DRAM bytes / algorithmic bytes over the SAME launches of the captured
                # window: the re-read factor (the capture's step mix is not this run's)
                "traffic_per_algorithmic_byte": traffic_ratio,
                "algorithmic_bytes_per_launch": kshare["bytes"] / max(kshare["launches"], 1),
                "algorithmic_flops_per_launch": kshare["flops"] / max(kshare["launches"], 1),
                "per_launch_algorithmic": per_launch,
                "avg_launch_ms": kshare["ms"] / max(kshare["launches"], 1),
                "launches": kshare["launches"], "peak_source": peak_src + peak_note,
                "ridge_flop_per_byte": ridge}

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
    engines = ", ".join(f"{p}: {len(es)} engine(s)" for p, es in rt.pool_engines.items())
    return {
        "metric": METRIC,
        "value": value,
        "unit": "workflows/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ramp_steps": ramp_steps,
        "ms_per_step": ms / max(steps, 1),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic: seeded NL2SQL trace (reference counter streams), random-init weights",
        "config": {"workload": desc, "model": cfg.name + "-shape",
                   "concurrency": rt.concurrency, "topology": arm.mode,
                   "engines": engines + (f" on {n_rep} replicas" if n_rep > 1
                                         else " sharing one GPU")
                   + (f"; TP = {args.tp} per replica" if args.tp > 1 else ""),
                   "l2": "inputs larger than L2 (16 GB of weights + KV streamed every step)"},
        "decode_tok_s": dec_tok / secs,
        "prefill_tok_s": pf_tok / secs,
        "workflows_finished_per_s": (completed + failed) / secs,
        "workflows_in_window": completed,
        "kv_occupancy": kv,
        "kernel_shares": {k: {"ms": v["ms"], "share": v["ms"] / max(prof_ms, 1e-9),
                              "launches": v["launches"]} for k, v in shares.items()},
        "roofline": roofline,
        "rooflines_by_class": rooflines,
        "rooflines_by_class_note": (f"{args.profile_steps} untimed steps right before the timed "
                                    "window, each class timed alone (the attention passes "
                                    "serialised on the main stream, no side-stream overlap)"),
        "clocks": clk,
        "e2e": {"value": completed / t_wall, "unit": "workflows/s",
                "h2d_bytes_per_step": h2d / max(steps, 1),
                "d2h_bytes_per_step": d2h / max(steps, 1)},
        "gpu_launches": int(launches),
    }


def window_tag(args) -> str:
    """Identifies the step mix of a timed window (profiles/traffic.json's `window`)."""
    return f"bench.py timed steps: {args.workload} {args.mode} {args.model} N=1"


def _follow(worker, tp_ring, dist, device, tp_comm, arms, args, spec, n_rep, replica, tp_rank,
            conc_total, max_batch) -> None:
    """TP follower rank: replay the leader's device calls until it stops; join the
    leader's collectives with zeros and each arm's link set-up collectives."""
    from paper_2510_14126_b200.tp import TpFollower

    pending = list(arms)

    def on_collective(kind, a) -> None:
        if kind == "barrier":
            dist.barrier()
        elif kind == "all_reduce":
            n, dtype, op = a
            dist.all_reduce(torch.zeros(n, dtype=getattr(torch, dtype.split(".")[-1]),
                                        device=device), op=op)
        elif kind == "arm":
            Arm(args, pending.pop(0), spec, worker, n_rep, replica, tp_rank, dist, conc_total,
                max_batch)
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
    return (time.perf_counter(), rt.blocks_in_use(),
            {h.engine_id: h.resident_prefix_tokens() for h in rt.all_engines})


def _kv_stats(rt, samples, cfg) -> dict:
    """Peak and time-weighted mean KV blocks per pool (the paper's key quantity,
    time-weighted as stagesim/simulation.py:445-453), plus the whole box."""
    out = {}
    pools = {p: [e.engine_id for e in es] for p, es in rt.pool_engines.items()}
    pools["total"] = [e.engine_id for e in rt.all_engines]
    for pool, eids in pools.items():
        vals = [sum(s[1][e] for e in eids) for s in samples]
        pre = [sum(s[2][e] for e in eids) for s in samples]
        ts = [s[0] for s in samples]
        if len(vals) < 2:
            continue
        integ = sum(vals[i] * (ts[i + 1] - ts[i]) for i in range(len(vals) - 1))
        mean = integ / (ts[-1] - ts[0])
        out[pool] = {"peak_blocks": max(vals), "mean_blocks": mean,
                     "peak_gib": max(vals) * cfg.kv_bytes_per_block / 2 ** 30,
                     "mean_gib": mean * cfg.kv_bytes_per_block / 2 ** 30,
                     "peak_resident_prefix_tokens": max(pre)}
    return out


if __name__ == "__main__":
    main()
