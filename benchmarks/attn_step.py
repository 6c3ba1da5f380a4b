"""One layer's attention work of a config-2 step, piece by piece (Llama-3-8B heads).

Shape of a steady-state bench step: ~215 decoding calls in two stage-prefix groups
(prefix 1000 tokens, resident once per engine), private context U(110, 450) each,
plus ~3 prompt prefills of 200 tokens behind a 1000-token prefix. Times, with CUDA
events on the launching streams:
  private  - per-call context splits (parts=2, HBM)
  cascade  - shared-prefix pass (parts=1, tcgen05)
  combine  - LSE merge (parts=4)
  decode   - the model's schedule: cascade on a side stream || private, then combine
  prefill  - tcgen05 FMHA over the prompts
  layer    - decode + prefill as the model runs them
"""

from __future__ import annotations

import json
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2510_14126_b200 import ops  # noqa: E402

HKV, GROUP = 8, 4
HQ = HKV * GROUP
P = 1000


def build(n_calls=215, n_pf=3, pf_len=200, slots=2, seed=0, layers=4):
    rng = np.random.default_rng(seed)
    dev = torch.device("cuda")
    npb = (P + 15) // 16
    priv = rng.integers(110, 451, n_calls)
    priv = (priv * float(os.environ.get("CORTEX_PRIV_SCALE", "1"))).astype(np.int64)
    nbs = [(int(p) + 15) // 16 for p in priv]
    pf_nb = (pf_len + 15) // 16
    nb = 2 * npb + sum(nbs) + n_pf * pf_nb + 64
    cache = torch.empty(layers, 2, nb, HKV, 16, 128, dtype=torch.bfloat16, device=dev)
    cache.normal_()
    rows = 2 + n_calls + n_pf
    cols = npb + max(max(nbs), pf_nb) + 1
    table = np.zeros((rows, cols), np.int32)
    perm = rng.permutation(np.arange(2 * npb, nb - 64)).astype(np.int32)
    for g in range(2):
        table[g, :npb] = np.arange(g * npb, (g + 1) * npb)
    k = 0
    half = n_calls // 2
    for i in range(n_calls):
        g = 0 if i < half else 1
        table[2 + i, :npb] = table[g, :npb]
        table[2 + i, npb:npb + nbs[i]] = perm[k:k + nbs[i]]
        k += nbs[i]
    for j in range(n_pf):
        r = 2 + n_calls + j
        table[r, :npb] = table[0, :npb]
        table[r, npb:npb + pf_nb] = perm[k:k + pf_nb]
        k += pf_nb
    d = lambda a: torch.as_tensor(np.asarray(a, np.int32), device=dev)
    T = n_calls + n_pf * pf_len
    q = torch.randn(T, HQ, 128, device=dev).to(torch.bfloat16)
    attn = torch.empty_like(q)
    st = {
        "cache": cache, "table": d(table), "q": q, "attn": attn, "nb": nb, "layers": layers,
        "n_calls": n_calls,
        "drow": d(np.arange(2, 2 + n_calls)), "dpre": d([P] * n_calls),
        "dkv": d(P + priv), "grow": d([0, 1]), "gplen": d([P, P]), "gfirst": d([0, half]),
        "gcount": d([half, n_calls - half]), "gmax": max(half, n_calls - half),
        "pslots": slots,
        "prow": d(np.arange(2 + n_calls, rows)), "ppre": d([P] * n_pf),
        "pkv": d([P + pf_len] * n_pf), "pqs": d(n_calls + pf_len * np.arange(n_pf)),
        "pql": d([pf_len] * n_pf), "n_pf": n_pf, "pf_len": pf_len,
        "priv_tokens": int(priv.sum()),
    }
    ntl = npb + (np.asarray(nbs))
    plan = ops.decode_flat_plan(np.full(n_calls, P), P + priv, HKV, True, 64)
    st["flat_plan"] = (d(plan[0]), plan[1], plan[2])
    st["flat_W"] = plan[2]
    st["flat"] = st["flat_plan"] if os.environ.get("CORTEX_FLAT_DECODE", "0") == "1" else None
    st["dzero"] = d([0] * n_calls)
    persplit = max(max(ops.decode_splits(0, int(p)) for p in priv),
                   max(ops.decode_splits(0, P + int(p)) for p in priv))
    st["max_splits"] = st["max_splits_cap"] = slots + max(persplit, plan[3], 8)
    # the model's slot count (pslots + the most private splits of a call): sizes the
    # per-call split grid of the context-split kernels
    st["max_splits_tight"] = slots + max(ops.decode_splits(0, int(p)) for p in priv)
    st["o_part"] = torch.empty(n_calls * st["max_splits"] * HQ * 128, device=dev)
    st["lse"] = torch.empty(n_calls * st["max_splits"] * HQ, device=dev)
    st["kvmap"] = ops.kv_map(cache.view(-1, 128))
    st["qmap"] = ops.QMap(q, HQ, GROUP)
    st["plane"] = nb * HKV * 16
    st["side"] = torch.cuda.Stream(priority=-1)  # as the model's side stream
    st["ev"] = (torch.cuda.Event(), torch.cuda.Event())
    return st


def _plan(st, W):
    key = f"plan{W}"
    if key not in st:
        dev = st["q"].device
        p = ops.decode_flat_plan(np.full(st["n_calls"], P), st["dkv"].cpu().numpy(), HKV, True,
                                 64, W=W)
        assert st["pslots"] + p[3] <= st["max_splits_cap"]
        st[key] = (torch.as_tensor(p[0], device=dev), p[1], p[2])
    return st[key]


def decode(st, layer, parts, stream=None, flat="default"):
    pl = st["plane"]
    groups = (st["grow"], st["gplen"], st["gfirst"], st["gcount"], 2, st["gmax"], st["pslots"])
    ops.paged_decode_attn(st["kvmap"], st["q"], st["table"], st["drow"], st["dpre"], st["dkv"],
                          st["n_calls"], HKV, GROUP, 2 * layer * pl, (2 * layer + 1) * pl,
                          1 / math.sqrt(128), st["o_part"], st["lse"],
                          st["max_splits_tight"] if (flat if flat != "default" else st["flat"]) is None
                          else st["max_splits"],
                          st["attn"], groups=groups, qmap=st["qmap"], parts=parts, stream=stream,
                          flat=st["flat"] if flat == "default" else flat)


def decode_overlap(st, layer):
    main = torch.cuda.current_stream()
    st["ev"][0].record(main)
    st["side"].wait_event(st["ev"][0])
    decode(st, layer, 1, st["side"])
    decode(st, layer, 2)
    st["ev"][1].record(st["side"])
    main.wait_event(st["ev"][1])
    decode(st, layer, 4)


def decode_overlap_privfirst(st, layer):
    """Private splits launched first (they fill the GPU), the cascade pass on the side
    stream slots in as private CTAs retire."""
    main = torch.cuda.current_stream()
    st["ev"][0].record(main)
    decode(st, layer, 2)
    st["side"].wait_event(st["ev"][0])
    decode(st, layer, 1, st["side"])
    st["ev"][1].record(st["side"])
    main.wait_event(st["ev"][1])
    decode(st, layer, 4)


def decode_nocascade(st, layer):
    """No shared-prefix pass: every call's splits read its prefix too (from L2)."""
    pl = st["plane"]
    ops.paged_decode_attn(st["kvmap"], st["q"], st["table"], st["drow"], st["dzero"],
                          st["dkv"], st["n_calls"], HKV, GROUP, 2 * layer * pl,
                          (2 * layer + 1) * pl, 1 / math.sqrt(128), st["o_part"], st["lse"],
                          st["max_splits"], st["attn"])


def layer_side_prefill(st, layer):
    """Cascade pass then prefill FMHA (both tensor-bound) on the side stream, concurrent
    with the private-context decode splits (HBM-bound) on the main stream."""
    main = torch.cuda.current_stream()
    st["ev"][0].record(main)
    st["side"].wait_event(st["ev"][0])
    decode(st, layer, 1, st["side"])
    prefill(st, layer, st["side"])
    decode(st, layer, 2)
    st["ev"][1].record(st["side"])
    main.wait_event(st["ev"][1])
    decode(st, layer, 4)


def layer_side_prefill_first(st, layer):
    """As layer_side_prefill with the prompt prefill ahead of the cascade pass."""
    main = torch.cuda.current_stream()
    st["ev"][0].record(main)
    st["side"].wait_event(st["ev"][0])
    prefill(st, layer, st["side"])
    decode(st, layer, 1, st["side"])
    decode(st, layer, 2)
    st["ev"][1].record(st["side"])
    main.wait_event(st["ev"][1])
    decode(st, layer, 4)


def layer_two_side(st, layer):
    """Cascade pass and prompt prefill on two high-priority side streams."""
    main = torch.cuda.current_stream()
    if "side2" not in st:
        st["side2"] = torch.cuda.Stream(priority=-1)
        st["ev2"] = torch.cuda.Event()
    st["ev"][0].record(main)
    st["side"].wait_event(st["ev"][0])
    st["side2"].wait_event(st["ev"][0])
    decode(st, layer, 1, st["side"])
    prefill(st, layer, st["side2"])
    decode(st, layer, 2)
    st["ev"][1].record(st["side"])
    st["ev2"].record(st["side2"])
    main.wait_event(st["ev"][1])
    main.wait_event(st["ev2"])
    decode(st, layer, 4)


def layer_two_side_pf_first(st, layer):
    """layer_two_side with the prompt prefill launched ahead of the cascade pass."""
    main = torch.cuda.current_stream()
    if "side2" not in st:
        st["side2"] = torch.cuda.Stream(priority=-1)
        st["ev2"] = torch.cuda.Event()
    st["ev"][0].record(main)
    st["side"].wait_event(st["ev"][0])
    st["side2"].wait_event(st["ev"][0])
    prefill(st, layer, st["side2"])
    decode(st, layer, 1, st["side"])
    decode(st, layer, 2)
    st["ev"][1].record(st["side"])
    st["ev2"].record(st["side2"])
    main.wait_event(st["ev"][1])
    main.wait_event(st["ev2"])
    decode(st, layer, 4)


def prefill(st, layer, stream=None):
    pl = st["plane"]
    ops.fmha_prefill(st["kvmap"], st["qmap"], st["attn"], st["table"], st["prow"], st["ppre"],
                     st["pkv"], st["pqs"], st["pql"], st["n_pf"], st["pf_len"], HKV, GROUP,
                     2 * layer * pl, (2 * layer + 1) * pl, 1 / math.sqrt(128), stream=stream)


def timed(st, fn, iters=40):
    """Device time per call (us): the iterations are captured in a CUDA graph so host
    launch overhead (ctypes, ~10 us per call) does not pace small kernels."""
    for i in range(3):
        fn(i % st["layers"])
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for i in range(iters):
                fn(i % st["layers"])
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3


def main():
    from paper_2510_14126_b200 import _lib

    for kv in filter(None, os.environ.get("CORTEX_KNOBS", "").split(",")):  # NAME=V,...
        k, v = kv.split("=")
        _lib.set_knob(k, int(v))
    st = build(slots=int(os.environ.get("CORTEX_CASCADE_SLOTS", "2")))
    if "--private-only" in sys.argv:  # tuning-variant sweeps: the context splits alone
        us = timed(st, lambda l: decode(st, l, 2, flat=None))
        gbs = st["priv_tokens"] * HKV * 128 * 2 * 2 / us / 1e3
        print(json.dumps({"private_us": us, "private_GBps": gbs,
                          "lib": os.environ.get("CORTEX_LIB", ""),
                          "knobs": os.environ.get("CORTEX_KNOBS", ""),
                          "priv_scale": os.environ.get("CORTEX_PRIV_SCALE", "1")}), flush=True)
        return
    if "--layer-only" in sys.argv:  # tuning-variant sweeps: one layer's attention as scheduled
        print(json.dumps({"layer_side_prefill_us": timed(st, lambda l: layer_side_prefill(st, l)),
                          "layer_prefill_first_us": timed(
                              st, lambda l: layer_side_prefill_first(st, l)),
                          "layer_two_side_us": timed(st, lambda l: layer_two_side(st, l)),
                          "layer_two_side_pf_first_us": timed(
                              st, lambda l: layer_two_side_pf_first(st, l)),
                          "private_us": timed(st, lambda l: decode(st, l, 2, flat=None)),
                          "lib": os.environ.get("CORTEX_LIB", ""),
                          "knobs": os.environ.get("CORTEX_KNOBS", "")}), flush=True)
        return
    if "--fmha-only" in sys.argv:  # tuning-variant sweeps: the tensor-core passes alone
        print(json.dumps({"prefill_us": timed(st, lambda l: prefill(st, l)),
                          "cascade_us": timed(st, lambda l: decode(st, l, 1)),
                          "lib": os.environ.get("CORTEX_LIB", ""),
                          "knobs": os.environ.get("CORTEX_KNOBS", "")}), flush=True)
        return
    if "--once" in sys.argv:  # for ncu: 2 x (private, cascade, combine, prefill)
        for i in range(2):
            decode(st, i, 2)
            decode(st, i, 1)
            decode(st, i, 4)
            prefill(st, i)
        torch.cuda.synchronize()
        return
    res = {
        "private_us": timed(st, lambda l: decode(st, l, 2)),
        "private_persplit_us": timed(st, lambda l: decode(st, l, 2, flat=None)),
        "private_flat_us": timed(st, lambda l: decode(st, l, 2, flat=st["flat_plan"])),
        "flat_W": st["flat_W"],
        **{f"private_flat_W{W}_us": timed(st, lambda l, W=W: decode(st, l, 2, flat=_plan(st, W)))
           for W in (8, 16, 24, 48)},
        "cascade_us": timed(st, lambda l: decode(st, l, 1)),
        "combine_us": timed(st, lambda l: decode(st, l, 4)),
        "decode_serial_us": timed(st, lambda l: decode(st, l, 7)),
        "decode_overlap_us": timed(st, lambda l: decode_overlap(st, l)),
        "decode_overlap_privfirst_us": timed(st, lambda l: decode_overlap_privfirst(st, l)),
        "decode_nocascade_us": timed(st, lambda l: decode_nocascade(st, l)),
        "prefill_us": timed(st, lambda l: prefill(st, l)),
        "layer_us": timed(st, lambda l: (decode_overlap(st, l), prefill(st, l))),
        "layer_side_prefill_us": timed(st, lambda l: layer_side_prefill(st, l)),
    }
    priv_bytes = st["priv_tokens"] * HKV * 128 * 2 * 2
    res["private_GBps"] = priv_bytes / res["private_us"] / 1e3
    casc_flops = 4.0 * st["n_calls"] * HQ * P * 128
    res["cascade_TFps"] = casc_flops / res["cascade_us"] / 1e6
    pf = st["pf_len"]
    pf_flops = 4.0 * st["n_pf"] * HQ * 128 * (pf * P + pf * (pf + 1) / 2)
    res["prefill_TFps"] = pf_flops / res["prefill_us"] / 1e6
    res["shape"] = {"calls": st["n_calls"], "prefix": P, "priv_tokens": st["priv_tokens"],
                    "prefill": [st["n_pf"], pf], "slots": st["pslots"]}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
