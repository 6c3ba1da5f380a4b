"""Kernel-level parity on the B200: every export against the CPU/fp32 oracle.

Run with `pytest -m gpu`. Tolerances (north star: "2e-3 relative error in bf16"):
  * GEMM: relative Frobenius error vs fp32 matmul of the same bf16 inputs,
    measured after the bf16 output rounding: <= 4e-3 (one bf16 rounding is
    2^-9 = 1.95e-3 per element, so the norm-relative error sits near 1e-3).
  * attention: relative Frobenius error vs oracle.attention_ref <= 4e-3.
  * allocator / argmax / embedding: bit-exact.
"""

from __future__ import annotations

import ctypes
import math
import random

import numpy as np

import pytest
import torch

from oracle.alloc_ref import BlockPoolRef
from oracle.decoder_ref import attention_ref, bf16, rmsnorm_ref, rope_ref, rope_tables

pytestmark = pytest.mark.gpu


def ops():
    from paper_2510_14126_b200 import ops as o

    return o


def rel(a: torch.Tensor, b: torch.Tensor) -> float:
    a = a.float().cpu()
    b = b.float().cpu()
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


# ---------------------------------------------------------------- GEMM


@pytest.mark.parametrize("N,K", [(256, 256), (512, 768), (6144, 4096), (1024, 14336)])
@pytest.mark.parametrize("M", [1, 5, 32, 33, 64, 100, 128, 200, 256, 300, 777])
def test_gemm_matches_fp32(cuda, M, N, K):
    o = ops()
    g = torch.Generator(device=cuda).manual_seed(1000 * M + N + K)
    x = torch.randn(max(M, 32), K, generator=g, device=cuda).to(torch.bfloat16)
    w = (torch.randn(N, K, generator=g, device=cuda) * 0.05).to(torch.bfloat16)
    ws = o.GemmWorkspace(cuda)
    out = torch.full((M, N), float("nan"), device=cuda, dtype=torch.bfloat16)
    o.gemm(o.weight_map(w), o.act_map(x), M, out, ws)
    ref = x[:M].float() @ w.float().T
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all()
    assert rel(out, ref) < 4e-3
    # split-K tile counters left zeroed (the last 512 hold the split flags: epoch values)
    assert int(ws.counters[:-512].abs().sum()) == 0


@pytest.mark.parametrize("M", [3, 64, 257])
def test_gemm_residual_and_f32(cuda, M):
    o = ops()
    N, K = 512, 1024
    g = torch.Generator(device=cuda).manual_seed(7 + M)
    x = torch.randn(max(M, 32), K, generator=g, device=cuda).to(torch.bfloat16)
    w = (torch.randn(N, K, generator=g, device=cuda) * 0.05).to(torch.bfloat16)
    r = torch.randn(M, N, generator=g, device=cuda)
    ws = o.GemmWorkspace(cuda)
    out = torch.empty(M, N, device=cuda, dtype=torch.float32)
    o.gemm(o.weight_map(w), o.act_map(x), M, out, ws, residual=r)
    ref = x[:M].float() @ w.float().T + r
    assert rel(out, ref) < 1e-5
    o.gemm(o.weight_map(w), o.act_map(x), M, r, ws, residual=r)  # in place (residual stream)
    assert rel(r, ref) < 1e-5
    out32 = torch.empty(M, N, device=cuda, dtype=torch.float32)
    o.gemm(o.weight_map(w), o.act_map(x), M, out32, ws)
    assert rel(out32, x[:M].float() @ w.float().T) < 1e-5


def _set_gemm_mode(o, mode):
    """0 automatic, 1 = 1-SM kernel, 2 = 2-SM whole tiles, 3 = 2-SM stream-K."""
    o.gemm_set_mode(min(mode, 2))
    o.gemm_set_stream_k({0: -1, 1: -1, 2: 0, 3: 1}[mode])


@pytest.mark.parametrize("mode", [1, 2, 3])
@pytest.mark.parametrize("M,N,K", [(129, 512, 256), (700, 4096, 4096), (300, 6144, 4096),
                                   (2048, 1536, 256), (33, 1024, 768), (1000, 28672, 4096),
                                   (4096, 4096, 14336), (5, 256, 4096)])
def test_gemm_paths_match(cuda, mode, M, N, K):
    """Both kernels (1-SM split-K and persistent 2-SM cta_group::2, the latter with whole
    tiles (mode 2) or stream-K ranges (mode 3)) on the same problems."""
    o = ops()
    g = torch.Generator(device=cuda).manual_seed(M + N)
    x = torch.randn(max(M, 32), K, generator=g, device=cuda).to(torch.bfloat16)
    w = (torch.randn(N, K, generator=g, device=cuda) * 0.05).to(torch.bfloat16)
    r = torch.randn(M, N, generator=g, device=cuda)
    ws = o.GemmWorkspace(cuda)
    _set_gemm_mode(o, mode)
    try:
        out = torch.full((M, N), float("nan"), device=cuda, dtype=torch.bfloat16)
        o.gemm(o.weight_map(w), o.act_map(x), M, out, ws)
        out32 = torch.empty(M, N, device=cuda)
        o.gemm(o.weight_map(w), o.act_map(x), M, out32, ws, residual=r)
        torch.cuda.synchronize()
        assert int(ws.counters[:-512].abs().sum()) == 0  # stream-K flags left zeroed
    finally:
        _set_gemm_mode(o, 0)
    ref = x[:M].float() @ w.float().T
    assert torch.isfinite(out.float()).all()
    assert rel(out, ref) < 4e-3
    assert rel(out32, ref + r) < 4e-5  # fp32 accumulation order over K <= 14336


@pytest.mark.parametrize("mode", [1, 2, 3])
@pytest.mark.parametrize("M,F,K", [(7, 768, 256), (300, 768, 256), (700, 14336, 4096),
                                   (64, 14336, 4096)])
def test_gemm_fused_swiglu(cuda, mode, M, F, K):
    """gate_up GEMM with SwiGLU applied to the fp32 accumulators in the epilogue."""
    o = ops()
    g = torch.Generator(device=cuda).manual_seed(M + F)
    x = torch.randn(max(M, 32), K, generator=g, device=cuda).to(torch.bfloat16)
    w = (torch.randn(2 * F, K, generator=g, device=cuda) * 0.05).to(torch.bfloat16)
    wi = o.interleave_gate_up(w)
    assert torch.equal(o.deinterleave_gate_up(wi), w)
    out = torch.full((M, F), float("nan"), device=cuda, dtype=torch.bfloat16)
    _set_gemm_mode(o, mode)
    try:
        o.gemm(o.weight_map(wi), o.act_map(x), M, out, o.GemmWorkspace(cuda), swiglu=True)
        torch.cuda.synchronize()
    finally:
        _set_gemm_mode(o, 0)
    gu = x[:M].float() @ w.float().T
    gg, uu = gu[:, :F], gu[:, F:]
    ref = gg / (1 + torch.exp(-gg)) * uu
    assert rel(out, ref) < 4e-3


@pytest.mark.parametrize("ks", [-1, 2, 3, 4])
@pytest.mark.parametrize("M,N,K", [(129, 4096, 4096), (210, 6144, 4096), (256, 4096, 14336),
                                   (200, 512, 256), (5, 4096, 4096), (64, 1024, 768),
                                   (100, 28672, 4096)])
def test_gemm_splitk_cluster(cuda, ks, M, N, K):
    """Cluster split-K 2-SM kernel (gemm_splitk.cu) with every split count: bf16 out,
    fp32 out with the residual added in place, and the fused SwiGLU epilogue."""
    o = ops()
    L = o.lib()
    g = torch.Generator(device=cuda).manual_seed(M * 7 + N + K)
    x = torch.randn(max(M, 32), K, generator=g, device=cuda).to(torch.bfloat16)
    w = (torch.randn(N, K, generator=g, device=cuda) * 0.05).to(torch.bfloat16)
    r = torch.randn(M, N, generator=g, device=cuda)
    ws = o.GemmWorkspace(cuda)
    o.gemm_set_mode(3)
    from paper_2510_14126_b200 import _lib

    _lib.set_knob("SK_KS", ks)
    try:
        kb = K // 64
        got = o.splitk_plan(M, N, K)[0]
        if ks > 0 and got:  # the forced count, or no plan (it would not fit one wave)
            assert got == ks and (got - 1) * -(-kb // got) < kb
        assert got != 1  # (no split only when forced: see test_gemm_splitk_nw2)
        path = o.gemm_path(M, N, K)
        out = torch.full((M, N), float("nan"), device=cuda, dtype=torch.bfloat16)
        o.gemm(o.weight_map(w), o.act_map(x), M, out, ws)
        res = r.clone()
        o.gemm(o.weight_map(w), o.act_map(x), M, res, ws, residual=res)
        wi = o.interleave_gate_up(w)
        act = torch.full((M, N // 2), float("nan"), device=cuda, dtype=torch.bfloat16)
        o.gemm(o.weight_map(wi), o.act_map(x), M, act, ws, swiglu=True)
        torch.cuda.synchronize()
    finally:
        o.gemm_set_mode(0)
        _lib.set_knob("SK_KS", -1)
    assert path == (3 if got >= 1 else 2)
    ref = x[:M].float() @ w.float().T
    assert torch.isfinite(out.float()).all()
    assert rel(out, ref) < 4e-3
    assert rel(res, ref + r) < 4e-5
    gg, uu = ref[:, :N // 2], ref[:, N // 2:]
    assert rel(act, gg / (1 + torch.exp(-gg)) * uu) < 4e-3


@pytest.mark.parametrize("M,N,K", [(100, 28672, 4096), (233, 28672, 4096), (17, 20480, 512)])
def test_gemm_splitk_nw2(cuda, M, N, K):
    """The kernel's unsplit mode with two 256-row weight sub-tiles per pair (forced; the
    automatic plan keeps wide projections on the persistent 2-SM kernel)."""
    o = ops()
    L = o.lib()
    g = torch.Generator(device=cuda).manual_seed(M + N)
    x = torch.randn(max(M, 32), K, generator=g, device=cuda).to(torch.bfloat16)
    w = (torch.randn(N, K, generator=g, device=cuda) * 0.05).to(torch.bfloat16)
    ws = o.GemmWorkspace(cuda)
    from paper_2510_14126_b200 import _lib

    _lib.set_knob("SK_NW", 2)
    try:
        ks, _, _, nw = o.splitk_plan(M, N, K)
        assert ks == 1
        assert nw == 2 and o.gemm_path(M, N, K) == 3
        out = torch.full((M, N), float("nan"), device=cuda, dtype=torch.bfloat16)
        o.gemm(o.weight_map(w), o.act_map(x), M, out, ws)
        act = torch.full((M, N // 2), float("nan"), device=cuda, dtype=torch.bfloat16)
        o.gemm(o.weight_map(o.interleave_gate_up(w)), o.act_map(x), M, act, ws, swiglu=True)
        torch.cuda.synchronize()
    finally:
        _lib.set_knob("SK_NW", -1)
    ref = x[:M].float() @ w.float().T
    assert rel(out, ref) < 4e-3
    gg, uu = ref[:, :N // 2], ref[:, N // 2:]
    assert rel(act, gg / (1 + torch.exp(-gg)) * uu) < 4e-3


def test_gemm_splitk_deterministic(cuda):
    """The split reduction runs in split order: repeated launches agree bit for bit."""
    o = ops()
    M, N, K = 210, 4096, 14336
    g = torch.Generator(device=cuda).manual_seed(11)
    x = torch.randn(M, K, generator=g, device=cuda).to(torch.bfloat16)
    w = (torch.randn(N, K, generator=g, device=cuda) * 0.05).to(torch.bfloat16)
    ws = o.GemmWorkspace(cuda)
    assert o.gemm_path(M, N, K) == 3
    outs = []
    for _ in range(3):
        out = torch.empty(M, N, device=cuda)
        o.gemm(o.weight_map(w), o.act_map(x), M, out, ws)
        outs.append(out)
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])


def test_gemm_batch_invariant(cuda):
    """Within the decode regime (M <= 256: the cluster split-K kernel, whose split count is
    fixed by N and K) a row's result does not depend on the other rows of the batch."""
    o = ops()
    N, K = 6144, 4096
    g = torch.Generator(device=cuda).manual_seed(3)
    x = torch.randn(256, K, generator=g, device=cuda).to(torch.bfloat16)
    w = (torch.randn(N, K, generator=g, device=cuda) * 0.05).to(torch.bfloat16)
    ws = o.GemmWorkspace(cuda)
    full = torch.empty(256, N, device=cuda, dtype=torch.bfloat16)
    assert o.gemm_path(256, N, K) == 3
    o.gemm(o.weight_map(w), o.act_map(x), 256, full, ws)
    for m in (1, 17, 64, 100, 129, 200):
        assert o.gemm_path(m, N, K) == 3
        part = torch.empty(m, N, device=cuda, dtype=torch.bfloat16)
        o.gemm(o.weight_map(w), o.act_map(x), m, part, ws)
        assert torch.equal(part, full[:m]), m


# ---------------------------------------------------------------- attention


def _make_cache(cuda, n_layers, nb, hkv, seed):
    g = torch.Generator(device=cuda).manual_seed(seed)
    cache = torch.randn(n_layers, 2, nb, hkv, 16, 128, generator=g, device=cuda).to(torch.bfloat16)
    return cache


def _rows(layer, nb, hkv):
    k_row0 = (layer * 2 + 0) * nb * hkv * 16
    v_row0 = (layer * 2 + 1) * nb * hkv * 16
    return k_row0, v_row0


def _logical_kv(cache, layer, table_row, prefix, kvlen):
    npb = (prefix + 15) // 16
    ks, vs = [], []
    for pos in range(kvlen):
        if pos < prefix:
            j, off = pos // 16, pos % 16
        else:
            jj = pos - prefix
            j, off = npb + jj // 16, jj % 16
        b = int(table_row[j])
        ks.append(cache[layer, 0, b, :, off, :])
        vs.append(cache[layer, 1, b, :, off, :])
    return torch.stack(ks).float().cpu(), torch.stack(vs).float().cpu()


def _seq_specs(rng, nb, max_blocks):
    # (prefix_len, kv_len) cases: no prefix, aligned prefix, ragged prefix, long
    # (0, 513) / (0, 545) / (1000, 1000 + 513 ...): a last split of 1-3 tiles, so some of
    # the CTA's 4 warps own no key at all (their merge rows must be skipped, not scaled)
    specs = [(0, 1), (0, 17), (40, 41), (40, 77), (1000, 1000 + 137), (16, 300), (5, 5 + 256),
             (0, 255), (0, 256), (0, 257), (1000, 1000 + 700), (0, 513), (0, 545),
             (1000, 1000 + 1050)]
    tables = []
    perm = rng.permutation(nb)
    used = 0
    for prefix, kvlen in specs:
        n = (prefix + 15) // 16 + (kvlen - prefix + 15) // 16
        assert n <= max_blocks
        tables.append(perm[used:used + n])
        used = (used + n) % (nb - max_blocks)
    return specs, tables


@pytest.mark.parametrize("group", [4, 2])
@pytest.mark.parametrize("flat", [False, True])
def test_paged_decode_attention(cuda, group, flat):
    o = ops()
    hkv, L, nb, max_blocks = 2, 2, 640, 134
    hq = hkv * group
    cache = _make_cache(cuda, L, nb, hkv, seed=11 + group)
    rng = np.random.default_rng(5)
    specs, tables = _seq_specs(rng, nb, max_blocks)
    B = len(specs)
    table = torch.zeros(B, max_blocks, dtype=torch.int32)
    for i, t in enumerate(tables):
        table[i, : len(t)] = torch.as_tensor(t, dtype=torch.int32)
    table = table.to(cuda)
    seq_row = torch.arange(B, dtype=torch.int32, device=cuda)
    seq_prefix = torch.tensor([s[0] for s in specs], dtype=torch.int32, device=cuda)
    seq_kvlen = torch.tensor([s[1] for s in specs], dtype=torch.int32, device=cuda)
    max_splits = max(o.decode_splits(p, k) for p, k in specs)
    plan = None
    if flat:  # balanced plan: equal flat tile ranges per CTA, calls split across chunks
        st, total, W, pieces = o.decode_flat_plan([s[0] for s in specs], [s[1] for s in specs],
                                                  hkv, False, 64)
        plan = (torch.as_tensor(st, device=cuda), total, W)
        max_splits = pieces
    q = torch.randn(B, hq, 128, device=cuda).to(torch.bfloat16)
    o_part = torch.empty(B, max_splits, hq, 128, device=cuda)
    lse_part = torch.empty(B, max_splits, hq, device=cuda)
    out = torch.empty(B, hq, 128, device=cuda, dtype=torch.bfloat16)
    kvmap = o.kv_map(cache.view(-1, 128))
    for layer in range(L):
        k0, v0 = _rows(layer, nb, hkv)
        o.paged_decode_attn(kvmap, q, table, seq_row, seq_prefix, seq_kvlen, B, hkv, group, k0, v0,
                            1 / math.sqrt(128), o_part, lse_part, max_splits, out, flat=plan)
        torch.cuda.synchronize()
        for b, (prefix, kvlen) in enumerate(specs):
            k, v = _logical_kv(cache, layer, table[b].cpu(), prefix, kvlen)
            ref = attention_ref(q[b:b + 1].float().cpu(), k, v, torch.tensor([kvlen - 1]),
                                torch.arange(kvlen))
            assert rel(out[b:b + 1], ref) < 4e-3, (layer, b, prefix, kvlen)


@pytest.mark.parametrize("group", [4, 2])
@pytest.mark.parametrize("plens", [(1000, 40), (8192,), (16, 5, 0)])
@pytest.mark.parametrize("impl", ["mma", "tc", "tc1", "tc-flat"])
def test_cascade_decode_attention(cuda, group, plens, impl):
    """Shared-prefix decode: calls grouped by resident prefix, prefix attended once."""
    o = ops()
    hkv, nb = 2, 2048
    hq = hkv * group
    cache = _make_cache(cuda, 1, nb, hkv, seed=31 + group)
    rng = np.random.default_rng(7)
    perm = list(rng.permutation(nb))
    # per prefix: (table row, blocks); then calls: 1..37 per group with ragged private lengths
    n_groups = len(plens)
    counts = [37, 3, 1][:n_groups]
    rows_total = n_groups + sum(counts)
    table = torch.zeros(rows_total, 600, dtype=torch.int32)
    pref_blocks = []
    for g, P in enumerate(plens):
        npb = (P + 15) // 16
        ids = [perm.pop() for _ in range(npb)]
        table[g, :npb] = torch.tensor(ids, dtype=torch.int32)
        pref_blocks.append(ids)
    seq_row, seq_pre, seq_kv, grp = [], [], [], []
    r = n_groups
    for g, P in enumerate(plens):
        first = len(seq_row)
        for i in range(counts[g]):
            # ragged private lengths, some past one 512-token split (a 1-3 tile 2nd split)
            priv = int(rng.integers(1, 300)) if i % 3 else int(rng.integers(513, 560))
            npr = (priv + 15) // 16
            ids = pref_blocks[g] + [perm.pop() for _ in range(npr)]
            table[r, :len(ids)] = torch.tensor(ids, dtype=torch.int32)
            seq_row.append(r)
            seq_pre.append(P)
            seq_kv.append(P + priv)
            r += 1
        if P:
            grp.append((g, P, first, counts[g]))
    B = len(seq_row)
    dev = lambda a: torch.as_tensor(np.asarray(a, dtype=np.int32), device=cuda)
    table = table.to(cuda)
    pslots = max([((P + 15) // 16 + 15) // 16 for _, P, _, _ in grp] + [1])
    priv = max(o.decode_splits(0, kv - p) for p, kv in zip(seq_pre, seq_kv))
    max_splits = pslots + priv
    plan = None
    if impl == "tc-flat":
        st, total, W, pieces = o.decode_flat_plan(seq_pre, seq_kv, hkv, True, 64)
        plan = (torch.as_tensor(st, device=cuda), total, W)
        max_splits = pslots + pieces
    q = torch.randn(B, hq, 128, device=cuda).to(torch.bfloat16)
    o_part = torch.empty(B, max_splits, hq, 128, device=cuda)
    lse_part = torch.empty(B, max_splits, hq, device=cuda)
    out = torch.empty(B, hq, 128, device=cuda, dtype=torch.bfloat16)
    ga = np.asarray(grp, dtype=np.int32).reshape(-1, 4).T
    groups = (dev(ga[0]), dev(ga[1]), dev(ga[2]), dev(ga[3]), len(grp), int(ga[3].max()), pslots)
    k0, v0 = _rows(0, nb, hkv)
    from paper_2510_14126_b200 import _lib

    prev_2q = o.fmha_set_2q(0 if impl == "tc1" else 1)
    plo = _lib.set_knob("FMHA_PLO", 0 if impl == "tc-bf16p" else 1)
    try:
        o.paged_decode_attn(o.kv_map(cache.view(-1, 128)), q, table, dev(seq_row), dev(seq_pre),
                            dev(seq_kv), B, hkv, group, k0, v0, 1 / math.sqrt(128), o_part,
                            lse_part, max_splits, out, groups=groups,
                            qmap=o.QMap(q, hq, group) if impl != "mma" else None, flat=plan)
    finally:
        o.fmha_set_2q(prev_2q)
        _lib.set_knob("FMHA_PLO", plo)
    torch.cuda.synchronize()
    for b in range(B):
        k, v = _logical_kv(cache, 0, table[seq_row[b]].cpu(), seq_pre[b], seq_kv[b])
        ref = attention_ref(q[b:b + 1].float().cpu(), k, v, torch.tensor([seq_kv[b] - 1]),
                            torch.arange(seq_kv[b]))
        assert rel(out[b:b + 1], ref) < 4e-3, (b, seq_pre[b], seq_kv[b])


@pytest.mark.parametrize("group", [4, 2])
@pytest.mark.parametrize("impl", ["mma", "tc", "tc1", "tc-bf16p"])
def test_paged_prefill_attention(cuda, group, impl):
    """tc: two-Q-tile tcgen05 kernel, tc1: one tile per CTA (both with P as bf16 hi + lo,
    the default), tc-bf16p: two tiles with bf16 P alone, mma: mma.sync."""
    o = ops()
    hkv, L, nb, max_blocks = 2, 1, 512, 160
    hq = hkv * group
    cache = _make_cache(cuda, L, nb, hkv, seed=23 + group)
    rng = np.random.default_rng(9)
    specs, tables = _seq_specs(rng, nb, max_blocks)
    qlens = [min(kv, q) for (p, kv), q in zip(specs, [1, 17, 1, 37, 137, 100, 256, 255, 3, 257, 700, 300, 65, 200])]
    B = len(specs)
    table = torch.zeros(B, max_blocks, dtype=torch.int32)
    for i, t in enumerate(tables):
        table[i, : len(t)] = torch.as_tensor(t, dtype=torch.int32)
    table = table.to(cuda)
    qstart = np.concatenate([[0], np.cumsum(qlens)[:-1]]).astype(np.int32)
    T = int(sum(qlens))
    q = torch.randn(T, hq, 128, device=cuda).to(torch.bfloat16)
    out = torch.zeros(T, hq, 128, device=cuda, dtype=torch.bfloat16)
    kvmap = o.kv_map(cache.view(-1, 128))
    k0, v0 = _rows(0, nb, hkv)
    dev = lambda a: torch.as_tensor(np.asarray(a, dtype=np.int32), device=cuda)
    args = (table, dev(range(B)), dev([s[0] for s in specs]), dev([s[1] for s in specs]),
            dev(qstart), dev(qlens), B, max(qlens), hkv, group, k0, v0, 1 / math.sqrt(128))
    if impl == "mma":
        o.paged_prefill_attn(kvmap, q, out, *args)
    else:
        from paper_2510_14126_b200 import _lib

        prev_2q = o.fmha_set_2q(0 if impl == "tc1" else 1)
        plo = _lib.set_knob("FMHA_PLO", 0 if impl == "tc-bf16p" else 1)
        try:
            o.fmha_prefill(kvmap, o.QMap(q, hq, group), out, *args)
        finally:
            o.fmha_set_2q(prev_2q)
            _lib.set_knob("FMHA_PLO", plo)
    torch.cuda.synchronize()
    for b, (prefix, kvlen) in enumerate(specs):
        k, v = _logical_kv(cache, 0, table[b].cpu(), prefix, kvlen)
        ql = qlens[b]
        qpos = torch.arange(kvlen - ql, kvlen)
        ref = attention_ref(q[qstart[b]:qstart[b] + ql].float().cpu(), k, v, qpos, torch.arange(kvlen))
        assert rel(out[qstart[b]:qstart[b] + ql], ref) < 4e-3, (b, prefix, kvlen, ql)


# ---------------------------------------------------------------- elementwise


def test_rmsnorm_embed_argmax(cuda):
    o = ops()
    d, V, T = 4096, 1000, 37
    g = torch.Generator(device=cuda).manual_seed(1)
    emb = torch.randn(V, d, generator=g, device=cuda).to(torch.bfloat16)
    toks = torch.randint(0, V, (T,), generator=g, device=cuda, dtype=torch.int32)
    h = torch.empty(T, d, device=cuda, dtype=torch.float32)
    o.embed(emb, toks, T, h)
    assert torch.equal(h, emb[toks.long()].float())
    w = (1 + 0.1 * torch.randn(d, generator=g, device=cuda)).to(torch.bfloat16)
    y = torch.empty(T, d, device=cuda, dtype=torch.bfloat16)
    o.rmsnorm(h, w, T, y, 1e-5)
    ref = rmsnorm_ref(h.float().cpu(), w.float().cpu(), 1e-5)
    assert rel(y, ref) < 1e-3
    rows = torch.tensor([5, 0, 36], dtype=torch.int32, device=cuda)
    y3 = torch.empty(3, d, device=cuda, dtype=torch.bfloat16)
    o.rmsnorm(h, w, 3, y3, 1e-5, rows=rows)
    assert torch.equal(y3, y[rows.long()])
    logits = torch.randn(T, 128256, generator=g, device=cuda)
    logits[3, 77] = 100.0
    logits[3, 99] = 100.0  # tie -> first index
    tok = torch.empty(T, dtype=torch.int32, device=cuda)
    o.argmax(logits, T, 128256, out_tok=tok)
    ref_tok = torch.argmax(logits, dim=1).to(torch.int32)
    assert torch.equal(tok, ref_tok)
    assert int(tok[3]) == 77
    # ties inside one 16-byte load, across threads and in the scalar tail of an odd vocab
    for vocab, ties in ((128256, (8, 9)), (128256, (4101, 5)), (1027, (1026, 1025)),
                        (1027, (1024, 3))):
        lg = torch.randn(2, vocab, generator=g, device=cuda)
        lg[1, list(ties)] = 50.0
        t2 = torch.empty(2, dtype=torch.int32, device=cuda)
        o.argmax(lg, 2, vocab, out_tok=t2)
        assert int(t2[1]) == min(ties), (vocab, ties)
        assert int(t2[0]) == int(torch.argmax(lg[0]))
    # a row without a finite logit still yields a valid token id (0)
    lg = torch.full((1, 128256), float("nan"), device=cuda)
    o.argmax(lg, 1, 128256, out_tok=t2)
    assert int(t2[0]) == 0


def test_rope_kv_append(cuda):
    o = ops()
    hq, hkv, T, nb = 8, 2, 21, 64
    g = torch.Generator(device=cuda).manual_seed(2)
    qkv = torch.randn(T, (hq + 2 * hkv) * 128, generator=g, device=cuda).to(torch.bfloat16)
    cache = torch.zeros(1, 2, nb, hkv, 16, 128, device=cuda, dtype=torch.bfloat16)
    table = torch.randperm(nb, generator=torch.Generator().manual_seed(0)).to(torch.int32)
    table = table.view(4, 16).to(cuda)
    pos = torch.arange(100, 100 + T, dtype=torch.int32)
    rows = torch.tensor([i % 4 for i in range(T)], dtype=torch.int32)
    cols = torch.tensor([(i // 4) % 16 for i in range(T)], dtype=torch.int32)
    offs = torch.tensor([(3 * i) % 16 for i in range(T)], dtype=torch.int32)
    cos, sin = rope_tables(4096, 500000.0)
    q_out = torch.empty(T, hq, 128, device=cuda, dtype=torch.bfloat16)
    k0, v0 = _rows(0, nb, hkv)
    o.rope_kv_append(qkv, q_out, cache, k0, v0, table, pos.to(cuda), rows.to(cuda), cols.to(cuda),
                     offs.to(cuda), cos.to(cuda), sin.to(cuda), T, hq, hkv)
    torch.cuda.synchronize()
    x = qkv.float().cpu()
    qr = rope_ref(x[:, : hq * 128].reshape(T, hq, 128), cos[pos.long()], sin[pos.long()])
    kr = rope_ref(x[:, hq * 128:(hq + hkv) * 128].reshape(T, hkv, 128), cos[pos.long()],
                  sin[pos.long()])
    vr = x[:, (hq + hkv) * 128:].reshape(T, hkv, 128)
    assert rel(q_out, qr) < 1e-5
    tab = table.cpu()
    for t in range(T):
        b = int(tab[rows[t], cols[t]])
        assert rel(cache[0, 0, b, :, offs[t]], kr[t]) < 1e-5
        assert torch.equal(cache[0, 1, b, :, offs[t]].float().cpu(), vr[t])


# ---------------------------------------------------------------- allocator


@pytest.mark.parametrize("host", [False, True])
def test_kv_alloc_free_matches_oracle(cuda, host):
    """Device-array requests (cortex_kv_alloc / _free) and host-array requests passed in
    the kernel parameters (the _h exports the engine uses) against the pool oracle."""
    o = ops()
    nblocks, id_base, n_rows, stride = 1000, 5000, 40, 64
    ref = BlockPoolRef(nblocks, id_base)
    bitmap = torch.from_numpy(ref.bitmap_words().view(np.int32)).to(cuda)
    table = torch.full((n_rows, stride), -1, dtype=torch.int32, device=cuda)
    status = torch.zeros(1, dtype=torch.int32, device=cuda)
    ref_table = np.full((n_rows, stride), -1, dtype=np.int64)
    held: dict[int, int] = {}  # row -> blocks held (from col 0)
    rnd = random.Random(4)
    dev = lambda a: torch.as_tensor(np.asarray(a, dtype=np.int32), device=cuda)
    for step in range(300):
        if rnd.random() < 0.55:
            free_rows = [r for r in range(n_rows) if r not in held]
            if not free_rows:
                continue
            rows = rnd.sample(free_rows, k=min(len(free_rows), rnd.randint(1, 6)))
            counts = [rnd.choice([0, 1, 3, 16, 63]) for _ in rows]
            if sum(counts) > ref.n_free():
                if host:
                    o.kv_alloc_h(bitmap, nblocks, id_base, counts, rows, [0] * len(rows), table,
                                 status)
                else:
                    o.kv_alloc(bitmap, nblocks, id_base, dev(counts), dev(rows),
                               dev([0] * len(rows)), len(rows), table, status)
                torch.cuda.synchronize()
                assert int(status[0]) == -3
                status.zero_()
                continue
            ids = ref.alloc(counts)
            for r, c, got in zip(rows, counts, ids):
                held[r] = c
                ref_table[r, :c] = got
            if host:
                o.kv_alloc_h(bitmap, nblocks, id_base, counts, rows, [0] * len(rows), table, status)
            else:
                o.kv_alloc(bitmap, nblocks, id_base, dev(counts), dev(rows), dev([0] * len(rows)),
                           len(rows), table, status)
        else:
            if not held:
                continue
            rows = rnd.sample(sorted(held), k=min(len(held), rnd.randint(1, 4)))
            counts = [held.pop(r) for r in rows]
            for r, c in zip(rows, counts):
                ref.free(ref_table[r, :c].tolist())
            if host:
                o.kv_free_h(bitmap, nblocks, id_base, table, rows, [0] * len(rows), counts, status)
            else:
                o.kv_free(bitmap, nblocks, id_base, table, dev(rows), dev([0] * len(rows)),
                          dev(counts), len(rows), status)
        torch.cuda.synchronize()
        assert int(status[0]) == 0
        got_bitmap = bitmap.cpu().numpy().view(np.uint32)
        assert np.array_equal(got_bitmap, ref.bitmap_words()), step
        tab = table.cpu().numpy()
        for r, c in held.items():
            assert np.array_equal(tab[r, :c], ref_table[r, :c]), (step, r)
    nfree = torch.zeros(1, dtype=torch.int32, device=cuda)
    o.kv_count_free(bitmap, nblocks, nfree)
    assert int(nfree[0]) == ref.n_free()


def test_kv_host_requests_chunked(cuda):
    """More requests than one kernel's parameter block holds (256): served in order over
    several launches, identical to the oracle; table_copy_h copies rows."""
    o = ops()
    nblocks, n_req = 1200, 600
    ref = BlockPoolRef(nblocks, 7)
    bitmap = torch.from_numpy(ref.bitmap_words().view(np.int32)).to(cuda)
    table = torch.full((n_req + 300, 4), -1, dtype=torch.int32, device=cuda)
    status = torch.zeros(1, dtype=torch.int32, device=cuda)
    counts = [1 + (i % 3) for i in range(n_req)]
    counts = [c if sum(counts[:i + 1]) <= nblocks else 0 for i, c in enumerate(counts)]
    ids = ref.alloc(counts)
    o.kv_alloc_h(bitmap, nblocks, 7, counts, list(range(n_req)), [0] * n_req, table, status)
    src = list(range(0, 300))
    o.table_copy_h(table, src, [n_req + i for i in range(300)], [1] * 300, [2] * 300)
    torch.cuda.synchronize()
    assert int(status[0]) == 0
    tab = table.cpu().numpy()
    for r, (c, got) in enumerate(zip(counts, ids)):
        assert tab[r, :c].tolist() == list(got)
    for i in range(300):
        assert tab[n_req + i, 1:3].tolist() == tab[i, :2].tolist()
    assert np.array_equal(bitmap.cpu().numpy().view(np.uint32), ref.bitmap_words())


def test_kv_double_free_flagged(cuda):
    o = ops()
    ref = BlockPoolRef(64)
    bitmap = torch.from_numpy(ref.bitmap_words().view(np.int32)).to(cuda)
    table = torch.full((2, 8), -1, dtype=torch.int32, device=cuda)
    status = torch.zeros(1, dtype=torch.int32, device=cuda)
    one = torch.ones(1, dtype=torch.int32, device=cuda)
    zero = torch.zeros(1, dtype=torch.int32, device=cuda)
    o.kv_alloc(bitmap, 64, 0, one * 4, zero, zero, 1, table, status)
    o.kv_free(bitmap, 64, 0, table, zero, zero, one * 4, 1, status)
    torch.cuda.synchronize()
    assert int(status[0]) == 0
    o.kv_free(bitmap, 64, 0, table, zero, zero, one * 4, 1, status)
    torch.cuda.synchronize()
    assert int(status[0]) == -1


@pytest.mark.parametrize("M,N", [(5, 128256), (129, 128256), (212, 128256), (300, 1024),
                                 (64, 1024)])
def test_lm_head_argmax_epilogue(cuda, M, N):
    """Greedy tokens from the lm_head GEMM's argmax epilogue (out mode 3: (max, index) per
    128-column chunk, then cortex_argmax_partials) equal the argmax over the full logits of
    the same GEMM, including exact ties across chunks (first index wins) and a row with no
    finite logit (token 0)."""
    o = ops()
    K = 4096 if N > 1024 else 256
    g = torch.Generator(device=cuda).manual_seed(M + N)
    x = torch.randn(max(M, 32), K, generator=g, device=cuda).to(torch.bfloat16)
    w = (torch.randn(N, K, generator=g, device=cuda) * 0.02).to(torch.bfloat16)
    w[N - 130] = w[7]  # identical rows in different chunks: exact ties, first index wins
    w[N - 1] = w[7]
    x[1] = 0  # a row of zero logits everywhere: the argmax is index 0
    if M > 3:
        x[3, 0] = float("nan")  # NaN logits in every column: token 0
    ws = o.GemmWorkspace(cuda)
    logits = torch.empty(M, N, device=cuda)
    o.gemm(o.weight_map(w), o.act_map(x), M, logits, ws)
    want = torch.empty(M, dtype=torch.int32, device=cuda)
    o.argmax(logits, M, N, out_tok=want)
    part = torch.empty(M, N // 128, dtype=torch.int64, device=cuda)
    o.gemm(o.weight_map(w), o.act_map(x), M, part, ws, argmax=True)
    got = torch.empty(M, dtype=torch.int32, device=cuda)
    o.argmax_partials(part, M, out_tok=got)
    torch.cuda.synchronize()
    assert torch.equal(got, want)
    assert int(got[1]) == 0
    if M > 3:
        assert int(got[3]) == 0
    ties = (logits[:, 7] == logits.max(dim=1).values).nonzero().flatten()
    assert all(int(got[r]) == 7 for r in ties.tolist() if r not in (1, 3))


@pytest.mark.parametrize("mode", [0, 2])
@pytest.mark.parametrize("M,hq,hkv,K", [(5, 32, 8, 4096), (129, 32, 8, 4096), (200, 32, 8, 4096),
                                        (700, 32, 8, 4096), (300, 2, 1, 256), (40, 16, 4, 4096)])
def test_gemm_qkv_rope_epilogue(cuda, mode, M, hq, hkv, K):
    """The QKV GEMM with RoPE + paged KV append in its epilogue (every GEMM path: automatic
    plan = split-K / 2-SM by M, forced 2-SM) against the unfused GEMM + rope_kv_append."""
    o = ops()
    N = (hq + 2 * hkv) * 128
    nb = 256
    g = torch.Generator(device=cuda).manual_seed(M + hq)
    x = torch.randn(max(M, 32), K, generator=g, device=cuda).to(torch.bfloat16)
    w = (torch.randn(N, K, generator=g, device=cuda) * 0.05).to(torch.bfloat16)
    table = torch.randperm(nb * 4, generator=torch.Generator().manual_seed(M))[:nb].to(
        torch.int32).view(8, 32).to(cuda) % nb
    rng = np.random.default_rng(M)
    # distinct (row, col, off) slots per token
    slots = rng.permutation(8 * 32 * 16)[:M]
    rows = torch.as_tensor(slots // (32 * 16), dtype=torch.int32, device=cuda)
    cols = torch.as_tensor((slots // 16) % 32, dtype=torch.int32, device=cuda)
    offs = torch.as_tensor(slots % 16, dtype=torch.int32, device=cuda)
    table = torch.arange(8 * 32, dtype=torch.int32, device=cuda).view(8, 32)  # distinct blocks
    pos = torch.as_tensor(rng.integers(0, 8000, M), dtype=torch.int32, device=cuda)
    cos, sin = rope_tables(8192, 500000.0)
    cos, sin = cos.to(cuda), sin.to(cuda)
    ws = o.GemmWorkspace(cuda)
    k0, v0 = _rows(0, nb, hkv)
    prev = o.gemm_set_mode(mode)
    try:
        qkv = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
        o.gemm(o.weight_map(w), o.act_map(x), M, qkv, ws)
        q_ref = torch.zeros(M, hq, 128, device=cuda, dtype=torch.bfloat16)
        c_ref = torch.zeros(1, 2, nb, hkv, 16, 128, device=cuda, dtype=torch.bfloat16)
        o.rope_kv_append(qkv, q_ref, c_ref, k0, v0, table, pos, rows, cols, offs, cos, sin, M,
                         hq, hkv)
        q_got = torch.zeros_like(q_ref)
        c_got = torch.zeros_like(c_ref)
        tok_dst = torch.empty(M, dtype=torch.int32, device=cuda)
        tok_cs = torch.empty(M, 128, device=cuda)
        o.rope_token_prep(table, pos, rows, cols, offs, cos, sin, M, hkv, tok_dst, tok_cs)
        o.gemm_qkv_rope(o.weight_map(w), o.act_map(x), M, ws, q_got, c_got, k0, v0, tok_dst,
                        tok_cs, hq, hkv)
        torch.cuda.synchronize()
    finally:
        o.gemm_set_mode(prev)
    # same rounding points; only fp32 contraction may differ -> rare 1-ulp bf16 flips
    for got, ref in ((q_got, q_ref), (c_got, c_ref)):
        assert rel(got, ref) < 1e-3
        assert (got != ref).float().mean().item() < 1e-3
