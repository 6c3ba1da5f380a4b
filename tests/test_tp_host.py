"""TP = 2 sharding (tp.py) checked on CPU in fp32: the two ranks' shards of one
decoder layer, each computing attention on its own heads and the MLP on its own
ffn slice, sum (after the O / down projections) to the unsharded layer."""

from __future__ import annotations

import pytest
import torch

from oracle.decoder_ref import attention_ref, rmsnorm_ref, rope_ref, rope_tables
from paper_2510_14126_b200.config import HEAD_DIM, LLAMA3_8B, TINY, TINY_TP
from paper_2510_14126_b200.tp import shard_config, shard_weights


def _weights(cfg, seed=0):
    g = torch.Generator().manual_seed(seed)
    d = cfg.d_model
    r = lambda *s: torch.randn(*s, generator=g) * 0.05  # noqa: E731
    return {"embed": r(cfg.vocab, d), "layers.0.attn_norm": 1 + r(d), "layers.0.mlp_norm": 1 + r(d),
            "layers.0.wqkv": r(cfg.qkv_dim, d), "layers.0.wo": r(d, cfg.n_heads * HEAD_DIM),
            "layers.0.wgu": r(2 * cfg.ffn, d), "layers.0.wd": r(d, cfg.ffn),
            "final_norm": 1 + r(d), "lm_head": r(cfg.vocab, d)}


def _attn(cfg, w, h, pos, cos, sin):
    """Attention contribution of layer 0 (O projection output, before the residual add)."""
    n = h.shape[0]
    hq, hkv = cfg.n_heads, cfg.n_kv_heads
    xn = rmsnorm_ref(h, w["layers.0.attn_norm"], cfg.eps)
    qkv = xn @ w["layers.0.wqkv"].T
    q = rope_ref(qkv[:, :hq * HEAD_DIM].reshape(n, hq, HEAD_DIM), cos, sin)
    k = rope_ref(qkv[:, hq * HEAD_DIM:(hq + hkv) * HEAD_DIM].reshape(n, hkv, HEAD_DIM), cos, sin)
    v = qkv[:, (hq + hkv) * HEAD_DIM:].reshape(n, hkv, HEAD_DIM)
    a = attention_ref(q, k, v, pos, pos).reshape(n, hq * HEAD_DIM)
    return a @ w["layers.0.wo"].T


def test_shard_config():
    s = shard_config(LLAMA3_8B, 2)
    assert (s.n_heads, s.n_kv_heads, s.ffn, s.group) == (16, 4, 7168, 4)
    assert s.d_model == LLAMA3_8B.d_model and s.vocab == LLAMA3_8B.vocab
    assert shard_config(TINY_TP, 2).n_kv_heads == 1
    assert shard_config(TINY, 1) is TINY
    with pytest.raises(ValueError):
        shard_config(TINY, 2)  # one kv head cannot be split


def test_shards_sum_to_the_full_layer():
    cfg = TINY_TP
    w = _weights(cfg)
    n = 12
    g = torch.Generator().manual_seed(1)
    h = torch.randn(n, cfg.d_model, generator=g)
    pos = torch.arange(n)
    cos, sin = rope_tables(64, cfg.rope_theta)
    cos, sin = cos[pos], sin[pos]
    full_attn = _attn(cfg, w, h, pos, cos, sin)
    sc = shard_config(cfg, 2)
    parts = [shard_weights(w, cfg, r, 2) for r in (0, 1)]
    for pw in parts:
        assert pw["layers.0.wqkv"].shape == (sc.qkv_dim, cfg.d_model)
        assert pw["layers.0.wo"].shape == (cfg.d_model, sc.n_heads * HEAD_DIM)
        assert pw["layers.0.wgu"].shape == (2 * sc.ffn, cfg.d_model)
        assert pw["layers.0.wd"].shape == (cfg.d_model, sc.ffn)
        assert pw["lm_head"] is w["lm_head"]  # replicated
    # attention: per-rank heads, partial O projections sum to the full one
    attn_parts = [_attn(sc, pw, h, pos, cos, sin) for pw in parts]
    torch.testing.assert_close(attn_parts[0] + attn_parts[1], full_attn, rtol=1e-5, atol=1e-5)
    # MLP on the all-reduced residual: partial down projections sum to the full one
    h2 = h + full_attn
    xn2 = rmsnorm_ref(h2, w["layers.0.mlp_norm"], cfg.eps)

    def mlp(c, ww):
        gu = xn2 @ ww["layers.0.wgu"].T
        gg, u = gu[:, :c.ffn], gu[:, c.ffn:]
        return (gg / (1 + torch.exp(-gg)) * u) @ ww["layers.0.wd"].T

    torch.testing.assert_close(mlp(sc, parts[0]) + mlp(sc, parts[1]), mlp(cfg, w), rtol=1e-5,
                               atol=1e-5)


# ------------------------------------------------------------------ replica host side


def _logging_worker(n_eng, conc):
    from harness import HostWorker
    from paper_2510_14126_b200.engine import EngineParams, blocks_for

    class LogWorker(HostWorker):
        def forward(self, plan):
            self.log.append(("forward", [(d.row, d.prefix_len, d.kv_len, d.hist_pos)
                                         for d in plan.decode],
                             [(s.row, s.prefix_len, s.kv_len, s.tokens.tolist(), s.out_row)
                              for s in plan.prefill]))
            return super().forward(plan)

    params = EngineParams(1000 + conc * 450, 5000.0, 0.02, 0.1, conc)
    return LogWorker(n_eng * blocks_for(params), n_eng * (conc + 4)), params


def _run_leader(worker, params, conc=8, n_wf=40, mid=None):
    from paper_2510_14126_b200.runtime import PoolRuntime
    from paper_2510_14126_b200.workflow import Constant, Nl2Sql

    spec = Nl2Sql(retry_budget=5, executor_service_time=Constant(0.0))
    rt = PoolRuntime(worker, spec, params, concurrency=conc, n_workflows=n_wf, seed=0,
                     prefill_budget=2048)
    rt.fill()
    rt.run_until(n_wf // 2)
    if mid is not None:
        mid()
    rt.run_until(n_wf)
    return sorted((wf.rid, wf.terminal, tuple(wf.history)) for wf in rt.finished)


def test_tp_leader_follower_mirror_in_process(tmp_path):
    """The follower replays exactly the leader's device calls; the proxy does not
    change scheduling (outcomes equal a TP = 1 run)."""
    from paper_2510_14126_b200.tp import ByteRing, TpFollower, TpLeader

    plain, params = _logging_worker(2, 8)
    out_plain = _run_leader(plain, params)
    lw, _ = _logging_worker(2, 8)
    fw, _ = _logging_worker(2, 8)
    ring = ByteRing(str(tmp_path / "ring"), create=True, cap=1 << 22)
    leader = TpLeader(lw, ring)
    fol = TpFollower(fw, ByteRing(str(tmp_path / "ring"), create=False, cap=1 << 22))
    drained = []

    def drain():  # the follower keeps up (single process: drain between steps)
        while (m := fol.ring.recv()) is not None:
            import pickle

            drained.append(fol.apply(pickle.loads(m)))

    orig = lw.forward

    def fwd(plan):
        n = orig(plan)
        drain()
        return n

    lw.forward = fwd
    out_tp = _run_leader(leader, params)
    leader.stop()
    drain()
    assert out_tp == out_plain
    assert drained[-1] is False and all(drained[:-1])
    assert len(lw.log) > 100
    assert fw.log == lw.log == plain.log
    assert fol.forwards == lw.steps
    ring.close()


def _two_rank(rank, port, path, out):
    import os
    import pickle

    import torch.distributed as dist

    from paper_2510_14126_b200.tp import ByteRing, TpFollower, TpLeader

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    w, params = _logging_worker(2, 8)
    if rank == 0:
        ring = ByteRing(path, create=True, cap=1 << 22)
        dist.barrier()
        leader = TpLeader(w, ring)

        def mid():
            leader.collective("barrier")
            dist.barrier()

        res = _run_leader(leader, params, mid=mid)
        leader.stop()
    else:
        dist.barrier()
        ring = ByteRing(path, create=False, cap=1 << 22)
        TpFollower(w, ring, on_collective=lambda kind, args: dist.barrier()).serve()
        res = None
    dist.barrier()
    with open(f"{out}.{rank}", "wb") as f:
        pickle.dump((res, w.log), f)
    ring.close()
    dist.destroy_process_group()


def test_tp_leader_follower_two_processes(tmp_path):
    import pickle
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "res")
    mp.start_processes(_two_rank, args=(port, str(tmp_path / "ring2"), out), nprocs=2,
                       join=True, start_method="spawn")
    (res0, log0), (_, log1) = [pickle.load(open(f"{out}.{r}", "rb")) for r in (0, 1)]
    plain, params = _logging_worker(2, 8)
    assert res0 == _run_leader(plain, params)
    assert log0 == log1 == plain.log
