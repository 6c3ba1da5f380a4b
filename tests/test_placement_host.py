"""Disjoint generator/fixer placement (placement.py) on CPU: world_size 2 over gloo,
host-only workers. Checks that handing workflows across ranks reproduces the
single-rank outcomes exactly (the same terminal states and stage histories) and
that the closed loop keeps its concurrency bound."""

from __future__ import annotations

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_14126_b200.engine import EngineParams, blocks_for
from paper_2510_14126_b200.placement import (
    ROLE_BOTH,
    ROLE_FIXER,
    ROLE_GENERATOR,
    PairChannel,
    open_pair_channel,
    role_of,
)
from paper_2510_14126_b200.runtime import PoolRuntime
from paper_2510_14126_b200.workflow import FIXER, Nl2Sql

from harness import HostWorker

N_WF = 48
CONC = 8


def _runtime(role, channel, n_eng):
    params = EngineParams(1000 + CONC * 450, 5000.0, 0.02, 0.1, CONC)
    bpe = blocks_for(params)
    w = HostWorker(n_eng * bpe, n_eng * (CONC + 4))
    spec = Nl2Sql(retry_budget=5, executor_service_time=_fast_exec())
    return PoolRuntime(w, spec, params, concurrency=CONC, n_workflows=N_WF, seed=0,
                       prefill_budget=2048, role=role, channel=channel)


def _fast_exec():
    from paper_2510_14126_b200.workflow import Constant

    return Constant(0.0)


def _summary(rt):
    return sorted((wf.rid, wf.terminal, tuple(wf.history)) for wf in rt.finished)


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    role, _, _ = role_of(rank, world)
    ch = open_pair_channel(dist, rank, world, cap=4 * CONC)
    rt = _runtime(role, ch, 1)
    rt.fill()
    if role == ROLE_GENERATOR:
        max_inflight = 0
        while rt._next_rid_i < N_WF or rt.workflows or rt.remote:
            rt.step()
            max_inflight = max(max_inflight, len(rt.workflows) + rt.remote)
        ch.phase = 1
    else:
        max_inflight = 0
        while ch.phase == 0:
            rt.step()
            max_inflight = max(max_inflight, len(rt.workflows))
        rt.step()
    q.put((rank, _summary(rt), rt.stats.handoffs, max_inflight, rt.worker.steps))
    dist.barrier()
    ch.close()
    dist.destroy_process_group()


def test_role_of():
    assert role_of(0, 1) == (ROLE_BOTH, 0, -1)
    assert role_of(0, 2) == (ROLE_GENERATOR, 0, 1)
    assert role_of(1, 2) == (ROLE_FIXER, 0, 0)
    assert role_of(5, 8) == (ROLE_FIXER, 1, 1)
    assert role_of(2, 3)[0] == ROLE_BOTH


def test_ring_roundtrip():
    ch = PairChannel(f"cortex_test_{os.getpid()}", create=True, cap=4)
    try:
        for i in range(3):
            ch.to_fixer.push(i, 0.5 * i)
        assert ch.to_fixer.pop_all() == [(0, 0.0), (1, 0.5), (2, 1.0)]
        assert ch.to_fixer.pop_all() == []
        for i in range(4):  # wraps
            ch.to_fixer.push(10 + i, 1.25)
        with pytest.raises(RuntimeError):
            ch.to_fixer.push(99, 0.0)
        assert [r for r, _ in ch.to_fixer.pop_all()] == [10, 11, 12, 13]
        ch.phase = 3
        assert ch.phase == 3 and ch.to_generator.pop_all() == []
    finally:
        ch.close()


def test_disjoint_pair_matches_single_rank():
    rt = _runtime(ROLE_BOTH, None, 2)
    rt.fill()
    rt.run_until(N_WF, max_seconds=120)
    want = _summary(rt)
    assert len(want) == N_WF

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        rank, summ, handoffs, inflight, steps = q.get(timeout=180)
        res[rank] = (summ, handoffs, inflight, steps)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    gen, fix = res[0], res[1]
    got = sorted(gen[0] + fix[0])
    assert got == want
    fixed = [s for s in want if any(st == FIXER for st, _ in s[2])]
    assert gen[1] == len(fixed) == len(fix[0]) and fixed
    assert gen[2] <= CONC
    assert fix[3] > 0
