"""Plugging GPU engines into the reference `Simulator`.

The reference constructs engines at exactly one seam,
`Simulator._add_engine(pool_id, params)` (stagesim/simulation.py:363-369, also
reached on autoscale scale-out at :799). `gpu_engine_factory` returns the
callable that seam needs: it carves the next engine's block range and table
rows out of a `GpuWorker` arena and returns a `GpuEngineState`. See
INTEGRATION.md for the three-line subclass a reference maintainer adds.
"""

from __future__ import annotations

from .engine import EngineObserver, EngineSlice, GpuEngineState, TokenSource, blocks_for
from .errors import InternalInvariantViolation


def gpu_engine_factory(worker, params_hint, seed: int = 0, n_prefix_rows: int = 4,
                       observer: EngineObserver | None = None):
    """Returns factory(engine_id, params, pool_id) -> GpuEngineState.

    Each engine gets blocks_for(params) blocks (enough that token admission can
    never be followed by block exhaustion) and max_batch + n_prefix_rows rows.
    """
    tokens = TokenSource(seed, worker.cfg.vocab)
    state = {"next_block": 0, "next_row": 0}

    def factory(engine_id: int, params, pool_id: str) -> GpuEngineState:
        nb = blocks_for(params, n_prefix_rows)
        rows = params.max_batch + n_prefix_rows
        b0, r0 = state["next_block"], state["next_row"]
        if b0 + nb > worker.n_blocks or r0 + rows > worker.table.shape[0]:
            raise InternalInvariantViolation(
                f"GPU arena exhausted creating engine {engine_id} for {pool_id}")
        if worker.table.shape[1] < nb:
            raise InternalInvariantViolation("block-table rows too short for the engine capacity")
        state["next_block"] += nb
        state["next_row"] += rows
        sl = EngineSlice(worker, b0, nb, list(range(r0, r0 + params.max_batch)),
                         list(range(r0 + params.max_batch, r0 + rows)), tokens)
        return GpuEngineState(engine_id, params, pool_id, sl, observer)

    factory.tokens = tokens
    return factory
