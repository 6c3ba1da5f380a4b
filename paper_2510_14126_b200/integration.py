"""Plugging GPU engines into the reference `Simulator`.

The reference constructs engines at exactly one seam,
`Simulator._add_engine(pool_id, params)` (stagesim/simulation.py:363-369, also
reached on autoscale scale-out at :799). `gpu_engine_factory` returns the
callable that seam needs: it carves the next engine's block range and table
rows out of a `GpuWorker` arena and returns a `GpuEngineState`. See
INTEGRATION.md for the subclass a reference maintainer adds.

Elastic pools. Borrowing (simulation.py:715-763) needs no
hook: a lent engine admits the borrower stage's calls through the ordinary
`admit`, which plants that stage's prefix cold on the engine's GPU blocks
(re-materialising the borrowed stage's schema prefix there) and serves it until
eviction. Autoscale scale-out (simulation.py:797-799) goes through
`_add_engine` like any engine. Scale-in (simulation.py:800-809) moves the idle
victim to `retired_engines` with no hook, so `gpu_simulator` also overrides
`_apply_scale`: after the reference's own decision, every engine that just
retired is closed (its resident prefixes' blocks return to its bitmap) and its
arena slice is recycled for the next scale-out. `gpu_simulator` also keeps a
per-sample block count beside the reference's `kv_usage.csv` samples
(`kv_blocks.csv`: the reference's columns plus `kv_blocks`).
"""

from __future__ import annotations

import csv
from pathlib import Path

from .engine import EngineObserver, EngineSlice, GpuEngineState, TokenSource, blocks_for
from .errors import InternalInvariantViolation


def gpu_engine_factory(worker, params_hint, seed: int = 0, n_prefix_rows: int = 4,
                       observer: EngineObserver | None = None):
    """Returns factory(engine_id, params, pool_id) -> GpuEngineState.

    Each engine gets blocks_for(params) blocks (enough that token admission can
    never be followed by block exhaustion) and max_batch + n_prefix_rows rows.
    `factory.release(engine)` closes a retired engine and recycles its slice; a
    new engine takes the lowest recycled slice of its size before fresh arena.
    `factory.assigned[engine_id]` = (block_base, n_blocks) of every engine made.
    """
    tokens = TokenSource(seed, worker.cfg.vocab)
    state = {"next_block": 0, "next_row": 0}
    free_slices: list[EngineSlice] = []
    assigned: dict[int, tuple[int, int]] = {}

    def factory(engine_id: int, params, pool_id: str) -> GpuEngineState:
        nb = blocks_for(params, n_prefix_rows)
        rows = params.max_batch + n_prefix_rows
        reuse = [s for s in free_slices
                 if s.n_blocks == nb and len(s.slot_rows) == params.max_batch
                 and len(s.prefix_rows) == n_prefix_rows]
        if reuse:
            sl = min(reuse, key=lambda s: s.block_base)
            free_slices.remove(sl)
        else:
            b0, r0 = state["next_block"], state["next_row"]
            if b0 + nb > worker.n_blocks or r0 + rows > worker.table.shape[0]:
                raise InternalInvariantViolation(
                    f"GPU arena exhausted creating engine {engine_id} for {pool_id}")
            if worker.table.shape[1] < nb:
                raise InternalInvariantViolation(
                    "block-table rows too short for the engine capacity")
            state["next_block"] += nb
            state["next_row"] += rows
            sl = EngineSlice(worker, b0, nb, list(range(r0, r0 + params.max_batch)),
                             list(range(r0 + params.max_batch, r0 + rows)), tokens)
        assigned[engine_id] = (sl.block_base, sl.n_blocks)
        return GpuEngineState(engine_id, params, pool_id, sl, observer)

    def release(engine: GpuEngineState) -> None:
        if engine.closed:
            return
        engine.close()
        free_slices.append(engine.gpu)

    factory.tokens = tokens
    factory.release = release
    factory.assigned = assigned
    return factory


KV_BLOCKS_HEADER = ["time", "pool", "engine", "kv_used_tokens", "resident_prefix_tokens",
                    "kv_blocks"]


def gpu_simulator(base, factory):
    """Subclass of the reference Simulator class `base` whose engines are GPU engines.

    Overrides (reference lines): `_add_engine` (simulation.py:363-369, the factory
    seam), `_apply_scale` (:796-809, closes engines the scale-in retired) and
    `_emit_kv_samples` (:455-463, records the block count of every sample the
    reference emits). Everything else — routing, borrowing, autoscale decisions,
    reports — is the reference's own code.
    """

    class GpuSimulator(base):
        def _add_engine(self, pool_id, params):
            engine = factory(self._next_engine_id, params, pool_id)
            engine.last_advance = self.clock
            self.engines[engine.engine_id] = engine
            self._kv_integral[engine.engine_id] = 0.0
            self._next_engine_id += 1
            return engine

        def _apply_scale(self, pool, decision):
            super()._apply_scale(pool, decision)
            for engine in self.retired_engines.values():
                if not engine.closed:
                    factory.release(engine)

        def _emit_kv_samples(self, force: bool = False):
            if not hasattr(self, "kv_block_samples"):
                self.kv_block_samples = []
            n0 = len(self.traces.kv_samples)
            super()._emit_kv_samples(force)
            for s in self.traces.kv_samples[n0:]:
                self.kv_block_samples.append((s, self.engines[s.engine_id].blocks_in_use))

        def write_kv_blocks(self, path) -> None:
            """kv_usage.csv's rows (its 9-decimal formatting, reporting.py:24-25) plus the
            engine's block count."""
            with Path(path).open("w", newline="") as f:
                w = csv.writer(f, lineterminator="\n")
                w.writerow(KV_BLOCKS_HEADER)
                for s, nb in getattr(self, "kv_block_samples", []):
                    w.writerow([f"{s.time:.9f}", s.pool, s.engine_id, f"{s.kv_used:.9f}",
                                s.resident_prefix_tokens, nb])

    GpuSimulator.__name__ = "Gpu" + base.__name__
    return GpuSimulator
