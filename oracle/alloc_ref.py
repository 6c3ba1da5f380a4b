"""CPU oracle of the KV block pool (test infrastructure only).

ORACLE — imported only by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline leg, as the checker. Never part of the product path.

The reference has no block allocator: its engine accounts KV as a token budget
(stagesim/engines.py:111-112, :142-166, :206-226) and the paper's non-goals
exclude "paged-attention block granularity". The block contract is
therefore the builder's, restated here in numpy:

  * a pool of `nblocks` blocks with ids id_base .. id_base+nblocks-1;
  * alloc(counts): all-or-nothing; request i receives the free blocks of global
    free-rank [off_i, off_i + counts[i]) in ascending id order (lowest free
    block first, requests served in the order given);
  * free(ids): returns blocks; freeing a free block or a foreign id is an error.

Parity status: pinned by construction (a contract, not a reference algorithm);
the GPU allocator must match it bit-exactly on every sequence the engine issues.
"""

from __future__ import annotations

import numpy as np


class OutOfBlocks(RuntimeError):
    pass


class BlockPoolRef:
    def __init__(self, nblocks: int, id_base: int = 0) -> None:
        self.nblocks = int(nblocks)
        self.id_base = int(id_base)
        self.free_mask = np.ones(self.nblocks, dtype=bool)

    def n_free(self) -> int:
        return int(self.free_mask.sum())

    def alloc(self, counts: list[int]) -> list[list[int]]:
        need = int(sum(counts))
        free_idx = np.flatnonzero(self.free_mask)
        if need > free_idx.size:
            raise OutOfBlocks(f"need {need} blocks, {free_idx.size} free")
        take = free_idx[:need]
        self.free_mask[take] = False
        out, pos = [], 0
        for c in counts:
            out.append([int(x) + self.id_base for x in take[pos:pos + c]])
            pos += c
        return out

    def free(self, ids) -> None:
        for gid in ids:
            i = int(gid) - self.id_base
            if not 0 <= i < self.nblocks:
                raise ValueError(f"block {gid} not in pool")
            if self.free_mask[i]:
                raise ValueError(f"double free of block {gid}")
            self.free_mask[i] = True

    def bitmap_words(self) -> np.ndarray:
        """The pool as 32-bit words, bit = 1 -> free (the device layout)."""
        nwords = (self.nblocks + 31) // 32
        bits = np.zeros(nwords * 32, dtype=np.uint64)
        bits[: self.nblocks] = self.free_mask
        w = bits.reshape(nwords, 32) << np.arange(32, dtype=np.uint64)
        return w.sum(axis=1).astype(np.uint32)
