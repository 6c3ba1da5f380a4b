"""Deterministic synthetic token ids for prefixes and prompts.

The reference draws one uniform per (seed, label, index) with SHA-256
(stagesim/rng.py:26-29); it never materialises token ids. Drawing millions of
ids that way in Python is far too slow, so token ids use a vectorised
counter-based generator keyed the same way: the 64-bit key is the first 8 bytes
of sha256("{seed}|{label}") and the ids are numpy Philox draws under that key.
Labels: "prefix:{stage_id}" for a stage's schema prefix and
"req:{rid}:tokens:{stage_id}:{visit}" for a call's prompt (visit = how many
times the workflow entered that stage before, the index the reference uses
for the same call's prompt/output length draws, stagesim/simulation.py:526-527).
"""

from __future__ import annotations

import hashlib

import numpy as np


def label_key(seed: int, label: str) -> int:
    return int.from_bytes(hashlib.sha256(f"{seed}|{label}".encode()).digest()[:8], "big")


def token_ids(seed: int, label: str, n: int, vocab: int) -> np.ndarray:
    gen = np.random.Generator(np.random.Philox(key=label_key(seed, label)))
    return gen.integers(0, vocab, size=n, dtype=np.int64).astype(np.int32)


def prefix_tokens(seed: int, stage_id: str, n: int, vocab: int) -> np.ndarray:
    return token_ids(seed, f"prefix:{stage_id}", n, vocab)


def prompt_tokens(seed: int, rid: int, stage_id: str, visit: int, n: int, vocab: int) -> np.ndarray:
    return token_ids(seed, f"req:{rid}:tokens:{stage_id}:{visit}", n, vocab)
