"""Uniform random initial colourings (`pkg/src/memcolor/init.py:49-54,67-71`).

``random_col_init(n, k, Stream.derive(seed, TAG_INIT, i))`` draws one
``below(k)`` per vertex in vertex order; ``random_col_assigns`` produces the
whole population at once with the same draws.
"""

from __future__ import annotations

import numpy as np

from .coloring import Coloring
from .rng import TAG_INIT, stream_keys, stream_values


def random_col_init(n, k, stream):
    if k < 1:
        raise ValueError("k must be at least 1")
    return Coloring(stream.below_many(k, n).astype(np.int32), k)


def random_col_assigns(n, k, p, master_seed, start=0):
    """int32[p, n]: row i == ``random_col_init(n, k, Stream.derive(seed,
    TAG_INIT, start + i)).assign``."""
    if k < 1:
        raise ValueError("k must be at least 1")
    keys = stream_keys_init(master_seed, p, start)
    v = stream_values(keys[:, None], np.arange(n, dtype=np.uint64)[None, :])
    return (v % np.uint64(k)).astype(np.int32)


def stream_keys_init(master_seed, p, start=0):
    """``stream_key(seed, TAG_INIT, i)`` (single index) for i in range."""
    from .rng import GOLDEN, MASK64, mix64, mix64_int
    base = mix64_int((int(master_seed) & MASK64) ^ ((TAG_INIT * GOLDEN) & MASK64))
    idx = np.arange(start, start + p, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(base) + idx * np.uint64(GOLDEN) + np.uint64(1)
    return mix64(z)


def init_col_population(n, k, p, master_seed):
    from dataclasses import dataclass

    assigns = random_col_assigns(n, k, p, master_seed)
    return InitOutcome(colorings=[Coloring(a, k) for a in assigns], k=k)


class InitOutcome:
    def __init__(self, colorings, k):
        self.colorings = colorings
        self.k = k


__all__ = ["random_col_init", "random_col_assigns", "init_col_population", "stream_keys"]
