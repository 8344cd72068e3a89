"""Batched GPX crossover -- drop-in for the kernel half of `memcolor.crossover`.

* ``build_offspring_batch``  `crossover.py:81-93` (keys stream_key(seed,
  TAG_CROSS, generation, job = i*K + j))
* ``gpx``                    `crossover.py:69-78` (single pair)
* ``gpx_batch``              `crossover.py:60-66` array-level operator

backed by `mcb_gpx_batch_host` (one warp per offspring on sm_100a).
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .coloring import Coloring
from .rng import TAG_CROSS, Stream, stream_keys


def gpx_batch(pop, matches, k, keys):
    """out[i, j] = GPX(pop[i], pop[matches[i, j]]) with stream keys[i*K+j]."""
    pop = np.ascontiguousarray(pop, dtype=np.int32)
    matches = np.ascontiguousarray(matches, dtype=np.int64)
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    p, n = pop.shape
    K = matches.shape[1]
    if matches.shape[0] != p or keys.shape[0] != p * K:
        raise ValueError("matches must be (p, K) and keys (p*K,)")
    out = np.empty((p, K, n), dtype=np.int32)
    L = N.lib()
    P = N.ptr
    N.check(L.mcb_gpx_batch_host(P(pop), p, n, P(matches), K, int(k), P(keys), P(out), 0, None))
    return out


def gpx(parent1, parent2, k, stream):
    """Single crossover of two colorings over the same vertex set."""
    pa = parent1.assign if isinstance(parent1, Coloring) else np.asarray(parent1)
    pb = parent2.assign if isinstance(parent2, Coloring) else np.asarray(parent2)
    if pa.shape != pb.shape:
        raise ValueError("parents must cover the same vertex set")
    key = stream.key if isinstance(stream, Stream) or hasattr(stream, "key") else int(stream)
    # a two-row batch: child (0, 0) = GPX(row 0, row 1) with `key`
    pop = np.stack([pa, pb]).astype(np.int32)
    out = gpx_batch(pop, np.array([[1], [0]], dtype=np.int64), k,
                    np.array([key, 0], dtype=np.uint64))
    return Coloring(out[0, 0], k)


def build_offspring_batch(pop_assigns, matches, k, master_seed, generation):
    """All p*K offspring; per-pair RNG streams keep the batch deterministic."""
    p, K = matches.shape
    keys = stream_keys(master_seed, TAG_CROSS, generation, p * K)
    return gpx_batch(np.asarray(pop_assigns).astype(np.int32), np.asarray(matches).astype(np.int64),
                     k, keys)
