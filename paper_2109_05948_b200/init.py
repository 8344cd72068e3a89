"""Initial populations (`pkg/src/memcolor/init.py`).

k-colouring (`:49-54,67-71`): ``random_col_init(n, k, Stream.derive(seed,
TAG_INIT, i))`` draws one ``below(k)`` per vertex in vertex order;
``random_col_assigns`` produces the whole population at once with the same
draws.

Weighted runs (`:23-46,57-64`): randomized greedy colourings, all p built at
once on the GPU by ``mcb_greedy_wvcp_init`` (csrc/init.cu), one warp per
individual, with the reference's streams -- identical colourings.
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
    assigns = random_col_assigns(n, k, p, master_seed)
    return InitOutcome(colorings=[Coloring(a, k) for a in assigns], k=k)


def greedy_order(g):
    """Vertices by weight desc, then degree desc, then id asc (`init.py:23-27`)."""
    return np.lexsort((np.arange(g.n), -np.asarray(g.degrees), -np.asarray(g.weights)))


def greedy_wvcp_assigns(g, keys, device=False):
    """int32[p, n] greedy colourings and int32[p] colours used, one per stream
    key (``keys[i] = stream_key(seed, TAG_INIT, i)``).  With ``device=True``
    the inputs/outputs are torch CUDA tensors and nothing leaves the GPU."""
    from . import _native as N

    order = np.ascontiguousarray(greedy_order(g), dtype=np.int32)
    if device:
        import torch

        dev = torch.device("cuda")
        keys_t = torch.as_tensor(np.asarray(keys, dtype=np.uint64).view(np.int64), device=dev)
        p = keys_t.shape[0]
        assigns = torch.empty((p, g.n), dtype=torch.int32, device=dev)
        used = torch.empty(p, dtype=torch.int32, device=dev)
        order_t = torch.as_tensor(order, device=dev)
        ip = torch.as_tensor(g.adj_indptr, device=dev)
        ix = torch.as_tensor(g.adj_indices if len(g.adj_indices) else np.zeros(1, np.int32), device=dev)
        N.check(N.lib().mcb_greedy_wvcp_init(N.ptr(order_t), N.ptr(ip), N.ptr(ix), g.n, N.ptr(keys_t), p,
                                            N.ptr(assigns), N.ptr(used),
                                            torch.cuda.current_stream().cuda_stream))
        return assigns, used
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    p = keys.shape[0]
    assigns = np.empty((p, g.n), dtype=np.int32)
    used = np.empty(p, dtype=np.int32)
    ip = np.ascontiguousarray(g.adj_indptr, dtype=np.int64)
    ix = np.ascontiguousarray(g.adj_indices if len(g.adj_indices) else np.zeros(1, np.int32), dtype=np.int32)
    N.check(N.lib().mcb_greedy_wvcp_init_host(N.ptr(order), N.ptr(ip), N.ptr(ix), g.n, N.ptr(keys), p,
                                             N.ptr(assigns), N.ptr(used), None))
    return assigns, used


def greedy_wvcp_init(g, stream):
    """One randomized greedy colouring (`init.py:30-46`), legal by
    construction; ``stream`` is a fresh ``Stream`` (its key is used)."""
    a, used = greedy_wvcp_assigns(g, np.array([stream.key], dtype=np.uint64))
    return Coloring(a[0], int(used[0]))


def init_wvcp_population(g, p, master_seed):
    """p greedy colourings re-padded to the common palette (`init.py:57-64`)."""
    assigns, used = greedy_wvcp_assigns(g, stream_keys_init(master_seed, p))
    k = int(used.max()) if p else 0
    return InitOutcome(colorings=[Coloring(a, k) for a in assigns], k=k)


class InitOutcome:
    def __init__(self, colorings, k):
        self.colorings = colorings
        self.k = k


__all__ = ["random_col_init", "random_col_assigns", "init_col_population", "stream_keys",
           "greedy_order", "greedy_wvcp_assigns", "greedy_wvcp_init", "init_wvcp_population"]
