"""Graph arrays consumed by the batched kernels.

Host mirror of ``WeightedGraph`` (`pkg/src/memcolor/graph.py:26-75`): the
kernels read exactly the arrays the reference passes to its numba kernels
(`pkg/src/memcolor/localsearch.py:418-424`):

* ``adj_indptr`` int64[n+1] / ``adj_indices`` int32[2m] -- CSR with every
  neighbour list sorted ascending (`graph.py:57-68`); TabuCol's conflict-list
  order depends on that sort, so it is part of the contract;
* ``edges`` int32[m, 2], lexicographically sorted, ``u < v`` (`graph.py:38-47`);
* ``weights`` int64[n] >= 1, ``weight_values`` (sorted distinct weights) and
  ``weight_ranks`` int32[n] (dense rank of each weight) (`graph.py:70-73`).

Construction is vectorised (the reference builds Python sets/lists), so the
1M-edge G(2000, 0.5) of config 5 builds in well under a second.  Any object
carrying these attributes -- including the reference's own ``WeightedGraph`` --
is accepted by the operator shims.
"""

from __future__ import annotations

import numpy as np

from .rng import batch_uniform, stream_values


class WeightedGraph:
    """Immutable undirected graph with positive integer vertex weights."""

    def __init__(self, n, edges, weights, name=""):
        if n <= 0:
            raise ValueError("graph must have at least one vertex")
        self.n = int(n)
        self.name = name
        e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
        if e.size:
            if (e[:, 0] == e[:, 1]).any():
                bad = int(e[e[:, 0] == e[:, 1]][0, 0])
                raise ValueError(f"self-loop on vertex {bad}")
            if (e < 0).any() or (e >= n).any():
                raise ValueError("edge endpoint out of range")
            lo = np.minimum(e[:, 0], e[:, 1])
            hi = np.maximum(e[:, 0], e[:, 1])
            code = np.unique(lo * self.n + hi)  # dedup + lexicographic sort
            e = np.stack([code // self.n, code % self.n], axis=1)
        self.edges = e.astype(np.int32).reshape(-1, 2)
        self.m = int(self.edges.shape[0])

        self.weights = np.asarray(weights, dtype=np.int64)
        if self.weights.shape != (self.n,):
            raise ValueError(f"expected {self.n} weights, got {self.weights.shape}")
        if (self.weights < 1).any():
            bad = int(np.argmax(self.weights < 1))
            raise ValueError(f"non-positive weight {self.weights[bad]} on vertex {bad}")

        # CSR with ascending neighbour lists: sort both directions by (src, dst)
        src = np.concatenate([self.edges[:, 0], self.edges[:, 1]]).astype(np.int64)
        dst = np.concatenate([self.edges[:, 1], self.edges[:, 0]]).astype(np.int64)
        order = np.argsort(src * self.n + dst, kind="stable")
        self.degrees = np.bincount(src, minlength=self.n).astype(np.int32)
        self.adj_indptr = np.zeros(self.n + 1, dtype=np.int64)
        np.cumsum(self.degrees, out=self.adj_indptr[1:])
        self.adj_indices = dst[order].astype(np.int32)

        self.max_weight = int(self.weights.max())
        self.weight_values = np.unique(self.weights)
        self.weight_ranks = np.searchsorted(self.weight_values, self.weights).astype(np.int32)
        self._adjacency = None

    @property
    def adjacency(self):
        if self._adjacency is None:
            self._adjacency = [
                self.adj_indices[self.adj_indptr[v]:self.adj_indptr[v + 1]]
                for v in range(self.n)
            ]
        return self._adjacency

    def neighbors(self, v):
        return self.adj_indices[self.adj_indptr[v]:self.adj_indptr[v + 1]]

    def has_edge(self, u, v):
        nb = self.neighbors(u)
        i = np.searchsorted(nb, v)
        return bool(i < nb.size and nb[i] == v)

    def density(self):
        possible = self.n * (self.n - 1) / 2
        return self.m / possible if possible else 0.0

    @property
    def max_degree(self):
        return int(self.degrees.max()) if self.n else 0

    def __eq__(self, other):
        return (
            hasattr(other, "edges")
            and self.n == other.n
            and np.array_equal(self.edges, other.edges)
            and np.array_equal(self.weights, other.weights)
        )

    def __repr__(self):
        return f"WeightedGraph(name={self.name!r}, n={self.n}, m={self.m})"


def rand_graph(seed, n, edge_prob=0.5, wmax=1, name=None):
    """Seeded G(n, p) with weights ``1 + below(wmax)``.

    Follows the reference test-oracle convention (`pkg/tests/oracles.py:15-22`):
    a raw-key ``Stream(seed)``; one ``uniform()`` per pair (u < v) in
    lexicographic order, edge iff ``< edge_prob``; then the weights continue
    the same stream.  Vectorised through ``batch_uniform`` (`rng.py:85-96`).
    """
    npairs = n * (n - 1) // 2
    u = batch_uniform(seed, 0, npairs)
    iu, iv = np.triu_indices(n, k=1)  # row-major (u, v), u < v == lexicographic
    mask = u < edge_prob
    edges = np.stack([iu[mask], iv[mask]], axis=1)
    w = stream_values(np.uint64(int(seed) & 0xFFFFFFFFFFFFFFFF),
                      np.arange(npairs, npairs + n, dtype=np.uint64))
    weights = (w % np.uint64(wmax)).astype(np.int64) + 1
    return WeightedGraph(n, edges, weights, name=name or f"rand{seed}")


def graph_arrays(g):
    """The kernel's graph inputs, contiguous (`localsearch.py:418-424`)."""
    return (
        np.ascontiguousarray(g.adj_indptr, dtype=np.int64),
        np.ascontiguousarray(g.adj_indices, dtype=np.int32),
        np.ascontiguousarray(g.edges[:, 0], dtype=np.int32),
        np.ascontiguousarray(g.edges[:, 1], dtype=np.int32),
    )
