"""Solution representation (host mirror of `pkg/src/memcolor/coloring.py:16-75`).

``Coloring`` is the I/O type of every operator: an int32 colour per vertex
over a palette of k slots, range-checked on construction (`coloring.py:24-25`).
``col_conflicts`` / ``wvcp_score`` are the from-scratch objectives the kernels'
incremental state must agree with.
"""

from __future__ import annotations

import numpy as np


class Coloring:
    """Per-vertex colour assignment over a fixed palette of k slots."""

    def __init__(self, assign, k):
        self.assign = np.asarray(assign, dtype=np.int32).copy()
        self.k = int(k)
        if self.assign.size == 0:
            raise ValueError("empty coloring")
        if (self.assign < 0).any() or (self.assign >= self.k).any():
            raise ValueError("color id out of range [0, k)")

    @property
    def n(self):
        return self.assign.size

    @property
    def group_sizes(self):
        return np.bincount(self.assign, minlength=self.k)

    def copy(self):
        return Coloring(self.assign, self.k)

    def __eq__(self, other):
        return (
            hasattr(other, "assign")
            and self.k == other.k
            and np.array_equal(self.assign, other.assign)
        )

    def __repr__(self):
        return f"Coloring(n={self.n}, k={self.k})"


def _as_assign(s):
    return s.assign if hasattr(s, "assign") else np.asarray(s)


def col_conflicts(g, s):
    """Number of monochromatic edges (`coloring.py:70-75`)."""
    assign = _as_assign(s)
    if g.m == 0:
        return 0
    return int((assign[g.edges[:, 0]] == assign[g.edges[:, 1]]).sum())


def col_conflicts_batch(g, assigns):
    """Conflicts of every row of an int[p, n] array."""
    assigns = np.asarray(assigns)
    if g.m == 0:
        return np.zeros(assigns.shape[0], dtype=np.int64)
    return (assigns[:, g.edges[:, 0]] == assigns[:, g.edges[:, 1]]).sum(axis=1).astype(np.int64)


def wvcp_score(g, s):
    """(score, conflicts): score = sum over non-empty classes of their max
    weight (`coloring.py:53-67`)."""
    assign = _as_assign(s)
    k = int(assign.max()) + 1 if not hasattr(s, "k") else s.k
    mx = np.zeros(k, dtype=np.int64)
    np.maximum.at(mx, assign, g.weights)
    return int(mx.sum()), col_conflicts(g, assign)


def wvcp_score_batch(g, assigns, k):
    assigns = np.asarray(assigns)
    p = assigns.shape[0]
    mx = np.zeros((p, k), dtype=np.int64)
    rows = np.repeat(np.arange(p), assigns.shape[1])
    np.maximum.at(mx, (rows, assigns.reshape(-1)), np.tile(g.weights, p))
    return mx.sum(axis=1), col_conflicts_batch(g, assigns)
