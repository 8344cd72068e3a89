"""Partition distances -- drop-in for `memcolor.distance`.

* ``pairwise_distances``        `distance.py:122-155` -> `mcb_pairwise_host`
* ``approx_partition_distance`` `distance.py:75-79`
* ``overlap_matrix``            `distance.py:30-37` (host helper, numpy)
* ``exact_partition_distance``  `distance.py:82-87` (Hungarian; scipy, not a
  hot-path operator -- kept for API completeness)

The value is the reference's greedy approximation, computed on the GPU by
`csrc/distance.cu` with bit-identical results (including its label dependence).
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .coloring import Coloring


def _as_assign_pair(a, b):
    aa = a.assign if isinstance(a, Coloring) else np.asarray(a, dtype=np.int32)
    bb = b.assign if isinstance(b, Coloring) else np.asarray(b, dtype=np.int32)
    if aa.shape != bb.shape:
        raise ValueError("colorings must cover the same vertex set")
    ka = (a.k if isinstance(a, Coloring) else int(aa.max()) + 1) if aa.size else 0
    kb = (b.k if isinstance(b, Coloring) else int(bb.max()) + 1) if bb.size else 0
    return aa, bb, max(ka, kb)


def overlap_matrix(a, b, k=None):
    """M[c, c'] = number of vertices in class c of `a` and class c' of `b`."""
    aa, bb, kk = _as_assign_pair(a, b)
    if k is None:
        k = kk
    m = np.zeros((k, k), dtype=np.int64)
    np.add.at(m, (aa, bb), 1)
    return m


def pairwise_raw(pop, off, k, job_begin=0, job_end=-1, cross=None, within=None):
    """Array-level operator (`_pairwise_kernel`, `distance.py:90-119`)."""
    pop = np.ascontiguousarray(pop, dtype=np.int32)
    off = np.ascontiguousarray(off, dtype=np.int32)
    p, q = pop.shape[0], off.shape[0]
    n = off.shape[1] if off.ndim == 2 else pop.shape[1]
    if pop.ndim == 2 and pop.shape[0] and pop.shape[1] != n:
        raise ValueError("colorings must cover the same vertex set")
    if cross is None:
        cross = np.zeros((p, q), dtype=np.int32)
    if within is None:
        within = np.zeros((q, q), dtype=np.int32)
    if p * q + q * (q - 1) // 2 == 0 or n == 0:
        return cross, within
    L = N.lib()
    P = N.ptr
    N.check(L.mcb_pairwise_host(P(pop), p, P(off), q, n, int(k), P(cross), P(within),
                                int(job_begin), int(job_end), 0, None))
    return cross, within


def pairwise_distances(pop, offspring, k=None, thread_count=None):
    """All pop-vs-offspring and offspring-vs-offspring approximate distances.

    Returns (cross, within): cross[i, j] = d(pop_i, off_j); within is the
    symmetric offspring matrix with a zero diagonal.  ``thread_count`` is
    accepted for API compatibility and ignored.
    """
    pop_arr = (np.stack([c.assign for c in pop])
               if len(pop) and isinstance(pop[0], Coloring) else np.asarray(pop))
    off_arr = (np.stack([c.assign for c in offspring])
               if len(offspring) and isinstance(offspring[0], Coloring) else np.asarray(offspring))
    pop_arr = pop_arr.astype(np.int32)
    off_arr = off_arr.astype(np.int32)
    if k is None:
        k = 1 + max(int(pop_arr.max()) if pop_arr.size else 0,
                    int(off_arr.max()) if off_arr.size else 0)
    if pop_arr.ndim == 1:
        pop_arr = pop_arr.reshape(0, off_arr.shape[1] if off_arr.ndim == 2 else 0)
    return pairwise_raw(pop_arr, off_arr, k)


def approx_partition_distance(a, b):
    """Greedy upper bound on the partition distance (`distance.py:75-79`)."""
    aa, bb, k = _as_assign_pair(a, b)
    if aa.size == 0:
        return 0
    cross, _ = pairwise_raw(aa[None, :], bb[None, :], k)
    return int(cross[0, 0])


def exact_partition_distance(a, b):
    """Exact partition distance via maximum-weight assignment."""
    from scipy.optimize import linear_sum_assignment

    aa, bb, k = _as_assign_pair(a, b)
    m = overlap_matrix(aa, bb, k)
    rows, cols = linear_sum_assignment(m, maximize=True)
    return int(aa.size - m[rows, cols].sum())
