"""Population update and parent matching -- drop-in for `memcolor.population`.

* ``min_spacing``              `mc/population.py:20-21`
* ``Population``               `:24-56` (same fields; ``from_colorings`` uses the
  GPU pairwise distances, `distance.py`)
* ``update_population``        `:59-127` -> `mcb_update_population_host`
* ``match_parents``            `:130-141` -> `mcb_match_parents_host`

Both operators run on the GPU (`csrc/population.cu`) with the reference's exact
semantics: candidates ranked by (fitness, origin, index), admitted while their
distance to every admitted one exceeds ``ms``, the best rejected ones filling
the remaining slots; neighbours ordered by (distance, index).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .coloring import Coloring


def min_spacing(n, divisor=10):
    return n // divisor


@dataclass
class Population:
    assigns: np.ndarray  # (p, n) int32
    k: int
    fitness: np.ndarray  # (p,) int64
    dist: np.ndarray  # (p, p) int32, symmetric, zero diagonal
    generation: int = 0
    admitted_by_rule: np.ndarray = None  # bool mask; False = fallback fill

    @property
    def p(self):
        return self.assigns.shape[0]

    @property
    def n(self):
        return self.assigns.shape[1]

    def colorings(self):
        return [Coloring(self.assigns[i], self.k) for i in range(self.p)]

    @classmethod
    def from_colorings(cls, colorings, fitness, generation=0):
        from .distance import pairwise_distances

        assigns = np.stack([c.assign for c in colorings]).astype(np.int32)
        k = colorings[0].k
        _, within = pairwise_distances(assigns[:0], assigns, k=k)
        return cls(assigns=assigns, k=k, fitness=np.asarray(fitness, dtype=np.int64), dist=within,
                   generation=generation, admitted_by_rule=np.ones(len(colorings), dtype=bool))


def _i32(a, shape, name):
    a = np.ascontiguousarray(a, dtype=np.int32)
    if a.shape != shape:
        raise ValueError(f"{name} must have shape {shape}, got {a.shape}")
    return a


def update_population(pop, improved_assigns, improved_fitness, cross, within, ms):
    """Merge the p incumbents and q newcomers, keep p (`population.py:59-127`)."""
    p, n = pop.assigns.shape
    improved_assigns = np.ascontiguousarray(improved_assigns, dtype=np.int32)
    improved_fitness = np.ascontiguousarray(improved_fitness, dtype=np.int64)
    q = improved_assigns.shape[0]
    if improved_assigns.ndim != 2 or (q and improved_assigns.shape[1] != n):
        raise ValueError("improved_assigns must be (q, n)")
    if improved_fitness.shape != (q,):
        raise ValueError("improved_fitness must be (q,)")
    pdist = _i32(pop.dist, (p, p), "pop.dist")
    cross = _i32(cross, (p, q), "cross")
    within = _i32(within, (q, q), "within")
    pa = np.ascontiguousarray(pop.assigns, dtype=np.int32)
    fit = np.ascontiguousarray(pop.fitness, dtype=np.int64)
    adm = np.empty(p, dtype=np.int32)
    rule = np.empty(p, dtype=np.uint8)
    new_dist = np.empty((p, p), dtype=np.int32)
    new_assigns = np.empty((p, n), dtype=np.int32)
    new_fit = np.empty(p, dtype=np.int64)
    P = N.ptr
    N.check(N.lib().mcb_update_population_host(
        P(pdist), P(cross), P(within), P(fit), P(improved_fitness), p, q, int(ms), P(pa),
        P(improved_assigns), n, P(adm), P(rule), P(new_dist), P(new_assigns), P(new_fit), None))
    return Population(assigns=new_assigns, k=pop.k, fitness=new_fit, dist=new_dist,
                      generation=pop.generation + 1, admitted_by_rule=rule.astype(bool))


def match_parents(pop, K):
    """K nearest neighbours of each individual, ties by lower index (`:130-141`)."""
    p = pop.p
    if not (0 < K < p):
        raise ValueError("need 0 < K < p")
    dist = _i32(pop.dist, (p, p), "pop.dist")
    matches = np.empty((p, K), dtype=np.int64)
    max_dist = int(pop.n)  # partition distances are <= n (distance.py:75-79)
    N.check(N.lib().mcb_match_parents_host(N.ptr(dist), p, int(K), max_dist, N.ptr(matches), None))
    return matches
