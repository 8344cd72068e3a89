"""CPU restatement of the reference's randomized greedy initialisation.

TEST INFRASTRUCTURE ONLY (the checker of csrc/init.cu): imported by tests/
only.  Restatement of `/root/reference/pkg/src/memcolor/init.py`:

* ``greedy_order``         :23-27  weight desc, degree desc, id asc
* ``greedy_wvcp_init``     :30-46  one draw ``below(len(allowed))`` per vertex
                                   that has an allowed open colour
* ``init_wvcp_population`` :57-64  streams ``Stream.derive(seed, TAG_INIT, i)``
"""

from __future__ import annotations

import numpy as np

GOLDEN = 0x9E3779B97F4A7C15
MASK64 = (1 << 64) - 1


def _mix64(z):
    z &= MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def greedy_order(weights, degrees):                                     # :23-27
    n = len(weights)
    return np.lexsort((np.arange(n), -np.asarray(degrees), -np.asarray(weights)))


def greedy_wvcp_init(indptr, indices, order, key):                      # :30-46
    n = len(indptr) - 1
    assign = -np.ones(n, dtype=np.int32)
    used, ctr = 0, 0
    for v in order:
        blocked = {int(assign[u]) for u in indices[indptr[v]:indptr[v + 1]] if assign[u] >= 0}
        allowed = [c for c in range(used) if c not in blocked]
        if allowed:
            r = _mix64(key + (ctr + 1) * GOLDEN) % len(allowed)  # Stream.below (rng.py:112-118)
            ctr += 1
            assign[v] = allowed[r]
        else:
            assign[v] = used
            used += 1
    return assign, used


def init_wvcp_population(indptr, indices, weights, degrees, keys):      # :57-64
    order = greedy_order(weights, degrees)
    rows = [greedy_wvcp_init(indptr, indices, order, int(k)) for k in keys]
    assigns = np.stack([r[0] for r in rows]) if rows else np.zeros((0, len(indptr) - 1), np.int32)
    used = np.array([r[1] for r in rows], dtype=np.int32)
    return assigns, used, int(used.max()) if len(used) else 0
