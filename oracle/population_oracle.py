"""CPU restatement of the reference's population update and parent matching.

TEST INFRASTRUCTURE ONLY (the checker of csrc/population.cu): imported by
tests/ only.  Line-by-line restatement of
`/root/reference/pkg/src/memcolor/population.py`:

* ``update_population``  :59-127  -> (admitted ids, by_rule, new_dist, new_assigns, new_fit)
* ``match_parents``      :130-141
"""

from __future__ import annotations

import numpy as np


def update_population(pdist, pop_fit, pop_assigns, improved_assigns, improved_fitness, cross, within, ms):
    p = pdist.shape[0]
    q = improved_assigns.shape[0]
    cand_fit = np.concatenate([pop_fit, improved_fitness]).astype(np.int64)           # :68
    origin = np.concatenate([np.zeros(p, dtype=np.int64), np.ones(q, dtype=np.int64)])  # :69
    index_in_origin = np.concatenate([np.arange(p), np.arange(q)])                      # :70
    order = np.lexsort((index_in_origin, origin, cand_fit))                             # :71

    def dist(i, j):                                                                      # :73-82
        if i < p and j < p:
            return pdist[i, j]
        if i < p:
            return cross[i, j - p]
        if j < p:
            return cross[j, i - p]
        return within[i - p, j - p]

    admitted, by_rule, rejected = [], [], []
    for cid in order:                                                                    # :87-95
        cid = int(cid)
        if len(admitted) == p:
            break
        if all(dist(cid, other) > ms for other in admitted):
            admitted.append(cid)
            by_rule.append(True)
        else:
            rejected.append(cid)
    for cid in rejected:                                                                 # :96-100
        if len(admitted) == p:
            break
        admitted.append(cid)
        by_rule.append(False)
    n = pop_assigns.shape[1]
    new_assigns = np.empty((p, n), dtype=np.int32)                                       # :102-108
    new_fit = np.empty(p, dtype=np.int64)
    for slot, cid in enumerate(admitted):
        new_assigns[slot] = pop_assigns[cid] if cid < p else improved_assigns[cid - p]
        new_fit[slot] = cand_fit[cid]
    new_dist = np.zeros((p, p), dtype=np.int32)                                          # :109-114
    for a in range(p):
        for b in range(a + 1, p):
            d = dist(admitted[a], admitted[b])
            new_dist[a, b] = d
            new_dist[b, a] = d
    return np.array(admitted, dtype=np.int32), np.array(by_rule, dtype=bool), new_dist, new_assigns, new_fit


def match_parents(dist, K):
    p = dist.shape[0]                                                                    # :130-141
    if not (0 < K < p):
        raise ValueError("need 0 < K < p")
    matches = np.empty((p, K), dtype=np.int64)
    idx = np.arange(p)
    for i in range(p):
        order = np.lexsort((idx, dist[i]))
        row = order[order != i][:K]
        matches[i] = row
    return matches
