"""Batched tabu search operators -- drop-in for `memcolor.localsearch`.

Same names, signatures, return values and error behaviour as the reference
module (`pkg/src/memcolor/localsearch.py`), with the numba kernels replaced by
the sm_100a kernels behind the C ABI (`mcb_tabucol_batch*`, `mcb_wvcp_batch*`):

* ``_run_tabucol_batch``  `localsearch.py:556-598`
* ``tabucol``             `localsearch.py:601-612`
* ``_run_wvcp_batch``     `localsearch.py:427-497`
* ``wvcp_tabu_search``    `localsearch.py:500-514`
* ``iterated_wvcp_ls``    `localsearch.py:517-553`
* ``improve_population``  `localsearch.py:615-682`

Host numpy arrays go through the ``*_host`` entry points (the library does the
host<->device copies); ``device.py`` holds the device-resident path.  The
`rng` keyword (default "splitmix") selects the reference's SplitMix64 streams
(bit-exact trajectories) or "philox" (production mode, statistically
equivalent).  There is no CPU fallback.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .coloring import Coloring
from .graph import graph_arrays
from .rng import TAG_LS, stream_keys

INF_SCORE = np.int64(1) << np.int64(62)

WVCP = "wvcp"
COL = "col"


@dataclass
class LsResult:
    """Outcome of improving one individual (`localsearch.py:33-43`)."""

    start: Coloring
    best: Coloring
    best_score: int
    iterations_used: int
    legal_found: bool
    end: Coloring
    phi_trajectory: list = field(default_factory=list)


def _flags(rng):
    if rng in (None, "splitmix", "validation"):
        return N.FLAG_DIAG
    if rng in ("philox", "production"):
        return N.FLAG_DIAG | N.FLAG_PRODUCTION
    raise ValueError(f"unknown rng {rng!r}")


def _check_assigns(assigns, k):
    if assigns.size and ((assigns < 0).any() or (assigns >= k).any()):
        raise ValueError("color id out of range [0, k)")


def default_wvcp_phi0(g, k):
    """Initial penalty coefficient: (k / (2 |V|)) * max weight (`:413-415`)."""
    return (k / (2.0 * g.n)) * g.max_weight


def _run_tabucol_batch(g, assigns, k, keys, depth, log_moves=False, *, rng=None, counters=False,
                       flags=0):
    """Batched TabuCol; mutates ``assigns`` (int32[p, n]) to the end state."""
    if assigns.dtype != np.int32 or not assigns.flags.c_contiguous:
        raise ValueError("assigns must be a C-contiguous int32 array")
    p = assigns.shape[0]
    n = g.n
    if assigns.shape[1] != n:
        raise ValueError("assigns must be (p, g.n)")
    _check_assigns(assigns, k)
    indptr, indices, eu, ev = graph_arrays(g)
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    best_assigns = assigns.copy()
    best_conflicts = np.empty(p, dtype=np.int64)
    end_conflicts = np.empty(p, dtype=np.int64)
    iters_used = np.zeros(p, dtype=np.int64)
    diag = np.zeros(p, dtype=np.int64)
    cap = depth if log_moves else 0
    log_v = np.zeros((p, max(cap, 1)), dtype=np.int32)
    log_iter = np.zeros((p, max(cap, 1)), dtype=np.int64)
    log_tt = np.zeros((p, max(cap, 1)), dtype=np.int64)
    log_cnt = np.zeros(p, dtype=np.int64)
    ctrs = np.zeros((p, 2), dtype=np.int64) if counters else None
    L = N.lib()
    P = N.ptr
    N.check(L.mcb_tabucol_batch_host(
        P(assigns), p, n, int(k), P(indptr), P(indices), P(eu), P(ev), g.m, int(depth), P(keys),
        P(best_assigns), P(best_conflicts), P(end_conflicts), P(iters_used), P(diag), cap,
        P(log_v) if cap else None, P(log_iter) if cap else None, P(log_tt) if cap else None,
        P(log_cnt), P(ctrs), _flags(rng) | flags, None))
    if diag.any():
        raise AssertionError("incremental evaluation diverged from scratch recomputation")
    out = {
        "end_assigns": assigns,
        "best_assigns": best_assigns,
        "best_conflicts": best_conflicts,
        "end_conflicts": end_conflicts,
        "iters_used": iters_used,
        "log": (log_v, log_iter, log_tt, log_cnt) if log_moves else None,
    }
    if counters:
        out["counters"] = ctrs
    return out


def tabucol(g, coloring, k, depth=None, key=0, log_moves=False):
    """Classic TabuCol on conflicting vertices; stops at zero conflicts."""
    if depth is None:
        depth = 128 * g.n
    assigns = coloring.assign[None, :].astype(np.int32).copy()
    keys = np.array([key], dtype=np.uint64)
    out = _run_tabucol_batch(g, assigns, k, keys, depth, log_moves=log_moves)
    end = Coloring(out["end_assigns"][0], k)
    best = Coloring(out["best_assigns"][0], k)
    if log_moves:
        return end, best, int(out["best_conflicts"][0]), out["log"]
    return end, best, int(out["best_conflicts"][0])


def _run_wvcp_batch(g, assigns, k, keys, depth, rounds, schedule_on, phi0, log_moves=False, *,
                    rng=None, flags=0):
    """Batched iterated weighted tabu search; mutates ``assigns``."""
    if assigns.dtype != np.int32 or not assigns.flags.c_contiguous:
        raise ValueError("assigns must be a C-contiguous int32 array")
    p, n = assigns.shape
    if n != g.n:
        raise ValueError("assigns must be (p, g.n)")
    _check_assigns(assigns, k)
    indptr, indices, eu, ev = graph_arrays(g)
    phi0s = np.full(p, float(phi0), dtype=np.float64)
    forced_phi = 2.0 * float(g.max_weight)
    tt_base = n // 5
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    wranks = np.ascontiguousarray(g.weight_ranks, dtype=np.int32)
    wvals = np.ascontiguousarray(g.weight_values, dtype=np.int64)
    weights = np.ascontiguousarray(g.weights, dtype=np.int64)
    best_assigns = assigns.copy()
    best_scores = np.empty(p, dtype=np.int64)
    end_scores = np.empty(p, dtype=np.int64)
    end_conflicts = np.empty(p, dtype=np.int64)
    phi_used = np.zeros((p, rounds + 1), dtype=np.float64)
    diag = np.zeros(p, dtype=np.int64)
    cap = rounds * depth if log_moves else 0
    log_v = np.zeros((p, max(cap, 1)), dtype=np.int32)
    log_iter = np.zeros((p, max(cap, 1)), dtype=np.int64)
    log_tt = np.zeros((p, max(cap, 1)), dtype=np.int64)
    log_asp = np.zeros((p, max(cap, 1)), dtype=np.int8)
    log_cnt = np.zeros(p, dtype=np.int64)
    L = N.lib()
    P = N.ptr
    N.check(L.mcb_wvcp_batch_host(
        P(assigns), p, n, int(k), P(indptr), P(indices), P(eu), P(ev), g.m, P(wranks), P(wvals),
        wvals.shape[0], P(weights), int(depth), int(rounds), int(bool(schedule_on)), P(phi0s),
        forced_phi, tt_base, P(keys), P(best_assigns), P(best_scores), P(end_scores),
        P(end_conflicts), P(phi_used), P(diag), cap, P(log_v) if cap else None,
        P(log_iter) if cap else None, P(log_tt) if cap else None, P(log_asp) if cap else None,
        P(log_cnt), _flags(rng) | flags, None))
    if diag.any():
        raise AssertionError("incremental evaluation diverged from scratch recomputation")
    return {
        "end_assigns": assigns,
        "best_assigns": best_assigns,
        "best_scores": best_scores,
        "end_scores": end_scores,
        "end_conflicts": end_conflicts,
        "phi_used": phi_used,
        "log": (log_v, log_iter, log_tt, log_asp, log_cnt) if log_moves else None,
    }


def wvcp_tabu_search(g, coloring, phi, depth, key, log_moves=False):
    """One fixed-phi search; returns (end coloring, best legal or None)."""
    assigns = coloring.assign[None, :].astype(np.int32).copy()
    keys = np.array([key], dtype=np.uint64)
    out = _run_wvcp_batch(g, assigns, coloring.k, keys, depth, 1, False, phi, log_moves=log_moves)
    end = Coloring(out["end_assigns"][0], coloring.k)
    best = None
    if out["best_scores"][0] < INF_SCORE:
        best = (Coloring(out["best_assigns"][0], coloring.k), int(out["best_scores"][0]))
    result = (end, best)
    if log_moves:
        result = (end, best, out["log"])
    return result


def iterated_wvcp_ls(g, coloring, key, depth=None, max_rounds=10, phi0=None, log_moves=False):
    """Successive tabu searches with the adaptive phi schedule (`:517-553`)."""
    k = coloring.k
    if depth is None:
        depth = 10 * g.n
    if phi0 is None:
        phi0 = default_wvcp_phi0(g, k)
    assigns = coloring.assign[None, :].astype(np.int32).copy()
    keys = np.array([key], dtype=np.uint64)
    out = _run_wvcp_batch(g, assigns, k, keys, depth, max_rounds, True, phi0, log_moves=log_moves)
    legal = bool(out["best_scores"][0] < INF_SCORE)
    best = Coloring(out["best_assigns"][0], k) if legal else coloring.copy()
    result = LsResult(
        start=coloring.copy(),
        best=best,
        best_score=int(out["best_scores"][0]) if legal else int(INF_SCORE),
        iterations_used=depth * max_rounds,
        legal_found=legal,
        end=Coloring(out["end_assigns"][0], k),
        phi_trajectory=list(out["phi_used"][0]),
    )
    if log_moves:
        return result, out["log"]
    return result


def improve_population(g, colorings, mode, master_seed, generation=0, thread_count=None, depth=None,
                       max_rounds=10, *, rng=None):
    """Improve every individual independently; deterministic and independent
    of ``thread_count`` (accepted and ignored: one CUDA stream per call)."""
    p = len(colorings)
    k = colorings[0].k
    n = g.n
    assigns = np.stack([c.assign for c in colorings]).astype(np.int32)
    keys = stream_keys(master_seed, TAG_LS, generation, p)
    starts = [c.copy() for c in colorings]

    if mode == WVCP:
        if depth is None:
            depth = 10 * n
        phi0 = default_wvcp_phi0(g, k)
        out = _run_wvcp_batch(g, assigns, k, keys, depth, max_rounds, True, phi0, rng=rng)
        results = []
        for i in range(p):
            legal = bool(out["best_scores"][i] < INF_SCORE)
            best = Coloring(out["best_assigns"][i], k) if legal else starts[i].copy()
            results.append(LsResult(
                start=starts[i],
                best=best,
                best_score=int(out["best_scores"][i]) if legal else int(INF_SCORE),
                iterations_used=depth * max_rounds,
                legal_found=legal,
                end=Coloring(out["end_assigns"][i], k),
                phi_trajectory=list(out["phi_used"][i]),
            ))
        return results

    if mode == COL:
        if depth is None:
            depth = 128 * n
        out = _run_tabucol_batch(g, assigns, k, keys, depth, rng=rng)
        results = []
        for i in range(p):
            results.append(LsResult(
                start=starts[i],
                best=Coloring(out["best_assigns"][i], k),
                best_score=int(out["best_conflicts"][i]),
                iterations_used=int(out["iters_used"][i]),
                legal_found=bool(out["best_conflicts"][i] == 0),
                end=Coloring(out["end_assigns"][i], k),
            ))
        return results

    raise ValueError(f"unknown mode {mode!r}")
