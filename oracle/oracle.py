"""ctypes front end of the C oracle (memcolor_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
CPU legs of bench.py, never by the product package.  Each wrapper returns the
same dict as the reference wrapper it restates:

* ``tabucol_batch``  -> `localsearch.py:556-598` (_run_tabucol_batch)
* ``wvcp_batch``     -> `localsearch.py:427-497` (_run_wvcp_batch)
* ``gpx_batch``      -> `crossover.py:60-66,81-93` (_gpx_batch)
* ``pairwise``       -> `distance.py:90-119,122-155` (_pairwise_kernel)
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "liboracle.so")
_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        I64 = C.c_int64
        L.orc_stream_value.restype = C.c_uint64
        L.orc_stream_value.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_max_threads.restype = C.c_int
        L.orc_tabucol_batch.restype = None
        L.orc_tabucol_batch.argtypes = [P, I64, I64, I64, P, P, P, P, I64, I64, P, P, P, P, P, P,
                                        I64, P, P, P, P, P, C.c_int]
        L.orc_wvcp_batch.restype = None
        L.orc_wvcp_batch.argtypes = [P, I64, I64, I64, P, P, P, P, I64, P, P, I64, P, I64, I64,
                                     C.c_int, P, C.c_double, I64, P, P, P, P, P, P, P, I64, P, P,
                                     P, P, P, C.c_int]
        L.orc_gpx_batch.restype = None
        L.orc_gpx_batch.argtypes = [P, I64, I64, P, I64, I64, P, P, C.c_int]
        L.orc_approx_distance.restype = I64
        L.orc_approx_distance.argtypes = [P, P, I64, I64]
        L.orc_pairwise.restype = None
        L.orc_pairwise.argtypes = [P, I64, P, I64, I64, I64, P, P, I64, I64, C.c_int]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _graph(g):
    return (np.ascontiguousarray(g.adj_indptr, dtype=np.int64),
            np.ascontiguousarray(g.adj_indices, dtype=np.int32),
            np.ascontiguousarray(g.edges[:, 0], dtype=np.int32),
            np.ascontiguousarray(g.edges[:, 1], dtype=np.int32))


def stream_value(key, ctr):
    return int(lib().orc_stream_value(int(key), int(ctr)))


def max_threads():
    return int(lib().orc_max_threads())


def tabucol_batch(g, assigns, k, keys, depth, log_moves=False, log_cap=None, threads=0,
                  counters=False):
    """Restates `_run_tabucol_batch` (`localsearch.py:556-598`); mutates
    ``assigns`` (int32, C-contiguous) to the end state like the reference."""
    assert assigns.dtype == np.int32 and assigns.flags.c_contiguous
    p, n = assigns.shape
    indptr, indices, eu, ev = _graph(g)
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    best_assigns = assigns.copy()
    best_conflicts = np.empty(p, np.int64)
    end_conflicts = np.empty(p, np.int64)
    iters_used = np.zeros(p, np.int64)
    diag = np.zeros(p, np.int64)
    cap = (depth if log_cap is None else log_cap) if log_moves else 0
    log_v = np.zeros((p, max(cap, 1)), np.int32)
    log_iter = np.zeros((p, max(cap, 1)), np.int64)
    log_tt = np.zeros((p, max(cap, 1)), np.int64)
    log_cnt = np.zeros(p, np.int64)
    ctrs = np.zeros((p, 2), np.int64) if counters else None
    lib().orc_tabucol_batch(_p(assigns), p, n, int(k), _p(indptr), _p(indices), _p(eu), _p(ev),
                            g.m, int(depth), _p(keys), _p(best_assigns), _p(best_conflicts),
                            _p(end_conflicts), _p(iters_used), _p(diag), cap, _p(log_v),
                            _p(log_iter), _p(log_tt), _p(log_cnt), _p(ctrs), int(threads))
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


def wvcp_batch(g, assigns, k, keys, depth, rounds, schedule_on, phi0, log_moves=False,
               threads=0, phi0s=None):
    """Restates `_run_wvcp_batch` (`localsearch.py:427-497`)."""
    assert assigns.dtype == np.int32 and assigns.flags.c_contiguous
    p, n = assigns.shape
    indptr, indices, eu, ev = _graph(g)
    if phi0s is None:
        phi0s = np.full(p, float(phi0), dtype=np.float64)
    phi0s = np.ascontiguousarray(phi0s, dtype=np.float64)
    forced_phi = 2.0 * float(g.max_weight)
    tt_base = n // 5
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    wranks = np.ascontiguousarray(g.weight_ranks, dtype=np.int32)
    wvals = np.ascontiguousarray(g.weight_values, dtype=np.int64)
    weights = np.ascontiguousarray(g.weights, dtype=np.int64)
    best_assigns = assigns.copy()
    best_scores = np.empty(p, np.int64)
    end_scores = np.empty(p, np.int64)
    end_conflicts = np.empty(p, np.int64)
    phi_used = np.zeros((p, rounds + 1), np.float64)
    diag = np.zeros(p, np.int64)
    cap = rounds * depth if log_moves else 0
    log_v = np.zeros((p, max(cap, 1)), np.int32)
    log_iter = np.zeros((p, max(cap, 1)), np.int64)
    log_tt = np.zeros((p, max(cap, 1)), np.int64)
    log_asp = np.zeros((p, max(cap, 1)), np.int8)
    log_cnt = np.zeros(p, np.int64)
    lib().orc_wvcp_batch(_p(assigns), p, n, int(k), _p(indptr), _p(indices), _p(eu), _p(ev), g.m,
                         _p(wranks), _p(wvals), wvals.shape[0], _p(weights), int(depth),
                         int(rounds), int(bool(schedule_on)), _p(phi0s), forced_phi, tt_base,
                         _p(keys), _p(best_assigns), _p(best_scores), _p(end_scores),
                         _p(end_conflicts), _p(phi_used), _p(diag), cap, _p(log_v), _p(log_iter),
                         _p(log_tt), _p(log_asp), _p(log_cnt), int(threads))
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


def gpx_batch(pop, matches, k, keys, threads=0):
    """Restates `_gpx_batch` (`crossover.py:60-66`) -> int32[p, K, n]."""
    pop = np.ascontiguousarray(pop, dtype=np.int32)
    matches = np.ascontiguousarray(matches, dtype=np.int64)
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    p, n = pop.shape
    K = matches.shape[1]
    out = np.empty((p, K, n), np.int32)
    lib().orc_gpx_batch(_p(pop), p, n, _p(matches), K, int(k), _p(keys), _p(out), int(threads))
    return out


def approx_distance(a, b, k):
    a = np.ascontiguousarray(a, dtype=np.int32)
    b = np.ascontiguousarray(b, dtype=np.int32)
    return int(lib().orc_approx_distance(_p(a), _p(b), a.size, int(k)))


def pairwise(pop, off, k, job_begin=0, job_end=-1, threads=0):
    """Restates `_pairwise_kernel` (`distance.py:90-119`) -> (cross, within)."""
    pop = np.ascontiguousarray(pop, dtype=np.int32)
    off = np.ascontiguousarray(off, dtype=np.int32)
    p, n = pop.shape
    q = off.shape[0]
    if n == 0:
        n = off.shape[1]
    cross = np.zeros((p, q), np.int32)
    within = np.zeros((q, q), np.int32)
    lib().orc_pairwise(_p(pop), p, _p(off), q, n, int(k), _p(cross), _p(within), int(job_begin),
                       int(job_end), int(threads))
    return cross, within
