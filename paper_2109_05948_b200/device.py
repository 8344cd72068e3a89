"""Device-resident path: the same kernels on torch CUDA tensors.

The multi-generation pipeline keeps the population, the graph and all
outputs in HBM and launches on the caller's current CUDA stream; nothing is
copied to the host.  Tensors use the reference dtypes (int32 assigns, int64
CSR/scalars); uint64 stream keys travel as int64 views (bit-identical).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .graph import graph_arrays


def _stream_handle():
    return torch.cuda.current_stream().cuda_stream


def keys_to_tensor(keys, device):
    return torch.from_numpy(np.ascontiguousarray(keys, dtype=np.uint64).view(np.int64)).to(device)


class DeviceGraph:
    """Graph arrays resident on one GPU (`localsearch.py:418-424` + weights)."""

    def __init__(self, g, device="cuda"):
        indptr, indices, eu, ev = graph_arrays(g)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(device)  # noqa: E731
        self.n, self.m = g.n, g.m
        self.indptr, self.indices, self.eu, self.ev = t(indptr), t(indices), t(eu), t(ev)
        self.wranks = t(np.asarray(g.weight_ranks, dtype=np.int32))
        self.wvals = t(np.asarray(g.weight_values, dtype=np.int64))
        self.weights = t(np.asarray(g.weights, dtype=np.int64))
        self.max_weight = int(g.max_weight)
        self.nranks = int(self.wvals.shape[0])
        self.device = device


def tabucol_batch(dg, assigns, k, keys, depth, *, flags=N.FLAG_DIAG, counters=False, log_cap=0):
    """Batched TabuCol on device tensors; ``assigns`` (int32 [p, n], CUDA) is
    overwritten with the end state.  Returns a dict of CUDA tensors."""
    assert assigns.is_cuda and assigns.dtype == torch.int32 and assigns.is_contiguous()
    p, n = assigns.shape
    dev = assigns.device
    i64 = dict(dtype=torch.int64, device=dev)
    out = {
        "end_assigns": assigns,
        "best_assigns": torch.empty_like(assigns),
        "best_conflicts": torch.empty(p, **i64),
        "end_conflicts": torch.empty(p, **i64),
        "iters_used": torch.zeros(p, **i64),
        "diag": torch.zeros(p, **i64),
        "counters": torch.zeros((p, 2), **i64) if counters else None,
    }
    logs = (None, None, None, None)
    if log_cap:
        logs = (torch.zeros((p, log_cap), dtype=torch.int32, device=dev),
                torch.zeros((p, log_cap), **i64), torch.zeros((p, log_cap), **i64),
                torch.zeros(p, **i64))
    P = N.ptr
    L = N.lib()
    N.check(L.mcb_tabucol_batch(
        P(assigns), p, n, int(k), P(dg.indptr), P(dg.indices), P(dg.eu), P(dg.ev), dg.m, int(depth),
        P(keys), P(out["best_assigns"]), P(out["best_conflicts"]), P(out["end_conflicts"]),
        P(out["iters_used"]), P(out["diag"]), int(log_cap), P(logs[0]), P(logs[1]), P(logs[2]),
        P(logs[3]), P(out["counters"]), int(flags), _stream_handle()))
    out["log"] = logs if log_cap else None
    return out


def tabucol_async_status():
    """Raise for the last asynchronous (FLAG_ASYNC) TabuCol call on the current
    stream (synchronises it): ValueError for colours outside [0, k)."""
    N.check(N.lib().mcb_tabucol_async_status(_stream_handle()))


def wvcp_batch(dg, assigns, k, keys, depth, rounds, schedule_on, phi0, *, flags=N.FLAG_DIAG):
    assert assigns.is_cuda and assigns.dtype == torch.int32 and assigns.is_contiguous()
    p, n = assigns.shape
    dev = assigns.device
    i64 = dict(dtype=torch.int64, device=dev)
    phi0s = torch.full((p,), float(phi0), dtype=torch.float64, device=dev)
    out = {
        "end_assigns": assigns,
        "best_assigns": assigns.clone(),
        "best_scores": torch.empty(p, **i64),
        "end_scores": torch.empty(p, **i64),
        "end_conflicts": torch.empty(p, **i64),
        "phi_used": torch.zeros((p, rounds + 1), dtype=torch.float64, device=dev),
        "diag": torch.zeros(p, **i64),
    }
    P = N.ptr
    L = N.lib()
    N.check(L.mcb_wvcp_batch(
        P(assigns), p, n, int(k), P(dg.indptr), P(dg.indices), P(dg.eu), P(dg.ev), dg.m,
        P(dg.wranks), P(dg.wvals), dg.nranks, P(dg.weights), int(depth), int(rounds),
        int(bool(schedule_on)), P(phi0s), 2.0 * dg.max_weight, n // 5, P(keys),
        P(out["best_assigns"]), P(out["best_scores"]), P(out["end_scores"]),
        P(out["end_conflicts"]), P(out["phi_used"]), P(out["diag"]), 0, None, None, None, None,
        None, int(flags), _stream_handle()))
    return out


def gpx_batch(pop, matches, k, keys, out=None):
    p, n = pop.shape
    K = matches.shape[1]
    if out is None:
        out = torch.empty((p, K, n), dtype=torch.int32, device=pop.device)
    N.check(N.lib().mcb_gpx_batch(N.ptr(pop), p, n, N.ptr(matches), K, int(k), N.ptr(keys),
                                  N.ptr(out), 0, _stream_handle()))
    return out


def pairwise(pop, off, k, job_begin=0, job_end=-1, cross=None, within=None):
    p, q = pop.shape[0], off.shape[0]
    n = off.shape[1]
    dev = off.device
    if cross is None:
        cross = torch.zeros((p, q), dtype=torch.int32, device=dev)
    if within is None:
        within = torch.zeros((q, q), dtype=torch.int32, device=dev)
    N.check(N.lib().mcb_pairwise(N.ptr(pop), p, N.ptr(off), q, n, int(k), N.ptr(cross),
                                 N.ptr(within), int(job_begin), int(job_end), 0, _stream_handle()))
    return cross, within


def pairwise_jobs(pop, off, k, job_begin, job_end, out=None):
    """Distances of the job range [job_begin, job_end) of the (pop, off) job
    space as a compact int16 vector (`mcb_pairwise_jobs`, the sharded path)."""
    p, q = pop.shape[0], off.shape[0]
    n = off.shape[1]
    if out is None:
        out = torch.empty(max(job_end - job_begin, 0), dtype=torch.int16, device=off.device)
    N.check(N.lib().mcb_pairwise_jobs(N.ptr(pop), p, N.ptr(off), q, n, int(k), N.ptr(out), int(job_begin),
                                      int(job_end), 0, _stream_handle()))
    return out


def pairwise_scatter(jobs, p, q, device):
    """The whole job space's int16 vector -> (cross p x q, within q x q) int32."""
    cross = torch.empty((p, q), dtype=torch.int32, device=device)
    within = torch.empty((q, q), dtype=torch.int32, device=device)
    N.check(N.lib().mcb_pairwise_scatter(N.ptr(jobs), p, q, N.ptr(cross), N.ptr(within), _stream_handle()))
    return cross, within


def gpx_rows(pop, matches_rows, row_off, k, keys_rows, out=None):
    """Offspring of population rows [row_off, row_off + rows) (sharded GPX,
    `mcb_gpx_rows`); `matches_rows` indexes the full population `pop`."""
    p, n = pop.shape
    rows, K = matches_rows.shape
    if out is None:
        out = torch.empty((rows, K, n), dtype=torch.int32, device=pop.device)
    N.check(N.lib().mcb_gpx_rows(N.ptr(pop), p, n, N.ptr(matches_rows), rows, int(row_off), K,
                                 int(k), N.ptr(keys_rows), N.ptr(out), 0, _stream_handle()))
    return out
