"""ctypes binding of the C ABI (include/memcolor_b200.h).

There is no fallback: if the shared library is missing or no CUDA device is
visible, every operator raises.  Status codes map onto the exception types the
reference raises for the same conditions (`localsearch.py:589-590,682`,
`crossover.py:73-74`, `distance.py:23-24`).
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from ._build import LIB

MCB_OK, MCB_ERR_VALUE, MCB_ERR_CUDA, MCB_ERR_UNSUPPORTED, MCB_ERR_RANGE = 0, 1, 2, 3, 4
FLAG_DIAG = 0x1
FLAG_PRODUCTION = 0x2
FLAG_FORCE_WIDE = 0x4
FLAG_FORCE_GLOBAL = 0x8
FLAG_PROFILE = 0x100
FLAG_WSTATS = 0x200
FLAG_ASYNC = 0x400
FLAG_FORCE_CLUSTER = 0x800

EXPORTS = [
    "mcb_version", "mcb_last_error", "mcb_device_count", "mcb_stream_values",
    "mcb_tabucol_batch", "mcb_tabucol_batch_host", "mcb_tabucol_async_status", "mcb_wvcp_batch", "mcb_wvcp_batch_host",
    "mcb_gpx_batch", "mcb_gpx_batch_host", "mcb_gpx_rows", "mcb_pairwise", "mcb_pairwise_host", "mcb_pairwise_jobs", "mcb_pairwise_scatter",
    "mcb_probe_smem_bandwidth", "mcb_probe_l2_bandwidth", "mcb_debug_phase_cycles", "mcb_debug_warp_stats", "mcb_debug_cluster_warps", "mcb_debug_group_stats", "mcb_debug_wvcp_stats",
    "mcb_debug_modcheck", "mcb_tabucol_describe",
    "mcb_update_population", "mcb_update_population_host", "mcb_match_parents", "mcb_match_parents_host",
    "mcb_greedy_wvcp_init", "mcb_greedy_wvcp_init_host", "mcb_segsum", "mcb_segsum_async",
    "mcb_colour_order", "mcb_segsum_sorted", "mcb_rowbias_affine_leaky",
]

_lib = None


class NativeUnavailable(RuntimeError):
    pass


def _declare(L):
    P, I64, U32, I32 = C.c_void_p, C.c_int64, C.c_uint32, C.c_int32
    L.mcb_version.restype = C.c_char_p
    L.mcb_last_error.restype = C.c_char_p
    L.mcb_device_count.restype = C.c_int
    L.mcb_stream_values.argtypes = [P, P, P, I64, P]
    tab = [P, I64, I64, I64, P, P, P, P, I64, I64, P, P, P, P, P, P, I64, P, P, P, P, P, U32, P]
    L.mcb_tabucol_batch.argtypes = tab
    L.mcb_tabucol_batch_host.argtypes = tab
    L.mcb_tabucol_async_status.argtypes = [P]
    wv = [P, I64, I64, I64, P, P, P, P, I64, P, P, I64, P, I64, I64, I32, P, C.c_double, I64, P,
          P, P, P, P, P, P, I64, P, P, P, P, P, U32, P]
    L.mcb_wvcp_batch.argtypes = wv
    L.mcb_wvcp_batch_host.argtypes = wv
    gp = [P, I64, I64, P, I64, I64, P, P, U32, P]
    L.mcb_gpx_batch.argtypes = gp
    L.mcb_gpx_batch_host.argtypes = gp
    L.mcb_gpx_rows.argtypes = [P, I64, I64, P, I64, I64, I64, I64, P, P, U32, P]
    pw = [P, I64, P, I64, I64, I64, P, P, I64, I64, U32, P]
    L.mcb_pairwise.argtypes = pw
    L.mcb_pairwise_host.argtypes = pw
    L.mcb_pairwise_jobs.argtypes = [P, I64, P, I64, I64, I64, P, I64, I64, U32, P]
    L.mcb_pairwise_scatter.argtypes = [P, I64, I64, P, P, P]
    L.mcb_probe_smem_bandwidth.argtypes = [P, P]
    L.mcb_probe_l2_bandwidth.argtypes = [P, P]
    L.mcb_debug_phase_cycles.argtypes = [P, C.c_int]
    L.mcb_debug_warp_stats.argtypes = [P]
    L.mcb_debug_cluster_warps.argtypes = [P, C.c_int]
    L.mcb_debug_group_stats.argtypes = [P]
    L.mcb_debug_wvcp_stats.argtypes = [P, C.c_int]
    L.mcb_debug_modcheck.argtypes = [I64, P]
    L.mcb_tabucol_describe.argtypes = [I64, I64, I64, C.c_char_p, C.c_int]
    up = [P, P, P, P, P, I64, I64, I64, P, P, I64, P, P, P, P, P, P]
    L.mcb_update_population.argtypes = up
    L.mcb_update_population_host.argtypes = up
    L.mcb_match_parents.argtypes = [P, I64, I64, I64, P, P]
    L.mcb_match_parents_host.argtypes = [P, I64, I64, I64, P, P]
    L.mcb_greedy_wvcp_init.argtypes = [P, P, P, I64, P, I64, P, P, P]
    L.mcb_greedy_wvcp_init_host.argtypes = [P, P, P, I64, P, I64, P, P, P]
    L.mcb_segsum.argtypes = [C.c_int, C.c_int, P, P, I64, I64, I64, I64, P, P]
    L.mcb_segsum_async.argtypes = [C.c_int, C.c_int, P, P, I64, I64, I64, I64, P, P]
    L.mcb_colour_order.argtypes = [P, I64, I64, I64, P, P, P]
    L.mcb_segsum_sorted.argtypes = [C.c_int, P, P, P, I64, I64, I64, I64, P, P, C.c_double, P, P]
    L.mcb_rowbias_affine_leaky.argtypes = [C.c_int, P, P, P, P, C.c_double, I64, I64, I64, P]
    for name in EXPORTS[3:]:
        getattr(L, name).restype = C.c_int


def load(path=None):
    """Load the library (no device needed).  Raises if it is not built."""
    global _lib
    if _lib is None:
        # MCB_LIB: an alternative build of the same ABI (A/B experiments, tools/)
        path = path or os.environ.get("MCB_LIB") or LIB
        if not os.path.exists(path):
            raise NativeUnavailable(
                f"{path} is missing: build it with `python -m paper_2109_05948_b200._build`")
        L = C.CDLL(path)
        _declare(L)
        _lib = L
    return _lib


def lib():
    """The library, with a CUDA device required (no CPU fallback)."""
    L = load()
    if L.mcb_device_count() < 1:
        raise NativeUnavailable("memcolor-b200 needs a CUDA device; none is visible")
    return L


def check(rc):
    if rc == MCB_OK:
        return
    msg = (load().mcb_last_error() or b"").decode(errors="replace")
    if rc in (MCB_ERR_VALUE, MCB_ERR_UNSUPPORTED, MCB_ERR_RANGE):
        raise ValueError(msg)
    raise RuntimeError(f"CUDA error: {msg}")


def ptr(a):
    """Address of a numpy array or torch tensor (None -> NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()
