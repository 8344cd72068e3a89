"""The BASELINE configs whose full shape the fixtures do not reach, pinned
bit-exact against the C restatement of `_tabucol_batch` (`mc/localsearch.py:
266-410`), move logs included:

* config 4 (C5): G(2000, .5), k = 150 -- the 2-CTA cluster kernel (gamma
  split over two SMs' shared memory), and the CTA kernel with its gamma table
  in per-CTA global (L2-resident) slices at both thread counts;
* config 2 (C3): G(1000, .5), k = 83 from random colourings at 20,000
  iterations -- tenures ~1,800 keep > 1,024 tabu entries live, so the
  individuals run on the warp kernel's SPILL variant (rows spilled to global
  memory) for most of the run.
"""
import ctypes

import numpy as np
import pytest

from paper_2109_05948_b200 import _native as N
from paper_2109_05948_b200 import localsearch as LS
from paper_2109_05948_b200.graph import rand_graph
from paper_2109_05948_b200.init import random_col_assigns
from paper_2109_05948_b200.rng import TAG_LS, stream_keys

pytestmark = pytest.mark.gpu


def _check(got, ref, tag):
    for key in ("end_assigns", "best_assigns", "best_conflicts", "end_conflicts", "iters_used", "counters"):
        np.testing.assert_array_equal(got[key], ref[key], err_msg=f"{tag}:{key}")
    for a, b in zip(got["log"], ref["log"]):
        np.testing.assert_array_equal(a, b, err_msg=f"{tag}:log")


@pytest.fixture(scope="module")
def c5_case(oracle_lib):
    g = rand_graph(1, 2000, 0.5)
    A = random_col_assigns(2000, 150, 4, 1)
    keys = stream_keys(1, TAG_LS, 0, 4)
    ref = oracle_lib.tabucol_batch(g, A.copy(), 150, keys, 3000, log_moves=True, counters=True)
    return g, A, keys, ref


@pytest.mark.parametrize("path", ["cluster", "l2-nt128", "l2-nt256"])
def test_c5_shape_vs_oracle(c5_case, path, monkeypatch):
    g, A, keys, ref = c5_case
    if path.startswith("l2"):
        monkeypatch.setenv("MCB_NO_CLUSTER", "1")
        monkeypatch.setenv("MCB_TC_NT", path[-3:])
    buf = ctypes.create_string_buffer(256)
    N.check(N.lib().mcb_tabucol_describe(2000, 150, 4, buf, 256))
    # k > 128 and gamma beyond one SM's shared memory: split over a 2-CTA
    # cluster by default, else the CTA kernel with gamma in L2
    assert (b"tabucol_cluster_kernel" if path == "cluster" else b"gamma in L2") in buf.value, buf.value
    got = LS._run_tabucol_batch(g, A.copy(), 150, keys, 3000, log_moves=True, counters=True)
    _check(got, ref, f"c5/{path}")
    assert (ref["iters_used"] == 3000).all()


def test_c3_20k_through_spill_vs_oracle(oracle_lib, monkeypatch):
    g = rand_graph(1, 1000, 0.5)
    A = random_col_assigns(1000, 83, 4, 1)
    keys = stream_keys(1, TAG_LS, 0, 4)
    ref = oracle_lib.tabucol_batch(g, A.copy(), 83, keys, 20000, log_moves=True, counters=True)
    monkeypatch.delenv("MCB_NO_SPILL", raising=False)
    got = LS._run_tabucol_batch(g, A.copy(), 83, keys, 20000, log_moves=True, counters=True, flags=N.FLAG_WSTATS)
    _check(got, ref, "c3/20k")
    buf = (ctypes.c_ulonglong * 40)()
    N.check(N.lib().mcb_debug_warp_stats(ctypes.addressof(buf)))
    assert buf[10] > 0, "no ring row spilled: the SPILL variant did not run"
    assert (ref["iters_used"] == 20000).all()
