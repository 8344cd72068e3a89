"""The 2-CTA cluster TabuCol kernel (csrc/tabucol_cluster.cu): colours split
between the two CTAs' shared memories, records / walk events / the chosen
column exchanged through DSMEM.  It must reproduce `_tabucol_batch`
(`mc/localsearch.py:266-410`) bit for bit -- move logs included -- on every
golden fixture (forced with MCB_FLAG_FORCE_CLUSTER, at 256 / 512 / 1024
threads per CTA), on random shapes against the C oracle (k up to 255: one
and two 64-colour mask words per half), at config 4's own shape where it is
the default kernel, and in production mode against the CTA kernel (same
Philox draws, so identical results)."""

import ctypes

import numpy as np
import pytest

from cases import check_tabucol, tabucol_case
from conftest import load_golden
from paper_2109_05948_b200 import _native as N
from paper_2109_05948_b200 import localsearch as LS
from paper_2109_05948_b200.coloring import col_conflicts_batch
from paper_2109_05948_b200.graph import rand_graph
from paper_2109_05948_b200.init import random_col_assigns
from paper_2109_05948_b200.rng import TAG_LS, stream_keys

pytestmark = pytest.mark.gpu
TAB = load_golden("tabucol")
KEYS = ("end_assigns", "best_assigns", "best_conflicts", "end_conflicts", "iters_used", "counters")


def _same(got, ref, tag):
    for key in KEYS:
        if key in ref:
            np.testing.assert_array_equal(got[key], ref[key], err_msg=f"{tag}:{key}")
    for a, b in zip(got.get("log") or (), ref.get("log") or ()):
        np.testing.assert_array_equal(a, b, err_msg=f"{tag}:log")


@pytest.mark.parametrize("nt", ["256", "512", "1024"])
@pytest.mark.parametrize("name", list(TAB["cases"]))
def test_cluster_golden_bit_exact(name, nt, monkeypatch):
    monkeypatch.setenv("MCB_CL_NT", nt)
    g, A, k, keys, depth, cap = tabucol_case(TAB, name)
    out = LS._run_tabucol_batch(g, A.copy(), k, keys, depth, log_moves=cap > 0, flags=N.FLAG_FORCE_CLUSTER)
    check_tabucol(TAB, name, out)


def test_cluster_vs_oracle_random(oracle_lib):
    rs = np.random.default_rng(11)
    for t in range(14):
        n = int(rs.integers(2, 700))
        pe = float(rs.uniform(0.05, 0.95))
        k = int(rs.integers(2, 256)) if t % 2 else int(rs.integers(2, 130))
        p = int(rs.integers(1, 24))
        depth = int(rs.integers(1, 2500))
        g = rand_graph(3000 + t, n, pe)
        A = random_col_assigns(n, k, p, 91 + t)
        keys = stream_keys(t, TAG_LS, 5, p)
        ref = oracle_lib.tabucol_batch(g, A.copy(), k, keys, depth, log_moves=True, counters=True)
        got = LS._run_tabucol_batch(g, A.copy(), k, keys, depth, log_moves=True, counters=True,
                                    flags=N.FLAG_FORCE_CLUSTER)
        _same(got, ref, f"case {t} n={n} k={k}")


def test_cluster_diag_flag(oracle_lib):
    """the O(m) scratch check every 1024 iterations (:398-405) finds no drift
    (the wrapper raises if any individual's diag count is non-zero)"""
    g = rand_graph(7, 300, 0.5)
    A = random_col_assigns(300, 30, 6, 7)
    keys = stream_keys(7, TAG_LS, 0, 6)
    got = LS._run_tabucol_batch(g, A.copy(), 30, keys, 4096, counters=True,
                                flags=N.FLAG_FORCE_CLUSTER | N.FLAG_DIAG)
    ref = oracle_lib.tabucol_batch(g, A.copy(), 30, keys, 4096, counters=True)
    _same(got, ref, "diag")


def test_cluster_production_matches_cta_kernel():
    """production mode (Philox4x32 draws, no event walks): the cluster and the
    single-CTA kernel draw the same numbers, so their results are identical"""
    g = rand_graph(2, 400, 0.5)
    A = random_col_assigns(400, 40, 12, 2)
    keys = stream_keys(2, TAG_LS, 0, 12)
    a = LS._run_tabucol_batch(g, A.copy(), 40, keys, 3000, counters=True,
                              flags=N.FLAG_PRODUCTION | N.FLAG_FORCE_CLUSTER)
    b = LS._run_tabucol_batch(g, A.copy(), 40, keys, 3000, counters=True,
                              flags=N.FLAG_PRODUCTION | N.FLAG_FORCE_GLOBAL)
    _same(a, b, "production")
    np.testing.assert_array_equal(col_conflicts_batch(g, a["best_assigns"]), a["best_conflicts"])


def test_cluster_overflow_reruns_wide(oracle_lib):
    """a vertex with > 254 neighbours of one colour overflows u8 gamma: the
    individual is re-run by the wide pass, results unchanged"""
    from paper_2109_05948_b200.graph import WeightedGraph

    n = 300
    edges = [(0, v) for v in range(1, n)] + [(v, v + 1) for v in range(1, n - 1, 3)]
    g = WeightedGraph(n, edges, [1] * n)
    A = np.zeros((3, n), np.int32)
    A[:, 0] = 1
    A[1, 1::2] = 1
    keys = stream_keys(3, TAG_LS, 0, 3)
    ref = oracle_lib.tabucol_batch(g, A.copy(), 3, keys, 500, log_moves=True, counters=True)
    got = LS._run_tabucol_batch(g, A.copy(), 3, keys, 500, log_moves=True, counters=True,
                                flags=N.FLAG_FORCE_CLUSTER)
    _same(got, ref, "overflow")


def test_cluster_is_the_config4_kernel():
    buf = ctypes.create_string_buffer(256)
    N.check(N.lib().mcb_tabucol_describe(2000, 150, 256, buf, 256))
    assert b"tabucol_cluster_kernel" in buf.value, buf.value


def test_cluster_k255_vs_oracle(oracle_lib):
    """k = 255, the ABI maximum: halves of 128 colours (32 words, every lane
    of the warp-cooperative scans, walks and locate busy)"""
    g = rand_graph(21, 420, 0.7)
    A = random_col_assigns(420, 255, 6, 21)
    keys = stream_keys(21, TAG_LS, 2, 6)
    ref = oracle_lib.tabucol_batch(g, A.copy(), 255, keys, 1500, log_moves=True, counters=True)
    got = LS._run_tabucol_batch(g, A.copy(), 255, keys, 1500, log_moves=True, counters=True,
                                flags=N.FLAG_FORCE_CLUSTER)
    _same(got, ref, "k255")


@pytest.mark.parametrize("n,k,kind", [(2000, 150, b"tabucol_cluster_kernel"), (2200, 150, b"gamma in L2"),
                                      (2600, 150, b"gamma in L2"), (2000, 200, b"gamma in L2"),
                                      (1000, 200, b"gamma in shared memory"), (1100, 200, b"tabucol_cluster_kernel")])
def test_cluster_dispatch_boundary(n, k, kind):
    """the cluster kernel serves exactly the shapes one CTA's shared memory
    cannot hold and the pair's can; beyond the pair, the L2 path"""
    buf = ctypes.create_string_buffer(256)
    N.check(N.lib().mcb_tabucol_describe(n, k, 64, buf, 256))
    assert kind in buf.value, buf.value


@pytest.mark.parametrize("hot", [0, 9], ids=["rank0-colour", "rank1-colour"])
def test_cluster_overflow_in_either_half(hot, oracle_lib):
    """a u8 count overflow seen by one CTA only (colour `hot` lives in rank 0's
    or rank 1's half at k = 10) stops both CTAs at the same barrier; the
    individual is re-run by the wide pass and the results match the oracle"""
    from paper_2109_05948_b200.graph import WeightedGraph

    n, k = 320, 10
    edges = [(0, v) for v in range(1, n)] + [(v, v + 2) for v in range(1, n - 2, 5)]
    g = WeightedGraph(n, edges, [1] * n)
    A = random_col_assigns(n, k, 4, 5)
    A[:, 1:] = np.where(np.arange(n - 1)[None, :] % 10 == 0, A[:, 1:], hot)  # ~287 leaves coloured `hot` (> 254)
    A[:, 0] = (hot + 1) % k
    keys = stream_keys(5, TAG_LS, 0, 4)
    ref = oracle_lib.tabucol_batch(g, A.copy(), k, keys, 800, log_moves=True, counters=True)
    got = LS._run_tabucol_batch(g, A.copy(), k, keys, 800, log_moves=True, counters=True,
                                flags=N.FLAG_FORCE_CLUSTER)
    _same(got, ref, f"overflow-{hot}")
