"""Randomised sweeps, every case bit-exact against the C oracle (oracle/, the
restatement pinned by the reference's fixtures): TabuCol over the whole warp-
kernel envelope (bitset rows of 8/16/32 chunks and CSR, gamma rows of 1..8 x 16
bytes, long tabu lists on the SPILL variant, the CTA-kernel fallbacks past it:
k > 128, n > 1024, gamma > 63), WVCP (u8 gamma and the u16 re-run), GPX and
distances (u8/u16 counters, every column-word count).  Sizes keep each case
around a second on the oracle."""

import numpy as np
import pytest

from paper_2109_05948_b200 import crossover as CX
from paper_2109_05948_b200 import distance as DI
from paper_2109_05948_b200 import localsearch as LS
from paper_2109_05948_b200.graph import rand_graph
from paper_2109_05948_b200.init import random_col_assigns
from paper_2109_05948_b200.rng import TAG_CROSS, TAG_LS, stream_keys

pytestmark = pytest.mark.gpu


def _tabucol_case(t):
    rs = np.random.default_rng(1000 + t)
    n = int(rs.choice([int(rs.integers(2, 64)), int(rs.integers(64, 600)), int(rs.integers(600, 1300))]))
    pe = float(rs.choice([rs.uniform(0.02, 0.2), rs.uniform(0.2, 0.6), rs.uniform(0.6, 0.98)]))
    k = int(rs.choice([int(rs.integers(2, 8)), int(rs.integers(8, 60)), int(rs.integers(60, 170))]))
    pop = int(rs.integers(1, 24))
    depth = int(rs.integers(1, max(2, 24_000_000 // max(1, n * pop))))
    return t, n, pe, k, pop, min(depth, 6000)


@pytest.mark.parametrize("case", [_tabucol_case(t) for t in range(36)], ids=lambda c: f"t{c[0]}n{c[1]}k{c[3]}")
def test_tabucol_fuzz(case, oracle_lib):
    t, n, pe, k, pop, depth = case
    g = rand_graph(50 + t, n, pe)
    A = random_col_assigns(n, k, pop, 70 + t)
    keys = stream_keys(t, TAG_LS, 0, pop)
    ref = oracle_lib.tabucol_batch(g, A.copy(), k, keys, depth, log_moves=True)
    got = LS._run_tabucol_batch(g, A.copy(), k, keys, depth, log_moves=True)
    for key in ("end_assigns", "best_assigns", "best_conflicts", "end_conflicts", "iters_used"):
        np.testing.assert_array_equal(got[key], ref[key], err_msg=key)
    for a, b in zip(got["log"], ref["log"]):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("t", range(12))
def test_wvcp_fuzz(t, oracle_lib):
    rs = np.random.default_rng(2000 + t)
    n = int(rs.integers(2, 700))
    pe = float(rs.uniform(0.02, 0.97))
    k = int(rs.integers(2, 90))
    wmax = int(rs.choice([1, 5, 100, 100000]))
    pop = int(rs.integers(1, 10))
    depth = int(rs.integers(1, max(2, 3_000_000 // max(1, n * pop))))
    rounds = int(rs.integers(1, 4))
    g = rand_graph(80 + t, n, pe, wmax=wmax)
    A = random_col_assigns(n, k, pop, 90 + t)
    keys = stream_keys(t, TAG_LS, 2, pop)
    phi0 = LS.default_wvcp_phi0(g, k) * float(rs.uniform(0.2, 4.0))
    sched = bool(rs.integers(0, 2))
    ref = oracle_lib.wvcp_batch(g, A.copy(), k, keys, depth, rounds, sched, phi0, log_moves=True)
    got = LS._run_wvcp_batch(g, A.copy(), k, keys, depth, rounds, sched, phi0, log_moves=True)
    for key in ("end_assigns", "best_assigns", "best_scores", "end_scores", "end_conflicts", "phi_used"):
        np.testing.assert_array_equal(got[key], ref[key], err_msg=key)
    for a, b in zip(got["log"], ref["log"]):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("t", range(10))
def test_distance_and_gpx_fuzz(t, oracle_lib):
    rs = np.random.default_rng(3000 + t)
    n = int(rs.integers(1, 2500))
    k = int(rs.integers(1, 256))
    p, q = int(rs.integers(0, 9)), int(rs.integers(1, 9))
    P = random_col_assigns(n, k, p, 5 + t) if p else np.zeros((0, n), np.int32)
    Q = random_col_assigns(n, k, q, 6 + t)
    if p and t % 2:  # related pairs: many overlap levels, large entries
        Q[: min(p, q)] = np.random.default_rng(t).permutation(k)[P[: min(p, q)]]
    c, w = DI.pairwise_distances(P, Q, k=k)
    rc, rw = oracle_lib.pairwise(P, Q, k)
    np.testing.assert_array_equal(c, rc)
    np.testing.assert_array_equal(w, rw)
    if q >= 2:
        K = int(rs.integers(1, q))
        matches = np.stack([np.random.default_rng(t + i).permutation(np.delete(np.arange(q), i))[:K]
                            for i in range(q)]).astype(np.int64)
        keys = stream_keys(t, TAG_CROSS, 0, q * K)
        np.testing.assert_array_equal(CX.gpx_batch(Q, matches, k, keys), oracle_lib.gpx_batch(Q, matches, k, keys))
