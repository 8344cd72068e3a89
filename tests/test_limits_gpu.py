"""Size limits fail loudly and cleanly (ValueError from MCB_ERR_UNSUPPORTED,
no crash, the library stays usable): TabuCol k <= 255 and n <= 32767, WVCP
k <= 255, distances k <= 255, greedy init n <= 32767 (Limits)."""

import numpy as np
import pytest

from paper_2109_05948_b200 import distance as DI
from paper_2109_05948_b200 import localsearch as LS
from paper_2109_05948_b200.graph import WeightedGraph, rand_graph
from paper_2109_05948_b200.init import greedy_wvcp_assigns, random_col_assigns, stream_keys_init
from paper_2109_05948_b200.rng import TAG_LS, stream_keys

pytestmark = pytest.mark.gpu


def _path_graph(n, wmax=1):
    e = np.stack([np.arange(n - 1), np.arange(1, n)], 1)
    return WeightedGraph(n, e, np.ones(n, np.int64) * wmax)


def test_colour_limits_raise():
    g = rand_graph(1, 40, 0.3)
    A = random_col_assigns(40, 256, 2, 1)
    keys = stream_keys(1, TAG_LS, 0, 2)
    with pytest.raises(ValueError, match="k<=255"):
        LS._run_tabucol_batch(g, A.copy(), 256, keys, 10)
    with pytest.raises(ValueError):
        LS._run_wvcp_batch(g, A.copy(), 256, keys, 10, 1, True, 1.0)
    with pytest.raises(ValueError):
        DI.pairwise_distances(A, A, k=256)
    # still usable afterwards
    out = LS._run_tabucol_batch(g, random_col_assigns(40, 5, 2, 1), 5, keys, 10)
    assert out["iters_used"].shape == (2,)


def test_vertex_limits_raise():
    """TabuCol: the CTA fallback keeps ~39 B per vertex in shared memory, so n
    is bounded near 5,900 (checked up front); greedy init: n <= 32767."""
    g = _path_graph(8000)
    A = np.zeros((1, 8000), np.int32)
    A[0, 1::2] = 1
    with pytest.raises(ValueError, match="per-vertex shared state"):
        LS._run_tabucol_batch(g, A, 2, stream_keys(1, TAG_LS, 0, 1), 5)
    g5 = _path_graph(5000)  # a large accepted n runs (CTA kernel, gamma in L2)
    A5 = np.zeros((2, 5000), np.int32)
    out = LS._run_tabucol_batch(g5, A5, 3, stream_keys(1, TAG_LS, 0, 2), 50)
    assert (out["best_conflicts"] < 4999).all()
    gl = _path_graph(32768)
    with pytest.raises(ValueError, match="n <= 32767"):
        greedy_wvcp_assigns(gl, stream_keys_init(1, 1))
    gm = _path_graph(32767)  # the largest greedy init: fewer warps per block
    a, used = greedy_wvcp_assigns(gm, stream_keys_init(1, 2))
    assert (a[:, :-1] != a[:, 1:]).all() and (used <= 3).all()


def test_shared_state_limits_raise_cleanly(oracle_lib):
    """WVCP and distances whose per-individual / per-pair shared-memory state
    cannot fit: a ValueError naming the limit, not a CUDA failure."""
    g = _path_graph(40000, wmax=3)
    A = np.zeros((1, 40000), np.int32)
    A[0, 1::2] = 1
    with pytest.raises(ValueError, match="shared memory"):
        LS._run_wvcp_batch(g, A, 3, stream_keys(1, TAG_LS, 0, 1), 5, 1, True, 1.0)
    # distances list only the cells reaching 2 (<= n / 2): n = 60000, k = 200
    # fits, u16 counters included (classes of ~300 vertices overflow u8)
    P = random_col_assigns(60000, 200, 2, 2)
    c, w = DI.pairwise_distances(P, P, k=200)
    rc, rw = oracle_lib.pairwise(P, P, 200)
    np.testing.assert_array_equal(c, rc)
    np.testing.assert_array_equal(w, rw)
    # u16 counters at n = 65535, k = 255 (~270 KB per pair) do not fit
    P = random_col_assigns(65535, 255, 1, 3)
    P[0, :600] = 0  # a class of >= 600 vertices: the u16 re-run is needed
    with pytest.raises(ValueError, match="shared memory"):
        DI.pairwise_distances(P, P, k=255)


@pytest.mark.parametrize("n,pe,k", [(1000, 0.9, 222), (1000, 0.5, 234)], ids=["dsjc1000.9-like", "r1000.5-like"])
def test_shapes_beyond_the_papers_runs(n, pe, k, oracle_lib):
    """Shapes the paper skipped (n k > 200,000, `PAPER.md:346`) run here,
    bit-exact vs the oracle: TabuCol on the CTA kernel (k > 128) and the
    distances (k^2 u8 counters: one warp per block)."""
    g = rand_graph(9, n, pe)
    A = random_col_assigns(n, k, 3, 9)
    keys = stream_keys(9, TAG_LS, 0, 3)
    ref = oracle_lib.tabucol_batch(g, A.copy(), k, keys, 400)
    got = LS._run_tabucol_batch(g, A.copy(), k, keys, 400)
    for key in ("best_assigns", "best_conflicts", "iters_used"):
        np.testing.assert_array_equal(got[key], ref[key])
    P, Q = got["best_assigns"], random_col_assigns(n, k, 2, 10)
    c, w = DI.pairwise_distances(P, Q, k=k)
    rc, rw = oracle_lib.pairwise(P, Q, k)
    np.testing.assert_array_equal(c, rc)
    np.testing.assert_array_equal(w, rw)
