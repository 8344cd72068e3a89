"""Greedy weighted initialisation: the CPU restatement (oracle/init_oracle.py)
against the reference's own colourings (tests/golden/init.npz, made by
tests/golden/make_golden.py from `mc/init.py:57-64`), and the package's
greedy order against the oracle's."""

import numpy as np

from conftest import load_golden
from oracle import init_oracle as IO
from paper_2109_05948_b200.graph import rand_graph
from paper_2109_05948_b200.init import greedy_order, stream_keys_init


def _case(G, name):
    seed, n, pe, wmax, p, ms = G[f"{name}__params"]
    g = rand_graph(int(seed), int(n), float(pe), wmax=int(wmax))
    return g, int(p), int(ms)


def test_oracle_matches_reference_fixtures():
    G = load_golden("init")
    for name in G["cases"]:
        g, p, ms = _case(G, name)
        a, used, k = IO.init_wvcp_population(g.adj_indptr, g.adj_indices, g.weights, g.degrees,
                                             stream_keys_init(ms, p))
        np.testing.assert_array_equal(a, G[f"{name}__assigns"], err_msg=str(name))
        assert k == int(G[f"{name}__k"])


def test_greedy_order_matches_oracle():
    for seed, n, pe, wmax in [(1, 125, 0.5, 100), (3, 50, 0.4, 1), (4, 300, 0.2, 3)]:
        g = rand_graph(seed, n, pe, wmax=wmax)
        np.testing.assert_array_equal(greedy_order(g), IO.greedy_order(g.weights, g.degrees))


def test_oracle_colourings_are_legal():
    g = rand_graph(2, 150, 0.6, wmax=20)
    a, used, k = IO.init_wvcp_population(g.adj_indptr, g.adj_indices, g.weights, g.degrees,
                                         stream_keys_init(4, 5))
    for row, u in zip(a, used):
        assert (row[g.edges[:, 0]] != row[g.edges[:, 1]]).all()
        assert row.max() == u - 1 and row.min() == 0
