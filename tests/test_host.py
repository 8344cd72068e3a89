"""Host-side logic (no GPU): stream contract, graph generator, initial
colourings, Coloring validation, and the C-ABI library's exports."""

import hashlib
import os
import re

import numpy as np
import pytest

from conftest import ROOT, load_golden
from paper_2109_05948_b200 import _native
from paper_2109_05948_b200.coloring import Coloring, col_conflicts, wvcp_score
from paper_2109_05948_b200.graph import WeightedGraph, rand_graph
from paper_2109_05948_b200.init import random_col_assigns, random_col_init
from paper_2109_05948_b200.rng import (TAG_INIT, TAG_LS, Stream, batch_uniform, stream_key,
                                       stream_keys, stream_value, stream_values)


def h(x):
    return hashlib.sha256(np.ascontiguousarray(x, dtype=np.int32).tobytes()).hexdigest()[:16]


def test_rng_golden():
    R = load_golden("rng")
    for spec, key, vals in zip(R["spec"], R["keys"], R["values"]):
        seed, tag, idx = eval(str(spec))
        assert stream_key(seed, tag, *idx) == int(key)
        assert [stream_value(int(key), c) for c in range(16)] == [int(v) for v in vals]
        np.testing.assert_array_equal(stream_values(key, np.arange(16, dtype=np.uint64)), vals)


def test_rng_known_answers():
    assert stream_key(1, TAG_LS, 0, 0) == 0xFAF75A0727F39370
    assert stream_key(1, TAG_INIT, 0) == 0x19438AE6B813B33D
    keys = stream_keys(1, TAG_LS, 5, 100)
    assert all(int(keys[i]) == stream_key(1, TAG_LS, 5, i) for i in range(100))


def test_batch_uniform_matches_stream():
    s = Stream(stream_key(7, TAG_INIT))
    seq = [s.uniform() for _ in range(50)]
    np.testing.assert_array_equal(batch_uniform(s.key, 0, 50), seq)


def test_graph_generator_pinned_to_reference():
    G = load_golden("graphs")
    for row in G["rows"]:
        seed, n, pe, wmax, m, de, dw, dp, di = eval(str(row))
        g = rand_graph(seed, n, pe, wmax=wmax)
        assert g.m == m
        assert (h(g.edges), h(g.weights), h(g.adj_indptr), h(g.adj_indices)) == (de, dw, dp, di)


def test_graph_appendix_a_sizes():
    for n, m, dmax in [(125, 4005, 77), (500, 62289, 280)]:
        g = rand_graph(1, n, 0.5)
        assert (g.m, g.max_degree) == (m, dmax)


def test_graph_validation():
    with pytest.raises(ValueError):
        WeightedGraph(3, [(0, 0)], [1, 1, 1])
    with pytest.raises(ValueError):
        WeightedGraph(3, [(0, 3)], [1, 1, 1])
    with pytest.raises(ValueError):
        WeightedGraph(2, [], [1, 0])
    g = WeightedGraph(4, [(1, 0), (0, 1), (2, 3)], [3, 1, 3, 2])
    assert g.m == 2 and g.edges.tolist() == [[0, 1], [2, 3]]
    assert g.weight_values.tolist() == [1, 2, 3] and g.weight_ranks.tolist() == [2, 0, 2, 1]


def test_initial_colourings_appendix_a():
    assert random_col_assigns(500, 48, 1, 1)[0, :8].tolist() == [21, 3, 7, 46, 21, 8, 1, 31]
    assert random_col_assigns(125, 18, 1, 1)[0, :8].tolist() == [9, 9, 1, 4, 9, 8, 1, 1]
    assert h(random_col_assigns(500, 48, 1, 1)[0]) == "7f5f3080ec2e8879"
    assert h(random_col_assigns(1000, 83, 1, 1)[0]) == "e0ea344fd0a74ea2"
    a = random_col_init(500, 48, Stream.derive(1, TAG_INIT, 0)).assign
    np.testing.assert_array_equal(a, random_col_assigns(500, 48, 1, 1)[0])


def test_coloring_and_objectives():
    with pytest.raises(ValueError):
        Coloring([0, 3], 3)
    with pytest.raises(ValueError):
        Coloring([], 3)
    g = WeightedGraph(3, [(0, 1), (1, 2)], [5, 3, 1])
    assert col_conflicts(g, Coloring([0, 0, 0], 1)) == 2
    assert wvcp_score(g, Coloring([0, 1, 0], 2)) == (8, 0)


def _header_symbols():
    text = open(os.path.join(ROOT, "include", "memcolor_b200.h")).read()
    return sorted(set(re.findall(r"\b(mcb_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_2109_05948_b200 import _build

    _build.build()
    L = _native.load()
    syms = _header_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(L, s), f"library does not export {s}"
    assert sorted(_native.EXPORTS) == syms
    assert b"sm_100a" in L.mcb_version()


def test_no_gpu_means_loud_failure():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    with pytest.raises(_native.NativeUnavailable):
        _native.lib()
