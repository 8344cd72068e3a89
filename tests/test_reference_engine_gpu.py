"""Drop-in proof against the reference's own caller: the unmodified
`memcolor` engine (`_generation_loop`, `mc/engine.py:171-319`, entered through
its public `run_col_fixed_k` and `run_wvcp`) runs whole generations -- local
search, surrogate training, distances, pool update, parent matching, GPX and
selection -- once with its numba operators and once with this package's
operators swapped in (INTEGRATION.md route 1: the engine's bindings of
`improve_population`, `pairwise_distances`, `Population`, `update_population`,
`match_parents`, and `memcolor.crossover.build_offspring_batch`).  The two run
records must be identical generation by generation.

The reference is imported from baseline/_ref (its pip install, which travels
to the GPU box with the repository) or /root/reference/pkg/src; the test is
skipped when neither is present or numba is missing."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    for c in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(c, "memcolor")):
            if c not in sys.path:
                sys.path.insert(0, c)
            break
    else:
        pytest.skip("reference package not installed (baseline/_ref)")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/mcb_numba_cache")
    pytest.importorskip("numba")
    import memcolor.crossover as X
    import memcolor.engine as E
    import memcolor.graph as G

    return E, X, G


def _swap(E, X, monkeypatch):
    from paper_2109_05948_b200 import crossover, distance, localsearch, population

    monkeypatch.setattr(E, "improve_population", localsearch.improve_population)
    monkeypatch.setattr(E, "pairwise_distances", distance.pairwise_distances)
    monkeypatch.setattr(E, "Population", population.Population)
    monkeypatch.setattr(E, "update_population", population.update_population)
    monkeypatch.setattr(E, "match_parents", population.match_parents)
    monkeypatch.setattr(X, "build_offspring_batch", crossover.build_offspring_batch)


def _graph(G, seed, n, pe, wmax):
    from paper_2109_05948_b200.graph import rand_graph

    g = rand_graph(seed, n, pe, wmax=wmax)
    return G.WeightedGraph(n, [tuple(e) for e in g.edges.tolist()], g.weights.tolist(), name=f"rand{seed}")


def _strip(record):
    gens = []
    for gen in record.generations:
        gens.append({k: v for k, v in gen.items() if k not in ("time", "wall_time_s")})
    return gens, record.best_score, record.best_assign, record.counters, record.stop_reason


def _same(a, b):
    ga, sa, aa, ca, ra = _strip(a)
    gb, sb, ab, cb, rb = _strip(b)
    assert len(ga) == len(gb)
    for i, (x, y) in enumerate(zip(ga, gb)):
        assert x.keys() == y.keys(), i
        for key in x:
            xv, yv = x[key], y[key]
            if isinstance(xv, float) or isinstance(yv, float):
                assert (xv == yv) or (np.isnan(xv) and np.isnan(yv)), (i, key, xv, yv)
            else:
                assert xv == yv, (i, key, xv, yv)
    assert sa == sb and aa == ab and ca == cb and ra == rb


@pytest.mark.parametrize("use_surrogate", [False, True], ids=["uniform-select", "surrogate"])
def test_col_generations_identical(ref, use_surrogate, monkeypatch):
    E, X, G = ref
    g = _graph(G, 3, 80, 0.5, 1)
    cfg = dict(problem="col", p=16, K=4, seed=3, max_generations=4, ls_depth_mult=8, epochs=2,
               batch_size=8, use_surrogate=use_surrogate)
    _, rec_ref = E.run_col_fixed_k(g, 9, E.RunConfig(**cfg))
    with monkeypatch.context() as m:
        _swap(E, X, m)
        _, rec_ours = E.run_col_fixed_k(g, 9, E.RunConfig(**cfg))
    assert len(rec_ref.generations) == 4
    _same(rec_ref, rec_ours)


def test_wvcp_generations_identical(ref, monkeypatch):
    E, X, G = ref
    g = _graph(G, 4, 70, 0.5, 20)
    cfg = dict(problem="wvcp", p=12, K=4, seed=5, max_generations=3, ls_depth_mult=3, max_ls_rounds=3,
               epochs=2, batch_size=6, use_surrogate=True)
    _, rec_ref = E.run_wvcp(g, E.RunConfig(**cfg))
    with monkeypatch.context() as m:
        _swap(E, X, m)
        _, rec_ours = E.run_wvcp(g, E.RunConfig(**cfg))
    assert len(rec_ref.generations) == 3
    _same(rec_ref, rec_ours)
