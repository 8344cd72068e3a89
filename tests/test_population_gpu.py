"""GPU population update / parent matching (csrc/population.cu) against the
reference fixtures and the CPU oracle (exact: admitted order, by-rule mask,
new distance matrix, assignments, fitness, neighbour order)."""

import numpy as np
import pytest

from conftest import load_golden
from oracle import population_oracle as PO
from paper_2109_05948_b200 import population as GP

pytestmark = pytest.mark.gpu
POP = load_golden("population")


def _pop(assigns, fit, dist, k):
    return GP.Population(assigns=np.ascontiguousarray(assigns, np.int32), k=k,
                         fitness=np.asarray(fit, np.int64), dist=np.ascontiguousarray(dist, np.int32))


@pytest.mark.parametrize("name", [str(c) for c in POP["cases"]])
def test_gpu_matches_reference_fixtures(name):
    pre = name + "__"
    seed, n, k, p, q, ms, K = (int(x) for x in POP[pre + "params"])
    pop = _pop(POP[pre + "pop_assigns"], POP[pre + "pop_fit"], POP[pre + "pop_dist"], k)
    res = GP.update_population(pop, POP[pre + "new_assigns"], POP[pre + "new_fit"], POP[pre + "cross"],
                               POP[pre + "within"], ms)
    np.testing.assert_array_equal(res.assigns, POP[pre + "res_assigns"])
    np.testing.assert_array_equal(res.fitness, POP[pre + "res_fit"])
    np.testing.assert_array_equal(res.dist, POP[pre + "res_dist"])
    np.testing.assert_array_equal(res.admitted_by_rule, POP[pre + "res_rule"].astype(bool))
    assert res.generation == 1
    np.testing.assert_array_equal(GP.match_parents(res, K), POP[pre + "matches"])


def _random_case(rs, p, q, n, clusters, fit_range):
    """Distances of colourings drawn around `clusters` centres (symmetric,
    zero diagonal, values in [0, n])."""
    cen = rs.integers(0, clusters, size=p + q)
    base = rs.integers(0, n // 3, size=(clusters, clusters))
    base = np.minimum(base + base.T + n // 2, n)
    D = base[cen][:, cen] + rs.integers(0, n // 8, size=(p + q, p + q))
    D = np.minimum((D + D.T) // 2, n).astype(np.int32)
    same = cen[:, None] == cen[None, :]
    D[same] = rs.integers(0, n // 10 + 3, size=int(same.sum()))
    D = np.minimum(D, D.T)
    np.fill_diagonal(D, 0)
    fit = rs.integers(0, fit_range, size=p + q).astype(np.int64)
    return D[:p, :p].copy(), D[:p, p:].copy(), D[p:, p:].copy(), fit[:p], fit[p:]


@pytest.mark.parametrize("p,q,n,clusters,fit_range", [(64, 64, 100, 5, 4), (200, 150, 300, 40, 10),
                                                       (150, 150, 60, 3, 3), (300, 1, 500, 300, 1000),
                                                       (100, 300, 200, 8, 2)])
def test_gpu_vs_oracle_random(p, q, n, clusters, fit_range):
    rs = np.random.default_rng(p * 7 + q)
    pd, cr, wi, fp, fq = _random_case(rs, p, q, n, clusters, fit_range)
    pa = rs.integers(0, 9, size=(p, 17)).astype(np.int32)
    na = rs.integers(0, 9, size=(q, 17)).astype(np.int32)
    ms = n // 10
    adm, rule, nd, nas, nf = PO.update_population(pd, fp, pa, na, fq, cr, wi, ms)
    res = GP.update_population(_pop(pa, fp, pd, 9), na, fq, cr, wi, ms)
    np.testing.assert_array_equal(res.assigns, nas)
    np.testing.assert_array_equal(res.fitness, nf)
    np.testing.assert_array_equal(res.dist, nd)
    np.testing.assert_array_equal(res.admitted_by_rule, rule)
    for K in (1, 7, min(31, p - 1), min(40, p - 1)):
        res.assigns = np.zeros((p, n), np.int32)  # n drives the histogram size
        np.testing.assert_array_equal(GP.match_parents(res, K), PO.match_parents(nd, K))


def test_gpu_large_properties():
    """p = q = 4096 (the oracle would take minutes): spacing rule, fill order,
    distance gather and neighbour order checked directly."""
    rs = np.random.default_rng(11)
    p = q = 4096
    n = 1000
    pd, cr, wi, fp, fq = _random_case(rs, p, q, n, 600, 50)
    ms = n // 10
    pa = np.zeros((p, n), np.int32)  # n bounds the distances
    na = np.zeros((q, n), np.int32)
    res = GP.update_population(_pop(pa, fp, pd, 2), na, fq, cr, wi, ms)
    full = np.block([[pd, cr], [cr.T, wi]])
    cand_fit = np.concatenate([fp, fq])
    order = np.lexsort((np.concatenate([np.arange(p), np.arange(q)]),
                        np.concatenate([np.zeros(p, np.int64), np.ones(q, np.int64)]), cand_fit))
    rank = np.empty(p + q, np.int64)
    rank[order] = np.arange(p + q)
    # recover admitted ids from the fitness + distance rows: the rule admissions
    # form a ms-separated set, listed in rank order, then the fill in rank order
    np.testing.assert_array_equal(np.sort(res.fitness[res.admitted_by_rule]), res.fitness[res.admitted_by_rule])
    assert (res.dist == res.dist.T).all() and (np.diag(res.dist) == 0).all()
    rule_block = res.dist[np.ix_(res.admitted_by_rule, res.admitted_by_rule)]
    off = rule_block[~np.eye(rule_block.shape[0], dtype=bool)]
    assert (off > ms).all()
    K = 16
    m = GP.match_parents(res, K)
    rows = np.arange(p)[:, None]
    d = res.dist[rows, m]
    assert (m != rows).all()
    assert ((d[:, 1:] > d[:, :-1]) | ((d[:, 1:] == d[:, :-1]) & (m[:, 1:] > m[:, :-1]))).all()
    kth = np.sort(np.where(np.eye(p, dtype=bool), 10 ** 9, res.dist), axis=1)[:, K - 1]
    assert (d[:, -1] == kth).all()


def test_match_parents_errors():
    pop = _pop(np.zeros((4, 3), np.int32), np.zeros(4), np.zeros((4, 4), np.int32), 2)
    with pytest.raises(ValueError):
        GP.match_parents(pop, 0)
    with pytest.raises(ValueError):
        GP.match_parents(pop, 4)
