"""One-off large randomised parity sweep (not part of the test suite): TabuCol
and WVCP on random shapes covering every kernel path, each bit-exact vs the C
oracle.  python tools/parity_sweep.py [--tabucol 200] [--wvcp 60] [--seed 0]"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle  # noqa: E402
from paper_2109_05948_b200 import localsearch as LS  # noqa: E402
from paper_2109_05948_b200.graph import rand_graph  # noqa: E402
from paper_2109_05948_b200.init import random_col_assigns  # noqa: E402
from paper_2109_05948_b200.rng import TAG_LS, stream_keys  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tabucol", type=int, default=200)
ap.add_argument("--wvcp", type=int, default=60)
ap.add_argument("--ops", type=int, default=60, help="cases each for distances, GPX, population, greedy init")
ap.add_argument("--seed", type=int, default=0)
a = ap.parse_args()
oracle.build()
bad = []
for t in range(a.tabucol):
    rs = np.random.default_rng(10_000 * a.seed + t)
    n = int(rs.choice([rs.integers(2, 100), rs.integers(100, 700), rs.integers(700, 2500)]))
    pe = float(rs.uniform(0.01, 0.98))
    k = int(rs.choice([rs.integers(2, 10), rs.integers(10, 90), rs.integers(90, 256)]))
    p = int(rs.integers(1, 40))
    depth = int(min(8000, max(1, rs.integers(1, max(2, 60_000_000 // max(1, n * p))))))
    g = rand_graph(t + 1, n, pe)
    A = random_col_assigns(n, k, p, t + 7)
    keys = stream_keys(t, TAG_LS, 1, p)
    ref = oracle.tabucol_batch(g, A.copy(), k, keys, depth)
    got = LS._run_tabucol_batch(g, A.copy(), k, keys, depth)
    ok = all(np.array_equal(got[x], ref[x]) for x in ("best_assigns", "best_conflicts", "end_assigns", "iters_used"))
    if not ok:
        bad.append(("tabucol", t, n, pe, k, p, depth))
for t in range(a.wvcp):
    rs = np.random.default_rng(20_000 * a.seed + t)
    n = int(rs.integers(2, 800))
    pe = float(rs.uniform(0.02, 0.97))
    k = int(rs.integers(2, 120))
    wmax = int(rs.choice([1, 3, 100, 10**6]))
    p = int(rs.integers(1, 12))
    depth = int(max(1, rs.integers(1, max(2, 2_000_000 // max(1, n * p)))))
    rounds = int(rs.integers(1, 5))
    sched = bool(rs.integers(0, 2))
    phi0 = float(rs.choice([LS.default_wvcp_phi0(rand_graph(t + 900, n, pe, wmax=wmax), k),
                            float(rs.integers(1, 40)) * 2.0 ** -int(rs.integers(0, 4)), float(rs.uniform(0.1, 50))]))
    g = rand_graph(t + 900, n, pe, wmax=wmax)
    A = random_col_assigns(n, k, p, t + 99)
    keys = stream_keys(t, TAG_LS, 2, p)
    ref = oracle.wvcp_batch(g, A.copy(), k, keys, depth, rounds, sched, phi0)
    got = LS._run_wvcp_batch(g, A.copy(), k, keys, depth, rounds, sched, phi0)
    ok = all(np.array_equal(got[x], ref[x]) for x in ("best_assigns", "best_scores", "end_scores", "phi_used"))
    if not ok:
        bad.append(("wvcp", t, n, pe, k, p, depth, phi0))
from oracle import init_oracle as IO  # noqa: E402
from oracle import population_oracle as PO  # noqa: E402
from paper_2109_05948_b200 import crossover as CX  # noqa: E402
from paper_2109_05948_b200 import distance as DI  # noqa: E402
from paper_2109_05948_b200 import population as PP  # noqa: E402
from paper_2109_05948_b200.init import greedy_wvcp_assigns, stream_keys_init  # noqa: E402
from paper_2109_05948_b200.rng import TAG_CROSS  # noqa: E402

for t in range(a.ops):
    rs = np.random.default_rng(30_000 * a.seed + t)
    n, k = int(rs.integers(1, 3000)), int(rs.integers(1, 256))
    p, q = int(rs.integers(0, 10)), int(rs.integers(1, 10))
    P = random_col_assigns(n, k, p, t + 3) if p else np.zeros((0, n), np.int32)
    Q = random_col_assigns(n, k, q, t + 4)
    if p and t % 2:
        Q[: min(p, q)] = rs.permutation(k)[P[: min(p, q)]]
    c, w = DI.pairwise_distances(P, Q, k=k)
    rc, rw = oracle.pairwise(P, Q, k)
    if not (np.array_equal(c, rc) and np.array_equal(w, rw)):
        bad.append(("distance", t, n, k, p, q))
    if q >= 2:
        K = int(rs.integers(1, q))
        m = rs.integers(0, q, size=(q, K)).astype(np.int64)
        ck = stream_keys(t, TAG_CROSS, 0, q * K)
        if not np.array_equal(CX.gpx_batch(Q, m, k, ck), oracle.gpx_batch(Q, m, k, ck)):
            bad.append(("gpx", t, n, k, q, K))
    # population update / matching on a random symmetric distance pool
    pp, qq, nn = int(rs.integers(2, 60)), int(rs.integers(1, 60)), int(rs.integers(2, 300))
    pa = random_col_assigns(nn, 5, pp, t + 5)
    ia = random_col_assigns(nn, 5, qq, t + 6)
    _, wpp = oracle.pairwise(pa[:0], pa, 5)
    cr, wi = oracle.pairwise(pa, ia, 5)
    pf = rs.integers(0, 20, pp).astype(np.int64)
    qf = rs.integers(0, 20, qq).astype(np.int64)
    ms = int(rs.integers(0, nn // 2 + 1))
    pop = PP.Population(assigns=pa, k=5, fitness=pf, dist=wpp)
    got = PP.update_population(pop, ia, qf, cr, wi, ms)
    radm, rrule, rdist, rassign, rfit = PO.update_population(wpp, pf, pa, ia, qf, cr, wi, ms)
    if not (np.array_equal(got.assigns, rassign) and np.array_equal(got.fitness, rfit) and np.array_equal(got.dist, rdist)):
        bad.append(("update_population", t, pp, qq, nn, ms))
    K = int(rs.integers(1, pp))
    if not np.array_equal(PP.match_parents(got, K), PO.match_parents(got.dist, K)):
        bad.append(("match_parents", t, pp, K))
    # greedy weighted initialisation
    gn = int(rs.integers(1, 400))
    gg = rand_graph(t + 17, gn, float(rs.uniform(0, 0.95)), wmax=int(rs.integers(1, 50)))
    keys = stream_keys_init(t, int(rs.integers(1, 8)))
    ga, gu = greedy_wvcp_assigns(gg, keys)
    ra, ru, _ = IO.init_wvcp_population(gg.adj_indptr, gg.adj_indices, gg.weights, gg.degrees, keys)
    if not (np.array_equal(ga, ra) and np.array_equal(gu, ru)):
        bad.append(("greedy_init", t, gn))
print(json.dumps({"tabucol_cases": a.tabucol, "wvcp_cases": a.wvcp, "op_cases": a.ops, "mismatches": bad}))
