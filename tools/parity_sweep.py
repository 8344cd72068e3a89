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
print(json.dumps({"tabucol_cases": a.tabucol, "wvcp_cases": a.wvcp, "mismatches": bad}))
