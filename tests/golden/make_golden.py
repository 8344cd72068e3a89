"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (where /root/reference exists and numba is
installed):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports the reference package (`/root/reference/pkg/src/memcolor`) and its
test oracles (`/root/reference/pkg/tests/oracles.py`) and records, for seeded
inputs, the outputs of the reference's own hot-path kernels:

* rng.npz       stream_key / stream_value / u64_below (`rng.py:56-82`)
* graphs.npz    rand_graph digests (`tests/oracles.py:15-22`)
* tabucol.npz   _run_tabucol_batch outputs + move logs (`localsearch.py:556`)
* wvcp.npz      _run_wvcp_batch outputs + move logs (`localsearch.py:427`)
* gpx.npz       build_offspring_batch / gpx (`crossover.py:69-93`)
* distance.npz  pairwise_distances / approx_partition_distance (`distance.py:75-155`)
* population.npz  update_population / match_parents (`population.py:59-141`)
* init.npz      init_wvcp_population greedy colourings (`init.py:23-64`)
* surrogate.npz SurrogateNet init / gradients / online training / predictions (`surrogate.py`)
* engine.npz    k-colouring generations without the surrogate, chained from the
                reference's own operators as `engine.py:_generation_loop` does
* improve.npz   improve_population LsResults, COL and WVCP, generations > 0 and
                the default depths (`localsearch.py:615-682`)

Inputs are regenerated in the tests from the recorded parameters with the
package's own generators (which are themselves pinned by graphs.npz and the
initial-colouring digests), so the fixtures stay small.  Nothing at test time
reads /root/reference.
"""

from __future__ import annotations

import hashlib
import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import numpy as np  # noqa: E402

from memcolor import crossover as RCX  # noqa: E402
from memcolor import distance as RDI  # noqa: E402
from memcolor import localsearch as RLS  # noqa: E402
from memcolor import population as RPOP  # noqa: E402
from memcolor import rng as RRNG  # noqa: E402
from memcolor.coloring import Coloring as RColoring  # noqa: E402
from oracles import rand_graph as ref_rand_graph  # noqa: E402

from paper_2109_05948_b200.graph import rand_graph  # noqa: E402
from paper_2109_05948_b200.init import random_col_assigns  # noqa: E402
from paper_2109_05948_b200.rng import TAG_CROSS, TAG_LS, stream_keys  # noqa: E402


def digest(x):
    return hashlib.sha256(np.ascontiguousarray(x, dtype=np.int32).tobytes()).hexdigest()[:16]


# --------------------------------------------------------------------------
# TabuCol cases: (name, seed, n, p_edge, k, pop, depth, log_cap, full_arrays)
# --------------------------------------------------------------------------
TABUCOL_CASES = [
    ("c1", 1, 125, 0.5, 18, 64, 10000, 10000, True),      # BASELINE config 0
    ("c2s", 1, 500, 0.5, 48, 4, 50000, 4000, True),       # config 1 shape, 4 individuals
    ("c2w", 1, 500, 0.5, 48, 32, 3000, 3000, True),       # config 1 shape, 32 x 3k
    ("c3s", 1, 1000, 0.5, 83, 2, 4000, 4000, True),       # config 2 shape
    ("k2dense", 5, 300, 0.9, 2, 4, 400, 400, True),       # gamma > 127: wide-table path
    ("k3", 7, 60, 0.3, 3, 16, 2000, 2000, True),
    ("k5sparse", 8, 200, 0.05, 5, 16, 5000, 5000, True),
    ("k8", 9, 90, 0.4, 8, 16, 3000, 3000, True),
    ("k40", 10, 200, 0.9, 40, 8, 4000, 4000, True),
    ("k64", 11, 400, 0.85, 64, 4, 3000, 3000, True),
    ("k70", 12, 400, 0.9, 70, 4, 3000, 3000, True),       # k > 64
    ("k150", 13, 700, 0.95, 150, 2, 1500, 1500, True),    # config 5 palette
    ("c5s", 1, 2000, 0.5, 150, 2, 2000, 2000, True),      # config 4 (C5) shape: the cluster kernel
    ("easy", 14, 80, 0.1, 6, 16, 5000, 5000, True),       # early exits
    ("k1", 15, 30, 0.3, 1, 4, 100, 100, True),            # k < 2: no iterations
    ("edgeless", 16, 40, 0.0, 4, 4, 100, 100, True),      # m = 0
    ("n1", 17, 1, 0.5, 3, 2, 10, 10, True),               # single vertex
    ("tenure", 18, 500, 0.9, 8, 2, 2500, 2500, True),     # long tenures (conflicts ~ 1e4)
    ("long", 19, 100, 0.5, 14, 4, 40000, 0, True),        # > 2x16384 iterations (stamp wrap)
    ("tenure32", 20, 800, 0.9, 4, 2, 300, 300, True),     # tenure > 16383 and gamma > 127
]

WVCP_CASES = [
    # name, seed, n, p_edge, wmax, k, pop, depth, rounds, schedule, phi0 (None=default), log
    ("c4s", 1, 500, 0.5, 100, 60, 2, 5000, 10, True, None, 4000),
    ("c4w", 1, 500, 0.5, 100, 60, 16, 300, 4, True, None, 1200),
    ("small", 21, 60, 0.4, 9, 10, 16, 400, 5, True, None, 2000),
    ("fixed", 22, 80, 0.3, 20, 12, 8, 600, 1, False, 3.0, 600),
    ("unit", 23, 100, 0.5, 1, 20, 8, 500, 3, True, None, 1500),
    ("k70", 24, 150, 0.5, 50, 70, 4, 300, 3, True, None, 900),
    ("legal", 25, 50, 0.1, 30, 12, 8, 400, 3, True, None, 1200),
]


def gen_tabucol(out):
    meta = []
    for name, seed, n, pe, k, pop, depth, cap, _ in TABUCOL_CASES:
        g = ref_rand_graph(seed, n, pe, wmax=1) if n <= 600 else None
        mine = rand_graph(seed, n, pe, wmax=1)
        if g is not None:
            assert np.array_equal(g.edges, mine.edges), name
        else:
            g = mine  # n > 600: ref rand_graph is a pure-Python n^2 loop
        if k >= 1:
            A = random_col_assigns(n, k, pop, seed)
        keys = stream_keys(seed, TAG_LS, 0, pop)
        r = RLS._run_tabucol_batch(g, A.copy(), k, keys, depth, log_moves=cap > 0)
        pre = f"{name}__"
        out[pre + "params"] = np.array([seed, n, int(pe * 1000), k, pop, depth, cap], np.int64)
        out[pre + "init_digest"] = np.array([digest(A)])
        out[pre + "best_conflicts"] = r["best_conflicts"]
        out[pre + "end_conflicts"] = r["end_conflicts"]
        out[pre + "iters_used"] = r["iters_used"]
        out[pre + "end_assigns"] = r["end_assigns"].astype(np.uint8)
        out[pre + "best_assigns"] = r["best_assigns"].astype(np.uint8)
        if cap > 0:
            lv, li, lt, lc = r["log"]
            out[pre + "log_cnt"] = lc
            nkeep = min(pop, 8)
            out[pre + "log_v"] = lv[:nkeep, :cap].astype(np.int16)
            out[pre + "log_iter"] = li[:nkeep, :cap].astype(np.int32)
            out[pre + "log_tt"] = lt[:nkeep, :cap].astype(np.int32)
        meta.append(name)
        print("tabucol", name, r["best_conflicts"][:4], r["iters_used"][:4])
    out["cases"] = np.array(meta)


def gen_wvcp(out):
    meta = []
    for name, seed, n, pe, wmax, k, pop, depth, rounds, sched, phi0, cap in WVCP_CASES:
        g = ref_rand_graph(seed, n, pe, wmax=wmax)
        mine = rand_graph(seed, n, pe, wmax=wmax)
        assert np.array_equal(g.edges, mine.edges) and np.array_equal(g.weights, mine.weights)
        A = random_col_assigns(n, k, pop, seed)
        keys = stream_keys(seed, TAG_LS, 0, pop)
        phi = RLS.default_wvcp_phi0(g, k) if phi0 is None else phi0
        r = RLS._run_wvcp_batch(g, A.copy(), k, keys, depth, rounds, sched, phi, log_moves=True)
        pre = f"{name}__"
        out[pre + "params"] = np.array([seed, n, int(pe * 1000), wmax, k, pop, depth, rounds,
                                        int(sched)], np.int64)
        out[pre + "phi0"] = np.array([phi], np.float64)
        for key in ["best_scores", "end_scores", "end_conflicts", "phi_used"]:
            out[pre + key] = r[key]
        out[pre + "end_assigns"] = r["end_assigns"].astype(np.uint8)
        out[pre + "best_assigns"] = r["best_assigns"].astype(np.uint8)
        lv, li, lt, la, lc = r["log"]
        nkeep = min(pop, 4)
        c = min(cap, lv.shape[1])
        out[pre + "log_cnt"] = lc
        out[pre + "log_v"] = lv[:nkeep, :c].astype(np.int16)
        out[pre + "log_iter"] = li[:nkeep, :c].astype(np.int32)
        out[pre + "log_tt"] = lt[:nkeep, :c].astype(np.int32)
        out[pre + "log_asp"] = la[:nkeep, :c]
        meta.append(name)
        print("wvcp", name, r["best_scores"][:4], r["end_scores"][:4])
    out["cases"] = np.array(meta)


def gen_gpx(out):
    meta = []
    cases = [("appA", 1, 1000, 83, 8, 4, "ring")]
    for s in range(12):
        st = RRNG.Stream(900 + s)
        n = 1 + st.below(300)
        k = 1 + st.below(40)
        p = 2 + st.below(6)
        K = 1 + st.below(p - 1) if p > 1 else 1
        cases.append((f"r{s}", 900 + s, n, k, p, K, "rand"))
    cases.append(("k150", 77, 2000, 150, 4, 3, "rand"))
    for name, seed, n, k, p, K, how in cases:
        P = random_col_assigns(n, k, p, seed)
        if how == "ring":
            matches = np.array([[(i + 1 + j) % p for j in range(K)] for i in range(p)], np.int64)
        else:
            st = RRNG.Stream(seed * 31 + 7)
            matches = np.array([[st.below(p) for _ in range(K)] for _ in range(p)], np.int64)
        o = RCX.build_offspring_batch(P, matches, k, seed, 0)
        keys = stream_keys(seed, TAG_CROSS, 0, p * K)
        # single-pair API on job 0 (`crossover.py:69-78`)
        single = RCX.gpx(RColoring(P[0], k), RColoring(P[matches[0, 0]], k), k,
                         RRNG.Stream(int(keys[0])))
        assert np.array_equal(single.assign, o[0, 0])
        pre = f"{name}__"
        out[pre + "params"] = np.array([seed, n, k, p, K], np.int64)
        out[pre + "matches"] = matches
        out[pre + "out"] = o.astype(np.uint8)
        meta.append(name)
    out["cases"] = np.array(meta)
    print("gpx", len(meta))


def gen_distance(out):
    meta = []
    cases = [("appA", 1, 1000, 83, 8, 8)]
    for s in range(16):
        st = RRNG.Stream(500 + s)
        cases.append((f"r{s}", 500 + s, 1 + st.below(200), 1 + st.below(40), st.below(6), 1 + st.below(7)))
    cases.append(("k150", 3, 2000, 150, 5, 6))
    cases.append(("near", 4, 300, 10, 6, 6))  # near-identical partitions
    for name, seed, n, k, p, q in cases:
        if name == "appA":
            P = random_col_assigns(n, k, p, seed)
            matches = np.array([[(i + 1 + j) % 8 for j in range(4)] for i in range(8)], np.int64)
            Q = RCX.build_offspring_batch(P, matches, k, seed, 0)[:, 0]
        elif name == "near":
            P = random_col_assigns(n, k, p, seed)
            Q = P.copy()
            st = RRNG.Stream(4444)
            for i in range(q):
                for _ in range(5):
                    Q[i, st.below(n)] = st.below(k)
        else:
            P = random_col_assigns(n, k, p, seed)
            Q = random_col_assigns(n, k, q, seed + 10_000)
        cross, within = RDI.pairwise_distances(P, Q, k=k)
        pre = f"{name}__"
        out[pre + "params"] = np.array([seed, n, k, p, q], np.int64)
        out[pre + "P"] = P.astype(np.uint8)
        out[pre + "Q"] = Q.astype(np.uint8)
        out[pre + "cross"] = cross
        out[pre + "within"] = within
        meta.append(name)
    # hand cases incl. the reference's known-bad expectation
    hand = [([0, 0, 1, 1], [0, 1, 0, 1], 2), ([0, 1, 2, 0], [0, 1, 2, 0], 3),
            ([0, 0, 1, 1, 2], [2, 2, 0, 0, 1], 3), ([0, 0, 1, 1, 2, 2], [0, 0, 1, 1, 2, 1], 3)]
    out["hand_values"] = np.array(
        [RDI.approx_partition_distance(RColoring(a, k), RColoring(b, k)) for a, b, k in hand])
    out["cases"] = np.array(meta)
    print("distance", len(meta), out["hand_values"])


# --------------------------------------------------------------------------
# population update / matching: (name, seed, n, k, p, q, n_close, fit_range, K)
#   n_close newcomers are perturbed copies of incumbents (distance <= ms), so
#   the spacing rule rejects and the fallback fill runs; fit_range small gives
#   fitness ties (origin / index tie-breaks)
# --------------------------------------------------------------------------
POP_CASES = [
    ("small", 3, 60, 6, 12, 12, 4, 5, 3),
    ("ties", 4, 80, 8, 20, 24, 10, 3, 5),
    ("crowded", 5, 50, 5, 16, 16, 16, 2, 4),   # many within ms: fill path
    ("wide", 6, 120, 10, 32, 32, 8, 40, 7),
    ("q0", 7, 40, 4, 10, 0, 0, 4, 2),          # no newcomers
    ("clones", 8, 50, 5, 12, 12, -1, 3, 3),    # all candidates near one colouring: fallback fill
    ("half", 9, 60, 6, 16, 16, -2, 4, 5),      # two clusters: 2 by the rule, the rest filled
]


def gen_population(out):
    from memcolor.distance import pairwise_distances as rpd

    for name, seed, n, k, p, q, n_close, fr, K in POP_CASES:
        rs = np.random.default_rng(seed)
        pop_a = rs.integers(0, k, size=(p, n)).astype(np.int32)
        new_a = rs.integers(0, k, size=(q, n)).astype(np.int32)
        ms = RPOP.min_spacing(n)
        if n_close < 0:
            # -1: every candidate a perturbation of one base colouring; -2: of two bases
            bases = rs.integers(0, k, size=(-n_close, n)).astype(np.int32)
            for arr in (pop_a, new_a):
                for t in range(arr.shape[0]):
                    arr[t] = bases[t % bases.shape[0]]
                    flip = rs.choice(n, size=1, replace=False)
                    arr[t, flip] = rs.integers(0, k, size=1)
        for t in range(max(0, min(n_close, q))):
            src = pop_a[rs.integers(0, p)] if t % 2 == 0 else new_a[rs.integers(0, max(t, 1))]
            new_a[t] = src
            flip = rs.choice(n, size=max(1, ms // 3), replace=False)
            new_a[t, flip] = rs.integers(0, k, size=flip.size)
        pop_f = rs.integers(0, fr, size=p).astype(np.int64)
        new_f = rs.integers(0, fr, size=q).astype(np.int64)
        cols = [RColoring(pop_a[i], k) for i in range(p)]
        pop = RPOP.Population.from_colorings(cols, pop_f)
        cross, within = rpd(pop_a, new_a, k=k)
        res = RPOP.update_population(pop, new_a, new_f, cross, within, ms)
        m = RPOP.match_parents(res, K)
        pre = name + "__"
        out[pre + "params"] = np.array([seed, n, k, p, q, ms, K], dtype=np.int64)
        out[pre + "pop_assigns"] = pop_a
        out[pre + "new_assigns"] = new_a
        out[pre + "pop_fit"] = pop_f
        out[pre + "new_fit"] = new_f
        out[pre + "pop_dist"] = pop.dist.astype(np.int32)
        out[pre + "cross"] = np.asarray(cross, dtype=np.int32)
        out[pre + "within"] = np.asarray(within, dtype=np.int32)
        out[pre + "res_assigns"] = res.assigns.astype(np.int32)
        out[pre + "res_fit"] = res.fitness.astype(np.int64)
        out[pre + "res_dist"] = res.dist.astype(np.int32)
        out[pre + "res_rule"] = res.admitted_by_rule.astype(np.uint8)
        out[pre + "matches"] = m.astype(np.int64)
    out["cases"] = np.array([c[0] for c in POP_CASES])


# --------------------------------------------------------------------------
# engine: generations of mc/engine.py:_generation_loop (:203-316) for COL with
# use_surrogate=False, chained from the reference's own functions
#   (name, seed, n, p_edge, k, p, K, depth, generations)
# --------------------------------------------------------------------------
ENGINE_CASES = [
    ("e1", 3, 70, 0.5, 9, 12, 3, 400, 4),
    ("e2", 5, 90, 0.3, 6, 16, 5, 600, 3),
]


def gen_engine(out):
    from memcolor.coloring import Coloring as RC
    from memcolor.coloring import col_conflicts as rcc
    from memcolor.crossover import build_and_select_offspring
    from memcolor.distance import pairwise_distances as rpd
    from memcolor.init import init_col_population

    for name, seed, n, pe, k, p, K, depth, G in ENGINE_CASES:
        g = ref_rand_graph(seed, n, pe)
        init = init_col_population(n, k, p, seed)
        fit = np.array([rcc(g, c) for c in init.colorings], dtype=np.int64)
        pop = RPOP.Population.from_colorings(init.colorings, fit)
        ms = RPOP.min_spacing(n)
        offspring = list(init.colorings)
        pre = name + "__"
        out[pre + "params"] = np.array([seed, n, int(pe * 1000), k, p, K, depth, G], dtype=np.int64)
        out[pre + "init"] = pop.assigns.astype(np.int32)
        for t in range(G):
            res = RLS.improve_population(g, offspring, RLS.COL, seed, generation=t, depth=depth)
            imp = np.stack([r.best.assign for r in res]).astype(np.int32)
            imp_fit = np.array([min(r.best_score, int(RLS.INF_SCORE)) for r in res], dtype=np.int64)
            cross, within = rpd(pop.assigns, imp, k=k)
            pop = RPOP.update_population(pop, imp, imp_fit, cross, within, ms)
            matches = RPOP.match_parents(pop, K)
            batch = build_and_select_offspring(pop, matches, None, seed, t, use_surrogate=False)
            offspring = [RC(batch.selected_assigns[i], k) for i in range(p)]
            out[pre + f"g{t}_improved"] = imp
            out[pre + f"g{t}_pop"] = pop.assigns.astype(np.int32)
            out[pre + f"g{t}_fit"] = pop.fitness.astype(np.int64)
            out[pre + f"g{t}_dist"] = pop.dist.astype(np.int32)
            out[pre + f"g{t}_matches"] = matches.astype(np.int64)
            out[pre + f"g{t}_selected"] = batch.selected_index.astype(np.int64)
            out[pre + f"g{t}_offspring"] = batch.selected_assigns.astype(np.int32)
    out["cases"] = np.array([c[0] for c in ENGINE_CASES])
    gen_engine_wvcp(out)
    gen_engine_surrogate(out)


ENGINE_SURROGATE_CASES = [  # (name, seed, n, p_edge, k, p, K, depth, G, epochs, batch)
    ("es1", 3, 60, 0.5, 8, 12, 4, 300, 3, 2, 5),
]


def gen_engine_surrogate(out):
    """k-colouring generations with the surrogate (`use_surrogate=True`,
    float64 net, arch "small"): training on (restart points, realized scores)
    with TAG_TRAIN streams (`engine.py:263-281`) and argmin selection
    (`crossover.py:114-118`)."""
    from memcolor.coloring import Coloring as RC
    from memcolor.coloring import col_conflicts as rcc
    from memcolor.crossover import build_and_select_offspring
    from memcolor.distance import pairwise_distances as rpd
    from memcolor.init import init_col_population
    from memcolor.rng import TAG_TRAIN
    from memcolor.rng import Stream as RStream
    from memcolor.surrogate import SurrogateNet as RNet

    for name, seed, n, pe, k, p, K, depth, G, epochs, bs in ENGINE_SURROGATE_CASES:
        g = ref_rand_graph(seed, n, pe)
        init = init_col_population(n, k, p, seed)
        fit = np.array([rcc(g, c) for c in init.colorings], dtype=np.int64)
        pop = RPOP.Population.from_colorings(init.colorings, fit)
        ms = RPOP.min_spacing(n)
        net = RNet(n, problem="col", arch="small", seed=seed, dtype=np.float64)
        offspring = list(init.colorings)
        pre = name + "__"
        out[pre + "params"] = np.array([seed, n, int(pe * 1000), k, p, K, depth, G, epochs, bs], dtype=np.int64)
        out[pre + "init"] = pop.assigns.astype(np.int32)
        for t in range(G):
            res = RLS.improve_population(g, offspring, RLS.COL, seed, generation=t, depth=depth)
            realized = np.array([r.best_score for r in res], dtype=np.float64)
            realized[realized >= float(RLS.INF_SCORE)] = np.nan
            mask = np.isfinite(realized)
            if mask.sum() >= 2:
                off = np.stack([c.assign for c in offspring])
                net.train_generation(off[mask], realized[mask], k, epochs, bs, RStream.derive(seed, TAG_TRAIN, t))
            imp = np.stack([r.best.assign for r in res]).astype(np.int32)
            imp_fit = np.array([min(r.best_score, int(RLS.INF_SCORE)) for r in res], dtype=np.int64)
            cross, within = rpd(pop.assigns, imp, k=k)
            pop = RPOP.update_population(pop, imp, imp_fit, cross, within, ms)
            matches = RPOP.match_parents(pop, K)
            batch = build_and_select_offspring(pop, matches, net, seed, t, use_surrogate=True)
            offspring = [RC(batch.selected_assigns[i], k) for i in range(p)]
            out[pre + f"g{t}_pop"] = pop.assigns.astype(np.int32)
            out[pre + f"g{t}_predicted"] = batch.predicted.astype(np.float64)
            out[pre + f"g{t}_selected"] = batch.selected_index.astype(np.int64)
            out[pre + f"g{t}_offspring"] = batch.selected_assigns.astype(np.int32)
    out["surrogate_cases"] = np.array([c[0] for c in ENGINE_SURROGATE_CASES])


ENGINE_WVCP_CASES = [  # (name, seed, n, p_edge, wmax, p, K, depth, rounds, G)
    ("w1", 2, 60, 0.5, 20, 10, 3, 120, 4, 3),
    ("w2", 4, 80, 0.3, 50, 12, 4, 160, 3, 3),
    ("w3", 6, 70, 0.7, 10, 8, 3, 1, 1, 3),  # too short to repair offspring: INF fitness
]


def gen_engine_wvcp(out):
    """Weighted generations: greedy init (`init.py:57-64`), fitness
    `wvcp_score` (`engine.py:332`), LS `improve_population(..., WVCP, ...)`."""
    from memcolor.coloring import Coloring as RC
    from memcolor.coloring import wvcp_score as rws
    from memcolor.crossover import build_and_select_offspring
    from memcolor.distance import pairwise_distances as rpd
    from memcolor.init import init_wvcp_population

    for name, seed, n, pe, wmax, p, K, depth, rounds, G in ENGINE_WVCP_CASES:
        g = ref_rand_graph(seed, n, pe, wmax=wmax)
        init = init_wvcp_population(g, p, seed)
        k = init.k
        fit = np.array([rws(g, c)[0] for c in init.colorings], dtype=np.int64)
        pop = RPOP.Population.from_colorings(init.colorings, fit)
        ms = RPOP.min_spacing(n)
        offspring = list(init.colorings)
        pre = name + "__"
        out[pre + "params"] = np.array([seed, n, int(pe * 1000), wmax, p, K, depth, rounds, G, k],
                                       dtype=np.int64)
        out[pre + "init"] = pop.assigns.astype(np.int32)
        out[pre + "init_fit"] = fit
        for t in range(G):
            res = RLS.improve_population(g, offspring, RLS.WVCP, seed, generation=t, depth=depth,
                                         max_rounds=rounds)
            imp = np.stack([r.best.assign for r in res]).astype(np.int32)
            imp_fit = np.array([min(r.best_score, int(RLS.INF_SCORE)) for r in res], dtype=np.int64)
            cross, within = rpd(pop.assigns, imp, k=k)
            pop = RPOP.update_population(pop, imp, imp_fit, cross, within, ms)
            matches = RPOP.match_parents(pop, K)
            batch = build_and_select_offspring(pop, matches, None, seed, t, use_surrogate=False)
            offspring = [RC(batch.selected_assigns[i], k) for i in range(p)]
            out[pre + f"g{t}_improved"] = imp
            out[pre + f"g{t}_imp_fit"] = imp_fit
            out[pre + f"g{t}_pop"] = pop.assigns.astype(np.int32)
            out[pre + f"g{t}_fit"] = pop.fitness.astype(np.int64)
            out[pre + f"g{t}_dist"] = pop.dist.astype(np.int32)
            out[pre + f"g{t}_offspring"] = batch.selected_assigns.astype(np.int32)
    out["wvcp_cases"] = np.array([c[0] for c in ENGINE_WVCP_CASES])


def gen_rng(out):
    rows = []
    for seed, tag, idx in [(1, 2, (0, 0)), (1, 1, (0,)), (2024, 2, (5, 11)), (7, 1, ()),
                           (0, 0, ()), (2**64 - 1, 7, (3, 2**40, 9)), (42, 3, (1, 2, 3, 4))]:
        key = RRNG.stream_key(seed, tag, *idx)
        vals = [int(RRNG.stream_value(np.uint64(key), np.uint64(c))) for c in range(16)]
        below = [int(RRNG.u64_below(np.uint64(key), np.uint64(c), np.uint64(c + 1))) for c in range(16)]
        rows.append((seed, tag, list(idx), key, vals, below))
    out["keys"] = np.array([r[3] for r in rows], np.uint64)
    out["values"] = np.array([r[4] for r in rows], np.uint64)
    out["below"] = np.array([r[5] for r in rows], np.uint64)
    out["spec"] = np.array([repr((r[0], r[1], tuple(r[2]))) for r in rows])


def gen_graphs(out):
    rows = []
    for seed, n, pe, wmax in [(1, 125, 0.5, 1), (1, 500, 0.5, 1), (1, 500, 0.5, 100), (3, 50, 0.4, 9),
                              (5, 300, 0.9, 1), (16, 40, 0.0, 4)]:
        g = ref_rand_graph(seed, n, pe, wmax=wmax)
        rows.append((seed, n, pe, wmax, g.m, digest(g.edges), digest(g.weights), digest(g.adj_indptr),
                     digest(g.adj_indices)))
    out["rows"] = np.array([repr(r) for r in rows])


INIT_CASES = [  # (name, seed, n, p_edge, wmax, p, master_seed)
    ("c125", 1, 125, 0.5, 100, 8, 11),
    ("c4shape", 1, 500, 0.5, 100, 6, 3),
    ("small", 3, 50, 0.4, 9, 10, 5),
    ("dense", 5, 300, 0.9, 1, 4, 2),
    ("edgeless", 16, 40, 0.0, 4, 3, 9),
    ("vdense", 7, 200, 0.97, 5, 3, 1),
]


def gen_init(out):
    from memcolor.init import init_wvcp_population as rinit

    for name, seed, n, pe, wmax, p, ms in INIT_CASES:
        g = ref_rand_graph(seed, n, pe, wmax=wmax)
        res = rinit(g, p, ms)
        out[f"{name}__params"] = np.array([seed, n, pe, wmax, p, ms], dtype=np.float64)
        out[f"{name}__assigns"] = np.stack([c.assign for c in res.colorings]).astype(np.int32)
        out[f"{name}__k"] = np.array(res.k)
    out["cases"] = np.array([c[0] for c in INIT_CASES])


SURROGATE_CASES = [  # (name, n, k, seed, dtype, use_bn, B, epochs, batch, generations)
    ("s64", 24, 5, 3, "float64", True, 40, 3, 8, 2),
    ("s32", 24, 5, 3, "float32", True, 40, 3, 8, 2),
    ("nobn", 20, 4, 7, "float64", False, 30, 2, 7, 2),
]


def surrogate_targets(assigns):
    """Deterministic synthetic targets for the surrogate fixtures."""
    a = assigns.astype(np.float64)
    return 3.0 * (assigns == 0).sum(axis=1) + 0.5 * a[:, 0] - 0.25 * a[:, -1] + 10.0


def gen_surrogate(out):
    from memcolor.rng import TAG_TRAIN
    from memcolor.rng import Stream as RStream
    from memcolor.surrogate import SurrogateNet as RNet

    for name, n, k, seed, dt, bn, B, epochs, bs, G in SURROGATE_CASES:
        pre = name + "__"
        net = RNet(n, problem="col", arch="small", seed=seed, dtype=np.dtype(dt), use_bn=bn)
        assigns = random_col_assigns(n, k, B, seed + 100)
        test = random_col_assigns(n, k, 16, seed + 200)
        y = surrogate_targets(assigns)
        out[pre + "params"] = np.array([n, k, seed, 1 if dt == "float64" else 0, int(bn), B, epochs, bs, G])
        out[pre + "pred0"] = net.predict_assigns(test, k)
        # one train-mode forward + hand-written backward on the first 8 rows
        x = net.one_hot(assigns[:8], k)
        pred = net.forward(x, mode="train", keep_cache=True, update_running=False)
        dout = (2.0 * (pred - ((y[:8] - y[:8].mean()) / y[:8].std())) / 8).astype(net.dtype)
        grads = net._backward(dout)
        for j, g in enumerate(grads):
            out[pre + f"grad{j}"] = np.asarray(g, dtype=np.float64)
        out[pre + "train_pred"] = pred.astype(np.float64)
        for layer in net.layers:
            layer.cache = None
        for t in range(G):
            losses = net.train_generation(assigns, y + t, k, epochs, bs, RStream.derive(seed, TAG_TRAIN, t))
            out[pre + f"g{t}_losses"] = np.array(losses)
            out[pre + f"g{t}_pred"] = net.predict_assigns(test, k)
        for i, layer in enumerate(net.layers):
            for nm in ("lam", "gam", "beta", "bn_scale", "bn_shift", "run_mean", "run_var"):
                out[pre + f"l{i}_{nm}"] = np.asarray(getattr(layer, nm), dtype=np.float64)
        out[pre + "adam_t"] = np.array(net.adam_t)
    out["cases"] = np.array([c[0] for c in SURROGATE_CASES])


# name, mode, seed, n, edge p, wmax, k, pop, generation, depth (0: default), max_rounds
IMPROVE_CASES = [
    ("col_g0", "col", 21, 120, 0.5, 1, 14, 6, 0, 3000, 0),
    ("col_g3", "col", 22, 200, 0.3, 1, 10, 5, 3, 5000, 0),
    ("col_default_depth", "col", 24, 60, 0.5, 1, 9, 4, 1, 0, 0),
    ("wvcp_g2", "wvcp", 23, 80, 0.4, 20, 12, 4, 2, 300, 3),
    ("wvcp_default", "wvcp", 25, 50, 0.5, 10, 10, 3, 0, 0, 2),
]


def gen_improve(out):
    """improve_population (`localsearch.py:615-682`): keys from the master
    seed and the generation, LsResult fields per individual."""
    meta = []
    for name, mode, seed, n, pe, wmax, k, pop, gen, depth, rounds in IMPROVE_CASES:
        g = ref_rand_graph(seed, n, pe, wmax=wmax)
        assert np.array_equal(g.edges, rand_graph(seed, n, pe, wmax=wmax).edges), name
        A = random_col_assigns(n, k, pop, seed)
        cols = [RColoring(A[i].copy(), k) for i in range(pop)]
        kw = {"depth": depth or None}
        if mode == "wvcp":
            kw["max_rounds"] = rounds
        res = RLS.improve_population(g, cols, RLS.WVCP if mode == "wvcp" else RLS.COL, seed, gen, **kw)
        pre = f"{name}__"
        out[pre + "params"] = np.array([seed, n, int(pe * 1000), wmax, k, pop, gen, depth, rounds], np.int64)
        out[pre + "mode"] = np.array([mode])
        out[pre + "init_digest"] = np.array([digest(A)])
        out[pre + "best"] = np.stack([r.best.assign for r in res]).astype(np.uint8)
        out[pre + "end"] = np.stack([r.end.assign for r in res]).astype(np.uint8)
        out[pre + "best_score"] = np.array([r.best_score for r in res], np.int64)
        out[pre + "iterations_used"] = np.array([r.iterations_used for r in res], np.int64)
        out[pre + "legal_found"] = np.array([r.legal_found for r in res], bool)
        if mode == "wvcp":
            out[pre + "phi"] = np.array([list(r.phi_trajectory) for r in res], np.float64)
        meta.append(name)
        print("improve", name, [r.best_score for r in res], [r.iterations_used for r in res])
    out["cases"] = np.array(meta)


def main():
    """python make_golden.py [name ...]  (default: every fixture)"""
    os.makedirs(HERE, exist_ok=True)
    only = set(sys.argv[1:])
    for fn, name in [(gen_rng, "rng"), (gen_graphs, "graphs"), (gen_tabucol, "tabucol"),
                     (gen_wvcp, "wvcp"), (gen_gpx, "gpx"), (gen_distance, "distance"),
                     (gen_population, "population"), (gen_engine, "engine"), (gen_init, "init"),
                     (gen_surrogate, "surrogate"), (gen_improve, "improve")]:
        if only and name not in only:
            continue
        out = {}
        fn(out)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print("done")


if __name__ == "__main__":
    main()
