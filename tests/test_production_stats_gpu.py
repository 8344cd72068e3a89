"""Production mode (Philox4x32 tie-break and tenure draws instead of the
reference's SplitMix64 streams): the best-found fitness distributions must be
statistically indistinguishable from the reference's: over
>= 2,048 individuals x 5 seeds (2..6), two-sample Kolmogorov-Smirnov and
Mann-Whitney U, alpha = 0.01.

The reference sample is the validation mode on the GPU, which reproduces
`_tabucol_batch` / `_wvcp_batch` (`mc/localsearch.py:266-410`, `:89-263`)
bit-for-bit -- the parity tests pin it, and each test here re-checks a
subsample of it against the CPU oracle.  That keeps the reference side at the
full scale (the CPU oracle alone would need ~25 min for C4).  With
MCB_STATS_OUT=<file> the p-values are also written as JSON."""

import json
import os

import numpy as np
import pytest
from scipy.stats import ks_2samp, mannwhitneyu

from paper_2109_05948_b200 import localsearch as LS
from paper_2109_05948_b200.graph import rand_graph
from paper_2109_05948_b200.init import random_col_assigns
from paper_2109_05948_b200.rng import TAG_LS, stream_keys

pytestmark = pytest.mark.gpu
ALPHA = 0.01
SEEDS = range(2, 7)
P = 2048
ANCHOR = 16  # validation individuals re-checked against the CPU oracle per test


def _record(name, res):
    out = os.environ.get("MCB_STATS_OUT")
    if not out:
        return
    data = {}
    if os.path.exists(out):
        data = json.load(open(out))
    data[name] = res
    json.dump(data, open(out, "w"), indent=1)


def _same_distribution(name, prod, ref, **info):
    a, b = np.concatenate(prod), np.concatenate(ref)
    ks = ks_2samp(a, b).pvalue
    mw = mannwhitneyu(a, b, alternative="two-sided").pvalue
    _record(name, dict(info, samples=int(a.size), ks_p=float(ks), mw_p=float(mw),
                       mean_production=float(a.mean()), mean_reference=float(b.mean()),
                       alpha=ALPHA))
    assert ks > ALPHA and mw > ALPHA, (ks, mw, a.mean(), b.mean())


def test_c1_iterations_to_zero(oracle_lib):
    """config 0: G(125,.5) k=18, iterations until a legal colouring."""
    g = rand_graph(1, 125, 0.5)
    prod, ref = [], []
    for seed in SEEDS:
        A = random_col_assigns(125, 18, P, seed)
        keys = stream_keys(seed, TAG_LS, 0, P)
        prod.append(LS._run_tabucol_batch(g, A.copy(), 18, keys, 20000, rng="philox")["iters_used"])
        val = LS._run_tabucol_batch(g, A.copy(), 18, keys, 20000)["iters_used"]
        ref.append(val)
    anchor = oracle_lib.tabucol_batch(g, A[:ANCHOR].copy(), 18, keys[:ANCHOR], 20000)["iters_used"]
    np.testing.assert_array_equal(val[:ANCHOR], anchor)
    _same_distribution("c1_iters_to_zero", prod, ref, shape="G(125,.5) k=18", depth=20000,
                       individuals=P, seeds=list(SEEDS))


@pytest.mark.parametrize("depth", [10000, 50000])
def test_c2_best_conflicts(depth, oracle_lib):
    """config 1: G(500,.5) k=48, best conflicts after 10k and after the
    config's 50k iterations."""
    g = rand_graph(1, 500, 0.5)
    prod, ref = [], []
    for seed in SEEDS:
        A = random_col_assigns(500, 48, P, seed)
        keys = stream_keys(seed, TAG_LS, 0, P)
        prod.append(LS._run_tabucol_batch(g, A.copy(), 48, keys, depth, rng="philox")["best_conflicts"])
        val = LS._run_tabucol_batch(g, A.copy(), 48, keys, depth)["best_conflicts"]
        ref.append(val)
    if depth == 10000:
        anchor = oracle_lib.tabucol_batch(g, A[:ANCHOR].copy(), 48, keys[:ANCHOR], depth)["best_conflicts"]
        np.testing.assert_array_equal(val[:ANCHOR], anchor)
    _same_distribution(f"c2_best_conflicts_{depth}", prod, ref, shape="G(500,.5) k=48", depth=depth,
                       individuals=P, seeds=list(SEEDS))


def test_c4_best_scores(oracle_lib):
    """config 3: weighted G(500,.5) w<=100, k=60, 10 rounds x 5000 iterations;
    the best legal score (the penalised end score when no legal colouring was
    reached)."""
    g = rand_graph(1, 500, 0.5, wmax=100)
    phi0 = LS.default_wvcp_phi0(g, 60)
    prod, ref = [], []
    fit = lambda r: np.where(r["best_scores"] < LS.INF_SCORE, r["best_scores"],  # noqa: E731
                             r["end_scores"] + 1000 * r["end_conflicts"])
    for seed in SEEDS:
        A = random_col_assigns(500, 60, P, seed)
        keys = stream_keys(seed, TAG_LS, 0, P)
        prod.append(fit(LS._run_wvcp_batch(g, A.copy(), 60, keys, 5000, 10, True, phi0, rng="philox")))
        val = LS._run_wvcp_batch(g, A.copy(), 60, keys, 5000, 10, True, phi0)
        ref.append(fit(val))
    anchor = oracle_lib.wvcp_batch(g, A[:ANCHOR].copy(), 60, keys[:ANCHOR], 5000, 10, True, phi0)
    np.testing.assert_array_equal(val["best_scores"][:ANCHOR], anchor["best_scores"])
    _same_distribution("c4_best_scores", prod, ref, shape="weighted G(500,.5) w<=100 k=60",
                       depth="10 rounds x 5000", individuals=P, seeds=list(SEEDS))
