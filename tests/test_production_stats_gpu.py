"""Production mode (Philox4x32 tie-break and tenure draws instead of the
reference's SplitMix64 streams): the best-found fitness distributions must be
statistically indistinguishable from the reference's:
two-sample Kolmogorov-Smirnov and Mann-Whitney U, alpha = 0.01, GPU production
vs the CPU oracle (which reproduces the reference bit-for-bit)."""

import numpy as np
import pytest
from scipy.stats import ks_2samp, mannwhitneyu

from paper_2109_05948_b200 import localsearch as LS
from paper_2109_05948_b200.graph import rand_graph
from paper_2109_05948_b200.init import random_col_assigns
from paper_2109_05948_b200.rng import TAG_LS, stream_keys

pytestmark = pytest.mark.gpu
ALPHA = 0.01


def _same_distribution(a, b):
    ks = ks_2samp(a, b).pvalue
    mw = mannwhitneyu(a, b, alternative="two-sided").pvalue
    assert ks > ALPHA and mw > ALPHA, (ks, mw, np.mean(a), np.mean(b))


def test_c1_iterations_to_zero(oracle_lib):
    """config 0: G(125,.5) k=18, iterations until a legal colouring."""
    g = rand_graph(1, 125, 0.5)
    gpu, cpu = [], []
    for seed in range(2, 7):
        A = random_col_assigns(125, 18, 512, seed)
        keys = stream_keys(seed, TAG_LS, 0, 512)
        gpu.append(LS._run_tabucol_batch(g, A.copy(), 18, keys, 20000, rng="philox")["iters_used"])
        cpu.append(oracle_lib.tabucol_batch(g, A.copy(), 18, keys, 20000)["iters_used"])
    _same_distribution(np.concatenate(gpu), np.concatenate(cpu))


def test_c2_best_conflicts(oracle_lib):
    """config 1 shape: G(500,.5) k=48, best conflicts after 2000 iterations."""
    g = rand_graph(1, 500, 0.5)
    gpu, cpu = [], []
    for seed in range(2, 7):
        A = random_col_assigns(500, 48, 410, seed)
        keys = stream_keys(seed, TAG_LS, 0, 410)
        gpu.append(LS._run_tabucol_batch(g, A.copy(), 48, keys, 2000, rng="philox")["best_conflicts"])
        cpu.append(oracle_lib.tabucol_batch(g, A.copy(), 48, keys, 2000)["best_conflicts"])
    _same_distribution(np.concatenate(gpu), np.concatenate(cpu))


def test_c4_best_scores(oracle_lib):
    """config 3 shape: weighted G(500,.5) w<=100, k=60, best legal score (or the
    end penalised score when no legal colouring was reached)."""
    g = rand_graph(1, 500, 0.5, wmax=100)
    phi0 = LS.default_wvcp_phi0(g, 60)
    gpu, cpu = [], []
    for seed in range(2, 7):
        A = random_col_assigns(500, 60, 64, seed)
        keys = stream_keys(seed, TAG_LS, 0, 64)
        rg = LS._run_wvcp_batch(g, A.copy(), 60, keys, 300, 4, True, phi0, rng="philox")
        rc = oracle_lib.wvcp_batch(g, A.copy(), 60, keys, 300, 4, True, phi0)
        gpu.append(rg["end_scores"] + 1000 * rg["end_conflicts"])
        cpu.append(rc["end_scores"] + 1000 * rc["end_conflicts"])
    _same_distribution(np.concatenate(gpu), np.concatenate(cpu))
