"""Weighted-colouring tabu search on the B200 vs the reference's golden
outputs and the CPU oracle: bit-exact scores, conflicts, phi trajectories,
end/best colourings and move logs (fp64 objective without FMA)."""

import numpy as np
import pytest

from cases import check_wvcp, wvcp_case
from conftest import load_golden
from paper_2109_05948_b200 import localsearch as LS
from paper_2109_05948_b200.coloring import Coloring, wvcp_score_batch
from paper_2109_05948_b200.graph import rand_graph
from paper_2109_05948_b200.init import random_col_assigns
from paper_2109_05948_b200.rng import TAG_LS, stream_keys

pytestmark = pytest.mark.gpu
WV = load_golden("wvcp")


@pytest.mark.parametrize("name", list(WV["cases"]))
def test_wvcp_golden_bit_exact(name):
    g, A, k, keys, depth, rounds, sched, phi0 = wvcp_case(WV, name)
    out = LS._run_wvcp_batch(g, A.copy(), k, keys, depth, rounds, sched, phi0, log_moves=True)
    check_wvcp(WV, name, out)


def test_wvcp_vs_oracle_random(oracle_lib):
    rs = np.random.default_rng(21)
    for t in range(8):
        n = int(rs.integers(2, 200))
        pe = float(rs.uniform(0.05, 0.9))
        wmax = int(rs.integers(1, 60))
        k = int(rs.integers(2, 40))
        p = int(rs.integers(1, 12))
        depth = int(rs.integers(1, 300))
        rounds = int(rs.integers(1, 5))
        sched = bool(rs.integers(0, 2))
        g = rand_graph(300 + t, n, pe, wmax=wmax)
        A = random_col_assigns(n, k, p, 31 + t)
        keys = stream_keys(t, TAG_LS, 1, p)
        phi0 = LS.default_wvcp_phi0(g, k) * float(rs.uniform(0.3, 3.0))
        ref = oracle_lib.wvcp_batch(g, A.copy(), k, keys, depth, rounds, sched, phi0, log_moves=True)
        got = LS._run_wvcp_batch(g, A.copy(), k, keys, depth, rounds, sched, phi0, log_moves=True)
        for key in ("end_assigns", "best_assigns", "best_scores", "end_scores", "end_conflicts",
                    "phi_used"):
            np.testing.assert_array_equal(got[key], ref[key], err_msg=f"case {t} {key}")
        for a, b in zip(got["log"], ref["log"]):
            np.testing.assert_array_equal(a, b, err_msg=f"case {t} log")


def test_wvcp_c4_properties():
    """Config 3 shape (G(500,.5), w in [1,100], k=60) at D=256: scores agree
    with scratch evaluation, legal bests only."""
    g = rand_graph(1, 500, 0.5, wmax=100)
    A = random_col_assigns(500, 60, 256, 1)
    keys = stream_keys(1, TAG_LS, 0, 256)
    out = LS._run_wvcp_batch(g, A.copy(), 60, keys, 500, 3, True, LS.default_wvcp_phi0(g, 60))
    sc, cf = wvcp_score_batch(g, out["end_assigns"], 60)
    np.testing.assert_array_equal(sc, out["end_scores"])
    np.testing.assert_array_equal(cf, out["end_conflicts"])
    legal = out["best_scores"] < int(LS.INF_SCORE)
    bs, bc = wvcp_score_batch(g, out["best_assigns"][legal], 60)
    np.testing.assert_array_equal(bs, out["best_scores"][legal])
    assert (bc == 0).all()


def test_wvcp_single_apis():
    g = rand_graph(5, 60, 0.3, wmax=20)
    c = Coloring(random_col_assigns(60, 12, 1, 5)[0], 12)
    end, best = LS.wvcp_tabu_search(g, c, 3.0, 300, 99)
    assert end.k == 12
    res = LS.iterated_wvcp_ls(g, c, 7, depth=200, max_rounds=3)
    assert len(res.phi_trajectory) == 4
    pop = LS.improve_population(g, [c, c, c], LS.WVCP, 3, depth=100, max_rounds=2)
    assert len(pop) == 3 and pop[0].iterations_used == 200


@pytest.mark.parametrize("case", ["init_overflow", "mixed"])
def test_wvcp_gamma_overflow_reruns_wide(case, oracle_lib, monkeypatch):
    """u8 gamma table first: individuals whose neighbour counts reach 256 re-run
    with u16.  `init_overflow`: degree ~570 on 2 colours (every individual
    overflows at the start); `mixed`: 3 colours where some starts stay below
    256 and moves push counts across it.  Both bit-exact vs the oracle, and
    identical to forcing u16 throughout (MCB_WVCP_WIDE)."""
    if case == "init_overflow":
        g, k, p, depth = rand_graph(41, 600, 0.95, wmax=7), 2, 4, 60
    else:
        g, k, p, depth = rand_graph(42, 800, 0.97, wmax=9), 3, 6, 80
    A = random_col_assigns(g.n, k, p, 5)
    keys = stream_keys(3, TAG_LS, 0, p)
    phi0 = LS.default_wvcp_phi0(g, k)
    ref = oracle_lib.wvcp_batch(g, A.copy(), k, keys, depth, 2, True, phi0, log_moves=True)
    monkeypatch.delenv("MCB_WVCP_WIDE", raising=False)
    got = LS._run_wvcp_batch(g, A.copy(), k, keys, depth, 2, True, phi0, log_moves=True)
    monkeypatch.setenv("MCB_WVCP_WIDE", "1")
    wide = LS._run_wvcp_batch(g, A.copy(), k, keys, depth, 2, True, phi0, log_moves=True)
    for key in ("end_assigns", "best_assigns", "best_scores", "end_scores", "end_conflicts", "phi_used"):
        np.testing.assert_array_equal(got[key], ref[key], err_msg=key)
        np.testing.assert_array_equal(wide[key], ref[key], err_msg=key)
    for a, b in zip(got["log"], ref["log"]):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("t", range(10))
def test_wvcp_dyadic_phi_vs_oracle(t, oracle_lib):
    """Random shapes with dyadic phi schedules (phi0 = t 2^-s: every reachable
    phi takes the exact 32-bit integer objective path of csrc/wvcp.cu);
    bit-exact vs the oracle, move logs included."""
    rs = np.random.default_rng(500 + t)
    n = int(rs.integers(2, 600))
    pe = float(rs.uniform(0.05, 0.9))
    k = int(rs.integers(2, 80))
    wmax = int(rs.choice([1, 7, 100]))
    p = int(rs.integers(1, 14))
    depth = int(rs.integers(1, max(2, 1_500_000 // max(1, n * p))))
    rounds = int(rs.integers(1, 5))
    sched = bool(rs.integers(0, 2))
    phi0 = float(rs.integers(1, 40)) * 2.0 ** -int(rs.integers(0, 4))
    g = rand_graph(700 + t, n, pe, wmax=wmax)
    A = random_col_assigns(n, k, p, 800 + t)
    keys = stream_keys(t, TAG_LS, 3, p)
    ref = oracle_lib.wvcp_batch(g, A.copy(), k, keys, depth, rounds, sched, phi0, log_moves=True)
    got = LS._run_wvcp_batch(g, A.copy(), k, keys, depth, rounds, sched, phi0, log_moves=True)
    for key in ("end_assigns", "best_assigns", "best_scores", "end_scores", "end_conflicts", "phi_used"):
        np.testing.assert_array_equal(got[key], ref[key], err_msg=f"{t} {key}")
    for a, b in zip(got["log"], ref["log"]):
        np.testing.assert_array_equal(a, b, err_msg=f"{t} log")
