"""The CPU oracle (oracle/memcolor_oracle.c) pinned against the reference's
own outputs (tests/golden/, made by make_golden.py from the reference) and the
SURVEY.md Appendix A known answers.  CPU only."""

import hashlib

import numpy as np
import pytest

from cases import check_tabucol, check_wvcp, tabucol_case, wvcp_case
from conftest import load_golden
from paper_2109_05948_b200.init import random_col_assigns
from paper_2109_05948_b200.rng import TAG_CROSS, TAG_LS, stream_keys, stream_key

TAB = load_golden("tabucol")
WV = load_golden("wvcp")


def h(x):
    return hashlib.sha256(np.ascontiguousarray(x, dtype=np.int32).tobytes()).hexdigest()[:16]


def test_oracle_rng_known_answers(oracle_lib):
    R = load_golden("rng")
    for key, vals in zip(R["keys"], R["values"]):
        for c, v in enumerate(vals):
            assert oracle_lib.stream_value(int(key), c) == int(v)
    k0 = stream_key(1, TAG_LS, 0, 0)
    assert k0 == 0xFAF75A0727F39370
    assert [oracle_lib.stream_value(k0, c) for c in range(3)] == [
        0x3C2FD00A61EEE31C, 0xDBE5E63AE4E33E4C, 0xCB08F94CB9907A2C]


FAST_TABU = [c for c in TAB["cases"] if c not in ("c2s", "long")]


@pytest.mark.parametrize("name", FAST_TABU)
def test_oracle_tabucol_golden(oracle_lib, name):
    g, A, k, keys, depth, cap = tabucol_case(TAB, name)
    out = oracle_lib.tabucol_batch(g, A.copy(), k, keys, depth, log_moves=cap > 0)
    check_tabucol(TAB, name, out)


@pytest.mark.parametrize("name", ["c2s", "long"])
def test_oracle_tabucol_golden_long(oracle_lib, name):
    g, A, k, keys, depth, cap = tabucol_case(TAB, name)
    out = oracle_lib.tabucol_batch(g, A.copy(), k, keys, depth, log_moves=cap > 0)
    check_tabucol(TAB, name, out)


def test_oracle_appendix_a_tabucol(oracle_lib):
    g, A, k, keys, depth, cap = tabucol_case(TAB, "c1")
    out = oracle_lib.tabucol_batch(g, A[:4].copy(), k, keys[:4], depth, log_moves=True)
    assert out["iters_used"].tolist() == [2681, 2128, 4023, 1906]
    assert out["best_conflicts"].tolist() == [0, 0, 0, 0]
    assert out["log"][0][0, :6].tolist() == [50, 119, 55, 90, 4, 40]
    assert out["log"][2][0, :6].tolist() == [121, 118, 114, 115, 111, 101]
    assert [h(out["end_assigns"][i]) for i in range(4)] == [
        "52d39fb0bdf92c00", "887a140ba18ae2f9", "3a80b5362eac47b9", "8474568000d574ae"]


@pytest.mark.parametrize("name", [c for c in WV["cases"] if c != "c4s"])
def test_oracle_wvcp_golden(oracle_lib, name):
    g, A, k, keys, depth, rounds, sched, phi0 = wvcp_case(WV, name)
    out = oracle_lib.wvcp_batch(g, A.copy(), k, keys, depth, rounds, sched, phi0, log_moves=True)
    check_wvcp(WV, name, out)


def test_oracle_gpx_golden(oracle_lib):
    G = load_golden("gpx")
    for name in G["cases"]:
        seed, n, k, p, K = (int(x) for x in G[f"{name}__params"])
        P = random_col_assigns(n, k, p, seed)
        keys = stream_keys(seed, TAG_CROSS, 0, p * K)
        out = oracle_lib.gpx_batch(P, G[f"{name}__matches"], k, keys)
        np.testing.assert_array_equal(out, G[f"{name}__out"].astype(np.int32), err_msg=name)
    # Appendix A
    P = random_col_assigns(1000, 83, 8, 1)
    m = np.array([[(i + 1 + j) % 8 for j in range(4)] for i in range(8)], np.int64)
    o = oracle_lib.gpx_batch(P, m, 83, stream_keys(1, TAG_CROSS, 0, 32))
    assert o[0, 0, :8].tolist() == [74, 40, 82, 66, 75, 3, 3, 25]
    assert h(o) == "f776d4aa28c9f7d3"


def test_oracle_distance_golden(oracle_lib):
    G = load_golden("distance")
    for name in G["cases"]:
        seed, n, k, p, q = (int(x) for x in G[f"{name}__params"])
        P = G[f"{name}__P"].astype(np.int32)
        Q = G[f"{name}__Q"].astype(np.int32)
        c, w = oracle_lib.pairwise(P, Q, k)
        np.testing.assert_array_equal(c, G[f"{name}__cross"], err_msg=name)
        np.testing.assert_array_equal(w, G[f"{name}__within"], err_msg=name)
    hand = [([0, 0, 1, 1], [0, 1, 0, 1], 2), ([0, 1, 2, 0], [0, 1, 2, 0], 3),
            ([0, 0, 1, 1, 2], [2, 2, 0, 0, 1], 3), ([0, 0, 1, 1, 2, 2], [0, 0, 1, 1, 2, 1], 3)]
    got = [oracle_lib.approx_distance(np.array(a), np.array(b), k) for a, b, k in hand]
    assert got == G["hand_values"].tolist() == [2, 0, 0, 1]


def test_oracle_distance_job_ranges(oracle_lib):
    """Sharding the linear job space reproduces the full pass."""
    P = random_col_assigns(60, 7, 5, 3)
    Q = random_col_assigns(60, 7, 6, 4)
    c_full, w_full = oracle_lib.pairwise(P, Q, 7)
    total = 5 * 6 + 6 * 5 // 2
    c = np.zeros_like(c_full)
    w = np.zeros_like(w_full)
    for b in range(0, total, 7):
        cc, ww = oracle_lib.pairwise(P, Q, 7, job_begin=b, job_end=min(total, b + 7))
        c += cc
        w += ww
    np.testing.assert_array_equal(c, c_full)
    np.testing.assert_array_equal(w, w_full)


def test_oracle_thread_count_independent(oracle_lib):
    g, A, k, keys, depth, cap = tabucol_case(TAB, "c2w")
    o1 = oracle_lib.tabucol_batch(g, A[:8].copy(), k, keys[:8], 500, threads=1)
    o8 = oracle_lib.tabucol_batch(g, A[:8].copy(), k, keys[:8], 500, threads=8)
    for key in ("end_assigns", "best_conflicts", "iters_used"):
        np.testing.assert_array_equal(o1[key], o8[key])
