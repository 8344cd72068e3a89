"""GPX crossover and pairwise partition distances on the B200 vs the
reference's golden outputs and the CPU oracle (bit-exact)."""

import numpy as np
import pytest

from conftest import load_golden
from paper_2109_05948_b200 import crossover as CX
from paper_2109_05948_b200 import distance as DI
from paper_2109_05948_b200.coloring import Coloring
from paper_2109_05948_b200.init import random_col_assigns
from paper_2109_05948_b200.rng import TAG_CROSS, Stream, stream_keys

pytestmark = pytest.mark.gpu


def test_gpx_golden():
    G = load_golden("gpx")
    for name in G["cases"]:
        seed, n, k, p, K = (int(x) for x in G[f"{name}__params"])
        P = random_col_assigns(n, k, p, seed)
        out = CX.build_offspring_batch(P, G[f"{name}__matches"], k, seed, 0)
        np.testing.assert_array_equal(out, G[f"{name}__out"].astype(np.int32), err_msg=name)
        keys = stream_keys(seed, TAG_CROSS, 0, p * K)
        m0 = int(G[f"{name}__matches"][0, 0])
        one = CX.gpx(Coloring(P[0], k), Coloring(P[m0], k), k, Stream(int(keys[0])))
        np.testing.assert_array_equal(one.assign, out[0, 0])


def test_gpx_vs_oracle_random(oracle_lib):
    rs = np.random.default_rng(11)
    for t in range(10):
        n, k, p = int(rs.integers(1, 2000)), int(rs.integers(1, 200)), int(rs.integers(2, 40))
        K = int(rs.integers(1, 17))
        P = random_col_assigns(n, k, p, t)
        matches = rs.integers(0, p, size=(p, K)).astype(np.int64)
        keys = stream_keys(t, TAG_CROSS, 2, p * K)
        np.testing.assert_array_equal(CX.gpx_batch(P, matches, k, keys),
                                      oracle_lib.gpx_batch(P, matches, k, keys), err_msg=str(t))


def test_gpx_errors():
    P = random_col_assigns(10, 3, 2, 1)
    with pytest.raises(ValueError):
        CX.gpx(P[0], P[1][:5], 3, 1)
    with pytest.raises(ValueError):
        CX.gpx_batch(P, np.array([[5], [0]]), 3, np.zeros(2, np.uint64))


def test_distance_golden():
    G = load_golden("distance")
    for name in G["cases"]:
        seed, n, k, p, q = (int(x) for x in G[f"{name}__params"])
        P = G[f"{name}__P"].astype(np.int32)
        Q = G[f"{name}__Q"].astype(np.int32)
        c, w = DI.pairwise_distances(P, Q, k=k)
        np.testing.assert_array_equal(c, G[f"{name}__cross"], err_msg=name)
        np.testing.assert_array_equal(w, G[f"{name}__within"], err_msg=name)
    hand = [([0, 0, 1, 1], [0, 1, 0, 1], 2), ([0, 1, 2, 0], [0, 1, 2, 0], 3),
            ([0, 0, 1, 1, 2], [2, 2, 0, 0, 1], 3), ([0, 0, 1, 1, 2, 2], [0, 0, 1, 1, 2, 1], 3)]
    got = [DI.approx_partition_distance(Coloring(a, k), Coloring(b, k)) for a, b, k in hand]
    assert got == G["hand_values"].tolist()


def test_distance_vs_oracle_random(oracle_lib):
    rs = np.random.default_rng(12)
    for t in range(12):
        n, k = int(rs.integers(1, 1200)), int(rs.integers(1, 160))
        p, q = int(rs.integers(0, 12)), int(rs.integers(1, 12))
        P = random_col_assigns(n, k, p, t) if p else np.zeros((0, n), np.int32)
        Q = random_col_assigns(n, k, q, 100 + t)
        if t % 3 == 0 and p:  # near-identical pairs: large overlap values
            Q[: min(p, q)] = P[: min(p, q)]
            Q[0, : n // 10] = (Q[0, : n // 10] + 1) % k
        c, w = DI.pairwise_distances(P, Q, k=k)
        rc, rw = oracle_lib.pairwise(P, Q, k)
        np.testing.assert_array_equal(c, rc, err_msg=str(t))
        np.testing.assert_array_equal(w, rw, err_msg=str(t))


def test_distance_job_range_sharding():
    P = random_col_assigns(300, 20, 9, 1)
    Q = random_col_assigns(300, 20, 11, 2)
    c_full, w_full = DI.pairwise_distances(P, Q, k=20)
    total = 9 * 11 + 11 * 10 // 2
    c = np.zeros_like(c_full)
    w = np.zeros_like(w_full)
    for b in range(0, total, 17):
        DI.pairwise_raw(P, Q, 20, b, min(total, b + 17), cross=c, within=w)
    np.testing.assert_array_equal(c, c_full)
    np.testing.assert_array_equal(w, w_full)
    assert (np.diagonal(w) == 0).all() and (w == w.T).all()


def test_gpx_rows_sharding_matches_full():
    import torch

    from paper_2109_05948_b200 import device as D

    P = random_col_assigns(700, 30, 10, 5)
    rs = np.random.default_rng(3)
    matches = rs.integers(0, 10, size=(10, 4)).astype(np.int64)
    keys = stream_keys(5, TAG_CROSS, 1, 40)
    full = CX.gpx_batch(P, matches, 30, keys)
    pop = torch.from_numpy(P).cuda()
    parts = []
    for lo, hi in ((0, 3), (3, 10)):
        m = torch.from_numpy(matches[lo:hi].copy()).cuda()
        kk = D.keys_to_tensor(keys[lo * 4:hi * 4], "cuda")
        parts.append(D.gpx_rows(pop, m, lo, 30, kk).cpu().numpy())
    np.testing.assert_array_equal(np.concatenate(parts), full)


@pytest.mark.parametrize("n,k", [(1100, 2), (700, 3), (1000, 12), (1000, 83), (3000, 200), (2000, 255)])
def test_distance_structured_vs_oracle(n, k, oracle_lib):
    """Permuted copies with noise: many overlap levels per pair, entries >= 32
    (small k), u8 counter overflow -> the u16 re-run (k = 2, 3), and every
    column-word count KWD = ceil(k / 32) up to 8."""
    rs = np.random.default_rng(n + k)
    P = random_col_assigns(n, k, 6, n)
    Q = np.empty((7, n), np.int32)
    for j in range(7):
        src = P[j % 6]
        Q[j] = rs.permutation(k)[src]
        noise = rs.random(n) < (0.05 + 0.1 * j)
        Q[j, noise] = rs.integers(0, k, int(noise.sum()))
    c, w = DI.pairwise_distances(P, Q, k=k)
    rc, rw = oracle_lib.pairwise(P, Q, k)
    np.testing.assert_array_equal(c, rc)
    np.testing.assert_array_equal(w, rw)


@pytest.mark.parametrize("k,noise", [(48, 0.02), (83, 0.1), (83, 0.3), (150, 0.05)])
def test_distance_converged_population_vs_oracle(k, noise, oracle_lib):
    """A converged population (every member one base colouring under its own
    colour permutation, a fraction recoloured): levels of a few large cells,
    taken in one step when their free cells have distinct rows and columns.
    Merged classes (two base colours onto one) and split classes (one base
    colour over two) put several cells of a level in one row or column, so
    the same pairs also take the round-based path."""
    n = 1000
    rs = np.random.default_rng(k + int(1000 * noise))
    base = random_col_assigns(n, k, 1, k)[0]
    M = np.empty((14, n), np.int32)
    for i in range(14):
        x = rs.permutation(k)[base]
        if i % 3 == 1:  # merge two classes
            a, b = rs.choice(k, 2, replace=False)
            x[x == a] = b
        if i % 3 == 2:  # split a class
            a = int(rs.integers(k))
            idx = np.flatnonzero(x == a)
            x[idx[::2]] = (a + 1) % k
        flip = rs.random(n) < noise
        x[flip] = rs.integers(0, k, int(flip.sum()))
        M[i] = x
    P, Q = M[:6], M[6:]
    c, w = DI.pairwise_distances(P, Q, k=k)
    rc, rw = oracle_lib.pairwise(P, Q, k)
    np.testing.assert_array_equal(c, rc)
    np.testing.assert_array_equal(w, rw)
