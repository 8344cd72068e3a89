"""Multi-GPU sharding logic on CPU: world size 2 over `gloo`, the CPU oracle as
the compute.  Sharded results must be bit-identical to the single-process
pass (individuals are independent and keyed by global index)."""

import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2109_05948_b200.graph import rand_graph
from paper_2109_05948_b200.init import random_col_assigns
from paper_2109_05948_b200.rng import TAG_CROSS, TAG_LS, stream_keys
from paper_2109_05948_b200.shard import (improve_col_sharded, offspring_sharded, pairwise_sharded,
                                         shard_range)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port):
    from oracle import oracle

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        g = rand_graph(3, 90, 0.4)
        k, p, depth = 8, 13, 400
        A = random_col_assigns(90, k, p, 3)
        ls = lambda g_, a, k_, keys, d: oracle.tabucol_batch(g_, a, k_, keys, d)  # noqa: E731
        got = improve_col_sharded(g, A, k, 3, 5, depth, ls)
        ref = oracle.tabucol_batch(g, A.copy(), k, stream_keys(3, TAG_LS, 5, p), depth)
        for key in ("best_assigns", "best_conflicts", "end_conflicts", "iters_used"):
            np.testing.assert_array_equal(got[key], ref[key], err_msg=key)

        P = random_col_assigns(90, k, 7, 11)
        Q = random_col_assigns(90, k, 9, 12)
        pf = lambda a, b, k_, lo, hi: oracle.pairwise(a, b, k_, lo, hi)  # noqa: E731
        c, w = pairwise_sharded(P, Q, k, pf)
        rc, rw = oracle.pairwise(P, Q, k)
        np.testing.assert_array_equal(c, rc)
        np.testing.assert_array_equal(w, rw)

        K = 3
        rs = np.random.default_rng(0)
        matches = rs.integers(0, 7, size=(7, K)).astype(np.int64)
        full_keys = stream_keys(3, TAG_CROSS, 2, 7 * K)

        def gx(pop, mrows, k_, keys, off):
            rows = mrows.shape[0]
            np.testing.assert_array_equal(keys, full_keys[off * K:(off + rows) * K])
            return oracle.gpx_batch(pop, matches, k_, full_keys)[off:off + rows]

        off = offspring_sharded(P, matches, k, 3, 2, gx)
        np.testing.assert_array_equal(off, oracle.gpx_batch(P, matches, k, full_keys))
    finally:
        dist.destroy_process_group()


def test_shard_ranges_cover_exactly():
    for total in (0, 1, 7, 100, 8192):
        for world in (1, 2, 3, 8):
            parts = [shard_range(total, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == total
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            assert max(h - l for l, h in parts) - min(h - l for l, h in parts) <= 1


def test_sharded_operators_gloo_world2(oracle_lib):
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    mp.spawn(_worker, args=(2, _free_port()), nprocs=2, join=True)


def test_single_process_passthrough(oracle_lib):
    g = rand_graph(4, 50, 0.3)
    A = random_col_assigns(50, 5, 6, 4)
    ls = lambda g_, a, k_, keys, d: oracle_lib.tabucol_batch(g_, a, k_, keys, d)  # noqa: E731
    got = improve_col_sharded(g, A, 5, 9, 0, 300, ls)
    ref = oracle_lib.tabucol_batch(g, A.copy(), 5, stream_keys(9, TAG_LS, 0, 6), 300)
    np.testing.assert_array_equal(got["best_assigns"], ref["best_assigns"])


def _gpx_rows_oracle(oracle, pop, mrows, k, keys, off):
    """Offspring rows [off, off + rows) with the whole-population oracle (first
    parent = the row's own individual): other rows get parent 0 and are dropped."""
    p, K = pop.shape[0], mrows.shape[1]
    m = np.zeros((p, K), np.int64)
    kk = np.zeros(p * K, np.uint64)
    m[off:off + mrows.shape[0]] = mrows
    kk[off * K:(off + mrows.shape[0]) * K] = keys
    return oracle.gpx_batch(pop, m, k, kk)[off:off + mrows.shape[0]]


def _gen_worker(rank, world, port):
    """World-2 sharded generations (oracle as the compute) reproduce the
    reference-chained generations of tests/golden/engine.npz bit for bit."""
    from conftest import load_golden
    from oracle import oracle
    from oracle import population_oracle as PO
    from paper_2109_05948_b200.population import min_spacing
    from paper_2109_05948_b200.shard import col_generation_sharded

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        ENG = load_golden("engine")
        ops = {"ls": lambda g_, a, k_, keys, d: oracle.tabucol_batch(g_, a, k_, keys, d),
               "pair": lambda a, b, k_, lo, hi: oracle.pairwise(a, b, k_, lo, hi),
               "gpx": lambda pop, mrows, k_, keys, off: _gpx_rows_oracle(oracle, pop, mrows, k_, keys, off),
               "update": PO.update_population, "match": PO.match_parents}
        for name in ENG["cases"]:
            pre = str(name) + "__"
            seed, n, pe, k, p, K, depth, G = (int(x) for x in ENG[pre + "params"])
            g = rand_graph(seed, n, pe / 1000.0)
            A = ENG[pre + "init"].astype(np.int32)
            fit = (A[:, g.edges[:, 0]] == A[:, g.edges[:, 1]]).sum(axis=1).astype(np.int64)
            pd = oracle.pairwise(A[:0], A, k)[1]
            off = A.copy()
            for t in range(G):
                A, fit, pd, off, imp = col_generation_sharded(g, A, fit, pd, off, k, seed, t, depth, K,
                                                              min_spacing(n), ops)
                np.testing.assert_array_equal(imp, ENG[pre + f"g{t}_improved"])
                np.testing.assert_array_equal(A, ENG[pre + f"g{t}_pop"])
                np.testing.assert_array_equal(fit, ENG[pre + f"g{t}_fit"])
                np.testing.assert_array_equal(pd, ENG[pre + f"g{t}_dist"])
                np.testing.assert_array_equal(off, ENG[pre + f"g{t}_offspring"])
    finally:
        dist.destroy_process_group()


def test_sharded_generations_world2():
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    mp.spawn(_gen_worker, args=(2, _free_port()), nprocs=2, join=True)
