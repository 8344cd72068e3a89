"""Device-resident k-colouring generations (paper_2109_05948_b200/engine.py)
against generations chained from the reference's own operators
(tests/golden/engine.npz, `mc/engine.py:_generation_loop` without the
surrogate): LS results, pool, fitness, distance matrix, parent matches,
selected offspring -- bit-identical after every generation."""

import numpy as np
import pytest
import torch

from conftest import load_golden
from paper_2109_05948_b200 import device as Dv
from paper_2109_05948_b200 import engine as E
from paper_2109_05948_b200.graph import rand_graph
from paper_2109_05948_b200.rng import TAG_LS, stream_keys  # noqa: F401

pytestmark = pytest.mark.gpu
ENG = load_golden("engine")


@pytest.mark.parametrize("name", [str(c) for c in ENG["cases"]])
def test_generations_match_reference(name):
    pre = name + "__"
    seed, n, pe, k, p, K, depth, G = (int(x) for x in ENG[pre + "params"])
    g = rand_graph(seed, n, pe / 1000.0)
    dg = Dv.DeviceGraph(g, "cuda")
    st = E.init_state(dg, ENG[pre + "init"], k)
    for t in range(G):
        ls = E.col_generation(dg, st, seed=seed, depth=depth, K=K)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(ls["best_assigns"].cpu().numpy(), ENG[pre + f"g{t}_improved"],
                                      err_msg=f"{name} g{t} LS")
        np.testing.assert_array_equal(st.pop_assigns.cpu().numpy(), ENG[pre + f"g{t}_pop"], err_msg=f"g{t} pop")
        np.testing.assert_array_equal(st.pop_fitness.cpu().numpy(), ENG[pre + f"g{t}_fit"], err_msg=f"g{t} fit")
        np.testing.assert_array_equal(st.pop_dist.cpu().numpy(), ENG[pre + f"g{t}_dist"], err_msg=f"g{t} dist")
        np.testing.assert_array_equal(st.offspring.cpu().numpy(), ENG[pre + f"g{t}_offspring"],
                                      err_msg=f"g{t} offspring")
    assert st.generation == G


@pytest.mark.parametrize("name", [str(c) for c in ENG["wvcp_cases"]])
def test_wvcp_generations_match_reference(name):
    """Weighted runs: greedy init on the GPU, iterated WVCP tabu, INF fitness
    for individuals that never reach a legal colouring (case w3)."""
    pre = name + "__"
    seed, n, pe, wmax, p, K, depth, rounds, G, k = (int(x) for x in ENG[pre + "params"])
    g = rand_graph(seed, n, pe / 1000.0, wmax=wmax)
    dg = Dv.DeviceGraph(g, "cuda")
    st = E.init_state_wvcp(dg, g, p, seed)
    assert st.k == k
    np.testing.assert_array_equal(st.pop_assigns.cpu().numpy(), ENG[pre + "init"])
    np.testing.assert_array_equal(st.pop_fitness.cpu().numpy(), ENG[pre + "init_fit"])
    for t in range(G):
        ls = E.generation(dg, st, seed=seed, depth=depth, K=K, max_rounds=rounds)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(ls["best_assigns"].cpu().numpy(), ENG[pre + f"g{t}_improved"],
                                      err_msg=f"{name} g{t} LS")
        np.testing.assert_array_equal(ls["best_scores"].cpu().numpy(), ENG[pre + f"g{t}_imp_fit"],
                                      err_msg=f"{name} g{t} LS fitness")
        np.testing.assert_array_equal(st.pop_assigns.cpu().numpy(), ENG[pre + f"g{t}_pop"], err_msg=f"g{t} pop")
        np.testing.assert_array_equal(st.pop_fitness.cpu().numpy(), ENG[pre + f"g{t}_fit"], err_msg=f"g{t} fit")
        np.testing.assert_array_equal(st.pop_dist.cpu().numpy(), ENG[pre + f"g{t}_dist"], err_msg=f"g{t} dist")
        np.testing.assert_array_equal(st.offspring.cpu().numpy(), ENG[pre + f"g{t}_offspring"],
                                      err_msg=f"g{t} offspring")


@pytest.mark.parametrize("name", [str(c) for c in ENG["surrogate_cases"]])
def test_surrogate_generations_match_reference(name):
    """Surrogate-guided generations (float64 net): online training on the LS
    start points, predictions of all p K candidates, argmin selection."""
    from paper_2109_05948_b200.surrogate import SurrogateNet

    pre = name + "__"
    seed, n, pe, k, p, K, depth, G, epochs, bs = (int(x) for x in ENG[pre + "params"])
    g = rand_graph(seed, n, pe / 1000.0)
    dg = Dv.DeviceGraph(g, "cuda")
    st = E.init_state(dg, ENG[pre + "init"], k)
    net = SurrogateNet(n, problem="col", arch="small", seed=seed, dtype=np.float64)
    for t in range(G):
        E.generation(dg, st, seed=seed, depth=depth, K=K, net=net, epochs=epochs, batch_size=bs)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(st.pop_assigns.cpu().numpy(), ENG[pre + f"g{t}_pop"], err_msg=f"g{t} pop")
        np.testing.assert_array_equal(st.offspring.cpu().numpy(), ENG[pre + f"g{t}_offspring"],
                                      err_msg=f"g{t} offspring")


def test_engine_selection_is_in_range_and_keeps_shapes():
    """A larger random k-colouring run: shapes, dtypes and invariants after
    two generations (distance matrix symmetric with zero diagonal, fitness =
    conflicts of the stored colourings)."""
    g = rand_graph(9, 150, 0.4)
    dg = Dv.DeviceGraph(g, "cuda")
    from paper_2109_05948_b200.init import random_col_assigns

    st = E.init_state(dg, random_col_assigns(150, 9, 64, 9), 9)
    for _ in range(2):
        E.generation(dg, st, seed=9, depth=300, K=5)
    d = st.pop_dist.cpu().numpy()
    assert (d == d.T).all() and (np.diagonal(d) == 0).all()
    a = st.pop_assigns.cpu().numpy()
    conf = (a[:, g.edges[:, 0]] == a[:, g.edges[:, 1]]).sum(axis=1)
    np.testing.assert_array_equal(conf, st.pop_fitness.cpu().numpy())
    assert st.offspring.shape == (64, 150) and st.generation == 2


def test_sharded_generation_composition_with_cuda_operators():
    """`shard.col_generation_sharded` (single process: world 1) with the CUDA
    operators as its compute reproduces the reference chain: the composition
    that the N-GPU run uses with NCCL."""
    from paper_2109_05948_b200 import distance as DI
    from paper_2109_05948_b200 import localsearch as LSm
    from paper_2109_05948_b200 import population as PP
    from paper_2109_05948_b200.population import min_spacing
    from paper_2109_05948_b200.shard import col_generation_sharded

    def upd(pdist, fit, pa, imp, imp_fit, cross, within, ms):
        pop = PP.Population(assigns=pa, k=0, fitness=fit, dist=pdist)
        out = PP.update_population(pop, imp, imp_fit, cross, within, ms)
        return None, out.admitted_by_rule, out.dist, out.assigns, out.fitness

    def gpx_rows(pop, mrows, k, keys, off):
        pt = torch.as_tensor(pop).cuda()
        mt = torch.as_tensor(mrows).cuda()
        kt = Dv.keys_to_tensor(keys, "cuda")
        return Dv.gpx_rows(pt, mt, off, k, kt).cpu().numpy()

    ops = {"ls": lambda g_, a, k_, keys, d: LSm._run_tabucol_batch(g_, a, k_, keys, d),
           "pair": lambda a, b, k_, lo, hi: DI.pairwise_raw(a, b, k_, lo, hi),
           "gpx": gpx_rows, "update": upd}
    for name in [str(c) for c in ENG["cases"]]:
        pre = name + "__"
        seed, n, pe, k, p, K, depth, G = (int(x) for x in ENG[pre + "params"])
        g = rand_graph(seed, n, pe / 1000.0)
        A = ENG[pre + "init"].astype(np.int32)
        fit = (A[:, g.edges[:, 0]] == A[:, g.edges[:, 1]]).sum(axis=1).astype(np.int64)
        pd = DI.pairwise_raw(A[:0], A, k)[1]
        off = A.copy()
        # match_parents bounds distances by the population's n
        ops["match"] = lambda d, K, n=n: PP.match_parents(
            PP.Population(assigns=np.zeros((d.shape[0], n), np.int32), k=0, fitness=None, dist=d), K)
        for t in range(G):
            A, fit, pd, off, imp = col_generation_sharded(g, A, fit, pd, off, k, seed, t, depth, K,
                                                          min_spacing(n), ops)
            np.testing.assert_array_equal(A, ENG[pre + f"g{t}_pop"], err_msg=f"{name} g{t}")
            np.testing.assert_array_equal(pd, ENG[pre + f"g{t}_dist"])
            np.testing.assert_array_equal(off, ENG[pre + f"g{t}_offspring"])


def test_device_sharded_generation_nccl_world1():
    """The device-resident sharded generation (`engine.generation(...,
    force_shard=True)`: LS shard + NCCL all-gathers, job-range distances +
    all-reduce, GPX rows) inside a one-rank NCCL group reproduces the
    reference chain; at world size N the same code splits the ranges."""
    import torch.distributed as dist

    from test_shard import _free_port

    if not dist.is_initialized():
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1)
    try:
        for name in [str(c) for c in ENG["cases"]]:
            pre = name + "__"
            seed, n, pe, k, p, K, depth, G = (int(x) for x in ENG[pre + "params"])
            g = rand_graph(seed, n, pe / 1000.0)
            dg = Dv.DeviceGraph(g, "cuda")
            st = E.init_state(dg, ENG[pre + "init"], k)
            for t in range(G):
                E.generation(dg, st, seed=seed, depth=depth, K=K, force_shard=True)
                torch.cuda.synchronize()
                np.testing.assert_array_equal(st.pop_assigns.cpu().numpy(), ENG[pre + f"g{t}_pop"], err_msg=f"g{t}")
                np.testing.assert_array_equal(st.pop_dist.cpu().numpy(), ENG[pre + f"g{t}_dist"])
                np.testing.assert_array_equal(st.offspring.cpu().numpy(), ENG[pre + f"g{t}_offspring"])
    finally:
        dist.destroy_process_group()


def _world2_worker(rank, port, out_path):
    import os
    import sys

    import torch.distributed as dist

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=2)
    try:
        eng = load_golden("engine")
        res = {}
        for name in [str(c) for c in eng["cases"]]:
            pre = name + "__"
            seed, n, pe, k, p, K, depth, G = (int(x) for x in eng[pre + "params"])
            g = rand_graph(seed, n, pe / 1000.0)
            dg = Dv.DeviceGraph(g, "cuda")
            st = E.init_state(dg, eng[pre + "init"], k)
            timings = {}
            for t in range(G):
                ls = E.generation(dg, st, seed=seed, depth=depth, K=K, timings=timings)
                torch.cuda.synchronize()
                res[f"{name}_g{t}_pop"] = st.pop_assigns.cpu().numpy()
                res[f"{name}_g{t}_dist"] = st.pop_dist.cpu().numpy()
                res[f"{name}_g{t}_offspring"] = st.offspring.cpu().numpy()
                for key in ("best_assigns", "best_conflicts", "end_assigns", "end_conflicts", "iters_used"):
                    res[f"{name}_g{t}_ls_{key}"] = ls[key].cpu().numpy()
            res[f"{name}_timing_stages"] = np.array(sorted(timings))
        if rank == 0:
            np.savez(out_path, **res)
    finally:
        dist.destroy_process_group()


def test_device_sharded_generation_world2(tmp_path):
    """The device-resident sharded generation at world size 2 (two processes
    on this GPU, gloo all-gathers with host staging -- the ranks' kernels never
    wait on each other): the same state after every generation as the
    reference chain, LS outputs gathered for the whole population, per-stage
    timings reported."""
    import torch.multiprocessing as mp

    from test_shard import _free_port

    out = str(tmp_path / "w2.npz")
    mp.start_processes(_world2_worker, args=(_free_port(), out), nprocs=2, join=True, start_method="spawn")
    res = np.load(out)
    for name in [str(c) for c in ENG["cases"]]:
        pre = name + "__"
        seed, n, pe, k, p, K, depth, G = (int(x) for x in ENG[pre + "params"])
        for t in range(G):
            np.testing.assert_array_equal(res[f"{name}_g{t}_pop"], ENG[pre + f"g{t}_pop"], err_msg=f"{name} g{t}")
            np.testing.assert_array_equal(res[f"{name}_g{t}_dist"], ENG[pre + f"g{t}_dist"])
            np.testing.assert_array_equal(res[f"{name}_g{t}_offspring"], ENG[pre + f"g{t}_offspring"])
            assert res[f"{name}_g{t}_ls_best_assigns"].shape == (p, n)
            assert res[f"{name}_g{t}_ls_iters_used"].shape == (p,)
        stages = set(res[f"{name}_timing_stages"].tolist())
        assert {"ls", "elite_allgather", "distances", "distance_allgather", "update_population"} <= stages
