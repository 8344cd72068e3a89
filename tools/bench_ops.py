"""Throughput of the secondary hot-path operators on one GPU, beside the CPU
restatement of the reference on this host (oracle/, OpenMP, all cores).

* WVCP moves/s      config 3 shape: G(500,.5) w in [1,100], k=60 (D, depth reduced)
* GPX offspring/s   config 2 shape: n=1000, k=83, parents (i, uniform j != i)
* distance pairs/s  config 2 shape: n=1000, k=83 pairwise_distances(P, P')
* update_population generations/s, config 2 size p = q = 16384 (n = 1000)
* match_parents     rows/s, p = 16384, K = 16

Each line: {"op", "gpu": units/s, "cpu": units/s, "cores", "sample", ...}.
Synthetic inputs; device-resident inputs, CUDA-event timing.
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle  # noqa: E402
from paper_2109_05948_b200 import _native as N  # noqa: E402
from paper_2109_05948_b200 import device as Dv  # noqa: E402
from paper_2109_05948_b200 import localsearch as LS  # noqa: E402
from paper_2109_05948_b200.graph import rand_graph  # noqa: E402
from paper_2109_05948_b200.init import random_col_assigns  # noqa: E402
from paper_2109_05948_b200.rng import TAG_CROSS, TAG_LS, TAG_MISC, stream_keys  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps, out


def bench_wvcp(a):
    g = rand_graph(1, 500, 0.5, wmax=100)
    k, D, depth, rounds = 60, a.wvcp_pop, a.wvcp_depth, 10
    A = random_col_assigns(500, k, D, 1)
    keys = stream_keys(1, TAG_LS, 0, D)
    dg = Dv.DeviceGraph(g, "cuda")
    kd = Dv.keys_to_tensor(keys, "cuda")
    a0 = torch.from_numpy(A).cuda()
    phi0 = LS.default_wvcp_phi0(g, k)
    t, _ = timed(lambda: Dv.wvcp_batch(dg, a0.clone(), k, kd, depth, rounds, True, phi0))
    moves = D * depth * rounds
    cores = os.cpu_count()
    nc = max(16, cores)
    t0 = time.perf_counter()
    oracle.wvcp_batch(g, A[:nc].copy(), k, keys[:nc], depth, rounds, True, phi0, threads=cores)
    tc = time.perf_counter() - t0
    return {"op": "wvcp", "unit": "moves/s", "gpu": moves / t, "cpu": nc * depth * rounds / tc,
            "cores": cores, "config": f"G(500,.5) w<=100 k=60 D={D} {rounds}x{depth}",
            "cpu_sample": f"{nc} individuals x {rounds}x{depth}", "gpu_ms": 1e3 * t}


def bench_gpx(a):
    n, k, p, K = 1000, 83, a.gpx_pop, 16
    P = random_col_assigns(n, k, p, 1)
    rs = np.random.default_rng(7)
    matches = (np.arange(p)[:, None] + 1 + rs.integers(0, p - 1, size=(p, K))) % p  # j != i
    keys = stream_keys(1, TAG_CROSS, 0, p * K)
    pop = torch.from_numpy(P).cuda()
    m = torch.from_numpy(matches.astype(np.int64)).cuda()
    kd = Dv.keys_to_tensor(keys, "cuda")
    out = torch.empty((p, K, n), dtype=torch.int32, device="cuda")
    t, _ = timed(lambda: Dv.gpx_batch(pop, m, k, kd, out))
    cores = os.cpu_count()
    pc = min(p, 512)
    t0 = time.perf_counter()
    oracle.gpx_batch(P[:pc], matches[:pc] % pc, k, keys[:pc * K], threads=cores)
    tc = time.perf_counter() - t0
    return {"op": "gpx", "unit": "offspring/s", "gpu": p * K / t, "cpu": pc * K / tc,
            "cores": cores, "config": f"n={n} k={k} p={p} K={K}",
            "cpu_sample": f"{pc}x{K} offspring", "gpu_ms": 1e3 * t,
            "alg_bytes_per_offspring": 3 * n}


def bench_distance(a):
    n, k, p = 1000, 83, a.dist_pop
    P = random_col_assigns(n, k, p, 1)
    Q = random_col_assigns(n, k, p, 2)
    if a.dist_related:
        # LS-like related pairs (a converged GA population): every colouring
        # is one base colouring under its own colour permutation with a
        # fraction of the vertices recoloured
        rng = np.random.default_rng(5)
        base = P[0].copy()
        for M in (P, Q):
            for i in range(p):
                M[i] = rng.permutation(k).astype(P.dtype)[base]
                flip = rng.random(n) < a.dist_related
                M[i, flip] = rng.integers(0, k, int(flip.sum()))
    pd, qd = torch.from_numpy(P).cuda(), torch.from_numpy(Q).cuda()
    cross = torch.zeros((p, p), dtype=torch.int32, device="cuda")
    within = torch.zeros((p, p), dtype=torch.int32, device="cuda")
    t, _ = timed(lambda: Dv.pairwise(pd, qd, k, cross=cross, within=within), reps=2)
    pairs = p * p + p * (p - 1) // 2
    cores = os.cpu_count()
    pc = 96
    t0 = time.perf_counter()
    oracle.pairwise(P[:pc], Q[:pc], k, threads=cores)
    tc = time.perf_counter() - t0
    return {"op": "distance", "unit": "pairs/s", "gpu": pairs / t,
            "cpu": (pc * pc + pc * (pc - 1) // 2) / tc, "cores": cores,
            "config": f"n={n} k={k} p=q={p} " + (f"(related pairs, {a.dist_related:.0%} recoloured)" if a.dist_related else "(random colourings)"), "cpu_sample": f"p=q={pc}",
            "gpu_ms": 1e3 * t, "alg_bytes_per_pair": 6 * n}


def _pop_case(p, q, n, seed=3):
    """Distance matrices with cluster structure (symmetric, zero diagonal)."""
    g = torch.Generator(device="cuda").manual_seed(seed)
    cen = torch.randint(0, max(2, (p + q) // 8), (p + q,), device="cuda", generator=g)
    D = torch.randint(n // 2, n + 1, (p + q, p + q), device="cuda", generator=g, dtype=torch.int32)
    D = torch.minimum(D, D.T)
    same = cen[:, None] == cen[None, :]
    D = torch.where(same, torch.randint(0, n // 10 + 3, (p + q, p + q), device="cuda", generator=g,
                                        dtype=torch.int32), D)
    D = torch.minimum(D, D.T)
    D.fill_diagonal_(0)
    fit = torch.randint(0, 40, (p + q,), device="cuda", generator=g, dtype=torch.int64)
    return (D[:p, :p].contiguous(), D[:p, p:].contiguous(), D[p:, p:].contiguous(), fit[:p].contiguous(),
            fit[p:].contiguous())


def bench_update_population(a):
    from oracle import population_oracle as PO

    p = q = a.pop_p
    n = 1000
    pd, cr, wi, fp, fq = _pop_case(p, q, n)
    ms = n // 10
    adm = torch.empty(p, dtype=torch.int32, device="cuda")
    rule = torch.empty(p, dtype=torch.uint8, device="cuda")
    nd = torch.empty((p, p), dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    P = N.ptr

    def run():
        N.check(N.lib().mcb_update_population(P(pd), P(cr), P(wi), P(fp), P(fq), p, q, ms, None, None, n,
                                             P(adm), P(rule), P(nd), None, None, stream))

    t, _ = timed(run, reps=2)
    pc = 384  # the reference loop is O(p^2) Python: bounded CPU sample
    pdc, crc, wic = pd[:pc, :pc].cpu().numpy(), cr[:pc, :pc].cpu().numpy(), wi[:pc, :pc].cpu().numpy()
    t0 = time.perf_counter()
    PO.update_population(pdc, fp[:pc].cpu().numpy(), np.zeros((pc, 1), np.int32), np.zeros((pc, 1), np.int32),
                         fq[:pc].cpu().numpy(), crc, wic, ms)
    tc = time.perf_counter() - t0
    return {"op": "update_population", "unit": "generations/s", "gpu": 1.0 / t,
            "cpu": 1.0 / (tc * (p / pc) ** 2), "cores": 1,
            "config": f"p=q={p}, n={n}, ms={ms} (clustered synthetic distances)",
            "cpu_sample": f"p=q={pc} with the restated reference loop, scaled by (p/{pc})^2 (O(p^2) loop)",
            "gpu_ms": 1e3 * t, "by_rule": int(rule.sum().item())}


def bench_match_parents(a):
    from oracle import population_oracle as PO

    p, K, n = a.pop_p, 16, 1000
    pd, _, _, _, _ = _pop_case(p, 1, n)
    m = torch.empty((p, K), dtype=torch.int64, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream

    def run():
        N.check(N.lib().mcb_match_parents(N.ptr(pd), p, K, n, N.ptr(m), stream))

    t, _ = timed(run, reps=3)
    rows = 256
    dc = pd.cpu().numpy()
    t0 = time.perf_counter()
    idx = np.arange(p)
    for i in range(rows):  # the reference row loop (population.py:137-140)
        order = np.lexsort((idx, dc[i]))
        order[order != i][:K]
    tc = time.perf_counter() - t0
    return {"op": "match_parents", "unit": "rows/s", "gpu": p / t, "cpu": rows / tc, "cores": 1,
            "config": f"p={p}, K={K}", "cpu_sample": f"{rows} rows of the reference loop", "gpu_ms": 1e3 * t,
            "alg_bytes_per_row": 4 * p}


def bench_greedy_init(a):
    """init_wvcp_population at the C4 shape: G(500,.5), w in [1,100], p = 8192."""
    from oracle import init_oracle as IO
    from paper_2109_05948_b200.graph import rand_graph
    from paper_2109_05948_b200.init import greedy_wvcp_assigns, stream_keys_init

    g = rand_graph(1, 500, 0.5, wmax=100)
    p = 8192
    keys = stream_keys_init(1, p)
    greedy_wvcp_assigns(g, keys[:8], device=True)

    def run():
        greedy_wvcp_assigns(g, keys, device=True)

    t, _ = timed(run, reps=3)
    pc = 8
    t0 = time.perf_counter()
    IO.init_wvcp_population(g.adj_indptr, g.adj_indices, g.weights, g.degrees, keys[:pc])
    tc = time.perf_counter() - t0
    return {"op": "greedy_init", "unit": "colourings/s", "gpu": p / t, "cpu": pc / tc, "cores": 1,
            "config": "G(500,.5) w in [1,100], p=8192 (C4 shape)",
            "cpu_sample": f"{pc} colourings with the restated reference loop (mc/init.py:30-46)",
            "gpu_ms": 1e3 * t}


def bench_surrogate(a):
    """Surrogate per generation at C3: predict p K = 16384 x 16 candidates
    (n = 1000, k = 83, arch "small", float32) + one training epoch on p rows."""
    from paper_2109_05948_b200.rng import TAG_TRAIN, Stream
    from paper_2109_05948_b200.surrogate import SurrogateNet

    n, k, p, K = 1000, 83, a.pop_p, 16
    net = SurrogateNet(n, problem="col", arch="small", seed=1)
    cands = torch.randint(0, k, (p * K, n), dtype=torch.int32, device="cuda")
    train = cands[:p]
    y = np.random.default_rng(1).random(p) * 100

    def run():
        net.train_generation(train, y, k, 1, 64, Stream.derive(1, TAG_TRAIN, 0))
        return net.predict_assigns_device(cands, k)

    t, _ = timed(run, reps=1)
    t_train, _ = timed(lambda: net.train_generation(train, y, k, 1, 64, Stream.derive(1, TAG_TRAIN, 0)), reps=1)
    t_train_eager, _ = timed(lambda: net.train_generation(train, y, k, 1, 64, Stream.derive(1, TAG_TRAIN, 0),
                                                          graphs=False), reps=1)
    net.tf32 = True  # opt-in tensor-core GEMMs (not the reference's float32 products)
    t_tf32, _ = timed(run, reps=1)
    net.tf32 = False
    # reference-style CPU cost: dense one-hot numpy forward, bounded sample
    lam = [l.lam.cpu().numpy() for l in net.layers]
    x = np.zeros((64, k, n), np.float32)
    a_ = cands[:64].cpu().numpy()
    x[np.arange(64)[:, None], a_, np.arange(n)[None, :]] = 1
    t0 = time.perf_counter()
    h = x
    for w in lam:
        h = np.maximum(h @ w, 0)
    tc = (time.perf_counter() - t0) / 64
    return {"op": "surrogate", "unit": "candidates/s", "gpu": p * K / t, "cpu": 1.0 / tc, "cores": os.cpu_count(),
            "config": f"n={n} k={k} arch small float32: predict {p}x{K} candidates + 1 epoch on {p} rows (batch 64)",
            "cpu_sample": "64 candidates, dense one-hot numpy matmuls (forward only, no BN: a lower bound)",
            "gpu_ms": 1e3 * t, "gpu_ms_tf32_opt_in": 1e3 * t_tf32,
            "train_epoch_ms_graphs": 1e3 * t_train, "train_epoch_ms_eager": 1e3 * t_train_eager}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ops", default="wvcp,gpx,distance")
    ap.add_argument("--wvcp-pop", type=int, default=592)
    ap.add_argument("--wvcp-depth", type=int, default=500)
    ap.add_argument("--gpx-pop", type=int, default=16384)
    ap.add_argument("--dist-pop", type=int, default=4096)
    ap.add_argument("--dist-related", type=float, default=0.0, help="recoloured fraction of related pairs (0: random)")
    ap.add_argument("--pop-p", type=int, default=16384)
    a = ap.parse_args()
    N.lib()
    oracle.build()
    for op in a.ops.split(","):
        r = {"wvcp": bench_wvcp, "gpx": bench_gpx, "distance": bench_distance,
             "update_population": bench_update_population, "match_parents": bench_match_parents,
             "greedy_init": bench_greedy_init, "surrogate": bench_surrogate}[op](a)
        r["speedup_vs_cpu"] = r["gpu"] / r["cpu"]
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
