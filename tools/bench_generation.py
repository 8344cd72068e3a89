"""One device-resident k-colouring generation at BASELINE config 2 shape
(G(1000,.5), k = 83, p = 16384, K = 16) with per-stage CUDA-event times:
LS (TabuCol), pairwise distances (p x p cross + p(p-1)/2 within), pool update,
parent matching, offspring (GPX p x K + selection).

    python tools/bench_generation.py [--p 16384] [--depth 2000] [--gens 2]
    torchrun --nproc-per-node N tools/bench_generation.py ...   (sharded over N GPUs, NCCL)

The LS stage scales linearly with depth (config 2 asks 100,000 iterations);
the other stages do not depend on it.
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_05948_b200 import device as Dv  # noqa: E402
from paper_2109_05948_b200 import engine as E  # noqa: E402
from paper_2109_05948_b200.graph import rand_graph  # noqa: E402
from paper_2109_05948_b200.init import random_col_assigns  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1000)
ap.add_argument("--k", type=int, default=83)
ap.add_argument("--p", type=int, default=16384)
ap.add_argument("--K", type=int, default=16)
ap.add_argument("--depth", type=int, default=2000)
ap.add_argument("--gens", type=int, default=2)
ap.add_argument("--surrogate", action="store_true", help="surrogate-guided selection (arch small, float32)")
ap.add_argument("--tf32", action="store_true", help="surrogate GEMMs on TF32 tensor cores (opt-in)")
ap.add_argument("--epochs", type=int, default=1)
a = ap.parse_args()
world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
if world > 1:
    import torch.distributed as dist

    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    dist.init_process_group("nccl")
t0 = time.time()
g = rand_graph(1, a.n, 0.5)
dg = Dv.DeviceGraph(g, "cuda")
A = random_col_assigns(a.n, a.k, a.p, 1)
st = E.init_state(dg, A, a.k)
net = None
if a.surrogate:
    from paper_2109_05948_b200.surrogate import SurrogateNet

    net = SurrogateNet(a.n, problem="col", arch="small", seed=1, tf32=a.tf32)
torch.cuda.synchronize()
for t in range(a.gens):
    tim = {}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ls = E.generation(dg, st, seed=1, depth=a.depth, K=a.K, timings=tim, net=net, epochs=a.epochs)
    e1.record()
    torch.cuda.synchronize()
    moves = int(ls["iters_used"].sum().item())
    if rank:
        continue
    print(json.dumps({"generation": t, "total_s": e0.elapsed_time(e1) / 1e3, "gpus": world,
                      "stages_s": {k_: round(v, 4) for k_, v in tim.items()},
                      "ls_moves": moves, "ls_moves_per_s": moves / tim["ls"] if "ls" in tim else None,
                      "best": st.best_score, "pop_fitness_mean": float(st.pop_fitness.float().mean()),
                      "config": f"G({a.n},.5) k={a.k} p={a.p} K={a.K} LS depth {a.depth}"
                                + (f", surrogate small{' tf32' if a.tf32 else ''} {a.epochs} epoch(s)" if net else "")}),
          flush=True)
