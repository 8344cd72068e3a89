"""A/B throughput probe of the TabuCol kernels under environment variants.

    python tools/warp_probe.py [--n 500 --k 48 --pop 1036 --depth 5000]
        [--var 'name:ENV=val,ENV2=val' ...]

Each variant sets its environment variables (read by the library at launch),
runs one warm-up and `--reps` timed launches (CUDA events) and prints moves/s.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_05948_b200 import _native as N  # noqa: E402
from paper_2109_05948_b200 import device as Dv  # noqa: E402
from paper_2109_05948_b200.graph import rand_graph  # noqa: E402
from paper_2109_05948_b200.init import random_col_assigns  # noqa: E402
from paper_2109_05948_b200.rng import TAG_LS, stream_keys  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=500)
ap.add_argument("--k", type=int, default=48)
ap.add_argument("--p", type=float, default=0.5)
ap.add_argument("--pop", type=int, default=1036)
ap.add_argument("--depth", type=int, default=5000)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--philox", action="store_true")
ap.add_argument("--var", action="append", default=[])
ap.add_argument("--stats", action="store_true")
ap.add_argument("--modcheck", type=int, default=0)
ap.add_argument("--warm", type=int, default=0, help="start from the end colourings of a WARM-iteration run")
a = ap.parse_args()

if a.modcheck:
    import ctypes
    bad = ctypes.c_ulonglong(0)
    N.lib().mcb_debug_modcheck(a.modcheck, ctypes.addressof(bad))
    print(json.dumps({"modcheck_pairs": a.modcheck, "mismatches": bad.value}), flush=True)
g = rand_graph(1, a.n, a.p)
A = random_col_assigns(a.n, a.k, a.pop, 1)
dg = Dv.DeviceGraph(g, "cuda")
keys = Dv.keys_to_tensor(stream_keys(1, TAG_LS, 0, a.pop), "cuda")
if a.warm:
    a_w = torch.from_numpy(A.copy()).cuda()
    Dv.tabucol_batch(dg, a_w, a.k, keys, a.warm)
    A = a_w.cpu().numpy()
    keys = Dv.keys_to_tensor(stream_keys(1, TAG_LS, 1, a.pop), "cuda")
flags = (N.FLAG_PRODUCTION if a.philox else 0) | (N.FLAG_WSTATS if a.stats else 0)
variants = a.var or ["default:"]
ref = None
for spec in variants:
    name, _, envs = spec.partition(":")
    saved = {}
    for kv in filter(None, envs.split(",")):
        k_, _, v_ = kv.partition("=")
        saved[k_] = os.environ.get(k_)
        os.environ[k_] = v_
    best = 0.0
    for r in range(a.reps + 1):
        a_dev = torch.from_numpy(A.copy()).cuda()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        out = Dv.tabucol_batch(dg, a_dev, a.k, keys, a.depth, flags=flags, counters=True)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        moves = int(out["iters_used"].sum().item())
        if r > 0:
            best = max(best, moves / (ms * 1e-3))
    res = {k_: out[k_].cpu().numpy() for k_ in ("best_conflicts", "end_conflicts", "iters_used")}
    same = None
    if ref is None:
        ref = res
    else:
        same = all(np.array_equal(ref[k_], res[k_]) for k_ in ref)
    c = out["counters"].cpu().numpy().sum(0)
    if a.stats:
        import ctypes
        buf = (ctypes.c_ulonglong * 40)()
        N.lib().mcb_debug_warp_stats(ctypes.addressof(buf))
        names = ["it", "rounds", "asp_rounds", "expire_rows", "supersede", "walk_passes", "draw_rounds",
                 "events", "removes", "best"] + [""] * 6 + ["cy_scan", "cy_select", "cy_move", "cy_update",
                                                           "cy_events", "cy_tail", "cy_expire",
                                                           "cy_rowmin", "cy_prefix", "cy_list", "cy_walk", "cy_p2",
                                                           "cy_draw", "cy_locrows", "ncl", "ncl_gt32", "ncl_gt144"]
        it_ = max(buf[0], 1)
        print(json.dumps({nm: round(buf[i] / it_, 3) for i, nm in enumerate(names) if nm}), flush=True)
    if os.environ.get("MCB_GSTATS"):
        import ctypes
        buf = (ctypes.c_ulonglong * 32)()
        N.lib().mcb_debug_group_stats(ctypes.addressof(buf))
        it_ = max(buf[15], 1)
        names = ["scan", "wscan+B1", "events", "cx+B2", "draws", "locate", "B4", "move", "update", "B5+list",
                 "expiry", "B6", "tail"]
        print(json.dumps({"gstats_" + nm: round(buf[i] / it_, 1) for i, nm in enumerate(names)}), flush=True)
    print(json.dumps({"variant": name, "moves_per_s": best, "ms": ms, "moves": moves,
                      "mean_C": float(c[0] / max(moves, 1)), "mean_deg": float(c[1] / max(moves, 1)),
                      "same_as_first": same}), flush=True)
    for k_, v_ in saved.items():
        if v_ is None:
            os.environ.pop(k_, None)
        else:
            os.environ[k_] = v_
