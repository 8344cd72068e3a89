"""Per-phase cycles of the WVCP kernel (MCB_FLAG_WSTATS, thread 0's clock64
between the CTA barriers), per iteration, at the config-4 shape.

    python tools/wvcp_probe.py [--pop 592 --depth 300 --rounds 2]
"""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_05948_b200 import _native as N  # noqa: E402
from paper_2109_05948_b200 import localsearch as LS  # noqa: E402
from paper_2109_05948_b200.graph import rand_graph  # noqa: E402
from paper_2109_05948_b200.init import random_col_assigns  # noqa: E402
from paper_2109_05948_b200.rng import TAG_LS, stream_keys  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--pop", type=int, default=592)
ap.add_argument("--depth", type=int, default=300)
ap.add_argument("--rounds", type=int, default=2)
ap.add_argument("--plain", action="store_true", help="throughput without instrumentation (CUDA events)")
a = ap.parse_args()
g = rand_graph(1, 500, 0.5, wmax=100)
k = 60
A = random_col_assigns(500, k, a.pop, 1)
keys = stream_keys(1, TAG_LS, 0, a.pop)
phi0 = LS.default_wvcp_phi0(g, k)
if a.plain:
    import torch

    from paper_2109_05948_b200 import device as Dv
    dg = Dv.DeviceGraph(g, "cuda")
    a0 = torch.from_numpy(A).cuda()
    kt = Dv.keys_to_tensor(keys, "cuda")
    best = 0.0
    for r in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = Dv.wvcp_batch(dg, a0.clone(), k, kt, a.depth, a.rounds, True, phi0)
        e1.record()
        torch.cuda.synchronize()
        if r:
            best = max(best, a.pop * a.depth * a.rounds / (e0.elapsed_time(e1) * 1e-3))
    print(json.dumps({"moves_per_s": best, "best_scores_sum": int(out["best_scores"].sum().item()),
                      "end_scores_sum": int(out["end_scores"].sum().item())}))
    sys.exit(0)
buf = (ctypes.c_ulonglong * 16)()
N.check(N.lib().mcb_debug_wvcp_stats(ctypes.addressof(buf), 1))
LS._run_wvcp_batch(g, A.copy(), k, keys, a.depth, a.rounds, True, phi0, flags=N.FLAG_WSTATS)
N.check(N.lib().mcb_debug_wvcp_stats(ctypes.addressof(buf), 1))
it = max(buf[0], 1)
names = ["pass1", "chunk_min", "prefix_walks", "warp0", "gamma_update", "refresh", "best", "tail"]
print(json.dumps({"iterations": buf[0], **{nm: round(buf[i + 1] / it, 1) for i, nm in enumerate(names)},
                  "total": round(sum(buf[1:9]) / it, 1),
                  "warp0_sub": {nm: round(buf[9 + i] / it, 1) for i, nm in
                                enumerate(["draws", "chunk_row", "colour_locate", "apply_move", "nbr_wait"])}}))
