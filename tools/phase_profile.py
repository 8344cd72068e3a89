"""Per-phase cycle breakdown of the TabuCol iteration (MCB_FLAG_PROFILE).
Usage: python tools/phase_profile.py [--pop P] [--depth D] [--workload c2]"""
import argparse
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_05948_b200 import _native as N  # noqa: E402
from paper_2109_05948_b200 import device as Dv  # noqa: E402
from paper_2109_05948_b200.graph import rand_graph  # noqa: E402
from paper_2109_05948_b200.init import random_col_assigns  # noqa: E402
from paper_2109_05948_b200.rng import TAG_LS, stream_keys  # noqa: E402

NAMES = {1: "pass1+sync", 2: "scan", 3: "draws", 4: "locate", 5: "apply(lane0)",
         6: "nbr update", 7: "events+best", 8: "end sync", 9: "diag/sweep"}
ap = argparse.ArgumentParser()
ap.add_argument("--pop", type=int, default=444)
ap.add_argument("--depth", type=int, default=20000)
ap.add_argument("--n", type=int, default=500)
ap.add_argument("--k", type=int, default=48)
ap.add_argument("--philox", action="store_true")
ap.add_argument("--cluster", action="store_true", help="force the 2-CTA cluster kernel (its own phase names)")
ap.add_argument("--nodiag", action="store_true")
a = ap.parse_args()
g = rand_graph(1, a.n, 0.5)
A = random_col_assigns(a.n, a.k, a.pop, 1)
dg = Dv.DeviceGraph(g, "cuda")
keys = Dv.keys_to_tensor(stream_keys(1, TAG_LS, 0, a.pop), "cuda")
buf = (ctypes.c_ulonglong * 16)()
N.lib().mcb_debug_phase_cycles(buf, 1)
wbuf = (ctypes.c_ulonglong * 96)()
N.lib().mcb_debug_cluster_warps(wbuf, 1)
flags = (0 if a.nodiag else N.FLAG_DIAG) | N.FLAG_PROFILE | (N.FLAG_PRODUCTION if a.philox else 0)
if a.cluster:
    flags |= N.FLAG_FORCE_CLUSTER
    NAMES = {1: "pass1+#1", 2: "prefix/walk+#2", 3: "draw/locate+#3", 4: "move+update", 5: "-",
             6: "list events", 7: "tail", 8: "(p1 work r0)", 9: "(p1 work r1)"}
t = torch.from_numpy(A).cuda()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
out = Dv.tabucol_batch(Dv.DeviceGraph(g, "cuda"), t, a.k, keys, a.depth, flags=flags, counters=True)
ev[1].record()
torch.cuda.synchronize()
N.check(N.lib().mcb_debug_phase_cycles(buf, 0))
its = buf[10]
tot = sum(buf[i] for i in range(1, 8 if a.cluster else 10))
print(f"iterations {its}, mean C {out['counters'][:,0].sum().item()/its:.1f}, "
      f"{tot/its:.0f} cycles/iteration (thread 0 view), kernel {ev[0].elapsed_time(ev[1]):.1f} ms")
for i in range(1, 10):
    print(f"  {NAMES[i]:14s} {buf[i]/its:9.1f} cycles  {100*buf[i]/tot:5.1f}%")
if a.cluster:
    print(f"  spilled rows/iteration (rank 0) {buf[11]/its:.1f}, walked half-rows/iteration {buf[12]/its:.2f}, "
          f"stale rescans {buf[13]/its:.1f}, masked scans {buf[14]/its:.2f} (rank 0); "
          f"init {buf[15]/a.pop:.0f} cycles per individual")
if a.cluster:
    N.check(N.lib().mcb_debug_cluster_warps(wbuf, 0))
    cl = a.pop // 1  # rank-0 CTAs: one per individual
    print("  per warp (rank 0, per iteration): pass-1 cycles / start delay / warp scans")
    print("   " + " ".join(f"{wbuf[w]/its:6.0f}" for w in range(32) if wbuf[w]))
    print("   " + " ".join(f"{wbuf[32+w]/its:6.0f}" for w in range(32) if wbuf[w]))
    print("   " + " ".join(f"{wbuf[64+w]/its:6.2f}" for w in range(32) if wbuf[w]))
    print("  warp0 pass-1 stage cycles: " + " ".join(f"{wbuf[80+i]/its:7.0f}" for i in range(4)))
