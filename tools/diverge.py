"""Find the first iteration where the warp kernel's move log diverges from the
legacy CTA kernel (same inputs).  Debug tool.
    python tools/diverge.py [--n 125 --k 18 --p 0.5 --pop 64 --depth 10000 --seed 1]"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_05948_b200 import localsearch as LS  # noqa: E402
from paper_2109_05948_b200.graph import rand_graph  # noqa: E402
from paper_2109_05948_b200.init import random_col_assigns  # noqa: E402
from paper_2109_05948_b200.rng import TAG_LS, stream_keys  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=125)
ap.add_argument("--k", type=int, default=18)
ap.add_argument("--p", type=float, default=0.5)
ap.add_argument("--pop", type=int, default=64)
ap.add_argument("--depth", type=int, default=10000)
ap.add_argument("--seed", type=int, default=1)
a = ap.parse_args()
g = rand_graph(a.seed, a.n, a.p)
A = random_col_assigns(a.n, a.k, a.pop, a.seed)
keys = stream_keys(a.seed, TAG_LS, 0, a.pop)
got = LS._run_tabucol_batch(g, A.copy(), a.k, keys, a.depth, log_moves=True)
os.environ["MCB_NO_WARP_KERNEL"] = "1"
ref = LS._run_tabucol_batch(g, A.copy(), a.k, keys, a.depth, log_moves=True)
lv, li, lt, lc = got["log"]
rv, ri, rt, rc = ref["log"]
nbad = 0
for i in range(a.pop):
    m = min(lc[i], rc[i], lv.shape[1])
    d = np.nonzero((lv[i, :m] != rv[i, :m]) | (lt[i, :m] != rt[i, :m]))[0]
    if len(d) or lc[i] != rc[i] or got["best_conflicts"][i] != ref["best_conflicts"][i]:
        nbad += 1
        j = int(d[0]) if len(d) else m
        print(f"ind {i}: first diff at move {j} (iter {ri[i, j] if j < m else '-'}), "
              f"got v={lv[i, j - 2:j + 3]} tt={lt[i, j - 2:j + 3]} | ref v={rv[i, j - 2:j + 3]} "
              f"tt={rt[i, j - 2:j + 3]}; cnt {lc[i]} vs {rc[i]}; best {got['best_conflicts'][i]} vs "
              f"{ref['best_conflicts'][i]}")
print(f"{nbad} of {a.pop} individuals differ")
