"""Regenerate the inputs of the golden cases (tests/golden/make_golden.py)
with the package's own generators (pinned by test_host.py)."""

import numpy as np

from paper_2109_05948_b200.graph import rand_graph
from paper_2109_05948_b200.init import random_col_assigns
from paper_2109_05948_b200.rng import TAG_LS, stream_keys


def tabucol_case(data, name):
    seed, n, pe, k, pop, depth, cap = (int(x) for x in data[f"{name}__params"])
    g = rand_graph(seed, n, pe / 1000.0, wmax=1)
    A = random_col_assigns(n, k, pop, seed)
    keys = stream_keys(seed, TAG_LS, 0, pop)
    return g, A, k, keys, depth, cap


def wvcp_case(data, name):
    seed, n, pe, wmax, k, pop, depth, rounds, sched = (int(x) for x in data[f"{name}__params"])
    g = rand_graph(seed, n, pe / 1000.0, wmax=wmax)
    A = random_col_assigns(n, k, pop, seed)
    keys = stream_keys(seed, TAG_LS, 0, pop)
    phi0 = float(data[f"{name}__phi0"][0])
    return g, A, k, keys, depth, rounds, bool(sched), phi0


def check_tabucol(data, name, out, nlog_rows=None):
    pre = f"{name}__"
    for key in ("best_conflicts", "end_conflicts", "iters_used"):
        np.testing.assert_array_equal(out[key], data[pre + key], err_msg=f"{name}:{key}")
    np.testing.assert_array_equal(out["end_assigns"], data[pre + "end_assigns"].astype(np.int32),
                                  err_msg=f"{name}:end_assigns")
    np.testing.assert_array_equal(out["best_assigns"], data[pre + "best_assigns"].astype(np.int32),
                                  err_msg=f"{name}:best_assigns")
    if out.get("log") is not None and pre + "log_v" in data:
        lv, li, lt, lc = out["log"]
        gv, gi, gt = data[pre + "log_v"], data[pre + "log_iter"], data[pre + "log_tt"]
        gc = data[pre + "log_cnt"]
        np.testing.assert_array_equal(np.minimum(lc, gv.shape[1]), np.minimum(gc, gv.shape[1]))
        for i in range(gv.shape[0]):
            c = int(min(gc[i], gv.shape[1]))
            np.testing.assert_array_equal(lv[i, :c], gv[i, :c], err_msg=f"{name}:log_v[{i}]")
            np.testing.assert_array_equal(li[i, :c], gi[i, :c], err_msg=f"{name}:log_iter[{i}]")
            np.testing.assert_array_equal(lt[i, :c], gt[i, :c], err_msg=f"{name}:log_tt[{i}]")


def check_wvcp(data, name, out):
    pre = f"{name}__"
    for key in ("best_scores", "end_scores", "end_conflicts"):
        np.testing.assert_array_equal(out[key], data[pre + key], err_msg=f"{name}:{key}")
    np.testing.assert_array_equal(out["phi_used"], data[pre + "phi_used"], err_msg=f"{name}:phi")
    np.testing.assert_array_equal(out["end_assigns"], data[pre + "end_assigns"].astype(np.int32))
    np.testing.assert_array_equal(out["best_assigns"], data[pre + "best_assigns"].astype(np.int32))
    if out.get("log") is not None:
        lv, li, lt, la, lc = out["log"]
        gv = data[pre + "log_v"]
        np.testing.assert_array_equal(lc, data[pre + "log_cnt"])
        c = gv.shape[1]
        for i in range(gv.shape[0]):
            cc = int(min(c, lc[i]))
            np.testing.assert_array_equal(lv[i, :cc], gv[i, :cc], err_msg=f"{name}:log_v[{i}]")
            np.testing.assert_array_equal(li[i, :cc], data[pre + "log_iter"][i, :cc])
            np.testing.assert_array_equal(lt[i, :cc], data[pre + "log_tt"][i, :cc])
            np.testing.assert_array_equal(la[i, :cc], data[pre + "log_asp"][i, :cc])
