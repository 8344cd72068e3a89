"""TabuCol on the B200 vs the reference (golden fixtures) and the CPU oracle.
Bit-exact: trajectories (move logs), end/best assignments, conflicts,
iterations -- through the C ABI (`mcb_tabucol_batch_host` / device path)."""

import numpy as np
import pytest

from cases import check_tabucol, tabucol_case
from conftest import load_golden
from paper_2109_05948_b200 import _native as N
from paper_2109_05948_b200 import localsearch as LS
from paper_2109_05948_b200.coloring import Coloring, col_conflicts_batch
from paper_2109_05948_b200.graph import rand_graph
from paper_2109_05948_b200.init import random_col_assigns
from paper_2109_05948_b200.rng import TAG_LS, stream_keys

pytestmark = pytest.mark.gpu
TAB = load_golden("tabucol")


@pytest.mark.parametrize("name", list(TAB["cases"]))
def test_tabucol_golden_bit_exact(name):
    g, A, k, keys, depth, cap = tabucol_case(TAB, name)
    out = LS._run_tabucol_batch(g, A.copy(), k, keys, depth, log_moves=cap > 0)
    check_tabucol(TAB, name, out)


@pytest.mark.parametrize("nt", ["128", "256"])
@pytest.mark.parametrize("flags", [N.FLAG_FORCE_WIDE, N.FLAG_FORCE_GLOBAL])
@pytest.mark.parametrize("name", ["c1", "c2w", "k70", "k3", "tenure"])
def test_tabucol_table_variants_bit_exact(name, flags, nt, monkeypatch):
    """int16/u32 tables and the L2-resident (global) tables give identical
    results, with 128 and with 256 threads per individual (MCB_TC_NT)."""
    monkeypatch.setenv("MCB_TC_NT", nt)
    g, A, k, keys, depth, cap = tabucol_case(TAB, name)
    out = LS._run_tabucol_batch(g, A.copy(), k, keys, depth, log_moves=cap > 0, flags=flags)
    check_tabucol(TAB, name, out)


def test_tabucol_vs_oracle_random(oracle_lib):
    rs = np.random.default_rng(5)
    for t in range(12):
        n = int(rs.integers(2, 300))
        pe = float(rs.uniform(0.05, 0.95))
        k = int(rs.integers(2, 90))
        p = int(rs.integers(1, 40))
        depth = int(rs.integers(1, 3000))
        g = rand_graph(1000 + t, n, pe)
        A = random_col_assigns(n, k, p, 77 + t)
        keys = stream_keys(t, TAG_LS, 3, p)
        ref = oracle_lib.tabucol_batch(g, A.copy(), k, keys, depth, log_moves=True, counters=True)
        got = LS._run_tabucol_batch(g, A.copy(), k, keys, depth, log_moves=True, counters=True)
        for key in ("end_assigns", "best_assigns", "best_conflicts", "end_conflicts", "iters_used",
                    "counters"):
            np.testing.assert_array_equal(got[key], ref[key], err_msg=f"case {t} {key}")
        for a, b in zip(got["log"], ref["log"]):
            np.testing.assert_array_equal(a, b, err_msg=f"case {t} log")


def test_tabucol_c2_subset_vs_oracle(oracle_lib):
    """BASELINE config 1 shape: 64 individuals x 5k iterations, bit-exact."""
    g = rand_graph(1, 500, 0.5)
    A = random_col_assigns(500, 48, 64, 1)
    keys = stream_keys(1, TAG_LS, 0, 64)
    ref = oracle_lib.tabucol_batch(g, A.copy(), 48, keys, 5000, counters=True)
    got = LS._run_tabucol_batch(g, A.copy(), 48, keys, 5000, counters=True)
    for key in ("end_assigns", "best_assigns", "best_conflicts", "end_conflicts", "iters_used",
                "counters"):
        np.testing.assert_array_equal(got[key], ref[key], err_msg=key)


def test_tabucol_full_size_properties():
    """Config 1 at D=1024 x 2k: outputs are consistent with scratch evaluation."""
    g = rand_graph(1, 500, 0.5)
    A = random_col_assigns(500, 48, 1024, 1)
    keys = stream_keys(1, TAG_LS, 0, 1024)
    start_conf = col_conflicts_batch(g, A)
    out = LS._run_tabucol_batch(g, A.copy(), 48, keys, 2000)
    np.testing.assert_array_equal(col_conflicts_batch(g, out["end_assigns"]), out["end_conflicts"])
    np.testing.assert_array_equal(col_conflicts_batch(g, out["best_assigns"]), out["best_conflicts"])
    assert (out["best_conflicts"] <= out["end_conflicts"]).all()
    assert (out["best_conflicts"] < start_conf).all()
    assert (out["iters_used"] == 2000).all()
    # determinism: same inputs, same outputs
    out2 = LS._run_tabucol_batch(g, A.copy(), 48, keys, 2000)
    np.testing.assert_array_equal(out["end_assigns"], out2["end_assigns"])


def test_tabucol_production_mode_sane():
    g = rand_graph(1, 125, 0.5)
    A = random_col_assigns(125, 18, 256, 2)
    keys = stream_keys(2, TAG_LS, 0, 256)
    out = LS._run_tabucol_batch(g, A.copy(), 18, keys, 10000, rng="philox")
    np.testing.assert_array_equal(col_conflicts_batch(g, out["best_assigns"]), out["best_conflicts"])
    assert (out["best_conflicts"] == 0).mean() > 0.9


def test_tabucol_api_and_errors():
    g = rand_graph(3, 40, 0.3)
    c = Coloring(random_col_assigns(40, 5, 1, 3)[0], 5)
    end, best, bc = LS.tabucol(g, c, 5, depth=500, key=123)
    assert bc == int(col_conflicts_batch(g, best.assign[None])[0])
    with pytest.raises(ValueError):
        LS._run_tabucol_batch(g, np.full((1, 40), 7, np.int32), 5, np.zeros(1, np.uint64), 10)
    with pytest.raises(ValueError):
        LS.improve_population(g, [c], "bogus", 1)
    res = LS.improve_population(g, [c, c], LS.COL, 1, depth=300)
    assert len(res) == 2 and res[0].start == c


def test_device_path_matches_host_path():
    import torch

    from paper_2109_05948_b200 import device as D

    g = rand_graph(1, 500, 0.5)
    A = random_col_assigns(500, 48, 32, 1)
    keys = stream_keys(1, TAG_LS, 0, 32)
    host = LS._run_tabucol_batch(g, A.copy(), 48, keys, 1500)
    dg = D.DeviceGraph(g, "cuda")
    a = torch.from_numpy(A.copy()).cuda()
    dev = D.tabucol_batch(dg, a, 48, D.keys_to_tensor(keys, "cuda"), 1500)
    torch.cuda.synchronize()
    for key in ("end_assigns", "best_assigns", "best_conflicts", "iters_used"):
        np.testing.assert_array_equal(dev[key].cpu().numpy(), host[key])


def test_host_path_leaves_unwritten_log_entries_alone():
    """The kernels write the first log_cnt[i] entries of each log row; the rest
    keeps the caller's content, as the numba kernel leaves it -- also when the
    device arena still holds a longer previous call's logs."""
    g = rand_graph(1, 125, 0.5)
    A = random_col_assigns(125, 18, 16, 1)
    keys = stream_keys(1, TAG_LS, 0, 16)
    LS._run_tabucol_batch(g, A.copy(), 18, keys, 3000, log_moves=True)  # long logs in the arena
    out = LS._run_tabucol_batch(g, A.copy(), 18, keys, 3000, log_moves=True)
    lv, li, lt, lc = out["log"]
    short = LS._run_tabucol_batch(g, A.copy(), 18, keys, 40, log_moves=True)
    sv, si, st, sc = short["log"]
    assert (sc == 40).all()
    np.testing.assert_array_equal(sv[:, :40], lv[:, :40])
    assert lv.shape[1] == 3000 and sv.shape[1] == 40
    # a caller-provided tail is preserved
    p, cap = 16, 200
    keep = np.full((p, cap), -7, np.int32)
    from paper_2109_05948_b200 import _native as NN
    Ac = A.copy()
    from paper_2109_05948_b200.graph import graph_arrays
    ip, ix, eu, ev = graph_arrays(g)
    best = A.copy()
    bc, ec, it, dg = (np.zeros(p, np.int64) for _ in range(4))
    li2, lt2, lcnt = np.zeros((p, cap), np.int64), np.zeros((p, cap), np.int64), np.zeros(p, np.int64)
    NN.check(NN.lib().mcb_tabucol_batch_host(
        Ac.ctypes.data, p, 125, 18, ip.ctypes.data, ix.ctypes.data, eu.ctypes.data, ev.ctypes.data, g.m, 50,
        keys.ctypes.data, best.ctypes.data, bc.ctypes.data, ec.ctypes.data, it.ctypes.data,
        dg.ctypes.data, cap, keep.ctypes.data, li2.ctypes.data, lt2.ctypes.data, lcnt.ctypes.data,
        None, 0, None))
    assert (lcnt == 50).all()
    assert (keep[:, 50:] == -7).all()
