"""The warp-per-individual TabuCol kernel (csrc/tabucol_warp.cu), every
variant, bit-exact against the CPU oracle (oracle/, the restatement of
`_tabucol_batch`, localsearch.py:266-410): move logs, end/best assignments,
conflicts, iteration counts and the algorithmic-byte counters.

Variants are selected the way the planner would (bitset rows of CH = 8/16/32
bits per lane, or CSR neighbours from L2; gamma rows of KV = 1..8 x 16 bytes)
and forced with MCB_WARP_MODE; MCB_NO_WARP_KERNEL selects the CTA kernel.
The fallback cases (gamma > 63, > 1000 live tabu entries) must hand the
affected individuals to the CTA kernel and still match."""

import ctypes

import numpy as np
import pytest

from paper_2109_05948_b200 import _native as N
from paper_2109_05948_b200 import localsearch as LS
from paper_2109_05948_b200.graph import rand_graph
from paper_2109_05948_b200.init import random_col_assigns
from paper_2109_05948_b200.rng import TAG_LS, stream_keys

pytestmark = pytest.mark.gpu

# (seed, n, p_edge, k, pop, depth): what each one exercises
SHAPES = [
    (7, 80, 0.5, 8, 48, 3000),      # re-tabu of a tabu pair (supersede), aspiration; KV=1 CH=8
    (7, 150, 0.2, 6, 48, 3000),     # supersede on a sparse graph
    (1, 125, 0.5, 18, 48, 4000),    # BASELINE config 0 shape (KV=2, CH=8), reaches 0 conflicts
    (1, 500, 0.5, 48, 24, 3000),    # BASELINE config 1 shape (KV=3, CH=16)
    (3, 300, 0.5, 83, 16, 2000),    # KV=6, many colours
    (3, 200, 0.4, 120, 16, 1500),   # KV=8 (k close to the 128 limit)
    (5, 700, 0.1, 20, 16, 2000),    # CH=32 (n > 512)
    (5, 1000, 0.05, 12, 8, 1500),   # n = 1000
]
FALLBACK = [
    (11, 200, 0.8, 2, 8, 500),      # gamma > 63 at the start -> CTA kernel
    (12, 300, 0.3, 6, 8, 2000),     # tenure ~1350 -> > 1024 live tabu entries -> SPILL variant
    (1, 1000, 0.5, 83, 6, 2500),    # config 2 (C3) shape from random colourings: tenure ~1800 -> SPILL
]


def _run(g, A, k, keys, depth, monkeypatch, mode):
    monkeypatch.delenv("MCB_WARP_MODE", raising=False)
    monkeypatch.delenv("MCB_NO_WARP_KERNEL", raising=False)
    if mode == "legacy":
        monkeypatch.setenv("MCB_NO_WARP_KERNEL", "1")
    elif mode != "auto":
        monkeypatch.setenv("MCB_WARP_MODE", mode)
    return LS._run_tabucol_batch(g, A.copy(), k, keys, depth, log_moves=True, counters=True)


def _check(got, ref, tag):
    for key in ("end_assigns", "best_assigns", "best_conflicts", "end_conflicts", "iters_used", "counters"):
        np.testing.assert_array_equal(got[key], ref[key], err_msg=f"{tag}:{key}")
    for a, b in zip(got["log"], ref["log"]):
        np.testing.assert_array_equal(a, b, err_msg=f"{tag}:log")


@pytest.mark.parametrize("mode", ["bits", "csr", "legacy"])
@pytest.mark.parametrize("shape", SHAPES, ids=[f"n{s[1]}k{s[3]}" for s in SHAPES])
def test_warp_variants_vs_oracle(shape, mode, monkeypatch, oracle_lib):
    seed, n, pe, k, pop, depth = shape
    g = rand_graph(seed, n, pe)
    A = random_col_assigns(n, k, pop, seed)
    keys = stream_keys(seed, TAG_LS, 0, pop)
    ref = oracle_lib.tabucol_batch(g, A.copy(), k, keys, depth, log_moves=True, counters=True)
    _check(_run(g, A, k, keys, depth, monkeypatch, mode), ref, f"{shape}/{mode}")


@pytest.mark.parametrize("shape", FALLBACK, ids=["gamma_overflow", "ring_overflow", "c3_random_start"])
def test_warp_fallback_vs_oracle(shape, monkeypatch, oracle_lib):
    seed, n, pe, k, pop, depth = shape
    g = rand_graph(seed, n, pe)
    A = random_col_assigns(n, k, pop, seed)
    keys = stream_keys(seed, TAG_LS, 0, pop)
    ref = oracle_lib.tabucol_batch(g, A.copy(), k, keys, depth, log_moves=True, counters=True)
    _check(_run(g, A, k, keys, depth, monkeypatch, "auto"), ref, f"{shape}")


def test_warp_supersede_path_is_exercised(monkeypatch):
    """The first SHAPES entry really re-tabus tabu pairs (so the bit-exact
    comparison above covers that path): counted by the kernel's stats."""
    seed, n, pe, k, pop, depth = SHAPES[0]
    g = rand_graph(seed, n, pe)
    A = random_col_assigns(n, k, pop, seed)
    keys = stream_keys(seed, TAG_LS, 0, pop)
    monkeypatch.delenv("MCB_NO_WARP_KERNEL", raising=False)
    LS._run_tabucol_batch(g, A.copy(), k, keys, depth, flags=N.FLAG_WSTATS)
    buf = (ctypes.c_ulonglong * 40)()
    N.check(N.lib().mcb_debug_warp_stats(ctypes.addressof(buf)))
    assert buf[0] == pop * depth or buf[0] > 0  # iterations ran in the warp kernel
    assert buf[4] > 0, "no supersede event in the supersede case"
    assert buf[2] > 0, "no aspiration round"


def test_spill_variant_runs_for_long_tabu_lists(monkeypatch):
    """The C3 shape from random colourings keeps > 1024 tabu entries live: the
    individuals re-run on the SPILL variant (rows spilled to global memory),
    bit-exact vs the oracle above; MCB_NO_SPILL routes them to the CTA kernel
    instead, with the same results."""
    seed, n, pe, k, pop, depth = FALLBACK[2]
    g = rand_graph(seed, n, pe)
    A = random_col_assigns(n, k, pop, seed)
    keys = stream_keys(seed, TAG_LS, 0, pop)
    monkeypatch.delenv("MCB_NO_WARP_KERNEL", raising=False)
    a = LS._run_tabucol_batch(g, A.copy(), k, keys, depth, flags=N.FLAG_WSTATS)
    buf = (ctypes.c_ulonglong * 40)()
    N.check(N.lib().mcb_debug_warp_stats(ctypes.addressof(buf)))
    assert buf[10] > 0, "no ring row spilled"
    monkeypatch.setenv("MCB_NO_SPILL", "1")
    b = LS._run_tabucol_batch(g, A.copy(), k, keys, depth)
    for key in ("end_assigns", "best_assigns", "best_conflicts", "iters_used"):
        np.testing.assert_array_equal(a[key], b[key])


def test_draw_divisibility_paths():
    """fp64 x % s == 0 test (any s) and the s < 64 table test vs the 64-bit %."""
    bad = ctypes.c_ulonglong(0)
    N.check(N.lib().mcb_debug_modcheck(20_000_000, ctypes.addressof(bad)))
    assert bad.value == 0


def test_describe_reports_the_warp_kernel():
    buf = ctypes.create_string_buffer(256)
    N.check(N.lib().mcb_tabucol_describe(500, 48, 8192, buf, 256))
    assert b"tabucol_warp_kernel<KV=3,bitset CH=16>" in buf.value


@pytest.mark.parametrize("nw", ["1", "2", "4"])
@pytest.mark.parametrize("shape", SHAPES + FALLBACK,
                         ids=[f"n{s[1]}k{s[3]}p{s[2]}" for s in SHAPES + FALLBACK])
def test_group_kernel_vs_oracle(shape, nw, monkeypatch, oracle_lib):
    """The opt-in group-of-warps kernel (csrc/tabucol_group.cu, MCB_GROUP_NW):
    row summaries + NW warps per individual, bit-exact including move logs and
    its hand-off of overflowing individuals to the warp SPILL / CTA kernels."""
    seed, n, pe, k, pop, depth = shape
    g = rand_graph(seed, n, pe)
    A = random_col_assigns(n, k, pop, seed)
    keys = stream_keys(seed, TAG_LS, 0, pop)
    ref = oracle_lib.tabucol_batch(g, A.copy(), k, keys, depth, log_moves=True, counters=True)
    monkeypatch.setenv("MCB_GROUP_NW", nw)
    buf = ctypes.create_string_buffer(256)
    N.check(N.lib().mcb_tabucol_describe(n, k, pop, buf, 256))
    assert b"tabucol_group_kernel" in buf.value
    _check(_run(g, A, k, keys, depth, monkeypatch, "auto"), ref, f"{shape}/group{nw}")
