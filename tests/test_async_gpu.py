"""MCB_FLAG_ASYNC TabuCol calls: no host synchronisation (per-stream scratch,
the SPILL and wide fallback passes always enqueued with device-side work
counts), so the call can be captured in a CUDA graph and overlap other
streams.  Results are identical to the synchronous path, including
individuals that take the fallback passes."""
import numpy as np
import pytest
import torch

from paper_2109_05948_b200 import _native as N
from paper_2109_05948_b200 import device as Dv
from paper_2109_05948_b200.graph import rand_graph
from paper_2109_05948_b200.init import random_col_assigns
from paper_2109_05948_b200.rng import TAG_LS, stream_keys

pytestmark = pytest.mark.gpu
KEYS = ("end_assigns", "best_assigns", "best_conflicts", "end_conflicts", "iters_used", "diag")

CASES = [
    (1, 500, 0.5, 48, 32, 2000),   # config 1 shape: warp kernel
    (12, 300, 0.3, 6, 8, 2000),    # > 1024 live tabu entries: the SPILL pass
    (11, 200, 0.8, 2, 8, 500),     # gamma > 63: the wide CTA pass
    (1, 2000, 0.5, 150, 4, 300),   # config 4 shape: CTA kernel, gamma in L2
]


def _inputs(seed, n, pe, k, p):
    g = rand_graph(seed, n, pe)
    dg = Dv.DeviceGraph(g, "cuda")
    a0 = torch.from_numpy(random_col_assigns(n, k, p, seed)).cuda()
    keys = Dv.keys_to_tensor(stream_keys(seed, TAG_LS, 0, p), "cuda")
    return dg, a0, keys


@pytest.mark.parametrize("case", CASES, ids=["c2", "spill", "wide", "c5"])
def test_async_matches_sync(case):
    seed, n, pe, k, p, depth = case
    dg, a0, keys = _inputs(seed, n, pe, k, p)
    ref = Dv.tabucol_batch(dg, a0.clone(), k, keys, depth)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        got = Dv.tabucol_batch(dg, a0.clone(), k, keys, depth, flags=N.FLAG_DIAG | N.FLAG_ASYNC)
        Dv.tabucol_async_status()
    torch.cuda.synchronize()
    for key in KEYS:
        assert torch.equal(got[key], ref[key]), key


def test_async_call_captured_in_a_cuda_graph():
    seed, n, pe, k, p, depth = CASES[0]
    dg, a0, keys = _inputs(seed, n, pe, k, p)
    ref = Dv.tabucol_batch(dg, a0.clone(), k, keys, depth)
    flags = N.FLAG_DIAG | N.FLAG_ASYNC
    a = a0.clone()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        Dv.tabucol_batch(dg, a, k, keys, depth, flags=flags)  # warm-up: sizes the stream's scratch
        Dv.tabucol_async_status()
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):  # the stream whose scratch the warm-up sized
        a.copy_(a0)
        out = Dv.tabucol_batch(dg, a, k, keys, depth, flags=flags)
    for _ in range(2):
        a.fill_(0)
        graph.replay()
        torch.cuda.synchronize()
        for key in KEYS:
            assert torch.equal(out[key], ref[key]), key


def test_async_range_error_reported():
    seed, n, pe, k, p, depth = CASES[0]
    dg, a0, keys = _inputs(seed, n, pe, k, p)
    bad = a0.clone()
    bad[3, 7] = k + 5
    Dv.tabucol_batch(dg, bad, k, keys, 50, flags=N.FLAG_DIAG | N.FLAG_ASYNC)
    with pytest.raises(ValueError, match="out of range"):
        Dv.tabucol_async_status()
    Dv.tabucol_batch(dg, a0.clone(), k, keys, 50, flags=N.FLAG_DIAG | N.FLAG_ASYNC)
    Dv.tabucol_async_status()  # a clean call clears the word
