"""`improve_population` (`mc/localsearch.py:615-682`) pinned directly against
the reference's own LsResults (tests/golden/improve.npz, made by
make_golden.py): TabuCol and WVCP, generations > 0 (the streams are keyed by
master seed, TAG_LS, generation and individual) and the default depths
(128 n for TabuCol, 10 n per WVCP round).  The oracle leg runs on CPU; the
package leg goes through the C-ABI on the GPU."""

import hashlib

import numpy as np
import pytest

from conftest import load_golden
from paper_2109_05948_b200 import localsearch as LS
from paper_2109_05948_b200.coloring import Coloring
from paper_2109_05948_b200.graph import rand_graph
from paper_2109_05948_b200.init import random_col_assigns
from paper_2109_05948_b200.rng import TAG_LS, stream_keys

IMP = load_golden("improve")


def _case(name):
    seed, n, pe, wmax, k, pop, gen, depth, rounds = (int(x) for x in IMP[f"{name}__params"])
    mode = str(IMP[f"{name}__mode"][0])
    g = rand_graph(seed, n, pe / 1000, wmax=wmax)
    A = random_col_assigns(n, k, pop, seed)
    d = hashlib.sha256(np.ascontiguousarray(A, dtype=np.int32).tobytes()).hexdigest()[:16]
    assert d == str(IMP[f"{name}__init_digest"][0]), "initial colourings differ from the fixture's"
    return mode, g, A, seed, k, pop, gen, depth, rounds


@pytest.mark.parametrize("name", list(IMP["cases"]))
def test_oracle_improve_population_golden(oracle_lib, name):
    """The restatement with improve_population's key derivation and default
    depths reproduces the reference's LsResults."""
    mode, g, A, seed, k, pop, gen, depth, rounds = _case(name)
    keys = stream_keys(seed, TAG_LS, gen, pop)
    pre = f"{name}__"
    if mode == "col":
        out = oracle_lib.tabucol_batch(g, A.copy(), k, keys, depth or 128 * g.n)
        np.testing.assert_array_equal(out["best_assigns"], IMP[pre + "best"])
        np.testing.assert_array_equal(out["end_assigns"], IMP[pre + "end"])
        np.testing.assert_array_equal(out["best_conflicts"], IMP[pre + "best_score"])
        np.testing.assert_array_equal(out["iters_used"], IMP[pre + "iterations_used"])
    else:
        phi0 = LS.default_wvcp_phi0(g, k)
        out = oracle_lib.wvcp_batch(g, A.copy(), k, keys, depth or 10 * g.n, rounds, True, phi0)
        legal = out["best_scores"] < LS.INF_SCORE
        np.testing.assert_array_equal(legal, IMP[pre + "legal_found"])
        np.testing.assert_array_equal(out["best_scores"][legal], IMP[pre + "best_score"][legal])
        np.testing.assert_array_equal(out["end_assigns"], IMP[pre + "end"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(IMP["cases"]))
def test_improve_population_golden(name):
    """The package's improve_population: every LsResult field equals the
    reference's (best / end colourings, scores, iterations, legality, the
    WVCP phi trajectory; start is the input colouring)."""
    mode, g, A, seed, k, pop, gen, depth, rounds = _case(name)
    cols = [Coloring(A[i].copy(), k) for i in range(pop)]
    kw = {"depth": depth or None}
    if mode == "wvcp":
        kw["max_rounds"] = rounds
    res = LS.improve_population(g, cols, LS.WVCP if mode == "wvcp" else LS.COL, seed, gen, **kw)
    pre = f"{name}__"
    assert len(res) == pop
    for i, r in enumerate(res):
        assert r.start == cols[i]
        np.testing.assert_array_equal(r.best.assign, IMP[pre + "best"][i], err_msg=f"{name} best {i}")
        np.testing.assert_array_equal(r.end.assign, IMP[pre + "end"][i], err_msg=f"{name} end {i}")
        assert r.best_score == int(IMP[pre + "best_score"][i])
        assert r.iterations_used == int(IMP[pre + "iterations_used"][i])
        assert r.legal_found == bool(IMP[pre + "legal_found"][i])
        if mode == "wvcp":
            np.testing.assert_array_equal(np.array(r.phi_trajectory, np.float64), IMP[pre + "phi"][i])
