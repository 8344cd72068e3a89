"""The CPU restatement of update_population / match_parents (oracle/)
against the reference's own outputs (tests/golden/population.npz, made by
tests/golden/make_golden.py from mc/population.py:59-141)."""

import numpy as np
import pytest

from conftest import load_golden
from oracle import population_oracle as PO

POP = load_golden("population")


@pytest.mark.parametrize("name", [str(c) for c in POP["cases"]])
def test_oracle_matches_reference_fixtures(name):
    pre = name + "__"
    seed, n, k, p, q, ms, K = (int(x) for x in POP[pre + "params"])
    adm, rule, nd, na, nf = PO.update_population(
        POP[pre + "pop_dist"], POP[pre + "pop_fit"], POP[pre + "pop_assigns"], POP[pre + "new_assigns"],
        POP[pre + "new_fit"], POP[pre + "cross"], POP[pre + "within"], ms)
    np.testing.assert_array_equal(na, POP[pre + "res_assigns"])
    np.testing.assert_array_equal(nf, POP[pre + "res_fit"])
    np.testing.assert_array_equal(nd, POP[pre + "res_dist"])
    np.testing.assert_array_equal(rule, POP[pre + "res_rule"].astype(bool))
    np.testing.assert_array_equal(PO.match_parents(nd, K), POP[pre + "matches"])


def test_fixtures_cover_the_fill_path():
    fills = [int((POP[str(c) + "__res_rule"] == 0).sum()) for c in POP["cases"]]
    assert max(fills) > 0 and min(fills) == 0
