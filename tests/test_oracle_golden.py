"""Pin the CPU oracle (oracle/rcp_oracle.py) to the reference's own outputs.

The fixtures in tests/golden/ were produced by running the reference package
(tests/golden/make_golden.py).  Same numpy/OpenBLAS in this image, so the
restatement must reproduce them bit for bit.
"""

import numpy as np
import pytest

from conftest import golden_names, load_golden
from oracle.rcp_oracle import OracleConfig, oracle_factor, oracle_solve


@pytest.mark.parametrize("name", golden_names())
def test_oracle_matches_reference_fixture(name):
    g = load_golden(name)
    cfg = dict(g["cfg"])
    res = oracle_factor(g["a"], OracleConfig(**cfg))
    assert np.array_equal(res.perm, g["perm"])
    assert np.array_equal(res.pattern, g["pattern"])
    assert np.array_equal(res.d_diag, g["d_diag"])
    assert np.array_equal(res.d_off, g["d_off"])
    if "L" in g:
        assert np.array_equal(res.L, g["L"])
    assert np.array_equal(res.L.sum(axis=1), g["L_rowsum"])
    assert res.rho_cheap == float(g["rho_cheap"])
    assert res.max_multiplier == float(g["max_multiplier"])
    assert res.recompute_count == int(g["recompute_count"])
    c = res.counters
    assert [c.mults, c.adds, c.divs, c.comps] == list(g["counters"])
    from paper_1710_00125_b200 import gallery
    x, sing = oracle_solve(res, gallery.rhs(g["a"].shape[0], 1))
    assert np.array_equal(x, g["x"])
    assert sing == bool(g["singular"])
