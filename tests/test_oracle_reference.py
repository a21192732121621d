"""Live cross-check of the oracle against the reference (build container only)."""

import sys
from pathlib import Path

import numpy as np
import pytest

REF = Path("/root/reference/pkg/src")
pytestmark = pytest.mark.skipif(not REF.exists(), reason="reference not mounted (GPU box)")


@pytest.fixture(scope="module")
def randldl():
    sys.path.insert(0, str(REF))
    import randldl as r
    return r


@pytest.mark.parametrize("n,b,p,seed", [(97, 8, 12, 0), (128, 16, 24, 5), (211, 32, 42, 9), (150, 4, 4, 2)])
def test_oracle_equals_reference(randldl, n, b, p, seed):
    from oracle.rcp_oracle import OracleConfig, oracle_factor
    from paper_1710_00125_b200 import gallery
    a = gallery.type6(n, seed + 100)
    f = randldl.factor(a, randldl.FactorConfig(strategy="rcp", b=b, q=b, p=p, seed=seed))
    o = oracle_factor(a, OracleConfig(b=b, q=b, p=p, seed=seed))
    assert np.array_equal(f.perm, o.perm)
    assert np.array_equal(f.L, o.L)
    assert np.array_equal(f.D.to_dense(), o.d_dense())
