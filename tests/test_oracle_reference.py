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


@pytest.mark.parametrize("strategy", ["bkpp", "bbk"])
@pytest.mark.parametrize("n,b,seed,kind", [(97, 8, 0, "type6"), (130, 16, 3, "type6"), (64, 1, 1, "type6"),
                                           (120, 32, 7, "kkt"), (90, 64, 2, "scaled")])
def test_oracle_bk_strategies_equal_reference(randldl, strategy, n, b, seed, kind):
    """The bkpp / bbk restatement (pivot.py:146-225 on factor.py's engine) is bit-identical."""
    from oracle.rcp_oracle import OracleConfig, oracle_factor
    from paper_1710_00125_b200 import gallery
    a = _bk_matrix(gallery, kind, n, seed)
    f = randldl.factor(a, randldl.FactorConfig(strategy=strategy, b=b, q=1, p=5, seed=seed))
    o = oracle_factor(a, OracleConfig(strategy=strategy, b=b, q=1, p=5, seed=seed))
    assert np.array_equal(f.perm, o.perm)
    assert np.array_equal(f.pattern, o.pattern)
    assert np.array_equal(f.L, o.L)
    assert np.array_equal(f.D.to_dense(), o.d_dense())
    c = f.stats.counters
    assert (c.mults, c.adds, c.divs, c.comps) == (o.counters.mults, o.counters.adds, o.counters.divs,
                                                  o.counters.comps)


def _bk_matrix(gallery, kind, n, seed):
    if kind == "type6":
        return gallery.type6(n, seed + 300)
    rng = np.random.default_rng(seed)
    if kind == "kkt":
        n1 = (4 * n) // 5
        g = rng.standard_normal((n1, n1))
        h = g.T @ g / n1 + np.eye(n1)
        h = np.tril(h) + np.tril(h, -1).T
        bm = rng.standard_normal((n - n1, n1))
        a = np.zeros((n, n))
        a[:n1, :n1] = h
        a[n1:, :n1] = bm
        a[:n1, n1:] = bm.T
        return a
    a = gallery.type6(n, seed + 500)
    d = 10.0 ** rng.uniform(-6, 6, n)
    a = (a * d[:, None]) * d[None, :]
    return np.tril(a) + np.tril(a, -1).T
