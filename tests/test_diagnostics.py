"""Experiment diagnostics: FactorConfig.track_growth="full" and
audit_sketch on the GPU against fixtures made by the reference itself
(tests/golden/make_golden.py --diag).

The reference forces width-1 panels for both (factor.py:294-296), takes a snapshot
(max|S|, largest column norm of S) of every active Schur complement at each step start
(factor.py:493-495, 605-606), records the sketch drift ||B - Omega S||_{1,2} / ||A||_{1,2}
after every panel (factor.py:497-504, 566-567) and derives rho_elem, rho_col, ||L||_1 and
||L^-1||_1 (factor.py:528-531, metrics.py:93-127).  Snapshots are functions of the computed
Schur complements, so they agree to rounding; the drift is itself a rounding-error measure
(~1e-14), so it is checked for count and size, not value."""

import json
from pathlib import Path

import numpy as np
import pytest

DIAG = Path(__file__).resolve().parent / "golden" / "diag"
NAMES = sorted(p.stem for p in DIAG.glob("d_*.npz"))


def _load(name):
    z = np.load(DIAG / f"{name}.npz", allow_pickle=False)
    d = {k: z[k] for k in z.files}
    d["cfg"] = json.loads(str(d["cfg"]))
    return d


def test_fixtures_present():
    assert len(NAMES) >= 6


def test_config_forces_eager_panels():
    from paper_1710_00125_b200 import api
    cfg = api.FactorConfig(strategy="rcp", b=16, q=16, p=24, track_growth="full")
    c = api._native_config(cfg)
    assert (c.b, c.q, c.p) == (1, 1, 24)
    cfg = api.FactorConfig(strategy="rcp", b=16, q=16, p=24, audit_sketch=True)
    assert (api._native_config(cfg).b, api._native_config(cfg).q) == (1, 1)
    cfg = api.FactorConfig(strategy="rcp", b=16, q=16, p=24)
    assert (api._native_config(cfg).b, api._native_config(cfg).q) == (16, 16)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_diagnostics_match_reference(cuda_ok, name):
    from paper_1710_00125_b200 import api
    g = _load(name)
    cfg = api.FactorConfig(**g["cfg"])
    fn = api.factor_robust if bool(g["robust"]) else api.factor
    f = fn(g["a"], cfg)
    assert np.array_equal(f.perm, g["perm"])
    assert np.array_equal(f.pattern, g["pattern"])
    assert tuple(int(x) for x in (f.stats.counters.mults, f.stats.counters.adds, f.stats.counters.divs,
                                  f.stats.counters.comps)) == tuple(int(x) for x in g["counters"])
    assert f.stats.recompute_count == int(g["recompute_count"])
    s = f.stats
    if bool(g["has_snapshots"]):
        snaps = np.array(s.snapshots, dtype=np.float64).reshape(-1, 2)
        assert snaps.shape == g["snapshots"].shape
        ref = g["snapshots"]
        assert np.allclose(snaps, ref, rtol=1e-11, atol=1e-13 * max(1.0, float(np.abs(ref).max()))), \
            float(np.abs(snaps - ref).max())
        for key in ("rho_elem", "rho_col", "L_norm1"):
            assert abs(getattr(s, key) - float(g[key])) <= 1e-11 * abs(float(g[key])), key
        assert abs(s.Linv_norm1 - float(g["Linv_norm1"])) <= 1e-9 * abs(float(g["Linv_norm1"]))
    else:
        assert s.snapshots is None and s.rho_elem is None
    if bool(g["has_drift"]):
        drift = np.array(s.sketch_drift, dtype=np.float64)
        assert drift.shape == g["drift"].shape
        assert np.isfinite(drift).all() and (drift >= 0).all()
        assert drift.max(initial=0.0) <= 1e-12, drift.max()
    else:
        assert s.sketch_drift is None
