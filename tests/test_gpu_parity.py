"""GPU parity: the CUDA path (through the C ABI) against the reference fixtures and the oracle.

Bar (BASELINE.json north_star): identical pivot sequence and 1x1/2x2 structure,
L and D within the stated tolerance ``conftest.l_tol(n)`` (10x the CPU rounding
noise floor), solve x within a conditioning-scaled tolerance, backward error and
growth within small factors of the reference.
"""

import numpy as np
import pytest

from conftest import golden_names, l_tol, load_golden

pytestmark = pytest.mark.gpu

ALL_CASES = golden_names()


def _gpu_factor(a, cfg, robust=False, trace=False):
    import torch

    from paper_1710_00125_b200 import api
    c = api.FactorConfig(**cfg)
    if robust and c.robust_r < 1:
        raise ValueError
    ad = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    df = api.factor_device(ad, c, trace=trace)
    torch.cuda.synchronize()
    return df


def _assert_factor_parity(g, f, n):
    assert np.array_equal(f.perm, g["perm"]), "pivot sequence differs"
    assert np.array_equal(f.pattern, g["pattern"]), "block structure differs"
    tol = l_tol(n)
    dd = np.concatenate([g["d_diag"], g["d_off"]])
    dscale = max(1.0, float(np.abs(dd).max()))
    got = np.concatenate([f.d_diag, f.d_off])
    assert np.abs(got - dd).max() <= tol * dscale
    # L relative to max|L| like D to max|D|: bkpp's multipliers are unbounded (1.7e11 on the scaled
    # C5 member), and perturbing the input by 1 ulp moves the reference's own L by ~1e-3 there
    lscale = max(1.0, float(np.abs(g["L_rowsum"]).max()) / n, float(np.abs(g["L"]).max()) if "L" in g else 1.0)
    if "L" in g:
        assert np.abs(f.L - g["L"]).max() <= tol * lscale
    assert np.abs(f.L.sum(axis=1) - g["L_rowsum"]).max() <= tol * n * lscale


@pytest.mark.parametrize("name", ALL_CASES)
def test_factor_matches_reference_fixture(cuda_ok, name):
    from paper_1710_00125_b200 import api
    g = load_golden(name)
    a = g["a"]
    n = a.shape[0]
    df = _gpu_factor(a, g["cfg"])
    hf = df.to_host()

    class F:  # flat view for the comparison helper
        perm = hf.perm
        pattern = hf.pattern
        L = hf.L
        d_diag = df.d_diag.cpu().numpy()
        d_off = df.d_off.cpu().numpy()

    _assert_factor_parity(g, F, n)
    assert hf.stats.recompute_count == int(g["recompute_count"])
    c = hf.stats.counters  # exact OpCounters parity (metrics.py:28-43)
    assert [c.mults, c.adds, c.divs, c.comps] == [int(x) for x in g["counters"]]
    rho_ref = float(g["rho_cheap"])
    assert abs(hf.stats.rho_cheap - rho_ref) <= l_tol(n) * max(1.0, rho_ref)
    mm_ref = float(g["max_multiplier"])
    assert abs(hf.stats.max_multiplier - mm_ref) <= l_tol(n) * 10 * max(1.0, mm_ref)
    # the reference's reconstruction criterion (test_factor.py:59-67), or within 100x of the
    # reference's own error where its multipliers are huge (bkpp on the scaled C5 member)
    perm = hf.perm
    den = float(np.abs(a).max()) or 1.0
    rec_tol = 1e-12
    if "L" in g:
        dref = np.zeros((n, n))
        np.fill_diagonal(dref, g["d_diag"])
        iu = np.arange(n - 1)
        dref[iu + 1, iu] = dref[iu, iu + 1] = g["d_off"][:-1]
        rref = g["L"] @ dref @ g["L"].T
        rec_tol = max(rec_tol, 100 * float(np.abs(rref - a[np.ix_(g["perm"], g["perm"])]).max()) / den)
    rec = hf.L @ hf.D.to_dense() @ hf.L.T
    assert float(np.abs(rec - a[np.ix_(perm, perm)]).max()) / den <= rec_tol
    # solve parity (solve.py:79-92)
    from paper_1710_00125_b200 import gallery
    rep = api.solve(hf, gallery.rhs(n, 1), a)
    assert rep.singular == bool(g["singular"])
    if not rep.singular:
        xr = g["x"]
        if mm_ref < 1e6:  # x itself is only comparable when the factors are well conditioned
            assert np.abs(rep.x - xr).max() <= 1e-8 * max(1.0, np.abs(xr).max())
        assert rep.backward_error <= max(1e-13, 100 * float(g["backward_error"]))


def test_trace_is_consistent_with_pattern(cuda_ok):
    g = load_golden("g_n300_b32")
    df = _gpu_factor(g["a"], g["cfg"], trace=True)
    kinds = df.trace_kind.cpu().numpy()
    pat = df.pattern.cpu().numpy()
    two = np.nonzero(kinds == 3)[0]
    assert np.all(pat[two] == 1) and np.all(pat[two + 1] == 2)
    assert df.stats["n_2x2"] == int((pat == 1).sum())


@pytest.mark.parametrize("n,b,p,seed", [(64, 8, 10, 0), (257, 16, 26, 1), (512, 32, 42, 2), (640, 64, 74, 3)])
def test_factor_matches_oracle_live(cuda_ok, n, b, p, seed):
    from oracle.rcp_oracle import OracleConfig, oracle_factor
    from paper_1710_00125_b200 import gallery
    a = gallery.type6(n, 1000 + seed)
    o = oracle_factor(a, OracleConfig(b=b, q=b, p=p, seed=seed))
    df = _gpu_factor(a, dict(strategy="rcp", b=b, q=b, p=p, seed=seed))
    hf = df.to_host()
    assert np.array_equal(hf.perm, o.perm)
    assert np.array_equal(hf.pattern, o.pattern)
    c, oc = hf.stats.counters, o.counters
    assert [c.mults, c.adds, c.divs, c.comps] == [oc.mults, oc.adds, oc.divs, oc.comps]
    assert np.abs(hf.L - o.L).max() <= l_tol(n)
    dref = o.d_dense()
    assert np.abs(hf.D.to_dense() - dref).max() <= l_tol(n) * max(1.0, np.abs(dref).max())


def test_input_validation_errors(cuda_ok):
    from paper_1710_00125_b200 import api
    with pytest.raises(ValueError, match="symmetric"):
        api.factor(np.array([[1.0, 2.0], [3.0, 4.0]]), strategy="rcp", b=2, q=2, p=2)
    with pytest.raises(ValueError):
        api.factor(np.array([[np.nan, 0.0], [0.0, 1.0]]), strategy="rcp", b=2, q=2, p=2)
    with pytest.raises(ValueError, match="NaN or Inf"):
        api.factor(np.array([[np.inf, 0.0], [0.0, 1.0]]), strategy="rcp", b=2, q=2, p=2)


def test_input_is_not_modified(cuda_ok):
    import torch

    from paper_1710_00125_b200 import api, gallery
    a = gallery.type6(130, 7)
    ad = torch.from_numpy(a).cuda()
    before = ad.clone()
    api.factor_device(ad, api.FactorConfig(b=16, q=16, p=20, seed=1))
    torch.cuda.synchronize()
    assert torch.equal(ad, before)


def test_solve_many_matches_columnwise(cuda_ok):
    from paper_1710_00125_b200 import api, gallery
    a = gallery.type6(200, 11)
    f = api.factor(a, strategy="rcp", b=16, q=16, p=20, seed=4)
    rhs = np.random.Generator(np.random.Philox(3)).standard_normal((200, 3))
    xm = api.solve_many(f, rhs)
    for j in range(3):
        xj = api.solve(f, rhs[:, j]).x
        assert np.allclose(xm[:, j], xj, rtol=1e-12, atol=1e-12)
    assert np.allclose(a @ xm, rhs, atol=1e-9)


def test_deficient_solve_flags_singular(cuda_ok):
    from paper_1710_00125_b200 import api
    g = load_golden("g_zero_tail")
    f = api.factor_robust(g["a"], api.FactorConfig(**{k: v for k, v in g["cfg"].items()}))
    first = int(np.nonzero(g["pattern"] == api.PAT_DEFICIENT)[0][0])   # reference: panel-aligned
    assert 40 <= first and f.deficient_from == first
    assert np.all(f.pattern[first:] == api.PAT_DEFICIENT)
    rep = api.solve(f, g["a"] @ np.ones(65), g["a"])
    assert rep.singular
    assert rep.backward_error <= 1e-12


@pytest.mark.parametrize("n,b,p,seed", [(96, 64, 5, 0), (200, 16, 8, 3), (333, 32, 5, 1), (130, 1, 5, 2)])
def test_q1_mode_matches_oracle_live(cuda_ok, n, b, p, seed):
    """q = 1 (per-step sketch pivoting, the reference's default FactorConfig mode)."""
    from oracle.rcp_oracle import OracleConfig, oracle_factor
    from paper_1710_00125_b200 import gallery
    a = gallery.type6(n, 2000 + seed)
    o = oracle_factor(a, OracleConfig(b=b, q=1, p=p, seed=seed))
    df = _gpu_factor(a, dict(strategy="rcp", b=b, q=1, p=p, seed=seed))
    hf = df.to_host()
    assert np.array_equal(hf.perm, o.perm)
    assert np.array_equal(hf.pattern, o.pattern)
    c, oc = hf.stats.counters, o.counters
    assert [c.mults, c.adds, c.divs, c.comps] == [oc.mults, oc.adds, oc.divs, oc.comps]
    assert np.abs(hf.L - o.L).max() <= l_tol(n)
    dref = o.d_dense()
    assert np.abs(hf.D.to_dense() - dref).max() <= l_tol(n) * max(1.0, np.abs(dref).max())


def test_default_config_is_supported(cuda_ok):
    """factor(a) with the reference's default FactorConfig (rcp, p=5, b=64, q=1)."""
    from oracle.rcp_oracle import OracleConfig, oracle_factor
    from paper_1710_00125_b200 import api, gallery
    a = gallery.type6(150, 77)
    f = api.factor(a)
    o = oracle_factor(a, OracleConfig())
    assert np.array_equal(f.perm, o.perm)
    assert np.abs(f.L - o.L).max() <= l_tol(150)


def test_q1_guard_detects_zero_tail(cuda_ok):
    """Reference test_factor.py:157-166 in the reference's own configuration (b=64, q=1, p=6)."""
    from oracle.rcp_oracle import OracleConfig, oracle_factor
    from paper_1710_00125_b200 import api, gallery
    a = np.zeros((65, 65))
    a[:40, :40] = gallery.type6(40, 5)
    f = api.factor_robust(a, strategy="rcp", p=6, seed=2)
    o = oracle_factor(a, OracleConfig(p=6, seed=2))
    assert f.deficient_from == 40
    assert np.all(f.pattern[40:] == api.PAT_DEFICIENT)
    assert f.stats.recompute_count == o.recompute_count == 1
    assert np.array_equal(f.perm, o.perm)
    assert np.array_equal(f.pattern, o.pattern)
    den = float(np.abs(a).max())
    rec = f.L @ f.D.to_dense() @ f.L.T
    assert float(np.abs(rec - a[np.ix_(f.perm, f.perm)]).max()) / den <= 1e-12


def test_large_panel_grid_reconstructs(cuda_ok):
    """n > 32 x #SMs: the panel CTA count G(m0) is capped by the SM count and is not monotone
    in m0 (regression: the launch grid must cover the largest G of every panel)."""
    import torch

    from paper_1710_00125_b200 import api, gallery
    n = 6144
    a = torch.from_numpy(gallery.type6(n, 3)).cuda()
    f = api.factor_device(a, api.FactorConfig(strategy="rcp", b=64, q=64, p=80, seed=1))
    rec = api.reconstruct_device(f)
    perm = f.perm
    err = float((rec - a[perm][:, perm]).abs().max()) / float(a.abs().max())
    assert err <= 1e-11
    x, sing = api.solve_device(f, torch.ones(n, dtype=torch.float64, device="cuda"))
    assert not sing
    r = float((a @ x - 1.0).abs().max()) / (float(a.abs().sum(dim=1).max()) * float(x.abs().max()))
    assert r <= 1e-13


@pytest.mark.parametrize("n", [2048, 3001])
def test_lower_to_host_is_exact(cuda_ok, n):
    """to_host(): only L's lower trapezoid crosses PCIe, the host writes the upper zeros; the
    result equals the device L exactly (including a ragged last block row)."""
    import torch

    from paper_1710_00125_b200 import api
    g = torch.Generator(device="cuda").manual_seed(n)
    lt = torch.tril(torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g), -1)
    lt += torch.eye(n, dtype=torch.float64, device="cuda")
    dev = api.DeviceFactorization(perm=torch.arange(n, device="cuda"), L=lt,
                                  d_diag=torch.ones(n, dtype=torch.float64, device="cuda"),
                                  d_off=torch.zeros(n, dtype=torch.float64, device="cuda"),
                                  pattern=torch.zeros(n, dtype=torch.int8, device="cuda"),
                                  stats={"rho_cheap": 1.0, "max_multiplier": 1.0, "counters": (0, 0, 0, 0),
                                         "recompute_count": 0})
    # poison a pinned block of the same size so stale host contents would show
    junk = torch.full((n, n), float("nan"), dtype=torch.float64, pin_memory=True)
    del junk
    f = dev.to_host()
    assert np.array_equal(f.L, lt.cpu().numpy())


@pytest.mark.parametrize("n,rank,robust,kw", [(2500, 2500, False, {}), (2300, 1500, True, {}),
                                              (2200, 2200, False, {"q": 1, "p": 12}),
                                              (2100, 2100, False, {"strategy": "bkpp", "q": 1, "p": 5}),
                                              (2049, 2049, False, {"strategy": "bbk", "q": 1, "p": 5})])
def test_streamed_host_l_matches_device(cuda_ok, n, rank, robust, kw):
    """factor(numpy) at n >= 2048 streams L into pinned memory while later panels run
    (rcp_factor_host_l): bit-identical to the device L, incl. a ragged last block row and the
    rows of a deficient tail (guarded, rank-deficient input)."""
    import torch

    from paper_1710_00125_b200 import api, gallery
    a = np.zeros((n, n))
    a[:rank, :rank] = gallery.type6(rank, 7)
    cfg = api.FactorConfig(**{"strategy": "rcp", "b": 64, "q": 64, "p": 80, "seed": 3,
                              "robust_r": 1 if robust else 0, **kw})
    f = api.factor(a, cfg)
    d = api.factor_device(torch.from_numpy(a).cuda(), cfg)
    assert np.array_equal(f.perm, d.perm.cpu().numpy())
    assert np.array_equal(f.L, d.L.cpu().numpy())
    assert np.array_equal(np.triu(f.L, 1), np.zeros((n, n)))
    assert np.all(np.diag(f.L) == 1.0)
    if robust:
        assert f.deficient_from is not None and 0 < f.deficient_from < n
    rec = f.L @ f.D.to_dense() @ f.L.T
    assert float(np.abs(rec - a[np.ix_(f.perm, f.perm)]).max()) / float(np.abs(a).max()) <= 1e-11


def test_host_input_symmetry_and_finiteness_large(cuda_ok):
    """factor(numpy) at n >= 2048: only the lower triangle goes to the device, so exact symmetry
    is checked on the host (core.py:48-53) and reported before anything else; NaN anywhere
    (also on the diagonal) fails it, Inf in a symmetric matrix is "NaN or Inf"."""
    from paper_1710_00125_b200 import api, gallery
    n = 2100
    a = gallery.type6(n, 11)
    for (i, j) in [(5, 2000), (2099, 0), (1000, 1001)]:  # one upper entry off by one ulp
        b = a.copy()
        b[min(i, j), max(i, j)] = np.nextafter(b[min(i, j), max(i, j)], np.inf)
        with pytest.raises(ValueError, match="symmetric"):
            api.factor(b, strategy="rcp", b=64, q=64, p=80)
    b = a.copy()
    b[17, 17] = np.nan
    with pytest.raises(ValueError, match="symmetric"):
        api.factor(b, strategy="rcp", b=64, q=64, p=80)
    b = a.copy()
    b[3, 1500] = b[1500, 3] = np.inf
    with pytest.raises(ValueError, match="NaN or Inf"):
        api.factor(b, strategy="rcp", b=64, q=64, p=80)


def test_supplied_omega_with_guard_recompute(cuda_ok):
    """Omega passed in (its draw is skipped lazily): a guard recompute must still continue the
    same normal stream (g_c5_scaled recomputes once)."""
    import torch

    from paper_1710_00125_b200 import api
    g = load_golden("g_c5_scaled")
    cfg = api.FactorConfig(**g["cfg"])
    n = g["a"].shape[0]
    om = np.random.Generator(np.random.Philox(cfg.seed)).standard_normal((cfg.p, n))
    a = torch.from_numpy(g["a"]).cuda()
    f = api.factor_device(a, cfg, omega=torch.from_numpy(om).cuda())
    assert f.stats["recompute_count"] == int(g["recompute_count"]) == 1
    assert np.array_equal(f.perm.cpu().numpy(), g["perm"])


@pytest.mark.parametrize("strategy", ["bkpp", "bbk"])
@pytest.mark.parametrize("n,b,seed,kind", [(512, 32, 0, "type6"), (1000, 64, 1, "type6"), (600, 16, 2, "kkt"),
                                           (257, 128, 3, "type6"), (300, 8, 4, "scaled")])
def test_bk_strategies_match_oracle_live(cuda_ok, strategy, n, b, seed, kind):
    """Bunch-Kaufman partial pivoting (pivot.py:146-171) and the rook search (pivot.py:189-218) on
    the same panel engine: same pivot sequence, block structure and op counters as the oracle
    (itself bit-exact vs the reference)."""
    from oracle.rcp_oracle import OracleConfig, oracle_factor
    from paper_1710_00125_b200 import gallery
    if kind == "type6":
        a = gallery.type6(n, 2000 + seed)
    elif kind == "kkt":
        a = gallery.kkt((4 * n) // 5, n - (4 * n) // 5, seed)
    else:
        a = gallery.scaled_member(n, seed, True)
    o = oracle_factor(a, OracleConfig(strategy=strategy, b=b, q=1, p=5, seed=seed))
    df = _gpu_factor(a, dict(strategy=strategy, b=b, q=1, p=5, seed=seed))
    hf = df.to_host()
    assert np.array_equal(hf.perm, o.perm)
    assert np.array_equal(hf.pattern, o.pattern)
    c, oc = hf.stats.counters, o.counters
    assert [c.mults, c.adds, c.divs, c.comps] == [oc.mults, oc.adds, oc.divs, oc.comps]
    assert np.abs(hf.L - o.L).max() <= l_tol(n) * max(1.0, np.abs(o.L).max())
    dref = o.d_dense()
    assert np.abs(hf.D.to_dense() - dref).max() <= l_tol(n) * max(1.0, np.abs(dref).max())
    assert hf.stats.recompute_count == 0
