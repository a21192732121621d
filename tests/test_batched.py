"""Batched C5 path (rcp_factor_batched / rcp_solve_batched) against the reference fixtures
and the oracle: every matrix of a batch must equal a separate ``factor`` call."""

import numpy as np
import pytest

from conftest import l_tol, load_golden

pytestmark = pytest.mark.gpu

C5 = dict(strategy="rcp", b=16, q=16, p=24, seed=0)


def _stack(mats):
    import torch
    return torch.from_numpy(np.ascontiguousarray(np.stack(mats))).cuda()


def _check_against(f, o, n):
    assert np.array_equal(f.perm, o.perm), "pivot sequence differs"
    assert np.array_equal(f.pattern, o.pattern), "block structure differs"
    assert np.abs(f.L - o.L).max() <= l_tol(n)
    dref = o.d_dense()
    assert np.abs(f.D.to_dense() - dref).max() <= l_tol(n) * max(1.0, np.abs(dref).max())
    c, oc = f.stats.counters, o.counters
    assert [c.mults, c.adds, c.divs, c.comps] == [oc.mults, oc.adds, oc.divs, oc.comps]
    assert f.stats.recompute_count == o.recompute_count


def test_batched_matches_reference_fixtures(cuda_ok):
    """The two C5 members stored from the reference itself (plain + scaled/guard trip)."""
    from paper_1710_00125_b200 import FactorConfig, batched
    gs = [load_golden("g_c5_plain"), load_golden("g_c5_scaled")]
    cfg = FactorConfig(**gs[0]["cfg"])
    bf = batched.factor_batched_device(_stack([g["a"] for g in gs]), cfg)
    fs = bf.to_host()
    for j, (f, g) in enumerate(zip(fs, gs)):
        n = g["a"].shape[0]
        assert np.array_equal(f.perm, g["perm"])
        assert np.array_equal(f.pattern, g["pattern"])
        assert np.abs(f.L - g["L"]).max() <= l_tol(n)
        dd = np.concatenate([g["d_diag"], g["d_off"]])
        got = np.concatenate([bf.d_diag[j].cpu().numpy(), bf.d_off[j].cpu().numpy()])
        assert np.abs(got - dd).max() <= l_tol(n) * max(1.0, np.abs(dd).max())
        assert f.stats.recompute_count == int(g["recompute_count"])
        c = f.stats.counters
        assert [c.mults, c.adds, c.divs, c.comps] == [int(x) for x in g["counters"]]
        assert abs(f.stats.rho_cheap - float(g["rho_cheap"])) <= l_tol(n) * max(1.0, float(g["rho_cheap"]))
        assert abs(f.stats.max_multiplier - float(g["max_multiplier"])) <= 10 * l_tol(n)


@pytest.mark.parametrize("n,b,p,seeds", [(256, 16, 24, range(0, 10)), (96, 8, 12, range(20, 26)),
                                         (61, 16, 24, range(30, 33)), (200, 32, 40, range(40, 43))])
def test_batched_matches_oracle(cuda_ok, n, b, p, seeds):
    from oracle.rcp_oracle import OracleConfig, oracle_factor
    from paper_1710_00125_b200 import FactorConfig, batched, gallery
    mats = [gallery.scaled_member(n, s, scaled=(s % 3 == 0)) for s in seeds]
    cfg = FactorConfig(strategy="rcp", b=b, q=b, p=p, seed=7)
    fs = batched.factor_batched_device(_stack(mats), cfg).to_host()
    for a, f in zip(mats, fs):
        o = oracle_factor(a, OracleConfig(b=b, q=b, p=p, seed=7))
        _check_against(f, o, n)


def test_batched_solve_matches_oracle(cuda_ok):
    from oracle.rcp_oracle import OracleConfig, oracle_factor, oracle_solve
    from paper_1710_00125_b200 import FactorConfig, batched, gallery
    n = 256
    mats = [gallery.scaled_member(n, s, scaled=(s == 2)) for s in range(4)]
    rhs = np.stack([gallery.rhs(n, 100 + s) for s in range(4)])
    import torch
    bf = batched.factor_batched_device(_stack(mats), FactorConfig(**C5))
    x, sing = batched.solve_batched_device(bf, torch.from_numpy(rhs).cuda())
    x = x.cpu().numpy()
    assert not sing.any().item()
    for i, a in enumerate(mats):
        o = oracle_factor(a, OracleConfig(b=16, q=16, p=24, seed=0))
        xo, so = oracle_solve(o, rhs[i])
        assert not so
        assert np.abs(x[i] - xo).max() <= 1e-8 * max(1.0, np.abs(xo).max())
        r = np.abs(a @ x[i] - rhs[i]).max() / (np.abs(a).sum(axis=1).max() * np.abs(x[i]).max())
        assert r <= 1e-13


def test_batched_errors_and_deficient(cuda_ok):
    from paper_1710_00125_b200 import FactorConfig, _native, batched, gallery
    good = gallery.scaled_member(64, 1, False)
    asym = good.copy()
    asym[3, 5] += 1.0
    nonfin = good.copy()
    nonfin[2, 2] = np.inf
    zero = np.zeros((64, 64))
    bf = batched.factor_batched_device(_stack([good, asym, nonfin, zero]),
                                       FactorConfig(strategy="rcp", b=8, q=8, p=12, seed=0), check=False)
    st = bf.stats["status"]
    assert list(st) == [_native.RCP_OK, _native.RCP_ERR_NOT_SYMMETRIC, _native.RCP_ERR_NONFINITE_INPUT,
                        _native.RCP_OK]
    fz = bf.factorization(3)
    assert (fz.pattern == 3).all() and fz.deficient_from == 0
    with pytest.raises(ValueError, match="matrix 1: A must be symmetric"):
        batched.factor_batched_device(_stack([good, asym]), FactorConfig(strategy="rcp", b=8, q=8, p=12, seed=0))


def test_batched_host_api_roundtrip(cuda_ok):
    from paper_1710_00125_b200 import FactorConfig, batched, factor, gallery, solve_batched
    mats = np.stack([gallery.scaled_member(128, s, scaled=False) for s in range(3)])
    cfg = FactorConfig(strategy="rcp", b=16, q=16, p=24, seed=3)
    fs = batched.factor_batched(mats, cfg)
    for a, f in zip(mats, fs):
        g = factor(a, cfg)  # the single-matrix GPU path
        assert np.array_equal(f.perm, g.perm)
        assert np.abs(f.L - g.L).max() <= l_tol(128)
    rhs = np.stack([gallery.rhs(128, s) for s in range(3)])
    x = solve_batched(fs, rhs)
    for i, a in enumerate(mats):
        assert np.abs(a @ x[i] - rhs[i]).max() <= 1e-10 * np.abs(rhs[i]).max() * np.abs(a).max() * 128


def test_batched_host_pipeline_equals_device(cuda_ok):
    """factor_batched_host (chunked upload / factor / download on three streams) returns the same
    bits as factor_batched_device on the resident stack: ragged last chunk, both slots reused,
    scaled members (guard recompute) and a failing matrix keep their per-matrix status."""
    import torch
    from paper_1710_00125_b200 import FactorConfig, _native, batched, gallery
    cfg = FactorConfig(**C5)
    a = gallery.c5_batch_device(301, 256, seed=7)
    a[150, 3, 5] += 1.0  # asymmetric member
    dev = batched.factor_batched_device(a, cfg, check=False)
    host = batched.factor_batched_host(a.cpu().pin_memory(), cfg, chunk=64, check=False)
    assert not host.L.is_cuda and host.L.is_pinned()
    assert np.array_equal(host.stats["status"], dev.stats["status"])
    ok = dev.stats["status"] == _native.RCP_OK
    assert ok.sum() == 300  # outputs of the failed member are unspecified
    okt = torch.from_numpy(ok)
    for name in ("perm", "L", "d_diag", "d_off", "pattern"):
        h, d = getattr(host, name)[okt], getattr(dev, name).cpu()[okt]
        bad = (h != d).reshape(len(h), -1).any(dim=1).nonzero().flatten().tolist()
        assert not bad, f"{name} differs in {len(bad)} matrices, first {bad[:5]}"
    for name in ("recompute_count", "n_2x2", "n_steps", "rho_cheap", "max_multiplier", "mults", "comps"):
        assert np.array_equal(host.stats[name][ok], dev.stats[name][ok]), name
    assert host.stats["status"][150] == _native.RCP_ERR_NOT_SYMMETRIC
    assert (host.stats["recompute_count"] > 0).sum() >= 25
    with pytest.raises(ValueError, match="matrix 150"):
        batched.factor_batched_host(a.cpu(), cfg, chunk=100)


def test_sharded_over_devices_equals_one_device(cuda_ok):
    """factor_batched_sharded: shards by matrix over the given devices (here the one GPU listed
    three times, so three host threads drive three shards concurrently) and merges the results;
    every matrix equals the single-device batched result bit for bit."""
    import torch
    from paper_1710_00125_b200 import FactorConfig, batched, gallery
    mats = [gallery.scaled_member(128, s, scaled=(s % 4 == 0)) for s in range(37)]
    a = torch.from_numpy(np.ascontiguousarray(np.stack(mats))).pin_memory()
    cfg = FactorConfig(strategy="rcp", b=16, q=16, p=24, seed=3)
    one = batched.factor_batched_host(a, cfg, chunk=8)
    sh = batched.factor_batched_sharded(a, cfg, devices=[0, 0, 0], chunk=5)
    for name in ("perm", "L", "d_diag", "d_off", "pattern"):
        assert torch.equal(getattr(one, name), getattr(sh, name)), name
    assert np.array_equal(one.stats, sh.stats)
