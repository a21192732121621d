"""BASELINE.json configurations at their full sizes on the GPU (C2 n=8192, C4 KKT n=20000,
C3 n=32768), pinned to the REFERENCE: tests/golden/g_full_{c2,c4,c3}.npz hold the outputs of
``randldl.factor`` itself on the same seeded inputs (tests/golden/make_golden_full.py, 8 BLAS
threads, build container).  Asserted against them: the identical pivot sequence (perm), 1x1/2x2
structure (pattern), op counters and recompute count; D within l_tol(n) * max|D|; the row and
column sums of L (a checksum of the dense L the fixture cannot hold); the solve x for the
seeded RHS; rho_cheap and max_multiplier.  A divergence reports the first divergent step and
the reference's decision margins there.

Besides the fixture comparison, size-independent properties are checked: perm is a
permutation, L has the reference's exact structure (unit diagonal, zero upper part,
L[k+1,k] = 0 inside every 2x2 block -- factor.py:287, 467), PAP^T = LDL^T to rounding
(tests/helpers.py:17-22 recon_error), the solve residual ||Ax-b||_inf / (||A||_inf ||x||_inf)
(metrics.py:151-167), and repeat factorizations are bit-identical."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _kkt_device(n1: int, n2: int, seed: int):
    """C4 input: gallery.kkt_c4 (H = G^T G / n1 + I with G on a 2^-8 grid, so G^T G is exact
    under any summation order: the same bits as the matrix the reference factored)."""
    import torch
    from paper_1710_00125_b200 import gallery
    return torch.from_numpy(gallery.kkt_c4(n1, n2, seed)).cuda()


def _golden(name):
    from pathlib import Path
    p = Path(__file__).resolve().parent / "golden" / f"g_full_{name}.npz"
    if not p.exists():
        pytest.skip(f"{p.name} not generated yet (tests/golden/make_golden_full.py {name})")
    z = np.load(p, allow_pickle=False)
    return {k: z[k] for k in z.files}


def _divergence_report(g, perm, pattern):
    """First step where the pivot sequence or the block structure differs, with the margins
    the reference saw at and before that step."""
    ref_perm, ref_pat = g["perm"].astype(np.int64), g["pattern"]
    bad = np.flatnonzero((ref_perm != perm) | (ref_pat != pattern))
    k = int(bad[0])
    ks = g["sbkp_k"]
    j = int(np.searchsorted(ks, k, side="right")) - 1
    lines = [f"first divergence at position k={k} of n={perm.size} ({bad.size} positions differ)"]
    for jj in range(max(0, j - 2), min(ks.size, j + 2)):
        lines.append(f"  reference SBKP decision at k={int(ks[jj])}: lambda top-2 gap {g['sbkp_lam_gap'][jj]:.3e}, "
                     f"|a_kk| vs alpha*lambda {g['sbkp_akk_margin'][jj]:.3e}, "
                     f"|d_r| vs alpha*lambda {g['sbkp_dr_margin'][jj]:.3e}")
    if g["qrcp_gap"].size:
        lines.append(f"  smallest QRCP residual-norm top-2 gap in the run: {np.nanmin(g['qrcp_gap']):.3e}")
    return "\n".join(lines)


def _compare_reference(f, g, a, name):
    """The GPU factorization against the reference's fixture (see module docstring)."""
    import torch
    from paper_1710_00125_b200 import api
    from conftest import l_tol
    n = f.n
    perm = f.perm.cpu().numpy()
    pattern = f.pattern.cpu().numpy()
    if not (np.array_equal(perm, g["perm"]) and np.array_equal(pattern, g["pattern"])):
        pytest.fail(f"{name}: pivot sequence / block structure differs from the reference\n"
                    + _divergence_report(g, perm, pattern))
    st = f.stats
    assert tuple(st["counters"]) == tuple(int(x) for x in g["counters"]), (st["counters"], g["counters"])
    assert st["recompute_count"] == int(g["recompute_count"])
    tol = l_tol(n)
    dd, doff = f.d_diag.cpu().numpy(), f.d_off.cpu().numpy()
    dmax = max(float(np.abs(g["d_diag"]).max()), float(np.abs(g["d_off"]).max()))
    err_d = max(float(np.abs(dd - g["d_diag"]).max()), float(np.abs(doff - g["d_off"]).max())) / dmax
    # L checksums: each sum adds <= n entries that each agree within l_tol(n)
    rows = f.L.sum(dim=1).cpu().numpy()
    cols = f.L.sum(dim=0).cpu().numpy()
    err_r = float(np.abs(rows - g["L_rowsum"]).max())
    err_c = float(np.abs(cols - g["L_colsum"]).max())
    rhs = torch.from_numpy(np.random.Generator(np.random.Philox(1)).standard_normal(n)).cuda()
    x, sing = api.solve_device(f, rhs)
    assert not sing and not bool(g["singular"])
    xr = g["x"]
    err_x = float(np.abs(x.cpu().numpy() - xr).max()) / float(np.abs(xr).max())
    err_rho = abs(st["rho_cheap"] - float(g["rho_cheap"])) / float(g["rho_cheap"])
    err_mm = abs(st["max_multiplier"] - float(g["max_multiplier"])) / float(g["max_multiplier"])
    print(f"{name}: n={n} perm/pattern/counters identical; |dD|/max|D| {err_d:.2e} (tol {tol:.1e}), "
          f"|d rowsum(L)| {err_r:.2e} |d colsum(L)| {err_c:.2e} (tol {tol * n:.1e}), |dx|/|x| {err_x:.2e}, "
          f"rho {err_rho:.1e}, max_mult {err_mm:.1e}")
    assert err_d <= tol, err_d
    assert err_r <= tol * n and err_c <= tol * n, (err_r, err_c)
    assert err_x <= 1e-8, err_x
    assert err_rho <= 1e-10 and err_mm <= tol, (err_rho, err_mm)


def _check(a, cfg, recon_tol, resid_tol, min_2x2=1):
    import torch
    from paper_1710_00125_b200 import PAT_PAIR_START, api
    n = a.shape[0]
    f = api.factor_device(a, cfg)
    perm = f.perm
    assert torch.equal(torch.sort(perm).values, torch.arange(n, device=perm.device))
    L = f.L
    assert bool((torch.diagonal(L) == 1.0).all())
    assert not bool(torch.triu(L, 1).any())
    pairs = (f.pattern == PAT_PAIR_START).nonzero().flatten()
    assert pairs.numel() >= min_2x2
    assert not bool(L[pairs + 1, pairs].any())
    # ||P A P^T - L D L^T||_max / ||A||_max, in row blocks (bounded temporaries)
    rec = api.reconstruct_device(f)
    amax = float(a.abs().max())
    err = 0.0
    for r0 in range(0, n, 4096):
        r1 = min(n, r0 + 4096)
        blk = a.index_select(0, perm[r0:r1]).index_select(1, perm)
        err = max(err, float((rec[r0:r1] - blk).abs().max()))
        del blk
    del rec
    assert err / amax <= recon_tol, err / amax
    rhs = torch.from_numpy(np.random.Generator(np.random.Philox(1)).standard_normal(n)).cuda()
    x, sing = api.solve_device(f, rhs)
    assert not sing
    resid = float((a @ x - rhs).abs().max()) / (float(a.abs().sum(dim=1).max()) * float(x.abs().max()))
    assert resid <= resid_tol, resid
    # determinism: a second factorization gives the same bits
    g = api.factor_device(a, cfg)
    for name in ("perm", "L", "d_diag", "d_off", "pattern"):
        assert torch.equal(getattr(f, name), getattr(g, name)), name
    return f


def test_c2_full_size(cuda_ok):
    import torch
    from paper_1710_00125_b200 import api, gallery
    g = _golden("c2")
    a = torch.from_numpy(gallery.type6(8192, 0)).cuda()
    f = _check(a, api.FactorConfig(strategy="rcp", b=64, q=64, p=74, seed=0), 1e-11, 1e-13, min_2x2=2000)
    _compare_reference(f, g, a, "C2")


def test_c4_kkt_full_size(cuda_ok):
    from paper_1710_00125_b200 import api
    g = _golden("c4")
    a = _kkt_device(16000, 4000, 0)
    f = _check(a, api.FactorConfig(strategy="rcp", b=64, q=64, p=74, seed=0), 1e-11, 1e-12, min_2x2=0)
    _compare_reference(f, g, a, "C4")


def test_c3_full_size(cuda_ok):
    import torch
    from paper_1710_00125_b200 import api, gallery
    g = _golden("c3")
    a = torch.from_numpy(gallery.type6(32768, 0)).cuda()
    f = _check(a, api.FactorConfig(strategy="rcp", b=128, q=128, p=144, seed=0), 1e-10, 1e-13, min_2x2=8000)
    assert f.stats["n_panels"] >= 32768 // 128
    _compare_reference(f, g, a, "C3")


@pytest.mark.parametrize("strategy", ["bkpp", "bbk"])
def test_c2_size_comparison_strategies(cuda_ok, strategy):
    """The reference grid's comparison strategies (bkpp, bbk) at the C2 size,
    pinned to the reference's own run like the rcp configurations."""
    import torch
    from paper_1710_00125_b200 import api, gallery
    g = _golden(f"c2_{strategy}")
    a = torch.from_numpy(gallery.type6(8192, 0)).cuda()
    f = _check(a, api.FactorConfig(strategy=strategy, b=64, q=1, p=5, seed=0), 1e-11, 1e-13, min_2x2=1000)
    _compare_reference(f, g, a, f"C2/{strategy}")
