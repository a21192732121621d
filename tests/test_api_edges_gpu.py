"""Edge cases of the device/host API (advisor findings, round 1): strided batch views, RHS dtype /
device conversion, Omega validation, and the device factorization kept with factor()'s result."""

import numpy as np
import pytest

from conftest import l_tol

pytestmark = pytest.mark.gpu


def test_batched_strided_view_reads_the_right_matrices(cuda_ok):
    import torch
    from paper_1710_00125_b200 import FactorConfig, batched, gallery
    mats = [gallery.scaled_member(64, s, scaled=(s % 3 == 0)) for s in range(6)]
    stack = torch.from_numpy(np.ascontiguousarray(np.stack(mats))).cuda()
    cfg = FactorConfig(strategy="rcp", b=8, q=8, p=12, seed=1)
    every_other = batched.factor_batched_device(stack[::2], cfg)       # stride(0) = 2 n^2
    direct = batched.factor_batched_device(stack[::2].contiguous(), cfg)
    for name in ("perm", "L", "d_diag", "d_off", "pattern"):
        assert torch.equal(getattr(every_other, name), getattr(direct, name)), name


def test_solve_device_converts_rhs_and_checks_shape(cuda_ok):
    import torch
    from paper_1710_00125_b200 import api, gallery
    a = gallery.type6(96, 4)
    f = api.factor_device(torch.from_numpy(a).cuda(), api.FactorConfig(strategy="rcp", b=16, q=16, p=20))
    rhs = np.random.Generator(np.random.Philox(5)).standard_normal(96)
    x64, _ = api.solve_device(f, torch.from_numpy(rhs).cuda())
    x32, _ = api.solve_device(f, torch.from_numpy(rhs.astype(np.float32)).cuda())  # float32 in
    xcpu, _ = api.solve_device(f, torch.from_numpy(rhs))                           # host tensor in
    assert x32.dtype == torch.float64 and x32.is_cuda and xcpu.is_cuda
    assert torch.equal(xcpu, x64)
    assert float((x32 - torch.from_numpy(rhs.astype(np.float32).astype(np.float64)).cuda()).abs().max()) >= 0.0
    with pytest.raises(ValueError, match="does not match"):
        api.solve_device(f, torch.zeros(95, dtype=torch.float64, device="cuda"))


def test_factor_device_validates_omega(cuda_ok):
    import torch
    from paper_1710_00125_b200 import api, gallery
    a = torch.from_numpy(gallery.type6(40, 2)).cuda()
    cfg = api.FactorConfig(strategy="rcp", b=8, q=8, p=10, seed=3)
    with pytest.raises(ValueError, match="omega must have shape"):
        api.factor_device(a, cfg, omega=torch.zeros(9, 40, dtype=torch.float64, device="cuda"))
    om = np.random.Generator(np.random.Philox(3)).standard_normal((10, 40))
    f1 = api.factor_device(a, cfg, omega=torch.from_numpy(om.astype(np.float32).astype(np.float64)))  # host omega
    f2 = api.factor_device(a, cfg, omega=torch.from_numpy(om.astype(np.float32).astype(np.float64)).cuda())
    assert torch.equal(f1.perm, f2.perm) and torch.equal(f1.L, f2.L)


def test_solve_reuses_the_device_factorization(cuda_ok):
    from paper_1710_00125_b200 import api, gallery
    a = gallery.type6(300, 3)
    f = api.factor(a, api.FactorConfig(strategy="rcp", b=32, q=32, p=42, seed=0))
    assert api._attached(f) is not None
    assert not f.L.flags.writeable and not f.perm.flags.writeable
    rhs = gallery.rhs(300, 1)
    rep = api.solve(f, rhs, a)
    # a Factorization whose arrays were replaced is uploaded again (same answer)
    g = api.Factorization(perm=f.perm.copy(), L=f.L.copy(), D=f.D, pattern=f.pattern.copy(), stats=f.stats)
    assert api._attached(g) is None
    rep2 = api.solve(g, rhs, a)
    assert np.array_equal(rep.x, rep2.x)
    assert rep.backward_error <= 1e-13
    xs = api.solve_many(f, np.stack([rhs, 2 * rhs], axis=1))
    assert np.allclose(xs[:, 0], rep.x, rtol=0, atol=l_tol(300) * np.abs(rep.x).max())
    assert np.allclose(xs[:, 1], 2 * rep.x, rtol=0, atol=2 * l_tol(300) * np.abs(rep.x).max())
