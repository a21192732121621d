"""The drop-in boundary on the GPU: the NumericalError path through the public API, and the
C ABI entry point ``rcp_factor`` called directly through ctypes the way INTEGRATION.md shows
a randldl maintainer binding it (no helper from this package on the call path)."""

import ctypes

import numpy as np
import pytest

from conftest import l_tol, load_golden

pytestmark = pytest.mark.gpu

# A 2x2 input whose first elimination overflows the trailing entry to -inf while the sketch
# Omega A stays finite (seed 0): the reference raises NumericalError("non-finite pivot data at
# step 1") from _eliminate's finiteness check (factor.py:455-456) for every mode below
# (established by running randldl.factor in the build container).
_X = 1e308
_OVERFLOW = np.array([[0.75 * _X, _X], [_X, -_X]])


@pytest.mark.parametrize("cfg", [
    dict(strategy="rcp", b=2, q=2, p=2),
    dict(strategy="rcp", b=1, q=1, p=2),
    dict(strategy="rcp", b=2, q=1, p=3),
    dict(strategy="bkpp", b=2, q=2, p=2),
    dict(strategy="bbk", b=2, q=2, p=2),
])
def test_nonfinite_pivot_data_raises_numerical_error(cuda_ok, cfg):
    from paper_1710_00125_b200 import NumericalError, api
    with pytest.raises(NumericalError, match=r"^non-finite pivot data at step 1$"):
        api.factor(_OVERFLOW, api.FactorConfig(seed=0, **cfg))


def test_device_path_raises_numerical_error_too(cuda_ok):
    import torch
    from paper_1710_00125_b200 import NumericalError, api
    with pytest.raises(NumericalError, match="non-finite pivot data at step 1"):
        api.factor_device(torch.from_numpy(_OVERFLOW).cuda(), api.FactorConfig(strategy="rcp", b=2, q=2, p=2))


class _Cfg(ctypes.Structure):  # rcp_config (include/rcp_b200.h)
    _fields_ = [("p", ctypes.c_int32), ("b", ctypes.c_int32), ("q", ctypes.c_int32),
                ("robust_r", ctypes.c_int32), ("strategy", ctypes.c_int32)]


_DRAW = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                         ctypes.POINTER(ctypes.c_double))


@pytest.mark.parametrize("name", ["g_n300_b32", "g_c5_scaled", "g_zero_tail"])
def test_rcp_factor_through_raw_ctypes(cuda_ok, name):
    """INTEGRATION.md section 2, verbatim in spirit: raw CDLL, own struct, own draw callback."""
    import torch
    from paper_1710_00125_b200._native import LIB_PATH
    g = load_golden(name)
    cfg = g["cfg"]
    a = g["a"]
    n = a.shape[0]
    lib = ctypes.CDLL(str(LIB_PATH))
    lib.rcp_workspace_bytes.restype = ctypes.c_size_t
    lib.rcp_workspace_bytes.argtypes = [ctypes.c_int64, ctypes.POINTER(_Cfg)]
    lib.rcp_factor.restype = ctypes.c_int
    gen = np.random.Generator(np.random.Philox(cfg["seed"]))
    omega = torch.from_numpy(gen.standard_normal((cfg["p"], n))).cuda()

    def draw(_ctx, rows, cols, out):
        z = gen.standard_normal((rows, cols))
        ctypes.memmove(out, z.ctypes.data, z.nbytes)
        return 0

    cb = _DRAW(draw)
    c = _Cfg(cfg["p"], cfg["b"], cfg["q"], cfg.get("robust_r", 1), 0)
    ws = torch.empty(int(lib.rcp_workspace_bytes(n, ctypes.byref(c))), dtype=torch.uint8, device="cuda")
    A = torch.from_numpy(a).cuda()
    perm = torch.empty(n, dtype=torch.int64, device="cuda")
    L = torch.empty(n, n, dtype=torch.float64, device="cuda")
    dd = torch.empty(n, dtype=torch.float64, device="cuda")
    doff = torch.empty(n, dtype=torch.float64, device="cuda")
    pat = torch.empty(n, dtype=torch.int8, device="cuda")
    st = (ctypes.c_byte * 1024)()
    vp = ctypes.c_void_p
    status = lib.rcp_factor(ctypes.byref(c), ctypes.c_int64(n), vp(A.data_ptr()), ctypes.c_int64(n),
                            vp(omega.data_ptr()), cb, None, vp(ws.data_ptr()), ctypes.c_size_t(ws.numel()),
                            vp(perm.data_ptr()), vp(L.data_ptr()), vp(dd.data_ptr()), vp(doff.data_ptr()),
                            vp(pat.data_ptr()), None, None, st,
                            vp(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    assert status == 0
    assert np.array_equal(perm.cpu().numpy(), g["perm"])
    assert np.array_equal(pat.cpu().numpy(), g["pattern"])
    dmax = max(1.0, float(np.abs(g["d_diag"]).max()))
    assert float(np.abs(dd.cpu().numpy() - g["d_diag"]).max()) <= l_tol(n) * dmax
    assert float(np.abs(L.cpu().numpy() - g["L"]).max()) <= l_tol(n)
