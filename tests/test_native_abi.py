"""The C-ABI library loads on CPU and exports every symbol include/rcp_b200.h declares."""

import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "rcp_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rcp_[a-z_0-9]+)\s*\(", text)) - {"rcp_draw_fn"})


@pytest.fixture(scope="module")
def lib():
    from paper_1710_00125_b200 import _native, build
    build.build()
    return _native.load()


def test_header_lists_expected_entry_points():
    from paper_1710_00125_b200 import _native
    assert declared_symbols() == sorted(_native.EXPORTED_SYMBOLS)


def test_library_exports_all_declared_symbols(lib):
    for sym in declared_symbols():
        assert hasattr(lib, sym), sym


def test_version_string_names_sm100a(lib):
    assert b"sm_100a" in lib.rcp_version()


def test_workspace_query_is_pure_host(lib):
    import ctypes
    from paper_1710_00125_b200 import _native
    c = _native.RcpConfig(144, 128, 128, 1)
    n = 32768
    need = lib.rcp_workspace_bytes(n, ctypes.byref(c))
    assert need >= 3 * n * n * 8          # two ping-pong trailing blocks + panel L store
    bad = _native.RcpConfig(5, 8, 3, 1)   # q not in {1, b}
    assert lib.rcp_workspace_bytes(100, ctypes.byref(bad)) == 0


def test_library_is_sm100a_only():
    import subprocess
    from paper_1710_00125_b200 import build
    out = build.build()
    res = subprocess.run(["cuobjdump", "--list-elf", str(out)], capture_output=True, text=True)
    if res.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in res.stdout
