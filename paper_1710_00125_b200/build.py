"""Build ``librcp_b200.so`` in-tree with nvcc for sm_100a.

``python -m paper_1710_00125_b200.build`` (also called by ``__graft_entry__.build``).
The library is rebuilt only when a source is newer than it (``force=True`` rebuilds).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT = PKG / "librcp_b200.so"

NVCC_FLAGS = [
    "-shared", "-Xcompiler", "-fPIC", "-std=c++17", "-O3", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def needs_build() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "rcp_b200.h"]
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False, out: Path | None = None, defines: list | None = None) -> Path:
    """Compile each .cu to an object in parallel (nvcc per file), then link the shared library.
    ``out`` / ``defines`` build an experiment variant (e.g. ``librcp_lower.so`` with
    ``-DRCP_FULL_STORAGE=0``), selected at run time with ``RCP_B200_LIB``."""
    target = Path(out) if out else OUT
    if out is None and not force and not needs_build():
        return OUT
    from concurrent.futures import ThreadPoolExecutor
    extra = ["-DRCP_PANEL_PROF=1"] if os.environ.get("RCP_PANEL_PROF") == "1" else []
    if os.environ.get("RCP_BATCH_PROF") == "1":
        extra.append("-DRCP_BATCH_PROF=1")
    extra += list(defines or [])
    objdir = ROOT / "build" / ("obj" if out is None else "obj_" + target.stem)
    objdir.mkdir(parents=True, exist_ok=True)
    compile_flags = [f for f in NVCC_FLAGS if f != "-shared"]
    nvcc = _nvcc()

    def one(src: Path) -> Path:
        obj = objdir / (src.stem + ".o")
        cmd = [nvcc, *compile_flags, *extra, "-c", str(src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True, cwd=str(ROOT))
        return obj

    with ThreadPoolExecutor(max_workers=max(1, min(len(sources()), os.cpu_count() or 1))) as ex:
        objs = list(ex.map(one, sources()))
    cmd = [nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(target) + ".tmp", *map(str, objs)]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=str(ROOT))
    os.replace(str(target) + ".tmp", target)
    return target


if __name__ == "__main__":
    # python -m paper_1710_00125_b200.build [--force] [--variant NAME -DFOO=1 ...]
    argv = sys.argv[1:]
    if "--variant" in argv:
        name = argv[argv.index("--variant") + 1]
        defs = [a for a in argv if a.startswith("-D")]
        p = build(verbose=True, out=PKG / f"librcp_{name}.so", defines=defs)
    else:
        p = build(force="--force" in argv, verbose=True)
    print(p)
