"""The trailing-update kernels are interchangeable bit for bit.

``schur_ws2_kernel`` (TMA operand ring, two MMA warps per sub-partition; the single-GPU default),
the same kernel with its cp.async producer (``RCP_SCHUR_TMA=0``) and the first-generation
``schur_ws_kernel`` (``RCP_SCHUR_V=1``; still used by the multi-GPU tile dealing) accumulate every
element of A22 - L21 W21^T in the same order (zero-initialised accumulators, k ascending, one add
into C-in), so a whole factorization must come out identical -- permutation, D and every bit of L.
The selection is read once per process, hence one subprocess per variant.  Shapes: n not a
multiple of 128 (ragged last supertile), P > 128 (two sketch supertiles per row block), a width-64
and a width-128 panel, and the q = 1 path (no fused sketch tiles).
"""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]

SCRIPT = r"""
import hashlib, json, sys
import numpy as np, torch
sys.path.insert(0, %r)
from paper_1710_00125_b200 import api, gallery
out = {}
for name, n, kw in (("n3001_b64", 3001, dict(b=64, q=64, p=74)),
                    ("n2304_b128", 2304, dict(b=128, q=128, p=144)),
                    ("n1500_q1", 1500, dict(b=32, q=1, p=5))):
    a = torch.from_numpy(gallery.type6(n, 7)).cuda()
    f = api.factor_device(a, api.FactorConfig(strategy="rcp", seed=3, **kw))
    torch.cuda.synchronize()
    h = hashlib.sha1()
    for t in (f.perm, f.L, f.d_diag, f.d_off, f.pattern):
        h.update(t.cpu().numpy().tobytes())
    out[name] = h.hexdigest()
print("HASHES " + json.dumps(out))
""" % str(ROOT)


def _run(env_extra):
    env = dict(os.environ)
    for k in ("RCP_SCHUR_V", "RCP_SCHUR_TMA", "RCP_SCHUR_HINTS"):
        env.pop(k, None)
    env.update(env_extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = next(l for l in r.stdout.splitlines() if l.startswith("HASHES "))
    return json.loads(line[len("HASHES "):])


def test_trailing_update_kernels_are_bit_identical():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    base = _run({})
    assert base == _run({"RCP_SCHUR_TMA": "0"}), "TMA and cp.async operand staging differ"
    assert base == _run({"RCP_SCHUR_V": "1"}), "schur_ws2_kernel and schur_ws_kernel differ"
    assert base == _run({"RCP_SCHUR_HINTS": "2"}), "L2 cache hints changed the result"
