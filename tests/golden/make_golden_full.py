"""Full-size golden fixtures for BASELINE.json configs 2, 3 and 4, made by running the
REFERENCE itself (``randldl`` from /root/reference; build container only).

    OPENBLAS_NUM_THREADS=8 python tests/golden/make_golden_full.py c2 [c4 c3]

Inputs are regenerated from their seeded spec on both sides, so only outputs are stored:
perm, pattern, D as (d_diag, d_off), row and column sums of L, the solve x for the
seeded RHS (gallery.rhs(n, 1)), rho_cheap / max_multiplier / recompute_count, the exact
op counters, and the per-decision margins the reference saw (the GPU parity test reports
the first divergent step together with the margin there):

* ``sbkp_k``/``sbkp_lam_gap``/``sbkp_akk_margin``/``sbkp_dr_margin``: per SBKP decision at
  step k, the relative top-2 gap of |c[1:]| (first-index argmax), ||a_kk| - alpha lam| /
  alpha lam and ||d_r| - alpha lam| / alpha lam (nan where the rule did not test it)
  -- pivot.py:111-128.
* ``qrcp_gap``: per residual-norm argmax inside ``partial_qrcp`` (sketch.py:152-154), the
  relative top-2 gap, in call order.

The recorders wrap ``randldl.factor._sbkp_from_data`` and ``randldl.sketch.column_norms``;
they only read values, so the factorization's bits are unchanged.

C4 (KKT) uses ``gallery.kkt_c4``: G's entries are N(0,1) draws rounded to multiples of 2^-8,
so that G^T G is exact in fp64 under ANY summation order -- the GPU test regenerates the
identical matrix with a device GEMM.
"""

from __future__ import annotations

import json
import math
import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE.parents[1]))

import randldl  # noqa: E402
rfactor = sys.modules["randldl.factor"]  # the module (randldl.factor the attribute is the function)
rsketch = sys.modules["randldl.sketch"]

from paper_1710_00125_b200 import gallery  # noqa: E402

CONFIGS = {
    # name: (generator spec, FactorConfig kwargs) -- SURVEY.md section 8 config mapping
    "c2": (dict(gen="type6", n=8192, seed=0), dict(strategy="rcp", b=64, q=64, p=74, seed=0)),
    "c4": (dict(gen="kkt_c4", n1=16000, n2=4000, seed=0), dict(strategy="rcp", b=64, q=64, p=74, seed=0)),
    "c3": (dict(gen="type6", n=32768, seed=0), dict(strategy="rcp", b=128, q=128, p=144, seed=0)),
    # the comparison strategies of the reference's benchmark grid at the C2 size
    "c2_bkpp": (dict(gen="type6", n=8192, seed=0), dict(strategy="bkpp", b=64, q=1, p=5, seed=0)),
    "c2_bbk": (dict(gen="type6", n=8192, seed=0), dict(strategy="bbk", b=64, q=1, p=5, seed=0)),
}


def make_input(spec):
    if spec["gen"] == "type6":
        return gallery.type6(spec["n"], spec["seed"])
    if spec["gen"] == "kkt_c4":
        return gallery.kkt_c4(spec["n1"], spec["n2"], spec["seed"])
    raise ValueError(spec)


class Recorder:
    def __init__(self):
        self.sbkp = []        # (k, lam_gap, akk_margin, dr_margin)
        self.qrcp = []

    def install(self):
        orig_sbkp = rfactor._sbkp_from_data
        orig_norms = rsketch.column_norms
        rec = self

        def sbkp(a_kk, sub, diag_at, k, params, counters):
            seen = {}

            def diag_spy(r):
                v = diag_at(r)
                seen["d"] = v
                return v

            dec = orig_sbkp(a_kk=a_kk, sub=sub, diag_at=diag_spy, k=k, params=params, counters=counters)
            lam_gap = akk_m = dr_m = math.nan
            if sub.size:
                lam = float(sub.max())
                if lam > 0.0:
                    if sub.size > 1:
                        top2 = np.partition(sub, sub.size - 2)[-2:]
                        lam_gap = float((top2[1] - top2[0]) / top2[1])
                    al = params.alpha * lam
                    akk_m = abs(abs(a_kk) - al) / al
                    if "d" in seen:
                        dr_m = abs(abs(seen["d"]) - al) / al
            rec.sbkp.append((k, lam_gap, akk_m, dr_m))
            return dec

        def norms(m, from_col=0):
            out = orig_norms(m, from_col=from_col)
            if out.size > 1:
                top2 = np.partition(out, out.size - 2)[-2:]
                rec.qrcp.append(float((top2[1] - top2[0]) / top2[1]) if top2[1] > 0 else math.nan)
            return out

        rfactor._sbkp_from_data = sbkp
        rsketch.column_norms = norms


def d_arrays(f):
    n = f.n
    dd, off = np.zeros(n), np.zeros(n)
    i = 0
    for blk in f.D.blocks:
        if blk.shape[0] == 1:
            dd[i] = blk[0, 0]
            i += 1
        else:
            dd[i], dd[i + 1], off[i] = blk[0, 0], blk[1, 1], blk[1, 0]
            i += 2
    return dd, off


def run(name):
    spec, cfg = CONFIGS[name]
    a = make_input(spec)
    n = a.shape[0]
    rec = Recorder()
    rec.install()
    t0 = time.perf_counter()
    f = randldl.factor(a, randldl.FactorConfig(**cfg))
    t_factor = time.perf_counter() - t0
    dd, off = d_arrays(f)
    rhs = gallery.rhs(n, 1)
    t0 = time.perf_counter()
    rep = randldl.solve(f, rhs, a)
    t_solve = time.perf_counter() - t0
    c = f.stats.counters
    sb = np.array(rec.sbkp, dtype=np.float64).reshape(-1, 4)
    out = dict(
        perm=f.perm.astype(np.int32), pattern=f.pattern, d_diag=dd, d_off=off, x=rep.x,
        singular=np.array(rep.singular), backward_error=np.array(rep.backward_error),
        rho_cheap=np.array(f.stats.rho_cheap), max_multiplier=np.array(f.stats.max_multiplier),
        recompute_count=np.array(f.stats.recompute_count),
        counters=np.array([c.mults, c.adds, c.divs, c.comps], dtype=np.int64),
        L_rowsum=f.L.sum(axis=1), L_colsum=f.L.sum(axis=0),
        sbkp_k=sb[:, 0].astype(np.int32), sbkp_lam_gap=sb[:, 1], sbkp_akk_margin=sb[:, 2],
        sbkp_dr_margin=sb[:, 3], qrcp_gap=np.array(rec.qrcp),
        cfg=np.array(json.dumps(cfg)), spec=np.array(json.dumps(spec)),
        t_factor_s=np.array(t_factor), t_solve_s=np.array(t_solve),
        blas_threads=np.array(os.environ.get("OPENBLAS_NUM_THREADS", "")),
    )
    np.savez_compressed(HERE / f"g_full_{name}.npz", **out)
    print(f"{name}: n={n} factor {t_factor:.1f} s solve {t_solve:.2f} s 2x2={int((f.pattern == 1).sum())} "
          f"rho={f.stats.rho_cheap:.4g} min sbkp gap={np.nanmin(sb[:, 1:]) if sb.size else 'nan'} "
          f"min qrcp gap={min(rec.qrcp) if rec.qrcp else 'nan'}", flush=True)


if __name__ == "__main__":
    for name in sys.argv[1:] or ["c2"]:
        run(name)
