"""Generate golden fixtures by running the REFERENCE implementation itself.

Run in the build container only (it imports ``randldl`` from /root/reference,
which does not exist on the GPU box):

    python tests/golden/make_golden.py

Each case stores the input matrix (small n) or its generator spec (C1), the
FactorConfig, and the reference outputs: perm, pattern, L (small n) or L
checksums (C1), D as (d_diag, d_off), rho_cheap, max_multiplier,
recompute_count, op counters, and a solve x for a seeded RHS.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE.parents[1]))

import randldl  # noqa: E402

from paper_1710_00125_b200 import gallery  # noqa: E402


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


def save(name, a, cfg, robust=False, store_a=True, store_l=True, spec=None):
    fn = randldl.factor_robust if robust else randldl.factor
    f = fn(a, randldl.FactorConfig(**cfg))
    dd, off = d_arrays(f)
    rhs = gallery.rhs(a.shape[0], 1)
    rep = randldl.solve(f, rhs, a)
    c = f.stats.counters
    out = dict(
        perm=f.perm, pattern=f.pattern, d_diag=dd, d_off=off, x=rep.x,
        singular=np.array(rep.singular), backward_error=np.array(rep.backward_error),
        rho_cheap=np.array(f.stats.rho_cheap), max_multiplier=np.array(f.stats.max_multiplier),
        recompute_count=np.array(f.stats.recompute_count),
        counters=np.array([c.mults, c.adds, c.divs, c.comps], dtype=np.int64),
        L_rowsum=f.L.sum(axis=1), L_colsum=f.L.sum(axis=0),
        cfg=np.array(json.dumps(cfg)), robust=np.array(robust),
        spec=np.array(json.dumps(spec or {})),
    )
    if store_a:
        out["a"] = a
    if store_l:
        out["L"] = f.L
    np.savez_compressed(HERE / f"{name}.npz", **out)
    print(name, a.shape[0], "2x2:", int((f.pattern == 1).sum()), "recompute:", f.stats.recompute_count)


def main():
    sym = gallery.type6
    # test_factor.py:59-67 shapes (q = b mode plus the q = 1 reference default)
    save("g_n100_b8", sym(100, 1), dict(strategy="rcp", b=8, q=8, p=8, seed=7))
    save("g_n100_b64", sym(100, 1), dict(strategy="rcp", b=64, q=64, p=64, seed=7))
    save("g_n100_q1_b1", sym(100, 1), dict(strategy="rcp", b=1, q=1, p=5, seed=7))
    save("g_n100_q1_b64", sym(100, 1), dict(strategy="rcp", b=64, q=1, p=5, seed=7))
    # odd sizes / ragged last panel
    save("g_n61_b8", sym(61, 2), dict(strategy="rcp", b=8, q=8, p=10, seed=3))
    save("g_n300_b32", sym(300, 3), dict(strategy="rcp", b=32, q=32, p=42, seed=0))
    # config-5 shaped members, including a guard trip + recompute
    save("g_c5_plain", gallery.scaled_member(256, 1, False), dict(strategy="rcp", b=16, q=16, p=24, seed=0))
    save("g_c5_scaled", gallery.scaled_member(256, 10, True), dict(strategy="rcp", b=16, q=16, p=24, seed=0))
    # KKT structure (config 4 shape, small)
    save("g_kkt_200", gallery.kkt(160, 40, 4), dict(strategy="rcp", b=16, q=16, p=26, seed=0))
    # structured / degenerate inputs from the reference tests
    save("g_identity8", np.eye(8), dict(strategy="rcp", b=8, q=8, p=8, seed=0))
    save("g_exchange4", np.eye(4)[::-1].copy(), dict(strategy="rcp", b=2, q=2, p=4, seed=0))
    save("g_one", np.array([[3.0]]), dict(strategy="rcp", b=4, q=4, p=4, seed=0))
    save("g_zero5", np.zeros((5, 5)), dict(strategy="rcp", b=4, q=4, p=4, seed=0))
    save("g_zero5_unguarded", np.zeros((5, 5)), dict(strategy="rcp", b=4, q=4, p=4, seed=0, robust_r=0))
    tail = np.zeros((65, 65))
    tail[:40, :40] = sym(40, 5)
    save("g_zero_tail", tail, dict(strategy="rcp", b=16, q=16, p=16, seed=2), robust=True)
    # C1 (configs[0]): perm / pattern / D / x / L checksums only
    save("g_c1", sym(1000, 0), dict(strategy="rcp", b=32, q=32, p=42, seed=0), store_a=False,
         store_l=False, spec=dict(gen="type6", n=1000, seed=0))


def main_bk():
    """Fixtures of the sketch-free bkpp strategy."""
    sym = gallery.type6
    save("g_bkpp_n100_b8", sym(100, 1), dict(strategy="bkpp", b=8, q=1, p=5, seed=7))
    save("g_bkpp_n300_b32", sym(300, 3), dict(strategy="bkpp", b=32, q=1, p=5, seed=0))
    save("g_bkpp_n64_b1", sym(64, 6), dict(strategy="bkpp", b=1, q=1, p=5, seed=0))
    save("g_bkpp_kkt_200", gallery.kkt(160, 40, 4), dict(strategy="bkpp", b=16, q=1, p=5, seed=0))
    save("g_bkpp_c5_scaled", gallery.scaled_member(256, 10, True), dict(strategy="bkpp", b=16, q=1, p=5, seed=0))
    save("g_bkpp_zero5", np.zeros((5, 5)), dict(strategy="bkpp", b=4, q=1, p=5, seed=0))
    save("g_bkpp_exchange4", np.eye(4)[::-1].copy(), dict(strategy="bkpp", b=2, q=1, p=5, seed=0))
    save("g_bbk_n100_b8", sym(100, 1), dict(strategy="bbk", b=8, q=1, p=5, seed=7))
    save("g_bbk_n300_b32", sym(300, 3), dict(strategy="bbk", b=32, q=1, p=5, seed=0))
    save("g_bbk_n64_b1", sym(64, 6), dict(strategy="bbk", b=1, q=1, p=5, seed=0))
    save("g_bbk_kkt_200", gallery.kkt(160, 40, 4), dict(strategy="bbk", b=16, q=1, p=5, seed=0))
    save("g_bbk_c5_scaled", gallery.scaled_member(256, 10, True), dict(strategy="bbk", b=16, q=1, p=5, seed=0))
    save("g_bbk_exchange4", np.eye(4)[::-1].copy(), dict(strategy="bbk", b=2, q=1, p=5, seed=0))


def save_diag(name, a, cfg, robust=False):
    """Diagnostics fixtures: track_growth="full" snapshots and the
    audit_sketch drift as the reference records them (factor.py:493-504, 514-531)."""
    fn = randldl.factor_robust if robust else randldl.factor
    f = fn(a, randldl.FactorConfig(**cfg))
    dd, off = d_arrays(f)
    s = f.stats
    c = s.counters
    out = dict(
        a=a, perm=f.perm, pattern=f.pattern, d_diag=dd, d_off=off, L=f.L,
        counters=np.array([c.mults, c.adds, c.divs, c.comps], dtype=np.int64),
        rho_cheap=np.array(s.rho_cheap), max_multiplier=np.array(s.max_multiplier),
        recompute_count=np.array(s.recompute_count),
        snapshots=np.array(s.snapshots if s.snapshots is not None else [], dtype=np.float64).reshape(-1, 2),
        has_snapshots=np.array(s.snapshots is not None),
        drift=np.array(s.sketch_drift if s.sketch_drift is not None else [], dtype=np.float64),
        has_drift=np.array(s.sketch_drift is not None),
        rho_elem=np.array(np.nan if s.rho_elem is None else s.rho_elem),
        rho_col=np.array(np.nan if s.rho_col is None else s.rho_col),
        L_norm1=np.array(np.nan if s.L_norm1 is None else s.L_norm1),
        Linv_norm1=np.array(np.nan if s.Linv_norm1 is None else s.Linv_norm1),
        cfg=np.array(json.dumps(cfg)), robust=np.array(robust),
    )
    np.savez_compressed(HERE / "diag" / f"{name}.npz", **out)
    print(name, "snapshots", len(s.snapshots or []), "drift", len(s.sketch_drift or []),
          "recompute", s.recompute_count)


def main_diag():
    (HERE / "diag").mkdir(exist_ok=True)
    sym = gallery.type6
    save_diag("d_full_n100", sym(100, 1), dict(strategy="rcp", b=8, q=8, p=8, seed=7, track_growth="full"))
    save_diag("d_audit_n100", sym(100, 1), dict(strategy="rcp", b=8, q=8, p=8, seed=7, audit_sketch=True))
    save_diag("d_both_n61", sym(61, 2), dict(strategy="rcp", b=16, q=1, p=10, seed=3, track_growth="full",
                                            audit_sketch=True))
    save_diag("d_both_c5_scaled", gallery.scaled_member(256, 10, True),
              dict(strategy="rcp", b=16, q=16, p=24, seed=0, track_growth="full", audit_sketch=True))
    tail = np.zeros((65, 65))
    tail[:40, :40] = sym(40, 5)
    save_diag("d_full_zero_tail", tail, dict(strategy="rcp", b=16, q=16, p=16, seed=2, track_growth="full",
                                             audit_sketch=True), robust=True)
    save_diag("d_full_bkpp", sym(80, 4), dict(strategy="bkpp", b=8, q=1, p=5, seed=0, track_growth="full"))
    save_diag("d_full_kkt", gallery.kkt(160, 40, 4), dict(strategy="rcp", b=16, q=16, p=26, seed=0,
                                                           track_growth="full"))


if __name__ == "__main__":
    if "--bk" in sys.argv:
        main_bk()
    elif "--diag" in sys.argv:
        main_diag()
    else:
        main()
