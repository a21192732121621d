"""Randomised parity sweep: the CUDA path against the live oracle on seeded random shapes.

Every case draws a size, a panel width, the sketch mode (q = b or q = 1), the oversampling, a
strategy and a matrix family (dense type-6, KKT saddle point, badly scaled, exactly rank-deficient
with the robust guard) from one seed, factors it on the GPU and with the oracle, and asserts the
same bar as the fixture tests: identical pivot sequence, 1x1/2x2 pattern, op counters and recompute
count; L and D within ``l_tol(n)``.  The default run takes a few dozen cases (seconds);
``RCP_SWEEP_CASES=600 RCP_SWEEP_MAXN=900`` is the long run recorded in profiles/.

Near-ties (north_star: "documented near-ties"; SURVEY.md section 7.3 noise-floor run): when the pivot
sequences differ at position k, the case is accepted only if the reference's own decision there is at
its rounding-noise level, by either of two measurable criteria:
  (a) the oracle re-run on the input perturbed by one ulp per entry (symmetrically) changes its OWN
      sequence at or before k;
  (b) sketch floor: the decision at k is a sketch-norm argmax (rcp) whose relative top-2 gap is below
      eps * n * max|Omega A| / ||b_top|| -- the error every trailing sketch column inherits from forming
      B = Omega A in floating point, which no later downdate removes.  This only opens on badly scaled
      inputs, where the trailing sketch columns lie many orders of magnitude below the initial sketch.
The case then still has to pass as a factorization (PAP^T = LDL^T componentwise to rounding) and is
printed as ``NEAR-TIE``.  Any other divergence fails.
"""

import os

import numpy as np
import pytest

from conftest import l_tol

pytestmark = pytest.mark.gpu

CASES = int(os.environ.get("RCP_SWEEP_CASES", "48"))
MAXN = int(os.environ.get("RCP_SWEEP_MAXN", "420"))
OFFSET = int(os.environ.get("RCP_SWEEP_OFFSET", "0"))


def _draw(seed):
    from paper_1710_00125_b200 import gallery
    g = np.random.Generator(np.random.Philox(90000 + seed))
    n = int(g.integers(2, MAXN + 1))
    b = int(g.choice([1, 2, 4, 8, 16, 32, 64, 128]))
    strategy = str(g.choice(["rcp", "rcp", "rcp", "bkpp", "bbk"]))
    q = b if (strategy != "rcp" or g.random() < 0.7) else 1
    p = (q if q > 1 else 1) + int(g.integers(2, 17))
    family = str(g.choice(["type6", "type6", "kkt", "scaled", "deficient"]))
    robust = 0
    if family == "type6":
        a = gallery.type6(n, 5000 + seed)
    elif family == "kkt":
        n2 = max(1, n // 5)
        a = gallery.kkt(n - n2, n2, 5000 + seed) if n - n2 >= 1 else gallery.type6(n, 5000 + seed)
    elif family == "scaled":
        a = gallery.scaled_member(n, 5000 + seed, True)
    else:  # exactly singular: z zero rows / columns scattered by a symmetric permutation (all later arithmetic
        # on them stays exactly zero, so both sides see the same deficient tail; rcp's guard must stop there)
        z = int(g.integers(1, max(2, n // 3 + 1)))
        a = np.zeros((n, n))
        if n - z >= 1:
            a[: n - z, : n - z] = gallery.type6(n - z, 5000 + seed)
        pm = g.permutation(n)
        a = np.ascontiguousarray(a[pm][:, pm])
        if strategy == "rcp":
            robust = int(g.integers(1, 11))
        else:
            a = a + np.diag(np.arange(1, n + 1, dtype=np.float64))  # bkpp / bbk have no guard: keep it regular
    cfg = dict(strategy=strategy, b=b, q=q, p=p, seed=int(g.integers(0, 1000)),
               robust_r=robust if robust else int(g.integers(0, 2)))
    return a, cfg, family


@pytest.mark.parametrize("seed", range(OFFSET, OFFSET + CASES))
def test_random_case_matches_oracle(cuda_ok, seed):
    import torch

    from oracle.rcp_oracle import OracleConfig, oracle_factor
    from paper_1710_00125_b200 import api
    a, cfg, family = _draw(seed)
    n = a.shape[0]
    o = oracle_factor(a, OracleConfig(**cfg))
    f = api.factor_device(torch.from_numpy(np.ascontiguousarray(a)).cuda(), api.FactorConfig(**cfg)).to_host()
    tag = f"seed {seed}: n={n} {family} {cfg}"
    if not (np.array_equal(f.perm, o.perm) and np.array_equal(f.pattern, o.pattern)):
        k = int(np.flatnonzero((f.perm != o.perm) | (f.pattern != o.pattern))[0])
        why = None
        g = np.random.Generator(np.random.Philox(777 + seed))
        e = np.tril(np.where(g.random((n, n)) < 0.5, -1.0, 1.0))
        e = e + np.tril(e, -1).T
        o2 = oracle_factor(a * (1.0 + np.finfo(np.float64).eps * e), OracleConfig(**cfg))
        moved = np.flatnonzero((o2.perm != o.perm) | (o2.pattern != o.pattern))
        if moved.size and int(moved[0]) <= k:
            why = f"the oracle's own sequence moves at k={int(moved[0])} under a 1-ulp input perturbation"
        elif cfg["strategy"] == "rcp":
            import oracle.rcp_oracle as orc
            rec, orig = [], orc.col_norms

            def spy(x, *args, **kw):
                out = orig(x, *args, **kw)
                if out.size > 1:
                    t = np.sort(out)[-2:]
                    rec.append((out.size, float((t[1] - t[0]) / t[1]) if t[1] > 0 else 0.0, float(t[1]),
                                float(np.abs(x).max())))
                return out
            orc.col_norms = spy
            try:
                oracle_factor(a, OracleConfig(**cfg))
            finally:
                orc.col_norms = orig
            b0 = rec[0][3]  # max |Omega A|
            at = [r for r in rec if r[0] == n - k] or [r for r in rec if r[0] in (n - k + 1, n - k - 1)]
            if at:
                gap, top = at[-1][1], at[-1][2]
                floor = np.finfo(np.float64).eps * n * b0 / top
                if gap <= floor:
                    why = (f"sketch floor: top-2 gap {gap:.2e} of the sketch norms at k={k} <= eps*n*max|Omega A|/||b|| "
                           f"= {floor:.2e} (||b_top|| = {top:.2e}, max|Omega A| = {b0:.2e})")
        assert why, f"{tag}: pivot sequence differs at k={k} and neither near-tie criterion holds"
        # a rounding-level tie of the reference itself: accept any valid factorization
        pa = a[f.perm][:, f.perm]
        rec = f.L @ f.D.to_dense() @ f.L.T
        scale = np.abs(f.L) @ np.abs(f.D.to_dense()) @ np.abs(f.L.T)
        err = float((np.abs(rec - pa) / np.maximum(scale, np.finfo(np.float64).tiny)).max())
        assert err <= 1e-10, f"{tag}: near-tie at k={k} but reconstruction error {err:.2e}"
        line = f"NEAR-TIE {tag}: first divergence at k={k} of n={n}; {why}; componentwise reconstruction {err:.1e}"
        print(line)
        if os.environ.get("RCP_SWEEP_LOG"):  # pytest-xdist swallows worker prints: keep a file as well
            with open(os.environ["RCP_SWEEP_LOG"], "a") as fh:
                fh.write(line + "\n")
        return
    fc, oc = f.stats.counters, o.counters
    assert [fc.mults, fc.adds, fc.divs, fc.comps] == [oc.mults, oc.adds, oc.divs, oc.comps], tag
    assert f.stats.recompute_count == o.recompute_count, tag
    tol = l_tol(n)
    lscale = max(1.0, float(np.abs(o.L).max()))
    assert np.abs(f.L - o.L).max() <= tol * lscale, tag
    dref = o.d_dense()
    assert np.abs(f.D.to_dense() - dref).max() <= tol * max(1.0, float(np.abs(dref).max())), tag


BATCHES = int(os.environ.get("RCP_SWEEP_BATCHES", "12"))


@pytest.mark.parametrize("seed", range(OFFSET, OFFSET + BATCHES))
def test_random_batch_matches_oracle(cuda_ok, seed):
    """The batched kernel (C5 path: n <= 256, b <= 32, p <= 64, q = b) on a random stack of mixed
    families: every member must equal the oracle's factorization of that matrix alone."""
    import torch

    from oracle.rcp_oracle import OracleConfig, oracle_factor
    from paper_1710_00125_b200 import api, batched, gallery
    g = np.random.Generator(np.random.Philox(70000 + seed))
    n = int(g.integers(2, 257))
    b = int(g.choice([2, 4, 8, 16, 32]))
    p = b + int(g.integers(2, 17))
    cfg = dict(strategy="rcp", b=b, q=b, p=p, seed=int(g.integers(0, 1000)), robust_r=int(g.integers(1, 11)))
    mats = []
    for j in range(6):
        fam = ["type6", "kkt", "scaled", "singular", "type6", "scaled"][j]
        sd = 8000 + 10 * seed + j
        if fam == "type6" or n < 3:
            a = gallery.type6(n, sd)
        elif fam == "kkt":
            n2 = max(1, n // 5)
            a = gallery.kkt(n - n2, n2, sd)
        elif fam == "scaled":
            a = gallery.scaled_member(n, sd, True)
        else:
            z = int(g.integers(1, max(2, n // 3 + 1)))
            a = np.zeros((n, n))
            a[: n - z, : n - z] = gallery.type6(n - z, sd)
            pm = g.permutation(n)
            a = np.ascontiguousarray(a[pm][:, pm])
        mats.append(a)
    fs = batched.factor_batched_device(torch.from_numpy(np.ascontiguousarray(np.stack(mats))).cuda(),
                                       api.FactorConfig(**cfg)).to_host()
    tol = l_tol(n)
    for j, (f, a) in enumerate(zip(fs, mats)):
        o = oracle_factor(a, OracleConfig(**cfg))
        tag = f"batch seed {seed} member {j}: n={n} {cfg}"
        assert np.array_equal(f.perm, o.perm), tag
        assert np.array_equal(f.pattern, o.pattern), tag
        fc, oc = f.stats.counters, o.counters
        assert [fc.mults, fc.adds, fc.divs, fc.comps] == [oc.mults, oc.adds, oc.divs, oc.comps], tag
        assert f.stats.recompute_count == o.recompute_count, tag
        assert np.abs(f.L - o.L).max() <= tol * max(1.0, float(np.abs(o.L).max())), tag
        dref = o.d_dense()
        assert np.abs(f.D.to_dense() - dref).max() <= tol * max(1.0, float(np.abs(dref).max())), tag
