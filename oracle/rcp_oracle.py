"""CPU oracle for the RCP block-LDL^T hot path (arXiv 1710.00125, reference ``randldl``).

TEST INFRASTRUCTURE ONLY.  This module is the *checker*: ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import it.  The product package
(``paper_1710_00125_b200``) never imports it; the CUDA path fails loudly if its
extension is missing instead of falling back here.

It is a NumPy restatement of the reference algorithm for the path named by
BASELINE.json ``north_star``: strategy ``rcp`` with the simplified
Bunch-Kaufman (SBKP) 1x1/2x2 rule, panels of width ``b``, sketch selection
either per panel (``q == b``, partial QRCP on the sketch) or per step
(``q == 1``), the guarded mode (sketch-collapse recompute / deficient tail),
the trailing Schur update, the sketch update, and the solve.  Every helper
cites the reference line range it follows (paths relative to
``/root/reference/pkg/src/randldl/``).

Parity pin: ``tests/golden/make_golden.py`` runs the *reference itself* (only
possible in the build container, where ``/root/reference`` exists) and stores
its outputs under ``tests/golden/``; ``tests/test_oracle_golden.py`` checks
this restatement against them bit-for-bit (perm, pattern, L, D, x).  The
restatement issues the same NumPy/SciPy primitives in the same order as the
reference, so OpenBLAS rounding is reproduced exactly on the same machine.

The Bunch-Kaufman partial-pivoting (``bkpp``) and rook (``bbk``) strategies run on the
same engine without a sketch (pivot.py:131-225).
Out of scope here: ``track_growth="full"`` snapshots and ``audit_sketch`` drift records.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
from scipy.linalg import solve_triangular

EPS = float(np.finfo(np.float64).eps)          # factor.py:91
ALPHA = math.sqrt(2.0) / 2.0                   # pivot.py:44 (SBKP_ALPHA)
BK_ALPHA = (1.0 + math.sqrt(17.0)) / 8.0       # pivot.py:47 (bkpp / bbk)

PAT_SINGLE, PAT_PAIR_START, PAT_PAIR_END, PAT_DEFICIENT = 0, 1, 2, 3   # factor.py:94-97

SKIP, ONE, ONE_SWAP, TWO = "skip", "1x1", "1x1-swap", "2x2"             # pivot.py:50-54


class OracleNumericalError(RuntimeError):
    """Mirror of ``randldl.NumericalError`` (factor.py:100-101)."""


@dataclass
class OracleConfig:
    """Knobs of ``FactorConfig`` used by the path (factor.py:116-149)."""

    strategy: str = "rcp"
    p: int = 5
    b: int = 64
    q: int = 1
    seed: int = 0
    robust_r: int = 1

    def __post_init__(self) -> None:
        if self.p < 1 or self.b < 1 or self.robust_r < 0:
            raise ValueError("bad config")
        if self.q not in (1, self.b) or self.p < self.q:
            raise ValueError("bad q/p")
        if self.strategy not in ("rcp", "bkpp", "bbk"):
            raise ValueError("bad strategy")


@dataclass
class OracleCounters:
    """Cost-model tallies, same charges as the reference (metrics.py:29-43)."""

    mults: int = 0
    adds: int = 0
    divs: int = 0
    comps: int = 0


@dataclass
class OracleResult:
    perm: np.ndarray
    L: np.ndarray
    blocks: list
    pattern: np.ndarray
    rho_cheap: float
    max_multiplier: float
    recompute_count: int
    counters: OracleCounters
    trace: list = field(default_factory=list)      # (k, kind, r) per decision
    panels: list = field(default_factory=list)     # (k0, k_end) per panel
    k_done: int = 0                                 # columns eliminated (== n unless stopped early)

    @property
    def d_diag(self) -> np.ndarray:
        return _blocks_to_arrays(self.blocks)[0]

    @property
    def d_off(self) -> np.ndarray:
        return _blocks_to_arrays(self.blocks)[1]

    def d_dense(self) -> np.ndarray:
        n = sum(b.shape[0] for b in self.blocks)
        out = np.zeros((n, n))
        i = 0
        for blk in self.blocks:
            s = blk.shape[0]
            out[i:i + s, i:i + s] = blk
            i += s
        return out


def _blocks_to_arrays(blocks):
    n = sum(b.shape[0] for b in blocks)
    dg, off = np.zeros(n), np.zeros(n)
    i = 0
    for blk in blocks:
        if blk.shape[0] == 1:
            dg[i] = blk[0, 0]
        else:
            dg[i], dg[i + 1], off[i] = blk[0, 0], blk[1, 1], blk[1, 0]
        i += blk.shape[0]
    return dg, off


# --------------------------------------------------------------------------- kernels

def col_norms(m: np.ndarray, start: int = 0) -> np.ndarray:
    """Scaled Euclidean column norms of ``m[:, start:]`` (core.py:122-142)."""
    blk = np.abs(m[:, start:])
    if blk.shape[1] == 0:
        return np.zeros(0)
    if blk.shape[0] == 0:
        return np.zeros(blk.shape[1])
    scale = blk.max(axis=0)
    div = np.where(scale > 0.0, scale, 1.0)
    sc = blk / div
    return scale * np.sqrt(np.einsum("ij,ij->j", sc, sc))


def sym_exchange(a: np.ndarray, i: int, j: int) -> None:
    """Exchange rows and columns i, j of a full symmetric array (core.py:100-112)."""
    if i != j:
        a[[i, j], :] = a[[j, i], :]
        a[:, [i, j]] = a[:, [j, i]]


def copy_lower_to_upper(a: np.ndarray, blk: int = 512) -> None:
    """a[j, i] = a[i, j] for i > j (core.py:115-119), done blockwise.

    Pure copies, so the result is bitwise identical to the reference's
    ``tril_indices`` fancy-index version but O(n^2) memory-friendly.
    """
    n = a.shape[0]
    for c0 in range(0, n, blk):
        c1 = min(n, c0 + blk)
        d = a[c0:c1, c0:c1]
        il = np.tril_indices(c1 - c0, -1)
        d[il[1], il[0]] = d[il]
        if c1 < n:
            a[c0:c1, c1:] = a[c1:, c0:c1].T


def qrcp_select(b: np.ndarray, q: int) -> list:
    """First q pivots of Householder QRCP on a copy of b (sketch.py:135-169)."""
    w = np.array(b, dtype=np.float64, copy=True)
    p, m = w.shape
    if not (1 <= q <= min(p, m)):
        raise ValueError("bad q for qrcp")
    order = np.arange(m)
    picks = []
    for s in range(q):
        nr = col_norms(w[s:, :], start=s)
        j = s + int(np.argmax(nr))                       # first index on ties
        if j != s:
            w[:, [s, j]] = w[:, [j, s]]
            order[[s, j]] = order[[j, s]]
        picks.append(int(order[s]))
        x = w[s:, s]
        xn = float(np.linalg.norm(x))
        if xn == 0.0:
            continue
        v = x.copy()
        v[0] += np.copysign(xn, x[0] if x[0] != 0.0 else 1.0)
        vv = float(v @ v)
        if vv == 0.0:
            continue
        w[s:, s:] -= np.outer(v, (2.0 / vv) * (v @ w[s:, s:]))
    return picks


def _multipliers(c0, c1):
    """1x1 / 2x2 multipliers and D block (factor.py:202-226)."""
    if c1 is None:
        d = float(c0[0])
        below = c0[1:]
        if below.size and float(np.abs(below).max()) != 0.0:
            if d == 0.0:
                raise OracleNumericalError("zero 1x1 pivot under a nonzero column")
            lc = (below / d)[:, None]
        else:
            lc = np.zeros((below.size, 1))
        return lc, np.array([[d]])
    d11, d21, d22 = float(c0[0]), float(c0[1]), float(c1[1])
    det = d11 * d22 - d21 * d21
    if det == 0.0:
        raise OracleNumericalError("singular 2x2 pivot block")
    a1, a2 = c0[2:], c1[2:]
    l1 = (a1 * d22 - d21 * a2) / det
    l2 = (d11 * a2 - d21 * a1) / det
    return np.column_stack([l1, l2]), np.array([[d11, d21], [d21, d22]])


# --------------------------------------------------------------------------- engine

class _State:
    """Mutable factorization state; mirrors _Engine (factor.py:273-634)."""

    def __init__(self, a: np.ndarray, cfg: OracleConfig, normal_source=None):
        a = np.asarray(a, dtype=np.float64)
        if a.ndim != 2 or a.shape[0] != a.shape[1]:
            raise ValueError("matrix must be square")
        if a.shape[0] == 0:
            raise ValueError("matrix must have at least one row")
        if not np.array_equal(a, a.T):
            raise ValueError("matrix must be symmetric (exact equality of triangles)")
        if not np.isfinite(a).all():
            raise ValueError("input matrix contains NaN or Inf")
        n = a.shape[0]
        self.n, self.cfg = n, cfg
        self.A = np.array(a, dtype=np.float64, copy=True)             # factor.py:285
        self.amax = float(np.abs(self.A).max())                        # factor.py:286
        self.L = np.eye(n)                                             # factor.py:287
        self.perm = np.arange(n, dtype=np.int64)
        self.pattern = np.zeros(n, dtype=np.int8)
        self.blocks: list = []
        self.cnt = OracleCounters()
        self.trace: list = []
        self.panels: list = []
        self.k = 0
        self.k0 = 0
        self.t = 0
        self.W = np.zeros((0, 0))
        self.P = cfg.p
        self.rcp = cfg.strategy == "rcp"
        self.alpha = ALPHA if self.rcp else BK_ALPHA                       # factor.py:299
        # One generator per factorization, advancing across recomputes (sketch.py:63-84).
        self.gen = normal_source or np.random.Generator(np.random.Philox(cfg.seed))
        # factor.py:306-310: only rcp draws a sketch
        self.B = self.gen.standard_normal((cfg.p, n)) @ self.A if self.rcp else np.zeros((cfg.p, 0))
        self.recomputes = 0
        self.armed = self.rcp and cfg.robust_r >= 1                        # factor.py:314
        self.delta = 1.0 / cfg.robust_r if self.armed else 0.0
        self.thr = EPS ** self.delta if self.armed else 0.0
        self.beta = float(col_norms(self.B).max()) if (self.armed and self.B.size) else 0.0
        self.stopped = False

    # -- relabel -----------------------------------------------------------
    def exchange(self, i: int, j: int) -> None:
        """Relabel positions i, j in A, L[:, :k], W, B, perm (factor.py:333-348)."""
        if i == j:
            return
        sym_exchange(self.A, i, j)
        if self.k:
            self.L[[i, j], :self.k] = self.L[[j, i], :self.k]
        if self.W.size:
            a, b = i - self.k0, j - self.k0
            self.W[[a, b], :] = self.W[[b, a], :]
        if self.rcp:
            self.B[:, [i, j]] = self.B[:, [j, i]]
        self.perm[[i, j]] = self.perm[[j, i]]

    # -- left-looking column formation ---------------------------------------
    def column(self, j: int) -> np.ndarray:
        """Column j of the current Schur complement, rows k: (factor.py:350-358)."""
        k, t = self.k, self.t
        c = self.A[k:, j].copy()
        if t:
            c -= self.L[k:, self.k0:self.k0 + t] @ self.W[j - self.k0, :t]
            self.cnt.mults += t * c.size
            self.cnt.adds += t * c.size
        return c

    def diag(self, j: int) -> float:
        """Diagonal entry j of the current Schur complement (factor.py:360-367)."""
        t = self.t
        v = float(self.A[j, j])
        if t:
            v -= float(self.L[j, self.k0:self.k0 + t] @ self.W[j - self.k0, :t])
            self.cnt.mults += t
            self.cnt.adds += t
        return v

    # -- pivot rule -----------------------------------------------------------
    def sbkp(self):
        """SBKP decision on the current leading column (factor.py:414-427, pivot.py:111-128)."""
        k = self.k
        c = self.column(k)
        below = np.abs(c[1:])
        if below.size:
            self.cnt.comps += below.size - 1
            j = int(np.argmax(below))
            lam = float(below[j])
        else:
            j, lam = 0, 0.0
        if below.size == 0 or lam == 0.0:
            return SKIP, 1, None
        r = k + 1 + j
        if abs(float(c[0])) >= ALPHA * lam:
            return ONE, 1, None
        if abs(self.diag(r)) >= ALPHA * lam:
            return ONE_SWAP, 1, r
        return TWO, 2, r

    def _scan(self, v: np.ndarray):
        """Max and its first index, charging the scan's comparisons (pivot.py:80-84)."""
        self.cnt.comps += max(v.size - 1, 0)
        j = int(np.argmax(v))
        return float(v[j]), j

    def bkpp(self):
        """Classic Bunch-Kaufman partial pivoting on the leading column (pivot.py:146-171)."""
        k = self.k
        c = self.column(k)
        sub = np.abs(c[1:])
        lam, j = self._scan(sub) if sub.size else (0.0, 0)
        if sub.size == 0 or lam == 0.0:
            return SKIP, 1, None, None
        r = k + 1 + j
        a_kk = float(c[0])
        if abs(a_kk) >= self.alpha * lam:
            return ONE, 1, None, None
        col_r = self.column(r)
        absr = np.abs(col_r)
        mask = np.ones(absr.size, dtype=bool)
        mask[r - k] = False
        sigma, _ = self._scan(absr[mask])
        a_rr = float(col_r[r - k])
        if abs(a_kk) * sigma >= self.alpha * lam * lam:
            return ONE, 1, None, None
        if abs(a_rr) >= self.alpha * sigma:
            return ONE_SWAP, 1, r, None
        return TWO, 2, r, None

    def bbk(self):
        """Rook search (bounded Bunch-Kaufman) on the leading column (pivot.py:189-218)."""
        k, n = self.k, self.n
        c = self.column(k)
        sub = np.abs(c[1:])
        lam, j = self._scan(sub) if sub.size else (0.0, 0)
        if sub.size == 0 or lam == 0.0:
            return SKIP, 1, None, None
        if abs(float(c[0])) >= self.alpha * lam:
            return ONE, 1, None, None
        p_idx, imax, colmax = k, k + 1 + j, lam
        for _ in range(n - k):
            col = self.column(imax)
            absc = np.abs(col)
            mask = np.ones(absc.size, dtype=bool)
            mask[imax - k] = False
            offsets = np.nonzero(mask)[0]
            rowmax, local = self._scan(absc[mask])
            jmax = k + int(offsets[local])
            if abs(float(col[imax - k])) >= self.alpha * rowmax:
                return ONE_SWAP, 1, imax, None
            if jmax == p_idx or rowmax <= colmax:
                return TWO, 2, imax, (None if p_idx == k else p_idx)
            p_idx, imax, colmax = imax, jmax, rowmax
        raise AssertionError("rook search failed to terminate")

    # -- elimination ----------------------------------------------------------
    def eliminate(self, kind: str, s: int) -> None:
        """Multipliers, checks and writes for one pivot block (factor.py:449-489)."""
        k, n = self.k, self.n
        c0 = self.column(k)
        c1 = self.column(k + 1) if s == 2 else None
        lc, dblk = _multipliers(c0, c1)
        if not np.isfinite(dblk).all() or not np.isfinite(lc).all():
            raise OracleNumericalError(f"non-finite pivot data at step {k}")
        if s == 2:
            d21 = abs(float(dblk[1, 0]))
            det = float(dblk[0, 0]) * float(dblk[1, 1]) - d21 * d21
            if abs(det) < (1.0 - self.alpha * self.alpha) * d21 * d21 * (1.0 - 1e-12):
                raise OracleNumericalError(f"2x2 block at step {k} violates its determinant bound")
        self.L[k + s:, k:k + s] = lc
        self.W[k - self.k0:, self.t] = c0
        if s == 2:
            self.W[k - self.k0:, self.t + 1] = c1
        self.blocks.append(dblk)
        if s == 1:
            self.pattern[k] = PAT_SINGLE
        else:
            self.pattern[k], self.pattern[k + 1] = PAT_PAIR_START, PAT_PAIR_END
        w = n - k - s
        if kind != SKIP:
            if s == 1:
                self.cnt.divs += w
            else:
                self.cnt.divs += 2 * w
                self.cnt.mults += 4 * w + 2
                self.cnt.adds += 2 * w + 1
        if self.rcp and self.cfg.q == 1 and w > 0:                 # per-step sketch downdate
            self.B[:, k + s:] -= self.B[:, k:k + s] @ lc.T
            self.cnt.mults += s * self.P * w
            self.cnt.adds += s * self.P * w

    # -- trailing update ----------------------------------------------------------
    def flush_panel(self) -> None:
        """Delayed panel update of the stored trailing block + mirror (factor.py:369-379)."""
        k, t = self.k, self.t
        m = self.n - k
        if t == 0 or m == 0:
            return
        blk = self.A[k:, k:]
        blk -= self.L[k:, self.k0:self.k0 + t] @ self.W[k - self.k0:, :t].T
        copy_lower_to_upper(blk)
        self.cnt.mults += t * (m * (m + 1)) // 2
        self.cnt.adds += t * (m * (m + 1)) // 2

    def finish_deficient(self) -> None:
        """Zero-block tail after a confirmed sketch collapse (factor.py:381-385)."""
        for j in range(self.k, self.n):
            self.blocks.append(np.zeros((1, 1)))
            self.pattern[j] = PAT_DEFICIENT
        self.stopped = True

    # -- guard -------------------------------------------------------------------
    def guard_trips(self, tsel: float) -> bool:
        return self.armed and tsel < self.thr * self.beta          # factor.py:389-390

    def resketch(self) -> str:
        """Fresh projection of the active block; "stop" or "go" (factor.py:392-410)."""
        k, m = self.k, self.n - self.k
        om = self.gen.standard_normal((self.P, m))
        self.B[:, k:] = om @ self.A[k:, k:]
        self.recomputes += 1
        self.delta += 1.0 / self.cfg.robust_r
        self.thr = EPS ** self.delta
        tsel = float(col_norms(self.B, start=k).max())
        return "stop" if tsel < self.thr * self.beta else "go"

    # -- panel-level selection -------------------------------------------------------
    def preselect(self, width: int) -> str:
        """Guard + partial QRCP + replay as symmetric exchanges (factor.py:570-600)."""
        k, n = self.k, self.n
        m = n - k
        if m <= 1:
            return "go"
        nr = col_norms(self.B, start=k)
        self.cnt.comps += m - 1
        self.cnt.mults += self.P * (m - 1)
        self.cnt.adds += self.P * (m - 1)
        if self.guard_trips(float(nr.max())):
            if self.resketch() == "stop":
                self.finish_deficient()
                return "stop"
        qn = min(self.cfg.q, width, m, self.P)
        picks = qrcp_select(self.B[:, k:], qn)
        where = np.arange(m)          # current slot of each pre-call column
        holder = np.arange(m)         # pre-call column currently in each slot
        for s, col in enumerate(picks):
            x = int(where[col])
            if x != s:
                self.exchange(k + s, k + x)
                moved = int(holder[s])
                holder[s], holder[x] = col, moved
                where[col], where[moved] = s, x
            self.cnt.comps += m - 1 - s
            self.cnt.mults += 2 * self.P * (m - s)
            self.cnt.adds += 2 * self.P * (m - s)
        return "go"

    def step(self, width: int) -> str:
        """One pivot decision + elimination inside a panel (factor.py:602-634)."""
        k, n, t = self.k, self.n, self.t
        m = n - k
        if self.rcp and self.cfg.q == 1 and m > 1:
            nr = col_norms(self.B, start=k)
            self.cnt.comps += m - 1
            self.cnt.mults += self.P * (m - 1)
            self.cnt.adds += self.P * (m - 1)
            jl = int(np.argmax(nr))
            if self.guard_trips(float(nr[jl])):
                if t > 0:
                    return "defer"
                if self.resketch() == "stop":
                    self.finish_deficient()
                    return "stop"
                jl = int(np.argmax(col_norms(self.B, start=k)))
            self.exchange(k, k + jl)
        pre = None
        if self.rcp:
            kind, s, r = self.sbkp()
        elif self.cfg.strategy == "bkpp":
            kind, s, r, pre = self.bkpp()
        else:
            kind, s, r, pre = self.bbk()
        if s == 2 and t > 0 and t + 2 > width:
            return "defer"
        self.trace.append((k, kind, r))
        if kind == ONE_SWAP:
            self.exchange(k, r)
        elif kind == TWO:
            if pre is not None:                                     # factor.py:628-629
                self.exchange(k, pre)
            if r != k + 1:
                self.exchange(k + 1, r)
        self.eliminate(kind, s)
        self.k += s
        self.t += s
        return "ok"

    def panel(self) -> None:
        """One panel: preselect, steps, trailing flush, sketch correction (factor.py:540-568)."""
        n = self.n
        self.k0 = self.k
        width = min(self.cfg.b, n - self.k0)
        self.t = 0
        self.W = np.zeros((n - self.k0, min(width + 1, n - self.k0)))
        if self.rcp and self.cfg.q > 1:
            if self.preselect(width) == "stop":
                self.W = np.zeros((0, 0))
                return
        while self.k < n and self.t < width:
            if self.step(width) != "ok":
                break
        self.flush_panel()
        if self.rcp and self.cfg.q > 1 and self.t > 0 and self.k < n:
            k0, k = self.k0, self.k
            z = solve_triangular(self.L[k0:k, k0:k], self.L[k:, k0:k].T,
                                 lower=True, unit_diagonal=True, trans="T")
            self.B[:, k:] -= self.B[:, k0:k] @ z
            w, t = n - k, k - k0
            self.cnt.mults += t * self.P * w + (t * (t - 1) // 2) * w
            self.cnt.adds += t * self.P * w + (t * (t - 1) // 2) * w
        self.panels.append((self.k0, self.k))
        self.W = np.zeros((0, 0))


def oracle_factor(a: np.ndarray, cfg: OracleConfig | None = None, max_panels: int | None = None,
                  **kw) -> OracleResult:
    """RCP factorization ``A[perm][:, perm] = L D L^T`` (factor.py:508-538, 637-647).

    ``max_panels`` stops after that many panels (used only to time a bounded
    CPU-baseline sample); the returned result is then partial (``k_done < n``).
    """
    cfg = cfg or OracleConfig(**kw)
    st = _State(a, cfg)
    n = st.n
    if st.armed and st.beta == 0.0:
        st.finish_deficient()
    npan = 0
    while st.k < n and not st.stopped:
        if max_panels is not None and npan >= max_panels:
            break
        st.panel()
        npan += 1
    dmax = max((float(np.abs(b).max()) for b in st.blocks), default=0.0)
    if st.amax == 0.0:
        rho = 1.0 if dmax == 0.0 else math.inf
    else:
        rho = dmax / st.amax
    mm = float(np.abs(np.tril(st.L, -1)).max()) if n > 1 else 0.0
    return OracleResult(perm=st.perm, L=st.L, blocks=st.blocks, pattern=st.pattern,
                        rho_cheap=rho, max_multiplier=mm, recompute_count=st.recomputes,
                        counters=st.cnt, trace=st.trace, panels=st.panels,
                        k_done=n if st.stopped else st.k)


# --------------------------------------------------------------------------- solve

def block_solve(blocks, z: np.ndarray):
    """D w = z blockwise; exact-zero blocks give zeros + singular flag (solve.py:34-66)."""
    w = np.array(z, dtype=np.float64, copy=True)
    sing = False
    i = 0
    for blk in blocks:
        if blk.shape[0] == 1:
            dv = float(blk[0, 0])
            if dv == 0.0:
                sing = True
                w[i] = 0.0
            else:
                w[i] /= dv
            i += 1
        else:
            d11, d21, d22 = float(blk[0, 0]), float(blk[1, 0]), float(blk[1, 1])
            det = d11 * d22 - d21 * d21
            if det == 0.0:
                sing = True
                w[i:i + 2] = 0.0
            else:
                z1 = np.array(w[i], copy=True)
                z2 = np.array(w[i + 1], copy=True)
                w[i] = (d22 * z1 - d21 * z2) / det
                w[i + 1] = (d11 * z2 - d21 * z1) / det
            i += 2
    return w, sing


def oracle_solve(res: OracleResult, rhs: np.ndarray):
    """x = P^T L^-T D^-1 L^-1 P b (solve.py:69-76); rhs may be (n,) or (n, k)."""
    y = np.asarray(rhs, dtype=np.float64)[res.perm]
    z = solve_triangular(res.L, y, lower=True, unit_diagonal=True)
    w, sing = block_solve(res.blocks, z)
    v = solve_triangular(res.L, w, lower=True, unit_diagonal=True, trans="T")
    x = np.empty_like(v)
    x[res.perm] = v
    return x, sing


def backward_error(a: np.ndarray, x: np.ndarray, b: np.ndarray) -> float:
    """|Ax - b|_inf / (|A|_inf |x|_inf) (metrics.py:151-167)."""
    resid = float(np.abs(a @ x - b).max())
    a_inf = float(np.abs(a).sum(axis=1).max())
    x_inf = float(np.abs(x).max()) if x.size else 0.0
    den = a_inf * x_inf
    if den == 0.0:
        return 0.0 if resid == 0.0 else math.inf
    return resid / den


def recon_error(a: np.ndarray, perm: np.ndarray, L: np.ndarray, d_dense: np.ndarray) -> float:
    """max |PAP^T - L D L^T| / max |A| (tests/helpers.py:17-22)."""
    permuted = a[np.ix_(perm, perm)]
    den = float(np.abs(a).max())
    err = float(np.abs(L @ d_dense @ L.T - permuted).max())
    return err / den if den else err
