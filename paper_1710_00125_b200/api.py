"""Drop-in mirror of the reference ``randldl`` factor/solve API, backed by CUDA.

Same names, fields, argument meaning and error behaviour as the reference
(paths relative to ``/root/reference/pkg/src/randldl/``):

* :class:`FactorConfig`       factor.py:116-149
* :class:`BlockDiag`          factor.py:152-173
* :class:`Factorization`      factor.py:176-199
* :class:`GrowthStats`        metrics.py:46-65,  :class:`OpCounters` metrics.py:28-43
* :class:`SolveReport`        solve.py:25-31
* :func:`factor` / :func:`factor_robust` / :func:`reconstruct`   factor.py:637-665
* :func:`solve` / :func:`solve_many`                              solve.py:79-107

Every numerical step runs in ``librcp_b200.so`` (``include/rcp_b200.h``) on the
GPU; this module only validates arguments, draws the Gaussian sketch with the
reference's generator (numpy ``Generator(Philox(seed))``, sketch.py:39-42) so
both implementations see identical bits, moves data and maps status codes to
the reference's exceptions.  There is no CPU fallback.

The device-resident entry points :func:`factor_device` / :func:`solve_device`
take and return CUDA tensors (used by the benchmark, whose timed region starts
with the matrix already in HBM).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from enum import Enum

import numpy as np
import torch

from . import _native

__all__ = [
    "Strategy", "GrowthTracking", "FactorConfig", "BlockDiag", "Factorization", "GrowthStats",
    "OpCounters", "SolveReport", "NumericalError", "PAT_SINGLE", "PAT_PAIR_START", "PAT_PAIR_END",
    "PAT_DEFICIENT", "SBKP_ALPHA", "factor", "factor_robust", "reconstruct", "solve", "solve_many",
    "DeviceFactorization", "factor_device", "solve_device", "reconstruct_device",
]

PAT_SINGLE = 0
PAT_PAIR_START = 1
PAT_PAIR_END = 2
PAT_DEFICIENT = 3
SBKP_ALPHA = math.sqrt(2.0) / 2.0


class NumericalError(RuntimeError):
    """Raised when the factorization meets a non-finite or impossible value (factor.py:100-101)."""


class Strategy(str, Enum):
    RCP = "rcp"
    BKPP = "bkpp"
    BBK = "bbk"


class GrowthTracking(str, Enum):
    CHEAP = "cheap"
    FULL = "full"


@dataclass
class FactorConfig:
    """Knobs for :func:`factor`; validation identical to factor.py:137-149."""

    strategy: Strategy = Strategy.RCP
    p: int = 5
    b: int = 64
    q: int = 1
    seed: int = 0
    robust_r: int = 1
    track_growth: GrowthTracking = GrowthTracking.CHEAP
    audit_sketch: bool = False

    def __post_init__(self) -> None:
        self.strategy = Strategy(self.strategy)
        self.track_growth = GrowthTracking(self.track_growth)
        if self.p < 1:
            raise ValueError("sketch size p must be positive")
        if self.b < 1:
            raise ValueError("panel width b must be positive")
        if self.q not in (1, self.b):
            raise ValueError(f"q must be 1 or b={self.b}, got {self.q}")
        if self.p < self.q:
            raise ValueError(f"sketch size p={self.p} must be at least q={self.q}")
        if self.robust_r < 0:
            raise ValueError("robust_r must be non-negative")


@dataclass
class OpCounters:
    mults: int = 0
    adds: int = 0
    divs: int = 0
    comps: int = 0

    def total_flops(self) -> int:
        return self.mults + self.adds + self.divs


@dataclass
class GrowthStats:
    rho_cheap: float
    max_multiplier: float
    counters: OpCounters = field(default_factory=OpCounters)
    rho_elem: float | None = None
    rho_col: float | None = None
    L_norm1: float | None = None
    Linv_norm1: float | None = None
    snapshots: list | None = None
    sketch_drift: list | None = None
    recompute_count: int = 0


@dataclass
class BlockDiag:
    """Block diagonal factor: an ordered list of (1,1) and (2,2) arrays."""

    blocks: list

    @property
    def dim(self) -> int:
        return sum(b.shape[0] for b in self.blocks)

    def to_dense(self) -> np.ndarray:
        n = self.dim
        d = np.zeros((n, n))
        i = 0
        for blk in self.blocks:
            s = blk.shape[0]
            d[i:i + s, i:i + s] = blk
            i += s
        return d

    def max_abs(self) -> float:
        return max((float(np.abs(b).max()) for b in self.blocks), default=0.0)


@dataclass
class Factorization:
    """Result of :func:`factor`: ``A[perm][:, perm] == L @ D @ L.T``."""

    perm: np.ndarray
    L: np.ndarray
    D: BlockDiag
    pattern: np.ndarray
    stats: GrowthStats
    # The device-resident factorization this result was copied from (factor() keeps it, so
    # solve() / solve_many() do not re-upload the dense L).  Its host arrays are made
    # read-only; solve() uses the device copy only while perm / L / D / pattern are still
    # the very objects factor() returned.
    _device: object = field(default=None, repr=False, compare=False)

    @property
    def n(self) -> int:
        return self.perm.size

    @property
    def deficient_from(self) -> int | None:
        hits = np.nonzero(self.pattern == PAT_DEFICIENT)[0]
        return int(hits[0]) if hits.size else None


@dataclass
class SolveReport:
    x: np.ndarray
    singular: bool
    backward_error: float | None = None


# --------------------------------------------------------------------------- helpers

def _require_square(a: np.ndarray, name: str = "A") -> np.ndarray:
    """core.py:33-45 (shape part; symmetry / finiteness: rcp_factor_host / the device)."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError(f"{name} must be square, got shape {a.shape}")
    if a.shape[0] == 0:
        raise ValueError(f"{name} must have at least one row")
    return a


_STRATEGY_CODE = {Strategy.RCP: 0, Strategy.BKPP: 1, Strategy.BBK: 2}  # rcp_b200.h RCP_STRATEGY_*


def _eager(cfg: FactorConfig) -> bool:
    """track_growth="full" and audit_sketch force width-1 panels (factor.py:294-296)."""
    return cfg.track_growth is GrowthTracking.FULL or cfg.audit_sketch


def _native_config(cfg: FactorConfig) -> _native.RcpConfig:
    b, q = (1, 1) if _eager(cfg) else (cfg.b, cfg.q)
    return _native.RcpConfig(cfg.p, b, q, cfg.robust_r, _STRATEGY_CODE[cfg.strategy])


def _check_supported(cfg: FactorConfig, batched: bool = False) -> None:
    if batched and cfg.strategy is not Strategy.RCP:
        raise ValueError(f"the batched kernel runs strategy 'rcp' only, got {cfg.strategy.value!r}")
    if batched and _eager(cfg):
        raise ValueError("track_growth='full' / audit_sketch run through factor(), not the batched kernel")


def _raise_status(status: int, st: _native.RcpStats | None) -> None:
    if status == _native.RCP_OK:
        return
    msg = st.message.decode(errors="replace") if st is not None else ""
    if status == _native.RCP_ERR_NOT_SYMMETRIC:
        raise ValueError("A must be symmetric (exact equality of triangles)")
    if status == _native.RCP_ERR_NONFINITE_INPUT:
        raise ValueError("input matrix contains NaN or Inf")
    if status == _native.RCP_ERR_NUMERICAL:
        kind, step = int(st.num_kind), int(st.num_step)
        if kind == _native.RCP_NUM_ZERO_1X1:
            raise NumericalError("zero 1x1 pivot under a nonzero column")
        if kind == _native.RCP_NUM_SINGULAR_2X2:
            raise NumericalError("singular 2x2 pivot block")
        if kind == _native.RCP_NUM_DET_BOUND:
            raise NumericalError(f"2x2 block at step {step} violates its determinant bound")
        raise NumericalError(f"non-finite pivot data at step {step}")
    if status == _native.RCP_ERR_INVALID_ARG:
        raise ValueError(f"invalid argument ({msg})")
    if status == _native.RCP_ERR_UNSUPPORTED:
        raise ValueError(f"unsupported configuration: {msg}")
    raise RuntimeError(f"rcp_b200 failed with status {status}: {msg}")


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


# --------------------------------------------------------------------------- device API

@dataclass
class DeviceFactorization:
    """GPU-resident factorization (all tensors on the CUDA device)."""

    perm: torch.Tensor      # int64 [n]
    L: torch.Tensor         # float64 [n, n] row-major, unit lower
    d_diag: torch.Tensor    # float64 [n]
    d_off: torch.Tensor     # float64 [n]
    pattern: torch.Tensor   # int8 [n]
    stats: dict
    trace_kind: torch.Tensor | None = None
    trace_r: torch.Tensor | None = None
    host_L: torch.Tensor | None = None  # pinned copy of L streamed during the factorization

    @property
    def n(self) -> int:
        return int(self.perm.numel())

    def blocks(self) -> list:
        return _blocks_from_arrays(self.d_diag.cpu().numpy(), self.d_off.cpu().numpy(),
                                   self.pattern.cpu().numpy())

    def to_host(self) -> Factorization:
        lh = self.host_L
        if lh is None and self.n >= 2048 and self.L.is_contiguous():
            # L into (cached) pinned memory: only its lower trapezoid crosses PCIe, the host zeroes
            # the strictly upper part meanwhile (rcp_lower_to_host)
            lh = torch.empty(tuple(self.L.shape), dtype=torch.float64, pin_memory=True)
            with torch.cuda.device(self.L.device):
                status = _native.load().rcp_lower_to_host(self.n, self.L.data_ptr(), lh.data_ptr(), _stream())
            if status != _native.RCP_OK:
                raise RuntimeError(f"rcp_lower_to_host failed (status {status})")
        pattern = self.pattern.cpu().numpy().astype(np.int8)
        blocks = _blocks_from_arrays(self.d_diag.cpu().numpy(), self.d_off.cpu().numpy(), pattern)
        s = self.stats
        stats = GrowthStats(rho_cheap=s["rho_cheap"], max_multiplier=s["max_multiplier"],
                            counters=OpCounters(*s["counters"]), recompute_count=s["recompute_count"],
                            rho_elem=s.get("rho_elem"), rho_col=s.get("rho_col"), L_norm1=s.get("L_norm1"),
                            Linv_norm1=s.get("Linv_norm1"), snapshots=s.get("snapshots"),
                            sketch_drift=s.get("sketch_drift"))
        perm = self.perm.cpu().numpy().astype(np.int64)
        if lh is not None:
            L = lh.numpy()
        else:
            L = self.L.cpu().numpy()
        return Factorization(perm=perm, L=L, D=BlockDiag(blocks), pattern=pattern, stats=stats)


def _blocks_from_arrays(dd: np.ndarray, doff: np.ndarray, pattern: np.ndarray) -> list:
    """The reference's list of (1,1)/(2,2) D blocks (factor.py:153-199) from the flat arrays.
    The blocks are views of two stacked arrays built vectorised (a Python-level np.array per
    block costs ~40 ms at n = 32768)."""
    n = pattern.size
    is2 = pattern == PAT_PAIR_START
    if n:
        is2[-1] = False
    consumed = np.zeros(n, dtype=bool)
    consumed[1:] = is2[:-1]
    starts = np.flatnonzero(~consumed)
    s2 = starts[is2[starts]]
    s1 = starts[~is2[starts]]
    two = np.empty((s2.size, 2, 2))
    two[:, 0, 0] = dd[s2]
    two[:, 0, 1] = doff[s2]
    two[:, 1, 0] = doff[s2]
    two[:, 1, 1] = dd[s2 + 1]
    one = np.ascontiguousarray(dd[s1], dtype=np.float64).reshape(-1, 1, 1)
    kind = is2[starts].tolist()
    blocks = []
    i1 = i2 = 0
    for k2 in kind:
        if k2:
            blocks.append(two[i2])
            i2 += 1
        else:
            blocks.append(one[i1])
            i1 += 1
    return blocks


class _NormalStream:
    """The reference's advancing generator (sketch.py:63-84) as a C callback."""

    def __init__(self, seed: int):
        self.gen = np.random.Generator(np.random.Philox(seed))
        self.draws = 0
        self.pending_skip = None  # (p, n): Omega was supplied; discard its draw on first use

        def _cb(_ctx, rows, cols, out):
            try:
                if self.pending_skip is not None:  # rare path (guard recompute): catch up first
                    self.gen.standard_normal(self.pending_skip)
                    self.pending_skip = None
                z = self.gen.standard_normal((int(rows), int(cols)))
                ctypes.memmove(out, z.ctypes.data, z.nbytes)
                self.draws += 1
                return 0
            except Exception:  # pragma: no cover - reported as a status code
                return 1

        self.cfunc = _native.DRAW_FN(_cb)

    def first(self, p: int, n: int) -> np.ndarray:
        return self.gen.standard_normal((p, n))

    def skip_first(self, p: int, n: int) -> None:
        """Omega was drawn elsewhere: advance past it lazily (only a recompute needs it)."""
        self.pending_skip = (p, n)


def _config(cfg: FactorConfig | None, overrides: dict) -> FactorConfig:
    if cfg is not None and overrides:
        raise ValueError("pass either cfg or keyword overrides, not both")
    if cfg is None:
        cfg = FactorConfig(**overrides)
    elif not isinstance(cfg, FactorConfig):  # e.g. the reference's own randldl.FactorConfig
        cfg = FactorConfig(strategy=getattr(cfg.strategy, "value", cfg.strategy), p=cfg.p, b=cfg.b, q=cfg.q,
                           seed=cfg.seed, robust_r=cfg.robust_r,
                           track_growth=getattr(cfg.track_growth, "value", cfg.track_growth),
                           audit_sketch=bool(cfg.audit_sketch))
    return cfg


def workspace_bytes(n: int, cfg: FactorConfig) -> int:
    lib = _native.load()
    c = _native_config(cfg)
    return int(lib.rcp_workspace_bytes(n, ctypes.byref(c)))


def factor_device(a: torch.Tensor, cfg: FactorConfig | None = None, *, omega: torch.Tensor | None = None,
                  trace: bool = False, workspace: torch.Tensor | tuple | None = None,
                  out: DeviceFactorization | None = None, world: int = 1, emulate: bool = False,
                  l_host: torch.Tensor | None = None, **overrides) -> DeviceFactorization:
    """Factor a CUDA float64 symmetric matrix; results stay on the device.

    ``omega`` (p x n, CUDA float64) may be passed pre-drawn; it must then be the
    first draw of ``Generator(Philox(cfg.seed))`` for results to match the
    reference.  ``workspace``/``out`` let a caller reuse device buffers (``workspace`` may also be a
    raw ``(device_pointer, nbytes)`` pair).  ``world > 1`` shares every trailing update with
    ``world - 1`` other GPUs running :func:`paper_1710_00125_b200.dist.schur_worker`
    (``emulate=True``: their parts run on this device, for testing; results are identical).
    ``l_host`` (pinned CPU float64 n x n, single GPU): L is also streamed into it while the
    factorization runs (``rcp_factor_host_l``); :meth:`DeviceFactorization.to_host` then uses it.
    """
    cfg = _config(cfg, overrides)
    _check_supported(cfg)
    lib = _native.load()
    if a.dim() != 2 or a.shape[0] != a.shape[1]:
        raise ValueError(f"A must be square, got shape {tuple(a.shape)}")
    n = int(a.shape[0])
    if n == 0:
        raise ValueError("A must have at least one row")
    if a.dtype != torch.float64 or not a.is_cuda:
        raise ValueError("factor_device expects a CUDA float64 tensor")
    if a.stride(1) != 1 and a.stride(0) != 1:
        a = a.contiguous()
    lda = a.stride(0) if a.stride(1) == 1 else a.stride(1)
    dev = a.device
    normals = _NormalStream(cfg.seed)
    if cfg.strategy is not Strategy.RCP:
        omega = None  # bkpp / bbk draw no sketch (factor.py:306-310)
    elif omega is None:
        omega = torch.from_numpy(normals.first(cfg.p, n)).to(dev)
    else:
        if tuple(omega.shape) != (cfg.p, n):
            raise ValueError(f"omega must have shape ({cfg.p}, {n}), got {tuple(omega.shape)}")
        normals.skip_first(cfg.p, n)  # advance past the supplied first draw when needed
        omega = omega.to(device=dev, dtype=torch.float64).contiguous()
    c = _native_config(cfg)
    need = int(lib.rcp_workspace_bytes(n, ctypes.byref(c)))
    if isinstance(workspace, tuple):
        ws_ptr, ws_bytes = int(workspace[0]), int(workspace[1])
        if ws_bytes < need:
            raise ValueError("workspace too small")
    else:
        if workspace is None or workspace.numel() < need:
            workspace = torch.empty(need, dtype=torch.uint8, device=dev)
        ws_ptr, ws_bytes = workspace.data_ptr(), workspace.numel()
    wws = None
    if world > 1 and emulate:
        wws = torch.empty(int(lib.rcp_worker_workspace_bytes(n, ctypes.byref(c))) * (world - 1),
                          dtype=torch.uint8, device=dev)
    if out is None:
        out = DeviceFactorization(
            perm=torch.empty(n, dtype=torch.int64, device=dev),
            L=torch.empty((n, n), dtype=torch.float64, device=dev),
            d_diag=torch.empty(n, dtype=torch.float64, device=dev),
            d_off=torch.empty(n, dtype=torch.float64, device=dev),
            pattern=torch.empty(n, dtype=torch.int8, device=dev),
            stats={},
        )
    if trace:
        out.trace_kind = torch.empty(n, dtype=torch.int8, device=dev)
        out.trace_r = torch.empty(n, dtype=torch.int32, device=dev)
    st = _native.RcpStats()
    diag = None
    if _eager(cfg):
        if world != 1 or l_host is not None:
            raise ValueError("track_growth='full' / audit_sketch run on a single GPU without l_host")
        cap = n + 1
        snaps = torch.zeros(cap, 2, dtype=torch.float64, device=dev)
        drift = torch.zeros(cap, dtype=torch.float64, device=dev)
        omega_orig = (torch.empty(cfg.p, n, dtype=torch.float64, device=dev)
                      if cfg.audit_sketch and cfg.strategy is Strategy.RCP else None)
        diag = _native.RcpDiag(int(cfg.track_growth is GrowthTracking.FULL), int(cfg.audit_sketch),
                               snaps.data_ptr(), drift.data_ptr(), _ptr(omega_orig), cap, 0, 0)
    with torch.cuda.device(dev):
        if diag is not None:
            out.host_L = None
            status = lib.rcp_factor_diag(
                ctypes.byref(c), n, a.data_ptr(), lda, 0 if omega is None else omega.data_ptr(), normals.cfunc, None,
                ws_ptr, ws_bytes, out.perm.data_ptr(), out.L.data_ptr(),
                out.d_diag.data_ptr(), out.d_off.data_ptr(), out.pattern.data_ptr(),
                _ptr(out.trace_kind if trace else None), _ptr(out.trace_r if trace else None),
                ctypes.byref(st), ctypes.byref(diag), _stream())
            _raise_status(status, st)
        elif l_host is not None:
            if world != 1 or l_host.dtype != torch.float64 or tuple(l_host.shape) != (n, n) \
                    or not l_host.is_pinned() or not l_host.is_contiguous():
                raise ValueError("l_host must be a contiguous pinned float64 (n, n) tensor (single GPU)")
            status = lib.rcp_factor_host_l(
                ctypes.byref(c), n, a.data_ptr(), lda, 0 if omega is None else omega.data_ptr(), normals.cfunc, None,
                ws_ptr, ws_bytes, out.perm.data_ptr(), out.L.data_ptr(),
                out.d_diag.data_ptr(), out.d_off.data_ptr(), out.pattern.data_ptr(),
                _ptr(out.trace_kind if trace else None), _ptr(out.trace_r if trace else None),
                ctypes.byref(st), l_host.data_ptr(), _stream())
            _raise_status(status, st)
            out.host_L = l_host
        else:
            out.host_L = None
            status = lib.rcp_factor_dist(
                ctypes.byref(c), n, a.data_ptr(), lda, 0 if omega is None else omega.data_ptr(), normals.cfunc, None,
                ws_ptr, ws_bytes, out.perm.data_ptr(), out.L.data_ptr(),
                out.d_diag.data_ptr(), out.d_off.data_ptr(), out.pattern.data_ptr(),
                _ptr(out.trace_kind if trace else None), _ptr(out.trace_r if trace else None),
                ctypes.byref(st), int(world), 1 if emulate else 0, _ptr(wws), 0 if wws is None else wws.numel(),
                _stream())
            _raise_status(status, st)
    out.stats = _stats_dict(st)
    if diag is not None:
        out.stats.update(_diag_stats(cfg, a, out, diag, snaps, drift))
    return out


def _max_col_norm(m: torch.Tensor) -> float:
    """norm_1_2 (metrics.py:83-90): the largest scaled Euclidean column norm (core.py:122-142)."""
    if m.numel() == 0:
        return 0.0
    scale = m.abs().amax(dim=0)
    safe = torch.where(scale > 0, scale, torch.ones_like(scale))
    return float((scale * torch.sqrt(((m / safe) ** 2).sum(dim=0))).max())


def _diag_stats(cfg, a, out, diag, snaps, drift) -> dict:
    """GrowthStats' diagnostic fields (factor.py:514-531; metrics.py:93-127) from the device
    snapshots / drift; rho_elem / rho_col, ||L||_1 and ||L^-1||_1 only with snapshots."""
    res = {"snapshots": None, "sketch_drift": None}
    if cfg.track_growth is GrowthTracking.FULL:
        k = int(diag.n_snapshots)
        res["snapshots"] = [tuple(map(float, r)) for r in snaps[:k].cpu().numpy()]
    if cfg.audit_sketch:
        k = int(diag.n_drift)
        norm12 = _max_col_norm(a) if cfg.strategy is Strategy.RCP else 0.0
        vals = drift[:k].cpu().numpy() if cfg.strategy is Strategy.RCP else np.zeros(0)
        res["sketch_drift"] = [float(v / norm12) if norm12 else float(v) for v in vals]
    if res["snapshots"]:
        sn = np.array(res["snapshots"])
        if sn[0, 0] == 0.0 or sn[0, 1] == 0.0:
            raise ValueError("snapshot of the input matrix is zero; growth undefined")
        res["rho_elem"] = float(sn[:, 0].max() / sn[0, 0])
        res["rho_col"] = float(sn[:, 1].max() / sn[0, 1])
        L = out.L
        res["L_norm1"] = float(L.abs().sum(dim=0).max())
        eye = torch.eye(L.shape[0], dtype=L.dtype, device=L.device)
        linv = torch.linalg.solve_triangular(L, eye, upper=False, unitriangular=True)
        res["Linv_norm1"] = float(linv.abs().sum(dim=0).max())
    return res


def _stats_dict(st) -> dict:
    return {
        "rho_cheap": float(st.rho_cheap), "max_multiplier": float(st.max_multiplier),
        "amax": float(st.amax), "dmax": float(st.dmax), "recompute_count": int(st.recompute_count),
        "n_panels": int(st.n_panels), "n_steps": int(st.n_steps), "n_2x2": int(st.n_2x2),
        "deficient_from": int(st.deficient_from), "t_factor_ms": float(st.t_factor_ms),
        "t_schur_ms": float(st.t_schur_ms), "t_panel_ms": float(st.t_panel_ms),
        "schur_flops": float(st.schur_flops), "n_launches": int(st.n_launches),
        "counters": (int(st.mults), int(st.adds), int(st.divs), int(st.comps)),
        "panel_prof_ms": dict(zip(("qrcp", "qrcp_exchange", "sbkp_gemv", "sbkp_exchange", "sbkp_eliminate",
                                   "next_pivot", "qrcp_reflect", "total", "sbkp_local_argmax",
                                   "qrcp_local_argmax", "qrcp_householder"),
                                  [round(float(x), 3) for x in st.panel_prof_ms])),
    }


def solve_device(f: DeviceFactorization, b: torch.Tensor, x: torch.Tensor | None = None,
                 workspace: torch.Tensor | None = None) -> tuple[torch.Tensor, bool]:
    """x = A^-1 b on the device; b is (n,) or (n, k) CUDA float64."""
    lib = _native.load()
    n = f.n
    if b.dim() not in (1, 2) or b.shape[0] != n:
        raise ValueError(f"right-hand side shape {tuple(b.shape)} does not match n={n}")
    vec = b.dim() == 1
    dev = f.L.device
    b = b.to(device=dev, dtype=torch.float64)  # the kernels read float64 on the factor's device
    nrhs = 1 if vec else int(b.shape[1])
    if nrhs == 0:
        return (torch.empty_like(b) if x is None else x), False
    bc = b.reshape(n, 1) if vec else b
    bcol = bc.t().contiguous()  # (k, n): column-major n x k
    xcol = torch.empty_like(bcol)
    need = int(lib.rcp_solve_workspace_bytes(n, nrhs))
    if workspace is None or workspace.numel() < need or workspace.device != dev:
        workspace = torch.empty(need, dtype=torch.uint8, device=dev)
    sing = ctypes.c_int32(0)
    with torch.cuda.device(dev):
        status = lib.rcp_solve(n, f.perm.data_ptr(), f.L.data_ptr(), f.d_diag.data_ptr(), f.d_off.data_ptr(),
                               f.pattern.data_ptr(), nrhs, bcol.data_ptr(), xcol.data_ptr(), workspace.data_ptr(),
                               workspace.numel(), ctypes.byref(sing), _stream())
    _raise_status(status, None)
    res = xcol.t()
    res = res.reshape(n) if vec else res.contiguous()
    if x is not None:
        x.copy_(res)
        res = x
    return res, bool(sing.value)


def reconstruct_device(f: DeviceFactorization) -> torch.Tensor:
    lib = _native.load()
    n = f.n
    out = torch.empty((n, n), dtype=torch.float64, device=f.L.device)
    with torch.cuda.device(f.L.device):
        status = lib.rcp_reconstruct(n, f.L.data_ptr(), f.d_diag.data_ptr(), f.d_off.data_ptr(),
                                     f.pattern.data_ptr(), out.data_ptr(), _stream())
    _raise_status(status, None)
    return out


# --------------------------------------------------------------------------- host API

def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise _native.NativeUnavailable("no CUDA device: the B200 build has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def factor(a: np.ndarray, cfg: FactorConfig | None = None, **overrides) -> Factorization:
    """Factor a dense symmetric matrix as ``A[perm][:, perm] = L D L.T`` (factor.py:637-647)."""
    cfg = _config(cfg, overrides)
    a = _require_square(a)
    _check_supported(cfg)
    _native.load()
    if _eager(cfg):  # diagnostics: exact symmetry / finiteness are checked on the device
        dev = _device()
        df = factor_device(torch.from_numpy(np.ascontiguousarray(a)).to(dev), cfg)
    else:
        df = _factor_host(np.ascontiguousarray(a), cfg, _device())
    return _attach(df.to_host(), df)


def _attach(f: Factorization, df: DeviceFactorization) -> Factorization:
    for arr in (f.perm, f.L, f.pattern):
        arr.flags.writeable = False
    f._device = (df, f.perm, f.L, f.D, f.pattern)
    return f


def _attached(f: Factorization) -> DeviceFactorization | None:
    ref = getattr(f, "_device", None)
    if ref is None:
        return None
    df, perm, L, D, pattern = ref
    if f.perm is perm and f.L is L and f.D is D and f.pattern is pattern:
        return df
    return None


def _factor_host(a: np.ndarray, cfg: FactorConfig, dev: torch.device) -> DeviceFactorization:
    """factor() on a C-contiguous float64 host array through ``rcp_factor_host``: the lower
    trapezoid goes to the device, exact symmetry is checked on host threads meanwhile, Omega is
    the first draw of the stream (drawn during the copies) and, for n >= 2048, L streams back into
    pinned memory while later panels run."""
    lib = _native.load()
    n = int(a.shape[0])
    if n == 0:
        raise ValueError("A must have at least one row")
    c = _native_config(cfg)
    workspace = torch.empty(int(lib.rcp_workspace_bytes(n, ctypes.byref(c))), dtype=torch.uint8, device=dev)
    out = DeviceFactorization(
        perm=torch.empty(n, dtype=torch.int64, device=dev),
        L=torch.empty((n, n), dtype=torch.float64, device=dev),
        d_diag=torch.empty(n, dtype=torch.float64, device=dev),
        d_off=torch.empty(n, dtype=torch.float64, device=dev),
        pattern=torch.empty(n, dtype=torch.int8, device=dev),
        stats={},
    )
    lh = torch.empty((n, n), dtype=torch.float64, pin_memory=True) if n >= 2048 else None
    normals = _NormalStream(cfg.seed)
    st = _native.RcpStats()
    with torch.cuda.device(dev):
        status = lib.rcp_factor_host(
            ctypes.byref(c), n, a.ctypes.data, n, None, normals.cfunc, None,
            workspace.data_ptr(), workspace.numel(), out.perm.data_ptr(), out.L.data_ptr(),
            out.d_diag.data_ptr(), out.d_off.data_ptr(), out.pattern.data_ptr(), None, None,
            ctypes.byref(st), _ptr(lh), _stream())
    _raise_status(status, st)
    out.host_L = lh
    out.stats = _stats_dict(st)
    return out


def factor_robust(a: np.ndarray, cfg: FactorConfig | None = None, **overrides) -> Factorization:
    """Like :func:`factor` with the sketch-collapse guard always armed (factor.py:650-660)."""
    cfg = _config(cfg, overrides)
    if cfg.strategy is not Strategy.RCP:
        raise ValueError("the guarded mode requires the rcp strategy")
    if cfg.robust_r < 1:
        raise ValueError("factor_robust needs robust_r >= 1")
    return factor(a, cfg)


def reconstruct(f: Factorization) -> np.ndarray:
    """Assemble ``L @ D @ L.T`` (factor.py:663-665)."""
    return f.L @ f.D.to_dense() @ f.L.T


def _device_from_host(f: Factorization) -> DeviceFactorization:
    dev = _device()
    n = f.n
    dd = np.zeros(n)
    doff = np.zeros(n)
    i = 0
    for blk in f.D.blocks:
        if blk.shape[0] == 1:
            dd[i] = blk[0, 0]
            i += 1
        else:
            dd[i], dd[i + 1], doff[i] = blk[0, 0], blk[1, 1], blk[1, 0]
            i += 2
    return DeviceFactorization(
        perm=torch.from_numpy(np.asarray(f.perm, dtype=np.int64)).to(dev),
        L=torch.from_numpy(np.ascontiguousarray(f.L, dtype=np.float64)).to(dev),
        d_diag=torch.from_numpy(dd).to(dev), d_off=torch.from_numpy(doff).to(dev),
        pattern=torch.from_numpy(np.asarray(f.pattern, dtype=np.int8)).to(dev), stats={})


def _backward_error(a: np.ndarray, x: np.ndarray, b: np.ndarray) -> float:
    """|Ax - b|_inf / (|A|_inf |x|_inf) (metrics.py:151-167)."""
    resid = float(np.abs(a @ x - b).max())
    a_inf = float(np.abs(a).sum(axis=1).max())
    x_inf = float(np.abs(x).max()) if x.size else 0.0
    den = a_inf * x_inf
    if den == 0.0:
        return 0.0 if resid == 0.0 else math.inf
    return resid / den


def solve(f: Factorization, b: np.ndarray, a: np.ndarray | None = None) -> SolveReport:
    """Solve ``A x = b`` given ``factor(A)`` (solve.py:79-92)."""
    b = np.asarray(b, dtype=np.float64)
    if b.shape != (f.n,):
        raise ValueError(f"right-hand side shape {b.shape} does not match n={f.n}")
    df = _attached(f) or _device_from_host(f)
    xd, sing = solve_device(df, torch.from_numpy(b).to(df.L.device))
    x = xd.cpu().numpy()
    err = _backward_error(np.asarray(a, dtype=np.float64), x, b) if a is not None else None
    return SolveReport(x=x, singular=sing, backward_error=err)


def solve_many(f: Factorization, b_rhs: np.ndarray) -> np.ndarray:
    """Column-wise :func:`solve` (solve.py:95-107)."""
    b_rhs = np.asarray(b_rhs, dtype=np.float64)
    if b_rhs.ndim != 2 or b_rhs.shape[0] != f.n:
        raise ValueError(f"right-hand sides must be ({f.n}, k), got {b_rhs.shape}")
    df = _attached(f) or _device_from_host(f)
    xd, _ = solve_device(df, torch.from_numpy(b_rhs).to(df.L.device))
    return xd.cpu().numpy()
