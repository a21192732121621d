"""Batched factor/solve of many small independent matrices (BASELINE config C5).

The reference has no batched entry point: a user factors a stack of matrices by
calling ``randldl.factor(a_i, cfg)`` in a loop (``factor.py:637-647``; one
``FactorConfig``, hence one seed, for all of them) and ``randldl.solve`` per
matrix (``solve.py:79-92``).  :func:`factor_batched` / :func:`solve_batched`
return exactly what that loop returns, computed by one persistent CUDA kernel
(``csrc/batched.cu``, C ABI ``rcp_factor_batched``) with no host round trip
per matrix.

Sketch stream: every ``factor`` call starts ``Generator(Philox(cfg.seed))``
afresh, draws Omega (``p x n``) and, on each guard recompute, the next ``p x m``
normals (``sketch.py:63-84``).  All matrices therefore read the same stream;
it is drawn once on the host and uploaded, with a budget of ``extra_draws``
full-size recomputes per matrix.  A matrix needing more (not seen on C5: its
scaled members recompute exactly once) is re-run through the single-matrix
path, which draws on demand.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .api import (BlockDiag, DeviceFactorization, Factorization, FactorConfig, GrowthStats, NumericalError,
                  OpCounters, _blocks_from_arrays, _check_supported, _config, _device, _raise_status, _stream,
                  factor_device)

__all__ = ["BatchedDeviceFactorization", "factor_batched_device", "factor_batched_host", "factor_batched", "solve_batched_device",
           "solve_batched", "batched_workspace_bytes", "normal_stream", "shard_range", "factor_batched_sharded"]

MAX_N = 256


@dataclass
class BatchedDeviceFactorization:
    """``count`` GPU-resident factorizations (leading dimension = matrix index)."""

    perm: torch.Tensor      # int64 [count, n]
    L: torch.Tensor         # float64 [count, n, n], row-major unit lower
    d_diag: torch.Tensor    # float64 [count, n]
    d_off: torch.Tensor     # float64 [count, n]
    pattern: torch.Tensor   # int8 [count, n]
    stats: np.ndarray       # structured array (_native.BATCH_STATS_DTYPE) [count]

    @property
    def count(self) -> int:
        return int(self.perm.shape[0])

    @property
    def n(self) -> int:
        return int(self.perm.shape[1])

    def factorization(self, i: int) -> Factorization:
        return self.to_host(range(i, i + 1))[0]

    def to_host(self, which=None) -> list:
        idx = range(self.count) if which is None else which
        sel = torch.as_tensor(list(idx), dtype=torch.int64, device=self.perm.device)
        perm = self.perm.index_select(0, sel).cpu().numpy()
        L = self.L.index_select(0, sel).cpu().numpy()
        dd = self.d_diag.index_select(0, sel).cpu().numpy()
        doff = self.d_off.index_select(0, sel).cpu().numpy()
        pat = self.pattern.index_select(0, sel).cpu().numpy().astype(np.int8)
        out = []
        for j, i in enumerate(idx):
            s = self.stats[i]
            stats = GrowthStats(rho_cheap=float(s["rho_cheap"]), max_multiplier=float(s["max_multiplier"]),
                                counters=OpCounters(int(s["mults"]), int(s["adds"]), int(s["divs"]),
                                                    int(s["comps"])),
                                recompute_count=int(s["recompute_count"]))
            out.append(Factorization(perm=perm[j].astype(np.int64), L=L[j],
                                     D=BlockDiag(_blocks_from_arrays(dd[j], doff[j], pat[j])),
                                     pattern=pat[j], stats=stats))
        return out


def _cfg_struct(cfg: FactorConfig) -> _native.RcpConfig:
    return _native.RcpConfig(cfg.p, cfg.b, cfg.q, cfg.robust_r, 0)


def batched_workspace_bytes(n: int, cfg: FactorConfig) -> int:
    lib = _native.load()
    c = _cfg_struct(cfg)
    return int(lib.rcp_batched_workspace_bytes(n, ctypes.byref(c)))


def normal_stream(cfg: FactorConfig, n: int, extra_draws: int = 4) -> np.ndarray:
    """The first ``p*n*(1 + extra_draws)`` values of ``Generator(Philox(cfg.seed)).standard_normal``."""
    gen = np.random.Generator(np.random.Philox(cfg.seed))
    return gen.standard_normal(cfg.p * n * (1 + extra_draws))


def _supported(cfg: FactorConfig, n: int) -> bool:
    return n <= MAX_N and cfg.q == cfg.b and cfg.q > 1 and cfg.b <= 32 and cfg.p <= 64


def _raise_matrix(i: int, s) -> None:
    st = _native.RcpStats()
    st.num_kind = int(s["num_kind"])
    st.num_step = int(s["num_step"])
    try:
        _raise_status(int(s["status"]), st)
    except (ValueError, NumericalError) as exc:
        raise type(exc)(f"matrix {i}: {exc}") from None


def factor_batched_device(a: torch.Tensor, cfg: FactorConfig | None = None, *, normals: torch.Tensor | None = None,
                          extra_draws: int = 4, workspace: torch.Tensor | None = None,
                          out: BatchedDeviceFactorization | None = None, check: bool = True,
                          **overrides) -> BatchedDeviceFactorization:
    """Factor ``a[i]`` (CUDA float64 ``[count, n, n]``, each exactly symmetric) for every i.

    Results equal ``[factor(a[i], cfg) for i in range(count)]``.  With ``check`` the first
    failing matrix raises the reference's exception (prefixed with its index); matrices that
    exhaust the pre-drawn normal stream are re-run through :func:`factor_device`.
    """
    cfg = _config(cfg, overrides)
    _check_supported(cfg, batched=True)
    lib = _native.load()
    if a.dim() != 3 or a.shape[1] != a.shape[2]:
        raise ValueError(f"expected a [count, n, n] stack, got shape {tuple(a.shape)}")
    if a.dtype != torch.float64 or not a.is_cuda:
        raise ValueError("factor_batched_device expects a CUDA float64 tensor")
    count, n = int(a.shape[0]), int(a.shape[1])
    if n == 0:
        raise ValueError("A must have at least one row")
    if not a.is_contiguous():  # the kernel reads matrix i at a + i * n * n
        a = a.contiguous()
    dev = a.device
    if out is None:
        out = BatchedDeviceFactorization(
            perm=torch.empty(count, n, dtype=torch.int64, device=dev),
            L=torch.empty(count, n, n, dtype=torch.float64, device=dev),
            d_diag=torch.empty(count, n, dtype=torch.float64, device=dev),
            d_off=torch.empty(count, n, dtype=torch.float64, device=dev),
            pattern=torch.empty(count, n, dtype=torch.int8, device=dev),
            stats=np.zeros(count, dtype=_native.BATCH_STATS_DTYPE))
    if not _supported(cfg, n):
        # outside the batched kernel's on-chip limits: the single-matrix GPU path, per matrix
        for i in range(count):
            f = factor_device(a[i], cfg)
            _copy_single(out, i, f)
        return out
    if normals is None:
        normals = torch.from_numpy(normal_stream(cfg, n, extra_draws)).to(dev)
    if workspace is None:
        workspace = torch.empty(batched_workspace_bytes(n, cfg), dtype=torch.uint8, device=dev)
    mstats = torch.empty(count * ctypes.sizeof(_native.RcpBatchStats), dtype=torch.uint8, device=dev)
    c = _cfg_struct(cfg)
    status = lib.rcp_factor_batched(ctypes.byref(c), count, n, a.data_ptr(), n, n * n, normals.data_ptr(),
                                    normals.numel(), workspace.data_ptr(), workspace.numel(), out.perm.data_ptr(),
                                    out.L.data_ptr(), out.d_diag.data_ptr(), out.d_off.data_ptr(),
                                    out.pattern.data_ptr(), mstats.data_ptr(), _stream())
    _raise_status(status, None)
    out.stats = mstats.cpu().numpy().view(_native.BATCH_STATS_DTYPE).copy()
    redo = np.nonzero(out.stats["status"] == _native.RCP_ERR_NEED_NORMALS)[0]
    for i in redo:
        f = factor_device(a[int(i)], cfg)
        _copy_single(out, int(i), f)
    if check:
        bad = np.nonzero(out.stats["status"] != _native.RCP_OK)[0]
        if bad.size:
            i = int(bad[0])
            _raise_matrix(i, out.stats[i])
    return out


def _copy_single(out: BatchedDeviceFactorization, i: int, f: DeviceFactorization) -> None:
    out.perm[i].copy_(f.perm)
    out.L[i].copy_(f.L)
    out.d_diag[i].copy_(f.d_diag)
    out.d_off[i].copy_(f.d_off)
    out.pattern[i].copy_(f.pattern)
    s = f.stats
    rec = out.stats[i]
    rec["status"] = _native.RCP_OK
    rec["recompute_count"] = s["recompute_count"]
    rec["deficient_from"] = s["deficient_from"]
    rec["n_2x2"] = s["n_2x2"]
    rec["n_steps"] = s["n_steps"]
    rec["n_panels"] = s["n_panels"]
    rec["rho_cheap"] = s["rho_cheap"]
    rec["max_multiplier"] = s["max_multiplier"]
    rec["amax"] = s["amax"]
    rec["dmax"] = s["dmax"]
    rec["mults"], rec["adds"], rec["divs"], rec["comps"] = s["counters"]


def factor_batched_host(a: torch.Tensor, cfg: FactorConfig | None = None, *, chunk: int = 296,
                        normals: torch.Tensor | None = None, extra_draws: int = 4,
                        workspace: torch.Tensor | None = None, out: BatchedDeviceFactorization | None = None,
                        check: bool = True, **overrides) -> BatchedDeviceFactorization:
    """Factor a host-resident stack ``a`` (CPU float64 ``[count, n, n]``, ideally pinned) into host memory.

    Same results as :func:`factor_batched_device` on ``a.cuda()``, with the PCIe traffic hidden
    behind the kernel: the batch runs in chunks of ``chunk`` matrices over two device slots, the
    upload of chunk i+1 (copy stream), the factorization of chunk i (compute stream) and the
    download of chunk i-1's perm/L/D/pattern (second copy stream) overlap.  The returned
    :class:`BatchedDeviceFactorization` holds pinned host tensors (``to_host`` works on it).
    """
    cfg = _config(cfg, overrides)
    _check_supported(cfg, batched=True)
    if a.dim() != 3 or a.shape[1] != a.shape[2]:
        raise ValueError(f"expected a [count, n, n] stack, got shape {tuple(a.shape)}")
    if a.dtype != torch.float64 or a.is_cuda:
        raise ValueError("factor_batched_host expects a host (CPU) float64 tensor")
    count, n = int(a.shape[0]), int(a.shape[1])
    if n == 0:
        raise ValueError("A must have at least one row")
    a = a.contiguous()
    dev = _device()
    pin = torch.cuda.is_available()
    if not _supported(cfg, n):  # single-matrix GPU path per matrix, results copied into `out`
        res = factor_batched_device(a.to(dev), cfg, check=check)
        if out is None:
            out = BatchedDeviceFactorization(
                perm=torch.empty(count, n, dtype=torch.int64, pin_memory=pin),
                L=torch.empty(count, n, n, dtype=torch.float64, pin_memory=pin),
                d_diag=torch.empty(count, n, dtype=torch.float64, pin_memory=pin),
                d_off=torch.empty(count, n, dtype=torch.float64, pin_memory=pin),
                pattern=torch.empty(count, n, dtype=torch.int8, pin_memory=pin),
                stats=np.zeros(count, dtype=_native.BATCH_STATS_DTYPE))
        for name in ("perm", "L", "d_diag", "d_off", "pattern"):
            getattr(out, name).copy_(getattr(res, name))
        out.stats = res.stats
        return out
    lib = _native.load()
    if out is None:
        out = BatchedDeviceFactorization(
            perm=torch.empty(count, n, dtype=torch.int64, pin_memory=pin),
            L=torch.empty(count, n, n, dtype=torch.float64, pin_memory=pin),
            d_diag=torch.empty(count, n, dtype=torch.float64, pin_memory=pin),
            d_off=torch.empty(count, n, dtype=torch.float64, pin_memory=pin),
            pattern=torch.empty(count, n, dtype=torch.int8, pin_memory=pin),
            stats=np.zeros(count, dtype=_native.BATCH_STATS_DTYPE))
    if normals is None:
        normals = torch.from_numpy(normal_stream(cfg, n, extra_draws)).to(dev)
    if workspace is None:
        workspace = torch.empty(batched_workspace_bytes(n, cfg), dtype=torch.uint8, device=dev)
    chunk = max(1, min(chunk, count))
    ssz = ctypes.sizeof(_native.RcpBatchStats)
    mstats = torch.empty(count * ssz, dtype=torch.uint8, device=dev)
    slots = [dict(a=torch.empty(chunk, n, n, dtype=torch.float64, device=dev),
                  L=torch.empty(chunk, n, n, dtype=torch.float64, device=dev),
                  perm=torch.empty(chunk, n, dtype=torch.int64, device=dev),
                  dd=torch.empty(chunk, n, dtype=torch.float64, device=dev),
                  doff=torch.empty(chunk, n, dtype=torch.float64, device=dev),
                  pat=torch.empty(chunk, n, dtype=torch.int8, device=dev)) for _ in range(2)]
    main = torch.cuda.current_stream(dev)
    up, comp, down = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    for s in (up, comp, down):
        s.wait_stream(main)  # normals / workspace / slots were made on the caller's stream
    ev_up = [torch.cuda.Event() for _ in range(2)]
    ev_comp = [torch.cuda.Event() for _ in range(2)]
    ev_down = [torch.cuda.Event() for _ in range(2)]
    c = _cfg_struct(cfg)
    for i, c0 in enumerate(range(0, count, chunk)):
        c1 = min(count, c0 + chunk)
        m, k, sl = c1 - c0, i % 2, slots[i % 2]
        if i >= 2:
            up.wait_event(ev_comp[k])     # slot k's A was consumed by chunk i-2
        with torch.cuda.stream(up):
            sl["a"][:m].copy_(a[c0:c1], non_blocking=True)
        ev_up[k].record(up)
        comp.wait_event(ev_up[k])
        if i >= 2:
            comp.wait_event(ev_down[k])   # slot k's outputs were downloaded
        status = lib.rcp_factor_batched(ctypes.byref(c), m, n, sl["a"].data_ptr(), n, n * n, normals.data_ptr(),
                                        normals.numel(), workspace.data_ptr(), workspace.numel(),
                                        sl["perm"].data_ptr(), sl["L"].data_ptr(), sl["dd"].data_ptr(),
                                        sl["doff"].data_ptr(), sl["pat"].data_ptr(),
                                        mstats.data_ptr() + c0 * ssz, comp.cuda_stream)
        _raise_status(status, None)
        ev_comp[k].record(comp)
        down.wait_event(ev_comp[k])
        with torch.cuda.stream(down):
            out.L[c0:c1].copy_(sl["L"][:m], non_blocking=True)
            out.perm[c0:c1].copy_(sl["perm"][:m], non_blocking=True)
            out.d_diag[c0:c1].copy_(sl["dd"][:m], non_blocking=True)
            out.d_off[c0:c1].copy_(sl["doff"][:m], non_blocking=True)
            out.pattern[c0:c1].copy_(sl["pat"][:m], non_blocking=True)
        ev_down[k].record(down)
    down.synchronize()
    comp.synchronize()
    out.stats = mstats.cpu().numpy().view(_native.BATCH_STATS_DTYPE).copy()
    redo = np.nonzero(out.stats["status"] == _native.RCP_ERR_NEED_NORMALS)[0]
    for i in redo:
        f = factor_device(a[int(i)].to(dev), cfg)
        _copy_single(out, int(i), f)
    if check:
        bad = np.nonzero(out.stats["status"] != _native.RCP_OK)[0]
        if bad.size:
            i = int(bad[0])
            _raise_matrix(i, out.stats[i])
    return out


def shard_range(count: int, rank: int, world: int) -> tuple:
    """Contiguous, balanced shard [start, stop) of ``count`` independent matrices for ``rank`` of
    ``world`` (config C5: sharded by matrix, no communication; the first count % world shards
    get one extra matrix)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"rank {rank} outside world {world}")
    base, extra = divmod(count, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def factor_batched_sharded(a: torch.Tensor, cfg: FactorConfig | None = None, *, devices=None,
                           chunk: int = 296, check: bool = True, **overrides) -> BatchedDeviceFactorization:
    """Factor a host stack (CPU float64 ``[count, n, n]``, ideally pinned) on several GPUs of this
    process: matrix shard ``shard_range(count, r, len(devices))`` goes to ``devices[r]`` (default:
    every visible GPU), each through :func:`factor_batched_host` in its own host thread (the
    native calls release the GIL), results land in one pinned host
    :class:`BatchedDeviceFactorization`.  Same results as :func:`factor_batched_host` on one GPU
    (every matrix restarts the same normal stream).  Under torchrun, give each rank its own
    ``shard_range`` slice instead."""
    import threading

    cfg = _config(cfg, overrides)
    _check_supported(cfg, batched=True)
    if a.dim() != 3 or a.shape[1] != a.shape[2] or a.is_cuda or a.dtype != torch.float64:
        raise ValueError("factor_batched_sharded expects a host (CPU) float64 [count, n, n] stack")
    if devices is None:
        devices = list(range(torch.cuda.device_count()))
    devices = [torch.device("cuda", d) if isinstance(d, int) else torch.device(d) for d in devices]
    if not devices:
        raise _native.NativeUnavailable("no CUDA device: the B200 build has no CPU fallback")
    count, n = int(a.shape[0]), int(a.shape[1])
    a = a.contiguous()
    pin = True
    out = BatchedDeviceFactorization(
        perm=torch.empty(count, n, dtype=torch.int64, pin_memory=pin),
        L=torch.empty(count, n, n, dtype=torch.float64, pin_memory=pin),
        d_diag=torch.empty(count, n, dtype=torch.float64, pin_memory=pin),
        d_off=torch.empty(count, n, dtype=torch.float64, pin_memory=pin),
        pattern=torch.empty(count, n, dtype=torch.int8, pin_memory=pin),
        stats=np.zeros(count, dtype=_native.BATCH_STATS_DTYPE))
    errors = [None] * len(devices)

    def work(r, dev):
        s0, s1 = shard_range(count, r, len(devices))
        if s1 <= s0:
            return
        try:
            with torch.cuda.device(dev):
                part = BatchedDeviceFactorization(out.perm[s0:s1], out.L[s0:s1], out.d_diag[s0:s1],
                                                  out.d_off[s0:s1], out.pattern[s0:s1], None)
                res = factor_batched_host(a[s0:s1], cfg, chunk=chunk, out=part, check=False)
                torch.cuda.synchronize(dev)
            out.stats[s0:s1] = res.stats
        except BaseException as exc:  # re-raised on the caller's thread
            errors[r] = exc

    threads = [threading.Thread(target=work, args=(r, d)) for r, d in enumerate(devices)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for exc in errors:
        if exc is not None:
            raise exc
    if check:
        bad = np.nonzero(out.stats["status"] != _native.RCP_OK)[0]
        if bad.size:
            _raise_matrix(int(bad[0]), out.stats[int(bad[0])])
    return out


def factor_batched(a: np.ndarray, cfg: FactorConfig | None = None, **overrides) -> list:
    """``[randldl.factor(a[i], cfg) for i in range(len(a))]`` in one device call."""
    cfg = _config(cfg, overrides)
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 3 or a.shape[1] != a.shape[2]:
        raise ValueError(f"expected a [count, n, n] stack, got shape {a.shape}")
    return factor_batched_host(torch.from_numpy(np.ascontiguousarray(a)), cfg).to_host()


def solve_batched_device(f: BatchedDeviceFactorization, b: torch.Tensor,
                         x: torch.Tensor | None = None) -> tuple:
    """x[i] = A_i^-1 b[i] (solve.py:34-76) for every factorization; returns (x, singular[count])."""
    lib = _native.load()
    count, n = f.count, f.n
    if tuple(b.shape) != (count, n):
        raise ValueError(f"right-hand sides must be ({count}, {n}), got {tuple(b.shape)}")
    b = b.to(dtype=torch.float64).contiguous()
    if x is None:
        x = torch.empty_like(b)
    sing = torch.zeros(count, dtype=torch.int32, device=b.device)
    if n > MAX_N:
        from .api import solve_device
        for i in range(count):
            df = DeviceFactorization(perm=f.perm[i], L=f.L[i], d_diag=f.d_diag[i], d_off=f.d_off[i],
                                     pattern=f.pattern[i], stats={})
            xi, si = solve_device(df, b[i])
            x[i].copy_(xi)
            sing[i] = int(si)
        return x, sing.bool()
    status = lib.rcp_solve_batched(count, n, f.perm.data_ptr(), f.L.data_ptr(), f.d_diag.data_ptr(),
                                   f.d_off.data_ptr(), f.pattern.data_ptr(), b.data_ptr(), x.data_ptr(),
                                   sing.data_ptr(), _stream())
    _raise_status(status, None)
    return x, sing.bool()


def solve_batched(fs: list, b: np.ndarray) -> np.ndarray:
    """``[randldl.solve(fs[i], b[i]).x for i]`` in one device call."""
    b = np.asarray(b, dtype=np.float64)
    if b.ndim != 2 or b.shape[0] != len(fs):
        raise ValueError(f"right-hand sides must be (count, n), got {b.shape}")
    dev = _device()
    n = b.shape[1]
    dd = np.zeros((len(fs), n))
    doff = np.zeros((len(fs), n))
    for i, f in enumerate(fs):
        j = 0
        for blk in f.D.blocks:
            if blk.shape[0] == 1:
                dd[i, j] = blk[0, 0]
                j += 1
            else:
                dd[i, j], dd[i, j + 1], doff[i, j] = blk[0, 0], blk[1, 1], blk[1, 0]
                j += 2
    bf = BatchedDeviceFactorization(
        perm=torch.from_numpy(np.stack([f.perm for f in fs]).astype(np.int64)).to(dev),
        L=torch.from_numpy(np.ascontiguousarray(np.stack([f.L for f in fs]))).to(dev),
        d_diag=torch.from_numpy(dd).to(dev), d_off=torch.from_numpy(doff).to(dev),
        pattern=torch.from_numpy(np.stack([f.pattern for f in fs]).astype(np.int8)).to(dev),
        stats=np.zeros(len(fs), dtype=_native.BATCH_STATS_DTYPE))
    x, _ = solve_batched_device(bf, torch.from_numpy(b).to(dev))
    return x.cpu().numpy()
