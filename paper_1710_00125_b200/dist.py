"""One factorization on several GPUs of one node (BASELINE config C3, "1/2/4/8 GPU").

One process per GPU (torchrun).  Rank 0 owns the matrix, runs the panels (pivot search,
QRCP, SBKP steps, sketch update: the latency-bound critical path, which needs random access
to every column of the trailing matrix at every step) and the bookkeeping; the trailing Schur
update of every panel -- the O(n^3) part -- is dealt tile-round-robin over all ranks, which
read C-in tiles from and write results into rank 0's matrix over NVLink peer memory (CUDA IPC
mapping of rank 0's workspace; protocol in ``csrc/dist.cuh``).  The reference has no
multi-process path (its ``factor`` is single-process, ``factor.py:637-647``); the result is
bit-identical to the single-GPU :func:`paper_1710_00125_b200.factor_device`.

Host orchestration (this module) is separated from the device calls (:class:`DeviceOps`) so the
protocol -- who allocates, prepares, exports, imports, and when each side may start and
stop -- is tested on CPU with the gloo backend (``tests/test_dist_host.py``).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _native
from .api import FactorConfig, _check_supported, _config, _stream, factor_device

__all__ = ["factor_distributed_device", "factor_distributed", "DeviceOps", "tile_plan"]


def tile_plan(mp: int, P: int, part: int, nparts: int, grid: int):
    """The trailing-update tiles device ``part`` of ``nparts`` processes for one panel (``mp``
    trailing rows, ``P`` fused sketch rows -- 0 when the update is shared), in its CTAs' order,
    as numpy arrays (m0, n0, is_sketch).  Computed by the C ABI (``rcp_schur_tile_plan``) with
    the same dealing functions the CUDA kernel runs; needs no GPU."""
    import numpy as np
    lib = _native.load()
    cnt = int(lib.rcp_schur_tile_plan(mp, P, part, nparts, grid, None, None, None, 0))
    if cnt < 0:
        raise ValueError("bad tile plan arguments")
    m0 = np.empty(cnt, dtype=np.int64)
    n0 = np.empty(cnt, dtype=np.int64)
    sk = np.empty(cnt, dtype=np.int8)
    lib.rcp_schur_tile_plan(mp, P, part, nparts, grid, m0.ctypes.data, n0.ctypes.data, sk.ctypes.data, cnt)
    return m0, n0, sk.astype(bool)


@dataclass
class _Plan:
    """What rank 0 broadcasts to the workers before the factorization."""

    handle: bytes
    n: int
    p: int
    b: int
    q: int
    robust_r: int
    world: int


class DeviceOps:
    """The CUDA side of the protocol (one instance per process)."""

    def __init__(self):
        self.lib = _native.load()
        self._ws = None       # rank 0: cached IPC-exportable workspace (ptr, bytes)
        self._imported = {}   # workers: handle -> mapped pointer
        self._wws = None

    def _cfg(self, plan_or_cfg):
        # workspace sizing and the Schur workers do not depend on the pivoting strategy
        return _native.RcpConfig(plan_or_cfg.p, plan_or_cfg.b, plan_or_cfg.q, plan_or_cfg.robust_r, 0)

    def alloc_workspace(self, n: int, cfg) -> tuple:
        c = self._cfg(cfg)
        need = int(self.lib.rcp_workspace_bytes(n, ctypes.byref(c)))
        if self._ws is not None and self._ws[1] >= need:
            return self._ws
        self.release()
        ptr = ctypes.c_void_p()
        if self.lib.rcp_device_alloc(need, ctypes.byref(ptr)) != 0:
            raise RuntimeError("rcp_device_alloc failed")
        self._ws = (int(ptr.value), need)
        return self._ws

    def prepare(self, n: int, cfg, ws) -> None:
        c = self._cfg(cfg)
        if self.lib.rcp_dist_prepare(n, ctypes.byref(c), ws[0], _stream()) != 0:
            raise RuntimeError("rcp_dist_prepare failed")

    def export(self, ws) -> bytes:
        buf = ctypes.create_string_buffer(64)
        if self.lib.rcp_ipc_export(ws[0], buf) != 0:
            raise RuntimeError("rcp_ipc_export failed")
        return buf.raw

    def free_workspace(self, ws) -> None:
        pass  # kept for the next call; release() frees it

    def release(self) -> None:
        if self._ws is not None:
            self.lib.rcp_device_free(self._ws[0])
            self._ws = None
        for ptr in self._imported.values():
            self.lib.rcp_ipc_close(ptr)
        self._imported = {}

    def factor(self, a, cfg, ws, world: int):
        return factor_device(a, cfg, workspace=ws, world=world)

    def import_(self, handle: bytes) -> int:
        if handle in self._imported:
            return self._imported[handle]
        ptr = ctypes.c_void_p()
        if self.lib.rcp_ipc_import(handle, ctypes.byref(ptr)) != 0:
            raise RuntimeError("rcp_ipc_import failed (peer access between these GPUs?)")
        self._imported[handle] = int(ptr.value)
        return int(ptr.value)

    def close(self, ptr: int) -> None:
        pass  # mappings are cached with the handle; release() closes them

    def worker(self, plan: _Plan, rank: int, rank0_ws: int) -> None:
        c = self._cfg(plan)
        wbytes = int(self.lib.rcp_worker_workspace_bytes(plan.n, ctypes.byref(c)))
        if self._wws is None or self._wws.numel() < wbytes:
            self._wws = torch.empty(wbytes, dtype=torch.uint8, device="cuda")
        wws = self._wws
        rc = self.lib.rcp_schur_worker(ctypes.byref(c), plan.n, rank, plan.world, rank0_ws, wws.data_ptr(),
                                       wws.numel(), _stream())
        if rc != 0:
            raise RuntimeError(f"rcp_schur_worker failed with status {rc}")


_DEFAULT_OPS: DeviceOps | None = None


def default_ops() -> DeviceOps:
    """Process-wide DeviceOps (keeps the IPC workspace / mappings between calls)."""
    global _DEFAULT_OPS
    if _DEFAULT_OPS is None:
        _DEFAULT_OPS = DeviceOps()
    return _DEFAULT_OPS


def factor_distributed_device(a: torch.Tensor | None, cfg: FactorConfig | None = None, *, group=None,
                              ops: DeviceOps | None = None, **overrides):
    """Collective: every rank of ``group`` calls it; rank 0 passes the matrix (CUDA float64),
    the others pass ``None``.  Returns the :class:`DeviceFactorization` on rank 0, ``None``
    elsewhere."""
    cfg = _config(cfg, overrides)
    _check_supported(cfg)
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    ops = ops if ops is not None else default_ops()
    if world == 1:
        return ops.factor(a, cfg, None, 1)
    src = 0 if group is None else dist.get_global_rank(group, 0)  # group rank 0 as a global rank
    if rank == 0:
        if a is None:
            raise ValueError("rank 0 must pass the matrix")
        n = int(a.shape[0])
        try:
            ws = ops.alloc_workspace(n, cfg)
            ops.prepare(n, cfg, ws)  # zero the signal block before any worker can look at it
            plan = _Plan(ops.export(ws), n, cfg.p, cfg.b, cfg.q, cfg.robust_r, world)
        except Exception as exc:  # release the workers (they wait in the broadcast) before raising
            dist.broadcast_object_list([("setup-failed", repr(exc))], src=src, group=group)
            raise
        try:
            dist.broadcast_object_list([plan], src=src, group=group)
            try:
                f = ops.factor(a, cfg, ws, world)
            finally:
                dist.barrier(group=group)  # every worker has detached (it saw "finished")
            return f
        finally:
            ops.free_workspace(ws)
    obj = [None]
    dist.broadcast_object_list(obj, src=src, group=group)
    if isinstance(obj[0], tuple) and obj[0] and obj[0][0] == "setup-failed":
        raise RuntimeError(f"rank 0 failed to set up the distributed factorization: {obj[0][1]}")
    plan: _Plan = obj[0]
    ptr = ops.import_(plan.handle)
    try:
        ops.worker(plan, rank, ptr)
    finally:
        ops.close(ptr)
        dist.barrier(group=group)
    return None


def factor_distributed(a, cfg: FactorConfig | None = None, *, group=None, ops: DeviceOps | None = None,
                       **overrides):
    """Host-level collective: rank 0 passes a numpy matrix and gets the reference's
    :class:`Factorization`; the other ranks pass ``None`` and get ``None``."""
    import numpy as np

    from .api import _device, _require_square
    a_dev = None
    if dist.get_rank(group) == 0:
        a = _require_square(a)
        a_dev = torch.from_numpy(np.ascontiguousarray(a)).to(_device())
    f = factor_distributed_device(a_dev, cfg, group=group, ops=ops, **overrides)
    return f.to_host() if f is not None else None
