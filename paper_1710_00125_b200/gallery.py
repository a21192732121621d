"""Seeded synthetic inputs of the BASELINE.json configurations.

* ``type6(n, seed)``: iid N(0,1) lower triangle mirrored to the upper one, the
  reference gallery's type 6 (gallery.py:163-166).  Large n is generated in row
  chunks from one generator (bit-identical to the one-shot draw) and mirrored
  without numpy's full-size temporaries.
* ``kkt(n1, n2, seed)``: saddle-point ``[[H, B^T], [B, 0]]`` with
  ``H = G^T G / n1 + I`` (config 4).  Not a reference family; generated here.
* ``scaled_member(n, seed, scaled)``: config-5 batch member: type6 and, for the
  scaled 10 %, ``D A D`` with ``D = diag(10^U(-6, 6))`` re-mirrored so the
  triangles are bitwise equal (the reference rejects asymmetric input).
"""

from __future__ import annotations

import numpy as np


def _gen(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(seed))


def mirror_lower_inplace(a: np.ndarray, blk: int = 2048) -> np.ndarray:
    """a[i, j] = a[j, i] for i < j (copy the lower triangle to the upper)."""
    n = a.shape[0]
    for c0 in range(0, n, blk):
        c1 = min(n, c0 + blk)
        d = a[c0:c1, c0:c1]
        il = np.tril_indices(c1 - c0, -1)
        d[il[1], il[0]] = d[il]
        if c1 < n:
            a[c0:c1, c1:] = a[c1:, c0:c1].T
    return a


def type6(n: int, seed: int = 0, chunk_rows: int = 1024) -> np.ndarray:
    """Symmetric Gaussian matrix identical to ``tril(g) + tril(g, -1).T``."""
    g = _gen(seed)
    if n <= 4096:
        m = g.standard_normal((n, n))
        return np.tril(m) + np.tril(m, -1).T
    a = np.empty((n, n))
    for r0 in range(0, n, chunk_rows):
        r1 = min(n, r0 + chunk_rows)
        a[r0:r1] = g.standard_normal((r1 - r0, n))
    return mirror_lower_inplace(a)


def kkt(n1: int, n2: int, seed: int = 0) -> np.ndarray:
    """[[H, B^T], [B, 0]] with H = G^T G / n1 + I, G (n1 x n1), B (n2 x n1) iid N(0,1)."""
    g = _gen(seed)
    G = g.standard_normal((n1, n1))
    Bm = g.standard_normal((n2, n1))
    H = G.T @ G / n1 + np.eye(n1)
    n = n1 + n2
    a = np.zeros((n, n))
    a[:n1, :n1] = H
    a[n1:, :n1] = Bm
    return mirror_lower_inplace(a)


def kkt_c4(n1: int = 16000, n2: int = 4000, seed: int = 0) -> np.ndarray:
    """Config 4 with an order-independent H: as :func:`kkt`, but G's N(0,1) draws are rounded
    to multiples of 2^-8.  Every product g_i g_j then has <= 22 significant bits and every
    partial sum of n1 <= 2^16 of them stays below 2^36 units of 2^-16, so G^T G is EXACT in
    fp64 under any summation order (OpenBLAS here, a device GEMM on the GPU box): both sides
    factor bit-identical matrices without shipping the 3.2 GB input."""
    assert n1 <= 1 << 16
    g = _gen(seed)
    G = np.round(g.standard_normal((n1, n1)) * 256.0) / 256.0
    Bm = g.standard_normal((n2, n1))
    H = G.T @ G
    del G
    H /= n1
    H += np.eye(n1)
    n = n1 + n2
    a = np.zeros((n, n))
    a[:n1, :n1] = H
    del H
    a[n1:, :n1] = Bm
    return mirror_lower_inplace(a)


def scaled_member(n: int, seed: int, scaled: bool) -> np.ndarray:
    """One matrix of the batched configuration (config 5)."""
    g = _gen(seed)
    m = g.standard_normal((n, n))
    a = np.tril(m) + np.tril(m, -1).T
    if scaled:
        d = 10.0 ** g.uniform(-6.0, 6.0, n)
        a = d[:, None] * a * d[None, :]
        a = np.tril(a) + np.tril(a, -1).T
    return a


def rhs(n: int, seed: int = 1) -> np.ndarray:
    return _gen(seed).standard_normal(n)


def c5_batch_device(count: int, n: int = 256, seed: int = 0, scaled_every: int = 10, device="cuda"):
    """Config-5 stack generated on the device (bench input; same distribution as
    :func:`scaled_member`, not the same bits): symmetrised N(0,1) matrices, every
    ``scaled_every``-th one scaled as D A D with D = diag(10^U(-6, 6)) and re-mirrored."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    a = torch.randn(count, n, n, dtype=torch.float64, device=device, generator=g)
    a = torch.tril(a) + torch.tril(a, -1).transpose(1, 2)
    if scaled_every:
        idx = torch.arange(0, count, scaled_every, device=device)
        d = 10.0 ** (torch.rand(idx.numel(), n, dtype=torch.float64, device=device, generator=g) * 12.0 - 6.0)
        s = d[:, :, None] * a[idx] * d[:, None, :]
        a[idx] = torch.tril(s) + torch.tril(s, -1).transpose(1, 2)
    return a
