"""Synthetic problem generators for BASELINE.json configs 1-5.

The reference ships only gen_synthetic (ĀᵀĀ, io.cpp:168-176) and the LIBSVM
ridge Hessian (io.cpp:123-166); the BASELINE generators are builder-defined
over the reference's RngStream (rng.hpp), one substream per object so the A
draw never aliases the sketch stream that run_inverter seeds with
RngStream(seed) (simi.cpp:275).  Inputs are synthetic stand-ins for the paper's
datasets (LIBSVM / UF), with their shapes, sizes and value distributions.

Dense configs return column-major float64 arrays; sparse configs return CSR
(rowptr int64, colind int32, val float64).

The module is importable on its own (bench.py's reference arm loads it by path,
without the package and its CUDA library): the RngStream class is injected
through `use_rng` (the oracle's and the library's streams are byte-identical,
tests/test_boundary_cpu.py) and defaults to the library's.  Input synthesis
is host-side numpy / BLAS only, so both bench arms build the same A bytes.
"""
from __future__ import annotations

import math

import numpy as np

_RNG = None


def use_rng(cls) -> None:
    """Select the RngStream implementation (a class with substream /
    gaussian_matrix / uniform_matrix, rng.hpp:13-71)."""
    global _RNG
    _RNG = cls


def RngStream(seed: int = 0):
    global _RNG
    if _RNG is None:
        from paper_1602_01768_b200.api import RngStream as _R

        _RNG = _R
    return _RNG(seed)


def config1_dense(n: int = 1024, seed: int = 0, m: int | None = None) -> np.ndarray:
    """A = BᵀB/m + 1e-3·I, B m×n i.i.d. N(0,1) (m = 2n; BASELINE config 1)."""
    m = 2 * n if m is None else m
    b = RngStream(seed).substream(1).gaussian_matrix(m, n)
    a = (b.T @ b) / m
    a[np.diag_indices(n)] += 1e-3
    return np.asfortranarray(0.5 * (a + a.T))


def config2_dense(n: int = 4096, seed: int = 0, m: int | None = None, density: float = 0.01) -> np.ndarray:
    """Ridge Gram A = BᵀB + I of sparse binary features, B m×n with P(1) = density
    (column-major draw order; BASELINE config 2 has m = 20000, n = 4096)."""
    m = int(round(n * 20000 / 4096)) if m is None else m
    u = RngStream(seed).substream(2).uniform_matrix(m, n)
    b = (u < density).astype(np.float64)
    a = b.T @ b
    a[np.diag_indices(n)] += 1.0
    return np.asfortranarray(a)


def config3_dense(n: int = 16384, seed: int = 0, reflectors: int = 8) -> np.ndarray:
    """A = Q·diag(λ)·Qᵀ, Q = H_8···H_1 Householder reflectors with N(0,1) vectors,
    λ_j = 10^(−3 + 3u_j) log-uniform in [1e-3, 1] (BASELINE config 3).

    Each reflector is applied two-sided in place on the upper triangle
    (A ← H A H = A − v uᵀ − u vᵀ, u = βAv − ½β²(vᵀAv)v: BLAS dsymv + dsyr2),
    then the upper triangle is mirrored, so A is exactly symmetric and no n×n
    temporary is made (≈5 s at n = 16384)."""
    from scipy.linalg import blas

    r = RngStream(seed).substream(3)
    v = r.gaussian_matrix(n, reflectors)
    lam = 10.0 ** (-3.0 + 3.0 * r.uniform_matrix(n, 1)[:, 0])
    a = np.zeros((n, n), order="F")
    a[np.diag_indices(n)] = lam
    for i in range(reflectors):
        vi = np.ascontiguousarray(v[:, i])
        beta = 2.0 / float(vi @ vi)
        p = blas.dsymv(1.0, a, vi, lower=0)
        u = beta * p - 0.5 * beta * beta * float(vi @ p) * vi
        a = blas.dsyr2(-1.0, vi, u, a=a, lower=0, overwrite_a=1)
    _mirror_upper(a)
    return a


def _mirror_upper(a: np.ndarray, blk: int = 2048) -> None:
    n = a.shape[0]
    for j0 in range(0, n, blk):
        j1 = min(j0 + blk, n)
        for i0 in range(j1, n, blk):
            i1 = min(i0 + blk, n)
            a[i0:i1, j0:j1] = a[j0:j1, i0:i1].T
        d = a[j0:j1, j0:j1]
        a[j0:j1, j0:j1] = np.triu(d) + np.triu(d, 1).T


def config3_dense_device(n: int = 16384, seed: int = 0, reflectors: int = 8, device: str = "cuda"):
    """config3_dense with the reflector applications done by torch on the GPU
    (same RngStream draws and formula; rounding differs from the numpy path).
    Input synthesis only -- returns a float64 CUDA tensor holding A column-major
    (the tensor is Aᵀ = A in row-major view)."""
    import torch

    r = RngStream(seed).substream(3)
    v = torch.from_numpy(r.gaussian_matrix(n, reflectors)).to(device)
    lam = torch.from_numpy(10.0 ** (-3.0 + 3.0 * r.uniform_matrix(n, 1)[:, 0])).to(device)
    a = torch.diag(lam)
    for i in range(reflectors):
        vi = v[:, i].contiguous()
        beta = 2.0 / float(vi @ vi)
        p = a @ vi
        u = beta * p - 0.5 * beta * beta * float(vi @ p) * vi
        a.sub_(torch.outer(vi, u)).sub_(torch.outer(u, vi))
    a = 0.5 * (a + a.T)
    return a.contiguous()


def config4_csr(n: int = 65536, shift: float = 1e-2):
    """2-D 5-point Dirichlet Laplacian on a g×g grid (g = √n) + shift·I (BASELINE config 4)."""
    g = int(round(math.sqrt(n)))
    if g * g != n:
        raise ValueError("config4: n must be a perfect square")
    idx = np.arange(n, dtype=np.int64)
    gi, gj = idx // g, idx % g
    rows, cols, vals = [idx], [idx], [np.full(n, 4.0 + shift)]
    for di, dj in ((-1, 0), (1, 0), (0, -1), (0, 1)):
        ni, nj = gi + di, gj + dj
        ok = (ni >= 0) & (ni < g) & (nj >= 0) & (nj < g)
        rows.append(idx[ok])
        cols.append((ni * g + nj)[ok])
        vals.append(np.full(int(ok.sum()), -1.0))
    return _coo_to_csr(n, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals))


def config5_csr(n: int = 98304, half_bandwidth: int = 64, seed: int = 0):
    """Banded random SPD: off-diagonals U(−1,1) within |i−j| ≤ b, symmetric,
    diagonal = 1 + row abs-sum (strict diagonal dominance; BASELINE config 5)."""
    b = half_bandwidth
    r = RngStream(seed).substream(5)
    # upper-band entries (i, i+d), d = 1..b, drawn diagonal by diagonal
    rows, cols, vals = [], [], []
    rowabs = np.zeros(n)
    for d in range(1, b + 1):
        cnt = n - d
        if cnt <= 0:
            break
        u = r.uniform_matrix(cnt, 1)[:, 0] * 2.0 - 1.0
        i = np.arange(cnt, dtype=np.int64)
        rows += [i, i + d]
        cols += [i + d, i]
        vals += [u, u]
        np.add.at(rowabs, i, np.abs(u))
        np.add.at(rowabs, i + d, np.abs(u))
    idx = np.arange(n, dtype=np.int64)
    rows.append(idx)
    cols.append(idx)
    vals.append(1.0 + rowabs)
    return _coo_to_csr(n, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals))


def _coo_to_csr(n, rows, cols, vals):
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rowptr, rows + 1, 1)
    rowptr = np.cumsum(rowptr).astype(np.int64)
    return rowptr, cols.astype(np.int32), vals.astype(np.float64)


def csr_to_dense(n, rowptr, colind, val) -> np.ndarray:
    a = np.zeros((n, n), order="F")
    for i in range(n):
        s, e = rowptr[i], rowptr[i + 1]
        a[i, colind[s:e]] += val[s:e]
    return a
