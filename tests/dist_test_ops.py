"""CPU test double for the sharded driver's panel ops (TEST INFRASTRUCTURE).

Implements the same contract as paper_1602_01768_b200.dist.CudaPanelOps on CPU
torch tensors with numpy arithmetic, and draws sketches from the oracle's
RngStream(seed).substream(draw), so the gloo tests exercise the row
decomposition, the collectives and the packing, against a single-process oracle
run on the same sketch sequence.
"""
import numpy as np
from numpy.lib.stride_tricks import as_strided

from oracle import oracle as O


def _view(t, rows, cols, ld, kmajor=False):
    a = t.numpy()
    if kmajor:  # element (r, c) at r*ld + c
        return as_strided(a, shape=(rows, cols), strides=(8 * ld, 8))
    return as_strided(a, shape=(rows, cols), strides=(8, 8 * ld))


class NumpyPanelOps:
    def __init__(self, a_dense=None):
        self.a = a_dense

    def gemm(self, M, N, K, A, lda, a_kmajor, B, ldb, b_kmajor, Cm, ldc, alpha=1.0, beta=0.0):
        a = _view(A, M, K, lda, a_kmajor)
        b = _view(B, K, N, ldb, not b_kmajor)  # b_kmajor: B(k,n) = B[k + n*ldb] -> column-major K×N
        c = _view(Cm, M, N, ldc)
        res = alpha * (a @ b)
        if beta != 0.0:
            res = res + beta * c
        c[...] = res

    def sketch(self, S, n, q, lds, seed, draw):
        s = O.RngStream(seed).substream(draw).gaussian_matrix(n, q)
        _view(S, n, q, lds)[...] = s

    def core(self, P, ldp, q, M, scratch):
        from paper_1602_01768_b200.api import GramRankDeficientError

        p = _view(P, q, 2 * q, ldp).copy()
        g = np.triu(p[:, :q]) + np.triu(p[:, :q], 1).T
        try:
            np.linalg.cholesky(g)
        except np.linalg.LinAlgError:
            raise GramRankDeficientError("bfgs_step: sketched Gram matrix is not positive definite")
        gi = np.linalg.inv(g)
        gi = 0.5 * (gi + gi.T)
        h = p[:, q:]
        m = np.zeros((2 * q, 2 * q))
        m[:q, :q] = gi + gi @ h @ gi
        m[:q, q:] = -gi
        m[q:, :q] = -gi
        _view(M, 2 * q, 2 * q, 2 * q)[...] = m

    def core_async(self, P, ldp, q, M, scratch, status):
        from paper_1602_01768_b200.api import GramRankDeficientError

        try:
            self.core(P, ldp, q, M, scratch)
            status[0] = 0
        except GramRankDeficientError:
            _view(M, 2 * q, 2 * q, 2 * q)[...] = 0.0
            status[0] = 1

    def residual_rows_sq(self, prob, m, r0, X, ldx):
        x = _view(X, m, self.a.shape[0], ldx)
        r = x @ self.a
        r[np.arange(m), r0 + np.arange(m)] -= 1.0
        return float((r * r).sum())

    # ---- AdaRBFGS panel ops (same contract as CudaPanelOps) ----
    def gather_columns(self, Lp, rows, ldl, idx, q, out):
        src, dst = Lp.numpy(), out.numpy()
        for j, c in enumerate(idx.numpy()[:q]):
            dst[j * rows:(j + 1) * rows] = src[c * ldl: c * ldl + rows]

    def ada_core(self, G, q, Z, n, idx, St, T, R, B, scratch):
        from paper_1602_01768_b200.api import GramRankDeficientError

        g = _view(G, q, q, q).copy()
        z = _view(Z, q, n, q).copy()
        try:
            r = O.sym_inv_sqrt(g)
            if St is None:
                t = np.zeros((q, n))
                t[np.arange(q), idx.numpy()[:q]] = 1.0
            else:
                st = _view(St, n, q, n).copy()
                t = O.sym_inv_sqrt(st.T @ st) @ st.T
                _view(T, q, n, q)[...] = t
        except O.NumericalError as e:
            raise GramRankDeficientError(str(e))
        _view(R, q, q, q)[...] = r
        _view(B, q, n, q)[...] = t - r @ z

    def pdiag_update(self, B, q, n, T, idx, d):
        b = _view(B, q, n, q)
        if T is None:
            t = np.zeros((q, n))
            t[np.arange(q), idx.numpy()[:q]] = 1.0
        else:
            t = _view(T, q, n, q)
        d.numpy()[:] += 2.0 * (t * b).sum(axis=0) - (b * b).sum(axis=0)

    def symupd(self, m, k, V, ldv, U, ldu, X, ldx):
        """X (m×m) += V·Uᵀ on the upper triangle, mirrored (the K-SYMUPD contract)."""
        x = _view(X, m, m, ldx)
        full = x + _view(V, m, k, ldv) @ _view(U, m, k, ldu).T
        x[...] = np.triu(full) + np.triu(full, 1).T

    def spmm(self, m, n, rowptr, colind, val, P, ldp, k, Y, ldy):
        import scipy.sparse as sp

        a = sp.csr_matrix((val.numpy(), colind.numpy().astype(np.int64), rowptr.numpy()), shape=(m, n))
        _view(Y, m, k, ldy)[...] = a @ _view(P, n, k, ldp)
