"""Row-sharded RBFGS host logic on CPU: world_size 1 and 2 over gloo, against a
single-process oracle run on the same sketch sequence."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(n, seed=3):
    rng = O.RngStream(seed)
    b = rng.gaussian_matrix(n, n)
    return np.asfortranarray(b @ b.T / n + np.eye(n))


def _oracle_run(a, q, iters, seed):
    n = a.shape[0]
    x = np.asfortranarray(np.eye(n))
    for draw in range(iters):
        s = O.RngStream(seed).substream(draw).gaussian_matrix(n, q)
        x = O.bfgs_step(x, a, s)
    return x


def _worker(rank, world, port, n, q, iters, seed, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        from dist_test_ops import NumpyPanelOps
        from paper_1602_01768_b200.dist import RowShardedRBFGS, row_partition

        a = _problem(n)
        starts = row_partition(n, world)
        r0, r1 = starts[rank], starts[rank + 1]
        a_rows = torch.from_numpy(np.asfortranarray(a[r0:r1, :]).reshape(-1, order="F").copy())
        solver = RowShardedRBFGS(NumpyPanelOps(a), n, q, a_rows, seed=seed)
        for _ in range(iters):
            solver.step()
        x = solver.gather_x().numpy().reshape((n, n), order="F")
        res = solver.residual()
        if rank == 0:
            out_q.put((x, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,q", [(1, 24, 4), (2, 37, 3), (2, 64, 8)])
def test_row_sharded_matches_oracle(world, n, q):
    iters, seed = 12, 5
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q, iters, seed, out_q)) for r in range(world)]
    for p in procs:
        p.start()
    x, res = out_q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a = _problem(n)
    ref = _oracle_run(a, q, iters, seed)
    assert np.linalg.norm(x - ref) / np.linalg.norm(ref) <= 1e-9
    assert res == pytest.approx(np.linalg.norm(np.eye(n) - a @ x), rel=1e-9)


def test_row_partition():
    from paper_1602_01768_b200.dist import row_partition

    assert row_partition(10, 3) == [0, 4, 7, 10]
    assert row_partition(8, 8) == list(range(9))


def _rows(a, r0, r1, sparse):
    if not sparse:
        return torch.from_numpy(np.asfortranarray(a[r0:r1, :]).reshape(-1, order="F").copy())
    import scipy.sparse as sp

    from paper_1602_01768_b200.dist import CsrRows

    c = sp.csr_matrix(a)
    return CsrRows.from_host(c.indptr.astype(np.int64), c.indices.astype(np.int32), c.data, r0, r1, "cpu")


def _sparse_problem(n):
    """A sparse SPD stand-in (banded, like config 5) as a dense array for the oracle."""
    rng = O.RngStream(11)
    a = np.zeros((n, n))
    for i in range(n):
        for j in range(max(0, i - 3), i):
            v = 2 * rng.uniform() - 1
            a[i, j] = a[j, i] = v
    a[np.arange(n), np.arange(n)] = 1.0 + np.abs(a).sum(axis=1)
    return a


def _ada_worker(rank, world, port, n, q, iters, seed, rule, use_l0, out_q, sparse=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        from dist_test_ops import NumpyPanelOps
        from paper_1602_01768_b200.dist import RowShardedAdaRBFGS, row_partition

        a = _sparse_problem(n) if sparse else _problem(n)
        starts = row_partition(n, world)
        r0, r1 = starts[rank], starts[rank + 1]
        a_rows = _rows(a, r0, r1, sparse)
        l0_rows = None
        if use_l0:
            l0 = _l0(n)
            l0_rows = torch.from_numpy(np.asfortranarray(l0[r0:r1, :]).reshape(-1, order="F").copy())
        solver = RowShardedAdaRBFGS(NumpyPanelOps(a), n, q, a_rows, rule=rule, seed=seed, l0_rows=l0_rows)
        for _ in range(iters):
            solver.step()
        lf = solver.gather_l().numpy().reshape((n, n), order="F")
        res = solver.residual()
        d = solver.d.numpy().copy() if solver.d is not None else None
        if rank == 0:
            out_q.put((lf, res, d))
    finally:
        dist.destroy_process_group()


def _l0(n):
    return np.eye(n) + 0.01 * O.RngStream(77).gaussian_matrix(n, n)


@pytest.mark.parametrize("world,n,q,rule,use_l0,sparse", [
    (1, 24, 4, "cols", False, False), (2, 37, 4, "cols", False, False), (2, 40, 6, "uniform", False, False),
    (2, 33, 3, "gauss", False, False), (2, 30, 5, "cols", True, False), (2, 41, 4, "cols", False, True),
    (2, 36, 4, "uniform", False, True),
])
def test_row_sharded_adarbfgs_matches_oracle(world, n, q, rule, use_l0, sparse):
    iters, seed = 15, 4
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ada_worker, args=(r, world, port, n, q, iters, seed, rule, use_l0, out_q, sparse))
             for r in range(world)]
    for p in procs:
        p.start()
    lf, res, d = out_q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a = _sparse_problem(n) if sparse else _problem(n)
    l0 = _l0(n) if use_l0 else None
    if rule == "gauss":  # same Philox-stand-in sketch sequence as the test double
        ref = np.asfortranarray(l0 if l0 is not None else np.eye(n))
        for draw in range(iters):
            ref = O.adarbfgs_update_factor(ref, a, O.RngStream(seed).substream(draw).gaussian_matrix(n, q))
    else:
        orule = O.ADA_COLS if rule == "cols" else O.ADA_COLS_UNIFORM
        ref = O.run_adarbfgs(a, q, rule=orule, tol=0.0, max_iters=iters, every_k=iters, seed=seed, l0=l0).x
    assert np.linalg.norm(lf - ref) / np.linalg.norm(ref) <= 1e-9
    assert res == pytest.approx(np.linalg.norm(np.eye(n) - a @ lf @ lf.T), rel=1e-9)
    if d is not None:  # the carried Eq. 8.2 diagonal equals the exact diag(LᵀAL)
        assert np.allclose(d, np.einsum("ij,ij->j", lf, a @ lf), rtol=1e-10, atol=0)


def _sym_worker(rank, world, port, n, q, iters, seed, out_q, sparse=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        from dist_test_ops import NumpyPanelOps
        from paper_1602_01768_b200.dist import SymmetricShardedRBFGS

        a = _sparse_problem(n) if sparse else _problem(n)

        def rows(r0, r1):
            return _rows(a, r0, r1, sparse)

        solver = SymmetricShardedRBFGS(NumpyPanelOps(a), n, q, rows, seed=seed)
        for _ in range(iters):
            solver.step()
        x = solver.gather_x().numpy().reshape((n, n), order="F")
        res = solver.residual()
        if rank == 0:
            out_q.put((x, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,q,sparse", [(1, 24, 4, False), (2, 37, 3, False), (3, 50, 5, False),
                                             (2, 45, 4, True)])
def test_symmetric_sharded_matches_oracle(world, n, q, sparse):
    iters, seed = 12, 5
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sym_worker, args=(r, world, port, n, q, iters, seed, out_q, sparse))
             for r in range(world)]
    for p in procs:
        p.start()
    x, res = out_q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a = _sparse_problem(n) if sparse else _problem(n)
    ref = _oracle_run(a, q, iters, seed)
    assert np.linalg.norm(x - ref) / np.linalg.norm(ref) <= 1e-9
    assert np.array_equal(x, x.T)
    assert res == pytest.approx(np.linalg.norm(np.eye(n) - a @ x), rel=1e-9)


def test_chunk_balance():
    from paper_1602_01768_b200.dist import chunk_bounds

    n, P = 16384, 8
    b = chunk_bounds(n, P)
    work = []
    for p in range(P):
        w = 0
        for c in (p, 2 * P - 1 - p):
            m = b[c + 1] - b[c]
            w += m * (n - b[c])  # trapezoid area
        work.append(w)
    assert max(work) / min(work) < 1.001


def _rejecting_ops(a, reject_calls):
    """NumpyPanelOps whose core rejects on the given call indices (forced non-PD Grams)."""
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from dist_test_ops import NumpyPanelOps
    from paper_1602_01768_b200.api import GramRankDeficientError

    class Ops(NumpyPanelOps):
        calls = 0

        def core(self, P, ldp, q, M, scratch):
            i = Ops.calls
            Ops.calls += 1
            if i in reject_calls:
                raise GramRankDeficientError("forced")
            super().core(P, ldp, q, M, scratch)

    Ops.calls = 0
    return Ops(a)


@pytest.mark.parametrize("reject,steps,max_redraws", [((), 7, 3), ((1,), 7, 3), ((0, 3, 4, 5, 9), 7, 3),
                                                      ((2, 3, 4), 6, 2), ((6,), 7, 1)])
def test_symmetric_deferred_pd_check_matches_sync(reject, steps, max_redraws):
    """The deferred PD read (update enqueued before the status is known, M = 0 on rejection)
    gives the synchronous loop's X, draw count and redraw count, also at the redraw limit."""
    from paper_1602_01768_b200.api import GramRankDeficientError
    from paper_1602_01768_b200.dist import SymmetricShardedRBFGS

    n, q, seed = 21, 3, 7
    a = _problem(n)

    def run(deferred):
        s = SymmetricShardedRBFGS(_rejecting_ops(a, set(reject)), n, q, lambda r0, r1: _rows(a, r0, r1, False),
                                  seed=seed, max_redraws=max_redraws, deferred=deferred)
        err = None
        try:
            for _ in range(steps):
                s.step()
            s.finalize()
        except GramRankDeficientError as e:
            err = e
        return s.gather_x().numpy().copy(), s.draw, s.redraws, err is not None

    xs, ds, rs, es = run(False)
    xd, dd, rd, ed = run(True)
    assert (dd, rd, ed) == (ds, rs, es)
    assert np.array_equal(xd, xs)
