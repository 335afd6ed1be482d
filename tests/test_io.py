"""Problem ingestion: MatrixMarket / LIBSVM readers and the
synthetic generator, following the reference's fixtures in
proj/tests/test_io_bench.cpp:35-137.

The CPU tests exercise the host parser through the C ABI (si_io_* — no device
work); the GPU tests build ProblemMatrix objects on the device and check them
against the same fixtures and against the oracle.
"""
import numpy as np
import pytest

import paper_1602_01768_b200 as si


def _fixture(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


COORD_SYM = ("%%MatrixMarket matrix coordinate real symmetric\n"
             "% running example\n"
             "2 2 3\n"
             "1 1 2.0\n"
             "2 1 1.0\n"
             "2 2 2.0\n")
TWO_ONE = np.array([[2.0, 1.0], [1.0, 2.0]])


# ------------------------------------------------------------------ host parser
def test_coordinate_symmetric_fixture(tmp_path):  # test_io_bench.cpp:35-49
    m, sym = si.read_matrix_market(_fixture(tmp_path, "coord.mtx", COORD_SYM))
    assert sym
    assert m.shape == (2, 2)
    assert np.array_equal(m, TWO_ONE)


def test_array_formats(tmp_path):  # test_io_bench.cpp:51-66
    g, sym = si.read_matrix_market(_fixture(tmp_path, "array.mtx",
                                            "%%MatrixMarket matrix array real general\n2 2\n1.0\n0.0\n0.0\n1.0\n"))
    assert not sym and np.array_equal(g, np.eye(2))
    s, sym = si.read_matrix_market(_fixture(tmp_path, "array_sym.mtx",
                                            "%%MatrixMarket matrix array real symmetric\n2 2\n2.0\n1.0\n2.0\n"))
    assert sym and np.array_equal(s, TWO_ONE)


def test_array_general_is_column_major(tmp_path):
    vals = "\n".join(str(v) for v in range(1, 10))
    m, _ = si.read_matrix_market(_fixture(tmp_path, "cm.mtx", "%%MatrixMarket matrix array real general\n3 3\n" + vals))
    assert np.array_equal(m, np.arange(1, 10, dtype=float).reshape(3, 3).T)


def test_several_values_per_line_and_integer_field(tmp_path):
    m, _ = si.read_matrix_market(_fixture(tmp_path, "int.mtx",
                                          "%%MatrixMarket MATRIX Array Integer General\n2 2\n4 0\n0 4\n"))
    assert np.array_equal(m, 4 * np.eye(2))


def test_duplicate_coordinate_last_wins(tmp_path):
    m, _ = si.read_matrix_market(_fixture(tmp_path, "dup.mtx",
                                          "%%MatrixMarket matrix coordinate real general\n2 2 3\n"
                                          "1 1 5.0\n1 1 7.0\n2 2 1.0\n"))
    assert np.array_equal(m, np.diag([7.0, 1.0]))


def test_error_reporting(tmp_path):  # test_io_bench.cpp:68-100
    trunc = _fixture(tmp_path, "trunc.mtx",
                     "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 2.0\n2 2 2.0\n")
    with pytest.raises(si.IoError, match="truncated file, expected 3 entries, got 2"):
        si.read_matrix_market(trunc)
    bad = _fixture(tmp_path, "malformed.mtx", "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 x 2.0\n")
    with pytest.raises(si.IoError, match=":3:"):
        si.read_matrix_market(bad)
    with pytest.raises(si.IoError):
        si.read_matrix_market("/nonexistent/file.mtx")
    rect = _fixture(tmp_path, "rect.mtx", "%%MatrixMarket matrix coordinate real general\n2 3 1\n1 1 1.0\n")
    with pytest.raises(si.IoError, match="matrix must be square"):
        si.read_matrix_market(rect)


@pytest.mark.parametrize("text,needle", [
    ("", "empty file"),
    ("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1\n", "unsupported field 'complex'"),
    ("%%MatrixMarket vector coordinate real general\n", "unsupported object 'vector'"),
    ("%%MatrixMarket matrix coordinate real hermitian\n", "unsupported symmetry 'hermitian'"),
    ("%%MatrixMarket matrix dense real general\n", "unsupported format 'dense'"),
    ("%MatrixMarket matrix coordinate real general\n", "missing %%MatrixMarket banner"),
    ("%%MatrixMarket matrix coordinate real general\n% only comments\n", "missing size line"),
    ("%%MatrixMarket matrix coordinate real general\n2 2\n", ":2: malformed coordinate size line"),
    ("%%MatrixMarket matrix array real general\nx\n", "malformed array size line"),
    ("%%MatrixMarket matrix coordinate real general\n0 0 0\n", "empty matrix"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n", ":3: index out of range"),
    ("%%MatrixMarket matrix array real general\n1 1\n1.0 2.0\n", ":3: surplus array entry"),
    ("%%MatrixMarket matrix array real general\n2 2\n1.0 abc\n", ":3: malformed array entry"),
    ("%%MatrixMarket matrix array real symmetric\n2 2\n1.0\n", "expected 3 entries, got 1"),
])
def test_header_and_body_errors(tmp_path, text, needle):
    with pytest.raises(si.IoError, match=needle):
        si.read_matrix_market(_fixture(tmp_path, "e.mtx", text))


def test_libsvm_scan_and_errors(tmp_path):  # test_io_bench.cpp:102-123
    assert si.libsvm_shape(_fixture(tmp_path, "ridge.libsvm", "1 1:1\n0 2:2\n")) == (2, 2)
    assert si.libsvm_shape(_fixture(tmp_path, "c.libsvm", "# header\n\n1 3:1 1:2\n")) == (1, 3)
    with pytest.raises(si.IoError, match=r"no features found \(n = 0\)"):
        si.libsvm_shape(_fixture(tmp_path, "empty.libsvm", "1\n0\n"))
    with pytest.raises(si.IoError, match=":2: malformed feature token 'nocolon'"):
        si.libsvm_shape(_fixture(tmp_path, "bad.libsvm", "1 1:1\n0 nocolon\n"))
    with pytest.raises(si.IoError, match="1-based"):
        si.libsvm_shape(_fixture(tmp_path, "zero.libsvm", "1 0:1\n"))
    with pytest.raises(si.IoError, match="malformed feature token"):
        si.libsvm_shape(_fixture(tmp_path, "v.libsvm", "1 1:abc\n"))


# ------------------------------------------------------------------ device ingestion
@pytest.mark.gpu
def test_gpu_load_matrix_market_sparse_and_dense(tmp_path):
    path = _fixture(tmp_path, "coord.mtx", COORD_SYM)
    for keep in (True, False):
        p = si.load_matrix_market(path, keep_sparse=keep)
        assert p.n() == 2 and p.is_symmetric() and p.sparse == keep
        assert np.array_equal(p.data(), TWO_ONE)


@pytest.mark.gpu
def test_gpu_matrix_market_solver_roundtrip(tmp_path):
    """A larger sparse SPD file read as CSR drives the solver to the same
    iterate as the dense ProblemMatrix of the same matrix (bit-level parity is
    asserted elsewhere; here: same problem, same X within round-off)."""
    rng = np.random.default_rng(5)
    n = 96
    a = np.zeros((n, n))
    for i in range(n):
        a[i, i] = 4.0
        j = rng.integers(0, n, 3)
        a[i, j] += 0.1
    a = (a + a.T) / 2
    lines = [f"{i + 1} {j + 1} {float(a[i, j])!r}" for j in range(n) for i in range(j, n) if a[i, j] != 0.0]
    path = _fixture(tmp_path, "spd.mtx", "%%MatrixMarket matrix coordinate real symmetric\n"
                    f"{n} {n} {len(lines)}\n" + "\n".join(lines) + "\n")
    sparse = si.load_matrix_market(path, symmetry=si.Symmetry.spd)
    assert sparse.sparse
    assert np.array_equal(sparse.data(), a)
    dense = si.ProblemMatrix(a, si.Symmetry.spd)
    cfg = dict(rule=si.SketchRule.gaussian(8), tol=0.0, max_iters=20, seed=3)
    r1 = si.run_inverter(si.InverterConfig(sparse, **cfg))
    r2 = si.run_inverter(si.InverterConfig(dense, **cfg))
    assert np.linalg.norm(r1.state.x - r2.state.x) <= 1e-10 * np.linalg.norm(r2.state.x)


@pytest.mark.gpu
def test_gpu_ridge_hessian(tmp_path):  # test_io_bench.cpp:102-111
    h = si.build_ridge_hessian(_fixture(tmp_path, "ridge.libsvm", "1 1:1\n0 2:2\n"), 1.0)
    assert np.array_equal(h.data(), np.array([[2.0, 0.0], [0.0, 5.0]]))
    h.validate_spd()
    with pytest.raises(si.ConfigError):
        si.build_ridge_hessian(_fixture(tmp_path, "r2.libsvm", "1 1:1\n"), -1.0)


@pytest.mark.gpu
def test_gpu_ridge_hessian_random_rows(tmp_path):
    """Σ x xᵀ + λI over ragged sparse rows (with a duplicated index) vs numpy."""
    rng = np.random.default_rng(11)
    n, m, lam = 150, 700, 0.5
    rows, dense = [], np.zeros((m, n))
    for s in range(m):
        idx = rng.choice(n, size=int(rng.integers(0, 9)), replace=False) + 1
        vals = np.round(rng.normal(size=idx.size), 6)
        toks = [f"{int(k)}:{float(v)!r}" for k, v in zip(idx, vals)]
        if idx.size and s % 50 == 0:  # duplicated feature: contributes (v1 + v2)² like the reference's pair loop
            toks.append(f"{idx[0]}:0.25")
            dense[s, idx[0] - 1] += 0.25
        dense[s, idx - 1] += vals
        rows.append("1 " + " ".join(toks))
    rows[-1] = f"0 {n}:1.0"  # pin the feature count
    dense[-1] = 0.0
    dense[-1, n - 1] = 1.0
    h = si.build_ridge_hessian(_fixture(tmp_path, "rand.libsvm", "\n".join(rows) + "\n"), lam)
    want = dense.T @ dense + lam * np.eye(n)
    got = h.data()
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()
    assert np.array_equal(got, got.T)


@pytest.mark.gpu
def test_gpu_synthetic_generator():  # test_io_bench.cpp:125-137
    a1, a2, a3 = si.gen_synthetic(10, 7), si.gen_synthetic(10, 7), si.gen_synthetic(10, 8)
    d1 = a1.data()
    assert np.array_equal(d1, a2.data())
    assert np.linalg.norm(d1 - a3.data()) > 0.0
    assert np.array_equal(d1, d1.T)
    a1.validate_spd()
    with pytest.raises(si.ConfigError):
        si.gen_synthetic(1, 0)
    # ĀᵀĀ with Ā from RngStream(7): same host draws as the oracle's RngStream
    from oracle import oracle as orc
    abar = orc.RngStream(7).uniform_matrix(10, 10)
    want = abar.T @ abar
    assert np.abs(d1 - want).max() <= 1e-13 * np.abs(want).max()
    big = si.gen_synthetic(300, 42).data()
    abar = orc.RngStream(42).uniform_matrix(300, 300)
    want = abar.T @ abar
    assert np.abs(big - want).max() <= 1e-12 * np.abs(want).max()
