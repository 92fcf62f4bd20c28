"""MatrixMarket I/O: exact round trips, scipy as an
independent reader/writer, symmetric / pattern / duplicate handling, vectors, errors."""
import numpy as np
import pytest
import scipy.io
import scipy.sparse as sp

from oracle import oracle as O
from paper_1901_01685_b200 import mmio
from paper_1901_01685_b200 import problems as P
from paper_1901_01685_b200._native import Csr


def csr_of(M):
    M = sp.csr_matrix(M)
    M.sort_indices()
    return Csr(M.shape[0], M.shape[1], M.indptr.astype(np.int32), M.indices.astype(np.int32),
               M.data.astype(np.float64))


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def test_round_trip_is_exact(tmp_path):
    rng = np.random.default_rng(0)
    M = sp.random(57, 43, density=0.2, random_state=1, format="csr")
    M.data = rng.standard_normal(M.nnz) * 10.0 ** rng.integers(-300, 300, M.nnz)
    A = csr_of(M)
    mmio.write_matrix(tmp_path / "a.mtx", A, comment="round trip")
    B = mmio.read_matrix(tmp_path / "a.mtx")
    assert (B.nrows, B.ncols) == (57, 43)
    np.testing.assert_array_equal(B.rowptr, A.rowptr)
    np.testing.assert_array_equal(B.col, A.col)
    np.testing.assert_array_equal(bits(B.val), bits(A.val))


def test_scipy_reads_ours_and_we_read_scipys(tmp_path):
    pb = P.build(1)
    A = pb.plevels[0].A  # an assembled operator (SPEC.md:193 export of A_k)
    mmio.write_matrix(tmp_path / "A.mtx", A)
    S = sp.csr_matrix(scipy.io.mmread(str(tmp_path / "A.mtx")))
    S.sort_indices()
    np.testing.assert_array_equal(S.indptr, A.rowptr)
    np.testing.assert_array_equal(S.indices, A.col)
    np.testing.assert_array_equal(bits(S.data), bits(A.val))
    M = sp.random(30, 30, density=0.1, random_state=3)
    M = (M + M.T).tocoo()
    scipy.io.mmwrite(str(tmp_path / "s.mtx"), M, symmetry="symmetric", precision=17)
    B = mmio.read_matrix(tmp_path / "s.mtx")
    R = csr_of(M)
    np.testing.assert_array_equal(B.rowptr, R.rowptr)
    np.testing.assert_array_equal(B.col, R.col)
    np.testing.assert_array_equal(bits(B.val), bits(R.val))


def test_read_operator_drives_the_solver_path(tmp_path):
    """A matrix read back from its export gives the same residual as the in-memory one."""
    pb = P.build(1)
    A = pb.plevels[0].A
    mmio.write_matrix(tmp_path / "A.mtx", A)
    B = mmio.read_matrix(tmp_path / "A.mtx")
    x = np.random.default_rng(1).uniform(-1, 1, A.ncols)
    np.testing.assert_array_equal(bits(O.residual(B, x, pb.f)), bits(O.residual(A, x, pb.f)))


def test_symmetric_skew_pattern_and_duplicates(tmp_path):
    (tmp_path / "m.mtx").write_text(
        "%%MatrixMarket matrix coordinate real skew-symmetric\n% comment\n3 3 2\n2 1 1.5\n3 2 -2\n")
    B = mmio.read_matrix(tmp_path / "m.mtx")
    D = np.zeros((3, 3))
    D[1, 0], D[0, 1], D[2, 1], D[1, 2] = 1.5, -1.5, -2.0, 2.0
    np.testing.assert_array_equal(sp.csr_matrix((B.val, B.col, B.rowptr), shape=(3, 3)).toarray(), D)
    (tmp_path / "p.mtx").write_text("%%MatrixMarket matrix coordinate pattern general\n2 3 3\n1 3\n2 1\n1 1\n")
    B = mmio.read_matrix(tmp_path / "p.mtx")
    np.testing.assert_array_equal(B.rowptr, [0, 2, 3])
    np.testing.assert_array_equal(B.col, [0, 2, 0])
    np.testing.assert_array_equal(B.val, [1.0, 1.0, 1.0])
    (tmp_path / "d.mtx").write_text("%%MatrixMarket matrix coordinate real general\n1 1 3\n1 1 0.1\n1 1 0.2\n1 1 0.3\n")
    B = mmio.read_matrix(tmp_path / "d.mtx")
    assert B.val[0] == (0.1 + 0.2) + 0.3  # duplicates summed in file order


def test_vectors(tmp_path):
    v = np.random.default_rng(2).standard_normal(101)
    mmio.write_vector(tmp_path / "v.mtx", v)
    np.testing.assert_array_equal(bits(mmio.read_vector(tmp_path / "v.mtx")), bits(v))
    (tmp_path / "v.txt").write_text("".join(f"{float(x)!r}\n" for x in v))  # plain text, one value per line
    np.testing.assert_array_equal(bits(mmio.read_vector(tmp_path / "v.txt")), bits(v))
    assert mmio.read_vector(tmp_path / "v.txt").size == 101


@pytest.mark.parametrize("text", ["not a header\n1 1 1\n", "%%MatrixMarket matrix array real general\n1 1\n1\n",
                                  "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n",
                                  "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n"])
def test_errors(tmp_path, text):
    (tmp_path / "bad.mtx").write_text(text)
    with pytest.raises(OSError):
        mmio.read_matrix(tmp_path / "bad.mtx")
    with pytest.raises(OSError):
        mmio.read_matrix(tmp_path / "missing.mtx")
