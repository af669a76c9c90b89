"""MatrixMarket output (assembly.py:304-320).  The writer is native host code
(no GPU): files read back bit-exactly (the reference's own round-trip test, test_assembly.py:182-190)
with the reference's header / symmetry conventions."""
import numpy as np
import pytest
import scipy.sparse as sp

from golden_io import load


def golden_matrix(case):
    import paper_1904_06971_b200 as pkg

    meta, arr = load(case)
    n = arr["indptr"].size - 1
    mat = sp.csr_matrix((arr["data"], arr["indices"], arr["indptr"]), shape=(n, n))
    return pkg.SparseMatrix(mat=mat, symmetric=bool(meta["symmetric"]))


@pytest.mark.parametrize("case", ["cfg1_full_poisson", "annulus_poisson_surr_general", "tri3d_poisson_p2"])
def test_matrix_market_round_trip_is_bitwise(case, tmp_path):
    import paper_1904_06971_b200 as pkg

    A = golden_matrix(case)
    path = tmp_path / "A.mtx"
    pkg.save_matrix_market(path, A, threads=3)
    text = path.read_text()
    assert text.startswith("%%MatrixMarket matrix coordinate real " + ("symmetric" if A.symmetric else "general"))
    B = pkg.load_matrix_market(path)
    assert B.symmetric == A.symmetric
    assert pkg.matrices_bitwise_equal(A, B)
    lines = text.splitlines()
    nr, nc, cnt = map(int, lines[2].split())
    expect = sp.tril(A.mat).nnz if A.symmetric else A.mat.nnz
    assert (nr, nc, cnt) == (A.shape[0], A.shape[1], expect) and len(lines) == 3 + cnt


def test_matrix_market_reads_like_scipy_output(tmp_path):
    # the reference writes through scipy.io.mmwrite(precision=16); both files describe the same matrix
    import scipy.io

    import paper_1904_06971_b200 as pkg

    A = golden_matrix("cfg1_full_poisson")
    ours, ref = tmp_path / "ours.mtx", tmp_path / "ref.mtx"
    pkg.save_matrix_market(ours, A)
    scipy.io.mmwrite(str(ref), A.mat, field="real", precision=16, symmetry="symmetric")
    a, b = pkg.load_matrix_market(ours), pkg.load_matrix_market(ref)
    assert np.array_equal(a.mat.indptr, b.mat.indptr) and np.array_equal(a.mat.indices, b.mat.indices)
    assert np.max(np.abs(a.mat.data - b.mat.data)) <= 1e-15 * np.max(np.abs(b.mat.data))


def test_matrix_market_rectangular_general(tmp_path):
    import paper_1904_06971_b200 as pkg

    rng = np.random.default_rng(3)
    M = sp.random(7, 11, density=0.4, random_state=rng, format="csr")
    M.data = rng.standard_normal(M.nnz) * 10.0 ** rng.integers(-300, 300, M.nnz)
    A = pkg.SparseMatrix(mat=M, symmetric=False)
    path = tmp_path / "R.mtx"
    pkg.save_matrix_market(path, A)
    B = pkg.load_matrix_market(path)
    assert B.shape == (7, 11) and pkg.matrices_bitwise_equal(A, B)
