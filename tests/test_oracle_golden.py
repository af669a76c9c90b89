"""Pin the CPU oracle against the reference's own outputs (golden vectors) -- CPU only."""
import numpy as np
import pytest

from golden_io import cases, load, oracle_problem
from oracle import surriga_oracle as O

TOL = 1e-12


@pytest.mark.parametrize("case", cases())
def test_oracle_matches_reference_golden(case):
    meta, arr = load(case)
    prob = oracle_problem(meta, arr)
    if meta["kind"] == "full":
        ip, ix, d, sym, pop = O.assemble(prob)
    elif meta["kind"] == "rows":
        ip, ix, d, sym, pop = O.assemble(prob, rows=arr["rows"])
        assert np.array_equal(pop, arr["populated_rows"])
    else:
        (ip, ix, d), sym, rep = O.surrogate(prob, meta["M"], meta["q"], meta["mode"])
        for k, v in meta["report"].items():
            assert rep[k] == v, (k, rep[k], v)
    assert sym == meta["symmetric"]
    assert np.array_equal(ip, arr["indptr"].astype(np.int64))
    assert np.array_equal(ix, arr["indices"])
    err = O.row_scaled_error(arr["indptr"], arr["indices"], arr["data"], ip, ix, d)
    assert err <= TOL, err


def test_oracle_p1_stencil_kat():
    # test_assembly.py:48-64: p=1 unit-square rows factor into 1D stencils
    meta, arr = load("unit_square_p1_poisson")
    prob = oracle_problem(meta, arr)
    import scipy.sparse as sp
    ip, ix, d, _, _ = O.assemble(prob)
    K = sp.csr_matrix((d, ix, ip), shape=(25, 25)).toarray()
    h = 0.25
    m1 = np.array([h / 6, 2 * h / 3, h / 6])
    k1 = np.array([-1 / h, 2 / h, -1 / h])
    row = K[2 + 2 * 5].reshape(5, 5, order="F")
    expect = np.zeros((5, 5))
    expect[1:4, 1:4] = np.outer(k1, m1) + np.outer(m1, k1)
    assert np.max(np.abs(row - expect)) < 1e-13


def test_oracle_skp_after_zero_drop_raises_like_reference():
    # the reference raises IndexError (surrogate.py:673-680 indexes an emptied row) for coefficient 0
    # in kernel-preserving mode; GENERAL mode gives the empty golden above
    meta, arr = load("annulus_poisson_surr_zero_general")
    prob = oracle_problem(meta, arr)
    with pytest.raises(IndexError):
        O.surrogate(prob, meta["M"], meta["q"], None)
