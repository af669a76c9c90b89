"""GPU parity of the full / row-restricted assembly against the reference's golden vectors and the oracle."""
import numpy as np
import pytest

from golden_io import cases, load, oracle_problem
from gpu_util import disc_from_golden, form_of
from oracle import surriga_oracle as O

TOL = 1e-12

FULL = [c for c in cases() if load(c)[0]["kind"] in ("full", "rows")]


@pytest.mark.gpu
@pytest.mark.parametrize("case", FULL)
def test_gpu_assembly_matches_reference_golden(case):
    import paper_1904_06971_b200 as pkg

    meta, arr = load(case)
    disc = disc_from_golden(meta, arr)
    rows = arr["rows"] if meta["kind"] == "rows" else None
    A = pkg.assemble(form_of(meta), disc, rows=rows, coefficient=meta.get("coefficient", 1.0))
    m = A.mat
    assert m.indptr.dtype == np.int32 and m.indices.dtype == np.int32 and m.data.dtype == np.float64
    assert np.array_equal(m.indptr, arr["indptr"]), "indptr differs"
    assert np.array_equal(m.indices, arr["indices"]), "indices differ"
    err = O.row_scaled_error(arr["indptr"], arr["indices"], arr["data"], m.indptr, m.indices, m.data)
    assert err <= TOL, err
    assert A.symmetric == meta["symmetric"]
    if rows is not None:
        assert np.array_equal(A.populated_rows, arr["populated_rows"])
    if A.symmetric:
        assert pkg.is_bitwise_symmetric(A)
