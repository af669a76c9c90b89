"""GPU parity of the load vector (assembly.py:728-759) against the reference's goldens and the oracle."""
import numpy as np
import pytest

from load_funcs import LOAD_FUNCS
from oracle import surriga_oracle as O
from test_oracle_load import load_cases, load_golden, problem

TOL = 1e-13


def disc_of(meta, arr):
    import paper_1904_06971_b200 as pkg
    from paper_1904_06971_b200.geometry import GeometryMap
    from paper_1904_06971_b200.spaces import NurbsWeights, make_tensor_space

    gsp = make_tensor_space(meta["geo_p"], meta["geo_ms"])
    geom = GeometryMap(space=gsp, weights=NurbsWeights(arr["geo_w"], polynomial_weight=True), control=arr["geo_ctrl"])
    p = meta["p"]
    space = make_tensor_space(p, [s + p for s in meta["spans"]])
    return pkg.Discretization(geom=geom, space=space, weights=NurbsWeights(arr["sol_w"]), gauss=meta["gauss"])


@pytest.mark.gpu
@pytest.mark.parametrize("case", load_cases())
def test_gpu_load_matches_reference_golden(case):
    import paper_1904_06971_b200 as pkg

    meta, arr = load_golden(case)
    vec = pkg.assemble_load(disc_of(meta, arr), LOAD_FUNCS[meta["func"]])
    ref = arr["vec"]
    assert vec.shape == ref.shape
    assert np.max(np.abs(vec - ref)) <= TOL * max(1.0, np.max(np.abs(ref)))


@pytest.mark.gpu
def test_gpu_load_constant_is_mass_row_sums():
    # f = 1: vec_i = sum_j M_ij (partition of unity), i.e. the mass matrix row sums
    import paper_1904_06971_b200 as pkg

    disc = pkg.make_discretization(pkg.twisted_cube_standin(), 2, (5, 4, 6))
    vec = pkg.assemble_load(disc, lambda x: np.ones(x.shape[:-1]))
    M = pkg.assemble(pkg.FormKind.MASS, disc).mat
    assert np.max(np.abs(vec - np.asarray(M.sum(axis=1)).ravel())) < 1e-14 * max(1.0, np.abs(vec).max())
    ref = O.load_vector(O.problem_from_disc("mass", disc), lambda x: np.ones(x.shape[:-1]))
    assert np.max(np.abs(vec - ref)) < 1e-13 * np.abs(ref).max()
