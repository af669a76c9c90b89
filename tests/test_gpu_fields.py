"""GPU parity of quadrature_fields (assembly.py:839-907) against the reference's goldens and the oracle."""
import numpy as np
import pytest

from oracle import surriga_oracle as O
from test_oracle_fields import check_fields, field_cases, field_golden, gauss_of


def disc_of(meta, arr):
    import paper_1904_06971_b200 as pkg
    from paper_1904_06971_b200.geometry import GeometryMap
    from paper_1904_06971_b200.spaces import NurbsWeights, make_tensor_space

    gsp = make_tensor_space(meta["geo_p"], meta["geo_ms"])
    geom = GeometryMap(space=gsp, weights=NurbsWeights(arr["geo_w"], polynomial_weight=True), control=arr["geo_ctrl"])
    p = meta["p"]
    space = make_tensor_space(p, [s + p for s in meta["spans"]])
    return pkg.Discretization(geom=geom, space=space, weights=NurbsWeights(arr["sol_w"]), gauss=p + 1)


@pytest.mark.gpu
@pytest.mark.parametrize("case", field_cases())
def test_gpu_fields_match_reference_golden(case):
    import paper_1904_06971_b200 as pkg

    meta, arr = field_golden(case)
    out = pkg.quadrature_fields(disc_of(meta, arr), arr["coefs"], nu=meta["nu"], gauss=meta["gauss"])
    check_fields(out, arr, meta["nu"])


@pytest.mark.gpu
@pytest.mark.parametrize("nu", [0, 1, 2])
def test_gpu_fields_vs_oracle_3d(nu):
    import paper_1904_06971_b200 as pkg

    disc = pkg.make_discretization(pkg.twisted_cube_standin(), 3, (6, 5, 7))
    c = np.cos(np.arange(disc.space.N) * 0.3)
    out = pkg.quadrature_fields(disc, c, nu=nu)
    ref = O.quadrature_fields(O.problem_from_disc("mass", disc), c, nu)
    x, w, v, g, h = ref
    arr = {"x": x, "w": w, "vals": v, "grads": g, "hesses": h}
    check_fields(out, arr, nu)


@pytest.mark.gpu
def test_gpu_fields_rational_gauss_override():
    import paper_1904_06971_b200 as pkg

    disc = pkg.make_discretization(pkg.quarter_annulus(1.0, 2.0), 2, (9, 7))
    c = np.sin(np.arange(disc.space.N) * 0.17)
    out = pkg.quadrature_fields(disc, c, nu=2, gauss=5)
    prob = O.problem_from_disc("mass", disc)
    prob.g = 5
    x, w, v, g, h = O.quadrature_fields(prob, c, 2)
    check_fields(out, {"x": x, "w": w, "vals": v, "grads": g, "hesses": h}, 2)
