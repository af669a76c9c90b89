"""CPU tests of the host-side mirror of the reference interface (no device calls)."""
from fractions import Fraction

import numpy as np
import pytest

import paper_1904_06971_b200 as pkg
from paper_1904_06971_b200 import surrogate as S
from paper_1904_06971_b200.spaces import basis_table, make_open_uniform_knots, make_tensor_space
from golden_io import cases, load, oracle_problem
from oracle import surriga_oracle as O


def test_spec_kat_offsets():
    # SPEC.md:322-325
    o = S.build_offsets(2, 2)
    assert o.count == 25 and o.canonical_half().size == 13
    o3 = S.build_offsets(1, 3)
    assert o3.count == 27
    sh = {tuple(x) for x in o3.shifts}
    assert all(tuple(-np.asarray(x)) in sh for x in sh)
    # colex order = ascending column order (surrogate.py:312-322)
    strides = np.array([1, 10, 100])
    assert np.all(np.diff(o3.shifts @ strides) > 0)


def test_spec_kat_tilde_and_lattice():
    t = S.tilde_domain(2, (21, 21))
    assert t.bounds[0] == (Fraction(7, 38), Fraction(31, 38))
    assert S.tilde_domain(2, (8,)).is_empty
    kvs = make_tensor_space(2, [21, 21]).kvs
    lat = S.build_sampling_lattice(kvs, 5)
    assert list(lat.indices[0]) == [4, 9, 14, 16]           # SPEC.md:341 (0-based)
    assert list(S.build_sampling_lattice(kvs, 1).indices[0]) == list(range(4, 17))
    assert list(S.build_sampling_lattice(kvs, 100).indices[0]) == [4, 16]


def test_spec_kat_mesh_dependent_M():
    assert S.mesh_dependent_M(S.MeshDependentSampling(0.0), 1 / 64, 2, 5) == 1
    assert S.mesh_dependent_M(S.MeshDependentSampling(3.0, 0.5), 1 / 64, 2, 5) == 16
    assert S.mesh_dependent_M(S.MeshDependentSampling(0.75, 0.5), 1 / 32, 2, 5) == 3
    with pytest.raises(ValueError):
        S.mesh_dependent_M(S.MeshDependentSampling(1.0), 0.1, 3, 3)
    with pytest.raises(TypeError):
        S.mesh_dependent_M(object(), 0.1, 2, 3)
    with pytest.raises(ValueError):
        S.mesh_dependent_M(S.ConstantSampling(0), 0.1, 2, 3)


def test_knots_and_basis_match_oracle():
    for p in (1, 2, 3, 4):
        kv = make_open_uniform_knots(p, 2 * p + 7)
        assert np.array_equal(kv.knots, O.open_uniform_knots(p, kv.m))
        x = np.linspace(0, 1, 37)
        s1, t1 = basis_table(kv.knots, p, x, 2)
        s2, t2 = O.basis_ders(kv.knots, p, x, 2)
        assert np.array_equal(s1, s2) and np.array_equal(t1, t2)
        assert np.allclose(t1[:, 0].sum(1), 1.0, atol=1e-14)


def test_geometry_builders_match_reference_fixture_nets():
    # the geometry nets stored with the goldens were produced by the reference's own builders
    for case in cases():
        meta, arr = load(case)
        g = meta["geometry"]
        if g.endswith(".geo"):
            ref = pkg.load_geometry(f"paper_1904_06971_b200/data/{g}")
        elif g == "annulus":
            ref = pkg.quarter_annulus(1.0, 2.0)
        else:
            ref = pkg.builtin_domain(g)
        assert np.allclose(ref.control, arr["geo_ctrl"], rtol=0, atol=1e-14), case
        assert np.allclose(ref.weights.weights, arr["geo_w"], rtol=0, atol=1e-15), case


def test_make_discretization_weights_match_reference():
    for case in ("cfg1_full_poisson", "annulus_mass_p3", "annulus_biharm_p3"):
        meta, arr = load(case)
        disc = pkg.make_discretization(pkg.quarter_annulus(1.0, 2.0), meta["p"], tuple(meta["spans"]))
        assert np.allclose(disc.weights.weights, arr["sol_w"], rtol=1e-14, atol=0)


@pytest.mark.parametrize("case", [c for c in cases() if load(c)[0]["kind"] == "surrogate"])
def test_surrogate_plan_matches_reference_report(case):
    meta, arr = load(case)
    from gpu_util import disc_from_golden

    disc = disc_from_golden(meta, arr)
    plan = S.surrogate_plan(disc, S.ConstantSampling(meta["M"]), meta["q"])
    rep = meta["report"]
    assert plan.active_elements == rep["active_elements"]
    if "surrogate=disabled" not in rep["flags"]:
        assert plan.interp_entries == rep["interp_entries"]
        assert plan.quad_entries == rep["quad_entries"]


def test_elements_for_rows_matches_oracle():
    ms, p = (9, 11, 7), 2
    rng = np.random.default_rng(0)
    rows = np.unique(rng.integers(0, np.prod(ms), 40))
    from paper_1904_06971_b200.assembly import _elements_for_rows

    assert np.array_equal(_elements_for_rows(ms, p, rows), O.elements_for_rows(ms, p, rows))


def test_argument_validation_messages():
    disc = pkg.make_discretization(pkg.unit_square(), 1, (4, 4))
    with pytest.raises(ValueError, match="assemble_divergence"):
        pkg.assemble(pkg.FormKind.STOKES_DIVERGENCE, disc)
    with pytest.raises(ValueError, match="fourth-order"):
        pkg.assemble(pkg.FormKind.BIHARMONIC, disc)
    with pytest.raises(ValueError, match="coefficient"):
        pkg.assemble(pkg.FormKind.MASS, pkg.make_discretization(pkg.unit_square(), 2, (4, 4)), coefficient=2.0)
    with pytest.raises(ValueError, match="kernel-preserving"):
        pkg.build_surrogate_matrix(pkg.FormKind.MASS, disc, mode=pkg.SurrogateMode.SYMMETRIC_KERNEL_PRESERVING)
    with pytest.raises(ValueError, match="build_surrogate_divergence"):
        pkg.build_surrogate_matrix(pkg.FormKind.STOKES_DIVERGENCE, disc)
    with pytest.raises(ValueError):
        pkg.make_discretization(pkg.unit_square(), 2, (4, 4), gauss=0)


@pytest.mark.parametrize("p,spans,M", [(2, (24, 24), 5), (3, (30, 29, 31), 4), (1, (12, 12, 12), 3), (3, (40,), 7),
                                       (2, (9, 10), 2), (3, (128, 128, 128), 16)])
def test_active_element_count_matches_row_dilation(p, spans, M):
    # the closed-form count of elements supporting a quadrature row equals the O(N) row-mask
    # dilation (_elements_for_rows of the quadrature rows, surrogate.py:590)
    from paper_1904_06971_b200.assembly import _elements_for_rows
    from paper_1904_06971_b200.spaces import make_tensor_space
    from paper_1904_06971_b200.surrogate import (_active_element_count, _flat, _masks, build_sampling_lattice,
                                                 tilde_domain)

    space = make_tensor_space(p, [s + p for s in spans])
    ms = tuple(kv.m for kv in space.kvs)
    tilde = tilde_domain(p, ms)
    lat = build_sampling_lattice(space.kvs, M, tilde)
    inb, smp = _masks(tilde, lat)
    quad = np.flatnonzero(~_flat(inb) | _flat(smp))
    assert _active_element_count(ms, p, tilde, lat) == _elements_for_rows(ms, p, quad).size
