"""GPU parity of the mixed divergence pairing (assembly.py:654-725) against the reference's goldens
(tests/golden/div) and the oracle; properties of test_assembly.py:154-178."""
import numpy as np
import pytest

from oracle import surriga_oracle as O
from test_oracle_divergence import check_component, div_cases, load_div, vel_problem

TOL = 1e-12


def stokes_from_golden(meta, arr):
    import paper_1904_06971_b200 as pkg
    from paper_1904_06971_b200.geometry import GeometryMap
    from paper_1904_06971_b200.spaces import NurbsWeights, make_tensor_space

    gsp = make_tensor_space(meta["geo_p"], meta["geo_ms"])
    geom = GeometryMap(space=gsp, weights=NurbsWeights(arr["geo_w"], polynomial_weight=True), control=arr["geo_ctrl"])
    st = pkg.stokes_subgrid_spaces(geom, meta["pp"], tuple(meta["spans"]))
    if st.velocity.gauss != meta["gauss"]:
        st = pkg.stokes_subgrid_spaces(geom, meta["pp"], tuple(meta["spans"]), gauss=meta["gauss"])
    return st


@pytest.mark.gpu
@pytest.mark.parametrize("case", [c for c in div_cases() if not c.startswith("sdiv_")])
def test_gpu_divergence_matches_reference_golden(case):
    import paper_1904_06971_b200 as pkg

    meta, arr = load_div(case)
    st = stokes_from_golden(meta, arr)
    rows = arr.get("rows")
    D = pkg.assemble_divergence(st, rows=rows)
    assert len(D) == meta["n"]
    for c, Dc in enumerate(D):
        m = Dc.mat
        assert m.indptr.dtype == np.int32 and m.indices.dtype == np.int32 and m.data.dtype == np.float64
        check_component(arr, c, m.indptr.astype(np.int64), m.indices, m.data)
        assert Dc.symmetric is False
        if rows is not None:
            assert np.array_equal(Dc.populated_rows, arr["populated_rows"])


@pytest.mark.gpu
def test_gpu_divergence_matches_oracle_larger_3d():
    import paper_1904_06971_b200 as pkg

    st = pkg.stokes_subgrid_spaces(pkg.twisted_cube_standin(), 2, (4, 3, 5))
    D = pkg.assemble_divergence(st)
    vel = O.problem_from_disc("stokes_divergence", st.velocity)
    ip, ix, data, _ = O.divergence(vel, 2)
    for c, Dc in enumerate(D):
        assert np.array_equal(Dc.mat.indptr, ip) and np.array_equal(Dc.mat.indices, ix)
        assert O.row_scaled_error(ip, ix, data[c], Dc.mat.indptr, Dc.mat.indices, Dc.mat.data) <= TOL


@pytest.mark.gpu
def test_gpu_divergence_rows_bitwise_and_constant_field():
    # test_assembly.py:154-160 and :173-178 on the GPU path
    import paper_1904_06971_b200 as pkg

    st = pkg.stokes_subgrid_spaces(pkg.builtin_domain("coons_quadratic"), 2, (6, 6))
    full = pkg.assemble_divergence(st)
    ones = np.ones(st.velocity.space.N)
    for Dc in full:
        assert np.max(np.abs(Dc.mat @ ones)) < 1e-13
    rows = np.array([0, 5, 17, 40])
    part = pkg.assemble_divergence(st, rows=rows)
    for Df, Dp in zip(full, part):
        assert pkg.matrices_bitwise_equal(Df, Dp, rows=rows)


@pytest.mark.gpu
@pytest.mark.parametrize("pp,spans", [(2, (14, 11)), (3, (9, 10))])
def test_gpu_divergence_rational_spaces(pp, spans):
    # NURBS velocity and pressure spaces (quarter annulus): the oracle's rational restatement (pinned
    # by the div_annulus_* goldens), partition of unity (constant velocity -> 0), rows bitwise
    import paper_1904_06971_b200 as pkg

    st = pkg.stokes_subgrid_spaces(pkg.quarter_annulus(1.0, 2.0), pp, spans)
    assert np.ptp(st.velocity.weights.weights) > 0 and np.ptp(st.pressure.weights.weights) > 0
    D = pkg.assemble_divergence(st)
    vel = O.problem_from_disc("stokes_divergence", st.velocity)
    ip, ix, data, _ = O.divergence(vel, pp, prs_w=st.pressure.weights.weights)
    ones = np.ones(st.velocity.space.N)
    for c, Dc in enumerate(D):
        assert np.array_equal(Dc.mat.indptr, ip) and np.array_equal(Dc.mat.indices, ix)
        assert O.row_scaled_error(ip, ix, data[c], Dc.mat.indptr, Dc.mat.indices, Dc.mat.data) <= TOL
        assert np.max(np.abs(Dc.mat @ ones)) < 1e-12 * np.max(np.abs(Dc.mat.data))
    rows = np.array([0, 7, 30, st.pressure.space.N - 1])
    part = pkg.assemble_divergence(st, rows=rows)
    for Df, Dp in zip(D, part):
        assert pkg.matrices_bitwise_equal(Df, Dp, rows=rows)


def check_zero_drop_tolerant(arr, c, A, tol=TOL, max_diff=4):
    """The surrogate merge drops exact zeros (scipy CSR add, surrogate.py:810).  A structurally zero
    entry is a rounding residue (|v| ~ 1e-19 of the row scale) whose exact-zero status depends on the
    summation order, so the patterns may differ in such entries only: every entry present in one
    matrix and absent from the other must be below ``tol`` x row max, and the values agree within
    ``tol`` row-scaled.  Everything else is compared exactly like the other parity tests."""
    import scipy.sparse as sp

    G = sp.csr_matrix((arr[f"data_{c}"], arr[f"indices_{c}"], arr[f"indptr_{c}"]), shape=A.shape)
    if np.array_equal(A.indptr, G.indptr) and np.array_equal(A.indices, G.indices):
        check_component(arr, c, A.indptr.astype(np.int64), A.indices, A.data)
        return
    diff = abs(A - G).tocsr()
    rmax = np.maximum(abs(G).max(axis=1).toarray().ravel(), abs(A).max(axis=1).toarray().ravel())
    rows = np.repeat(np.arange(A.shape[0]), np.diff(diff.indptr))
    assert np.all(diff.data <= tol * rmax[rows]), "values differ beyond tolerance"
    ga = set(zip(*A.nonzero()))
    gg = set(zip(*G.nonzero()))
    for r, cc in ga ^ gg:
        v = A[r, cc] if (r, cc) in ga else G[r, cc]
        assert abs(v) <= tol * rmax[r], (r, cc, v)
    assert len(ga ^ gg) <= max_diff, f"{len(ga ^ gg)} pattern differences"


@pytest.mark.gpu
@pytest.mark.parametrize("case", [c for c in div_cases() if c.startswith("sdiv_")])
def test_gpu_surrogate_divergence_matches_reference_golden(case):
    import paper_1904_06971_b200 as pkg

    meta, arr = load_div(case)
    st = stokes_from_golden(meta, arr)
    D, rep = pkg.build_surrogate_divergence(st, pkg.ConstantSampling(meta["M"]), q=meta["q"])
    for k, v in meta["report"].items():
        assert getattr(rep, k) == v, (k, getattr(rep, k), v)
    for c, Dc in enumerate(D):
        check_zero_drop_tolerant(arr, c, Dc.mat)
        assert Dc.symmetric is False


@pytest.mark.gpu
def test_gpu_surrogate_divergence_matches_oracle_3d():
    import paper_1904_06971_b200 as pkg

    st = pkg.stokes_subgrid_spaces(pkg.twisted_cube_standin(), 1, (10, 9, 11))
    D, rep = pkg.build_surrogate_divergence(st, pkg.ConstantSampling(4))
    mats, orep = O.surrogate_divergence(O.problem_from_disc("stokes_divergence", st.velocity), 1, 4, 3)
    assert rep.interp_entries == orep["interp_entries"] and rep.quad_entries == orep["quad_entries"]
    for Dc, (ip, ix, d) in zip(D, mats):
        assert np.array_equal(Dc.mat.indptr, ip) and np.array_equal(Dc.mat.indices, ix)
        assert O.row_scaled_error(ip, ix, d, Dc.mat.indptr, Dc.mat.indices, Dc.mat.data) <= TOL


def thick_annulus():
    """3D NURBS domain: the quarter annulus (the reference's net, data/quarter_annulus_1_2.geo)
    extruded linearly in z over [0, 1] with degree 2 (rational weights vary in y, not in z)."""
    import paper_1904_06971_b200 as pkg
    from paper_1904_06971_b200.geometry import GeometryMap
    from paper_1904_06971_b200.spaces import NurbsWeights, make_tensor_space

    a = pkg.quarter_annulus(1.0, 2.0)
    space = make_tensor_space(2, tuple(a.space.shape) + (5,))
    zg = space.kvs[2].greville()
    n2 = a.space.N
    w = np.tile(a.weights.weights, zg.size)
    ctrl = np.column_stack([np.tile(a.control, (zg.size, 1)), np.repeat(zg, n2)])
    return GeometryMap(space=space, weights=NurbsWeights(w, polynomial_weight=True), control=ctrl, name="thick_annulus")


@pytest.mark.gpu
def test_gpu_divergence_rational_3d():
    import paper_1904_06971_b200 as pkg

    st = pkg.stokes_subgrid_spaces(thick_annulus(), 2, (3, 4, 3))
    assert np.ptp(st.velocity.weights.weights) > 0
    D = pkg.assemble_divergence(st)
    vel = O.problem_from_disc("stokes_divergence", st.velocity)
    ip, ix, data, _ = O.divergence(vel, 2, prs_w=st.pressure.weights.weights)
    for c, Dc in enumerate(D):
        assert np.array_equal(Dc.mat.indptr, ip) and np.array_equal(Dc.mat.indices, ix)
        assert O.row_scaled_error(ip, ix, data[c], Dc.mat.indptr, Dc.mat.indices, Dc.mat.data) <= TOL


@pytest.mark.gpu
@pytest.mark.parametrize("geo,pp,spans", [("coons_quadratic", 2, (9, 8)), ("annulus", 2, (7, 9)), ("twisted", 1, (4, 5, 6))])
def test_gpu_divergence_row_slabs_stitch_bitwise(geo, pp, spans):
    # SURVEY §8e for the mixed pairing: per-GPU pressure-row slabs (velocity halo recomputed, no
    # exchange) reproduce every component bit for bit
    import paper_1904_06971_b200 as pkg
    from paper_1904_06971_b200.assembly import assemble_divergence_device
    from paper_1904_06971_b200.slabs import plane_slabs, stitch

    g = {"coons_quadratic": lambda: pkg.builtin_domain("coons_quadratic"), "annulus": lambda: pkg.quarter_annulus(1.0, 2.0),
         "twisted": pkg.twisted_cube_standin}[geo]()
    st = pkg.stokes_subgrid_spaces(g, pp, spans)
    full = pkg.assemble_divergence(st)
    ms = tuple(kv.m for kv in st.pressure.space.kvs)
    for world in (2, 3):
        parts = [[] for _ in full]
        for lo, hi in plane_slabs(ms, world):
            res, _ = assemble_divergence_device(st, slab=(lo, hi))
            for c, r in enumerate(res):
                parts[c].append(r.to_host())
                r.free()
        for c, Dc in enumerate(full):
            ip, ix, d = stitch(parts[c])
            assert np.array_equal(ip, Dc.mat.indptr) and np.array_equal(ix, Dc.mat.indices)
            assert np.array_equal(d.view(np.int64), Dc.mat.data.view(np.int64))


@pytest.mark.gpu
def test_gpu_surrogate_divergence_rational_3d():
    # general-mode surrogate pairing on NURBS spaces in 3D against the oracle (2D: sdiv_annulus_p2 golden)
    import paper_1904_06971_b200 as pkg

    st = pkg.stokes_subgrid_spaces(thick_annulus(), 2, (12, 11, 13))
    D, rep = pkg.build_surrogate_divergence(st, pkg.ConstantSampling(3))
    assert rep.interp_entries > 0
    mats, orep = O.surrogate_divergence(O.problem_from_disc("stokes_divergence", st.velocity), 2, 3, 3,
                                        prs_w=st.pressure.weights.weights)
    assert rep.interp_entries == orep["interp_entries"] and rep.quad_entries == orep["quad_entries"]
    # the extruded map makes many entries structural zeros whose exact-zero status (and hence the
    # merge's drop, surrogate.py:810) depends on the summation order: patterns may differ only in
    # entries below 1e-12 x the row maximum
    for c, (Dc, (ip, ix, d)) in enumerate(zip(D, mats)):
        ref = {f"indptr_{c}": ip, f"indices_{c}": ix, f"data_{c}": d}
        check_zero_drop_tolerant(ref, c, Dc.mat, max_diff=ix.size // 100)


@pytest.mark.gpu
@pytest.mark.parametrize("geo,pp,spans,M", [("coons_quadratic", 2, (20, 22), 4), ("twisted", 1, (10, 9, 11), 4)])
def test_gpu_surrogate_divergence_row_slabs_stitch_bitwise(geo, pp, spans, M):
    # each slab assembles its quadrature rows plus the lattice rows and interpolates only
    # its own rows; the stitched slabs equal the whole-matrix surrogate bit for bit
    import paper_1904_06971_b200 as pkg
    from paper_1904_06971_b200.slabs import plane_slabs, stitch
    from paper_1904_06971_b200.surrogate import surrogate_divergence_device

    g = pkg.builtin_domain("coons_quadratic") if geo == "coons_quadratic" else pkg.twisted_cube_standin()
    st = pkg.stokes_subgrid_spaces(g, pp, spans)
    full, rep = pkg.build_surrogate_divergence(st, pkg.ConstantSampling(M))
    assert rep.interp_entries > 0
    ms = tuple(kv.m for kv in st.pressure.space.kvs)
    for world in (2, 3):
        parts = [[] for _ in full]
        for lo, hi in plane_slabs(ms, world):
            for c, r in enumerate(surrogate_divergence_device(st, pkg.ConstantSampling(M), slab=(lo, hi))):
                parts[c].append(r.to_host())
                r.free()
        for c, Dc in enumerate(full):
            ip, ix, d = stitch(parts[c])
            assert np.array_equal(ip, Dc.mat.indptr) and np.array_equal(ix, Dc.mat.indices)
            assert np.array_equal(d.view(np.int64), Dc.mat.data.view(np.int64))
