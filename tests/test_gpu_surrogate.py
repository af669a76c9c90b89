"""GPU parity of the surrogate assembly against the reference's golden vectors and the oracle."""
import numpy as np
import pytest

from golden_io import cases, load, oracle_problem
from gpu_util import disc_from_golden, form_of
from oracle import surriga_oracle as O

TOL = 1e-12
SURR = [c for c in cases() if load(c)[0]["kind"] == "surrogate"]


@pytest.mark.gpu
@pytest.mark.parametrize("case", SURR)
def test_gpu_surrogate_matches_reference_golden(case):
    import paper_1904_06971_b200 as pkg

    meta, arr = load(case)
    disc = disc_from_golden(meta, arr)
    mode = None if meta["mode"] is None else pkg.SurrogateMode(meta["mode"])
    A, rep = pkg.build_surrogate_matrix(form_of(meta), disc, pkg.ConstantSampling(meta["M"]), q=meta["q"], mode=mode,
                                        coefficient=meta.get("coefficient", 1.0))
    m = A.mat
    assert m.indptr.dtype == np.int32 and m.indices.dtype == np.int32
    assert np.array_equal(m.indptr, arr["indptr"]), "indptr differs"
    assert np.array_equal(m.indices, arr["indices"]), "indices differ"
    err = O.row_scaled_error(arr["indptr"], arr["indices"], arr["data"], m.indptr, m.indices, m.data)
    assert err <= TOL, err
    assert A.symmetric == meta["symmetric"]
    for k, v in meta["report"].items():
        assert getattr(rep, k) == v, (k, getattr(rep, k), v)
    if A.symmetric:
        assert pkg.is_bitwise_symmetric(A)


@pytest.mark.gpu
@pytest.mark.parametrize("M,mode", [(1, None), (3, "general"), (5, None), (2, "symmetric")])
def test_gpu_surrogate_vs_oracle_3d(M, mode):
    import paper_1904_06971_b200 as pkg

    disc = pkg.make_discretization(pkg.twisted_cube_standin(), 2, (12, 13, 14))
    fk = pkg.FormKind.POISSON
    md = None if mode is None else pkg.SurrogateMode(mode)
    A, rep = pkg.build_surrogate_matrix(fk, disc, pkg.ConstantSampling(M), mode=md)
    (ip, ix, d), sym, r2 = O.surrogate(O.problem_from_disc(fk, disc), M, 3, mode)
    m = A.mat
    assert np.array_equal(m.indptr, ip) and np.array_equal(m.indices, ix)
    assert O.row_scaled_error(ip, ix, d, m.indptr, m.indices, m.data) <= TOL
    assert rep.interp_entries == r2["interp_entries"] and rep.active_elements == r2["active_elements"]
    if M == 1:
        full = pkg.assemble(fk, disc)
        assert pkg.matrices_bitwise_equal(full, A)


@pytest.mark.gpu
def test_gpu_surrogate_skp_kernel_and_symmetry():
    # SPEC acceptance 7: SKP -> A 1 = 0 to 1e-12 ||A||, bitwise symmetric; GENERAL breaks the kernel
    import paper_1904_06971_b200 as pkg

    disc = pkg.make_discretization(pkg.builtin_domain("coons_rational"), 2, (40, 40))
    A, _ = pkg.build_surrogate_matrix(pkg.FormKind.POISSON, disc, pkg.ConstantSampling(5))
    assert pkg.is_bitwise_symmetric(A)
    assert np.max(np.abs(A.row_sums())) <= 1e-12 * A.max_abs()
    G, _ = pkg.build_surrogate_matrix(pkg.FormKind.POISSON, disc, pkg.ConstantSampling(5),
                                      mode=pkg.SurrogateMode.GENERAL)
    assert np.max(np.abs(G.row_sums())) > 1e-10 * G.max_abs()


ROWS3 = [(2, (26, 27, 25), 8, "poisson", None), (2, (26, 27, 25), 8, "poisson", "general"),
         (3, (28, 29, 27), 8, "mass", None)]


@pytest.mark.gpu
@pytest.mark.parametrize("p,spans,M,form,mode", ROWS3)
def test_gpu_surrogate_rows3_kernel_vs_oracle(p, spans, M, form, mode):
    # 3D interpolation degree 3 with M >= 8 runs the row-staged K7 kernel (interp_rows3)
    import paper_1904_06971_b200 as pkg
    from paper_1904_06971_b200 import _lib

    disc = pkg.make_discretization(pkg.twisted_cube_standin(), p, spans)
    fk = pkg.FormKind(form)
    md = None if mode is None else pkg.SurrogateMode(mode)
    A, rep = pkg.build_surrogate_matrix(fk, disc, pkg.ConstantSampling(M), mode=md)
    assert "interp_rows3" in [n for n, _ in _lib.last_kernel_times()]
    (ip, ix, d), sym, r2 = O.surrogate(O.problem_from_disc(fk, disc), M, 3, mode)
    m = A.mat
    assert np.array_equal(m.indptr, ip) and np.array_equal(m.indices, ix)
    assert O.row_scaled_error(ip, ix, d, m.indptr, m.indices, m.data) <= TOL
    assert rep.interp_entries == r2["interp_entries"] and rep.quad_entries == r2["quad_entries"]
    assert A.symmetric == sym
    if sym:
        assert pkg.is_bitwise_symmetric(A)


@pytest.mark.gpu
@pytest.mark.parametrize("p,spans,form", [(1, (30, 29, 31), "poisson"), (4, (37, 38, 36), "mass"), (4, (37, 38, 36), "poisson")])
def test_gpu_rows3_kernel_matches_64row_kernel(p, spans, form, monkeypatch):
    # degrees 1 and 4 of the row-staged kernel against the 64-row-tile kernel (SG_INTERP_FIX=1) on
    # the same surrogate: identical pattern and counts, values within 1e-12 row-scaled
    import paper_1904_06971_b200 as pkg
    from paper_1904_06971_b200 import _lib

    disc = pkg.make_discretization(pkg.twisted_cube_standin(), p, spans)
    fk = pkg.FormKind(form)
    A, rep = pkg.build_surrogate_matrix(fk, disc, pkg.ConstantSampling(8))
    assert "interp_rows3" in [n for n, _ in _lib.last_kernel_times()]
    monkeypatch.setenv("SG_INTERP_FIX", "1")
    B, rep2 = pkg.build_surrogate_matrix(fk, disc, pkg.ConstantSampling(8))
    assert "interp_rows3" not in [n for n, _ in _lib.last_kernel_times()]
    a, b = A.mat, B.mat
    assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)
    assert O.row_scaled_error(b.indptr, b.indices, b.data, a.indptr, a.indices, a.data) <= TOL
    assert rep.interp_entries == rep2.interp_entries and rep.quad_entries == rep2.quad_entries
    if A.symmetric:
        assert pkg.is_bitwise_symmetric(A)


ZERO = [("annulus", 2, (14, 13), 4), ("twisted", 2, (26, 27, 25), 8)]


@pytest.mark.gpu
@pytest.mark.parametrize("geom,p,spans,M", ZERO)
def test_gpu_surrogate_exact_zero_drop(geom, p, spans, M):
    # coefficient 0: every merged entry is an exact zero and scipy's CSR add drops it
    # (surrogate.py:670).  GENERAL: empty pattern, report counts unchanged, as the reference gives;
    # SKP: the positional reset (surrogate.py:673-680) then indexes an empty row -- IndexError in the
    # reference, the oracle and here alike.
    import paper_1904_06971_b200 as pkg

    g = pkg.quarter_annulus(1.0, 2.0) if geom == "annulus" else pkg.twisted_cube_standin()
    disc = pkg.make_discretization(g, p, spans)
    fk = pkg.FormKind.POISSON
    prob = O.problem_from_disc(fk, disc, coefficient=0.0)
    A, rep = pkg.build_surrogate_matrix(fk, disc, pkg.ConstantSampling(M), mode=pkg.SurrogateMode.GENERAL,
                                        coefficient=0.0)
    (ip, ix, d), sym, r2 = O.surrogate(prob, M, 3, "general")
    assert d.size == 0 and A.mat.nnz == 0 and np.array_equal(A.mat.indptr, ip)
    assert rep.interp_entries == r2["interp_entries"] and rep.quad_entries == r2["quad_entries"]
    with pytest.raises(IndexError):
        O.surrogate(prob, M, 3, None)
    with pytest.raises(IndexError):
        pkg.build_surrogate_matrix(fk, disc, pkg.ConstantSampling(M), coefficient=0.0)
    # the library stays usable after the failed call
    B, _ = pkg.build_surrogate_matrix(fk, disc, pkg.ConstantSampling(M))
    assert B.mat.nnz > 0


@pytest.mark.gpu
def test_gpu_surrogate_exact_zero_drop_row_slabs():
    # the zero-drop compaction per row slab: GENERAL slabs stitch to the full result;
    # SKP's positional reset (surrogate.py:673-680) past a slab's end is refused, past the matrix's
    # end it is the reference's IndexError
    import paper_1904_06971_b200 as pkg
    from paper_1904_06971_b200._lib import NativeError
    from paper_1904_06971_b200.slabs import plane_slabs, stitch
    from paper_1904_06971_b200.surrogate import surrogate_device

    disc = pkg.make_discretization(pkg.twisted_cube_standin(), 2, (26, 27, 25))
    fk = pkg.FormKind.POISSON
    full, st, _ = surrogate_device(fk, disc, 8, 3, "general", coefficient=0.0)
    fip, fix, fd = full.to_host()
    full.free()
    assert st.n_zero_dropped > 0 and fd.size == 0
    ms = tuple(kv.m for kv in disc.space.kvs)
    parts = []
    slabs = plane_slabs(ms, 3)
    for lo, hi in slabs:
        res, _, _ = surrogate_device(fk, disc, 8, 3, "general", slab=(lo, hi), coefficient=0.0)
        parts.append(res.to_host())
        res.free()
    ip, ix, d = stitch(parts)
    assert np.array_equal(ip, fip) and ix.size == 0 and d.size == 0
    with pytest.raises(NativeError):
        surrogate_device(fk, disc, 8, 3, "symmetric_kernel_preserving", slab=slabs[0], coefficient=0.0)
    with pytest.raises(IndexError):
        surrogate_device(fk, disc, 8, 3, "symmetric_kernel_preserving", slab=slabs[-1], coefficient=0.0)
