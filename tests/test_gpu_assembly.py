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


@pytest.mark.gpu
@pytest.mark.parametrize("form,geom,p,spans", [("poisson", "twisted", 3, (7, 6, 9)), ("mass", "twisted", 2, (6, 5, 8)),
                                               ("biharmonic", "sinmap", 3, (20, 17))])
def test_gpu_row_slabs_stitch_bitwise(form, geom, p, spans):
    # per-GPU row slabs (halo recomputed, no exchange) reproduce the full matrix bit for bit
    import paper_1904_06971_b200 as pkg
    from paper_1904_06971_b200.slabs import plane_slabs, stitch

    g = pkg.twisted_cube_standin() if geom == "twisted" else pkg.sin_map_standin()
    disc = pkg.make_discretization(g, p, spans)
    fk = pkg.FormKind(form)
    full = pkg.assemble(fk, disc).mat
    ms = tuple(kv.m for kv in disc.space.kvs)
    for world in (2, 3):
        parts = []
        for lo, hi in plane_slabs(ms, world):
            res, _, _ = pkg.assemble_device(fk, disc, slab=(lo, hi))
            parts.append(res.to_host())
            res.free()
        ip, ix, d = stitch(parts)
        assert np.array_equal(ip, full.indptr) and np.array_equal(ix, full.indices)
        assert np.array_equal(d.view(np.int64), full.data.view(np.int64))


@pytest.mark.gpu
def test_gpu_surrogate_row_slabs():
    import paper_1904_06971_b200 as pkg
    from paper_1904_06971_b200.slabs import plane_slabs, stitch
    from paper_1904_06971_b200.surrogate import surrogate_device

    disc = pkg.make_discretization(pkg.twisted_cube_standin(), 2, (14, 13, 15))
    fk = pkg.FormKind.POISSON
    A, _ = pkg.build_surrogate_matrix(fk, disc, pkg.ConstantSampling(4))
    ms = tuple(kv.m for kv in disc.space.kvs)
    parts = []
    for lo, hi in plane_slabs(ms, 3):
        res, st, _ = surrogate_device(fk, disc, 4, 3, "symmetric_kernel_preserving", slab=(lo, hi))
        parts.append(res.to_host())
        res.free()
    ip, ix, d = stitch(parts)
    assert np.array_equal(ip, A.mat.indptr) and np.array_equal(ix, A.mat.indices)
    assert np.array_equal(d.view(np.int64), A.mat.data.view(np.int64))


@pytest.mark.gpu
def test_gpu_matrix_market_from_device_result(tmp_path):
    # the device-resident result writes the same file as its host copy
    import paper_1904_06971_b200 as pkg

    disc = pkg.make_discretization(pkg.twisted_cube_standin(), 2, (6, 5, 4))
    res, sym, _ = pkg.assemble_device(pkg.FormKind.POISSON, disc)
    try:
        pkg.save_matrix_market(tmp_path / "dev.mtx", res, symmetric=sym)
    finally:
        res.free()
    A = pkg.assemble(pkg.FormKind.POISSON, disc)
    pkg.save_matrix_market(tmp_path / "host.mtx", A)
    assert (tmp_path / "dev.mtx").read_bytes() == (tmp_path / "host.mtx").read_bytes()
    assert pkg.matrices_bitwise_equal(A, pkg.load_matrix_market(tmp_path / "dev.mtx"))


@pytest.mark.gpu
@pytest.mark.parametrize("form", ["poisson", "mass"])
def test_gpu_surrogate_weighted_slabs_rows3(form):
    # cost-weighted slabs (bench.py's surrogate split) on the row-staged K7 path stitch bitwise
    import paper_1904_06971_b200 as pkg
    from paper_1904_06971_b200.slabs import job_slabs, stitch
    from paper_1904_06971_b200.surrogate import DEFAULT_MODE, build_sampling_lattice, surrogate_device

    disc = pkg.make_discretization(pkg.twisted_cube_standin(), 3, (28, 29, 27))
    fk = pkg.FormKind(form)
    mode = DEFAULT_MODE[form].value
    full, _, _ = surrogate_device(fk, disc, 8, 3, mode)
    fip, fix, fd = full.to_host()
    full.free()
    ms = tuple(kv.m for kv in disc.space.kvs)
    lat = build_sampling_lattice(disc.space.kvs, 8)
    parts = []
    for lo, hi in job_slabs(ms, 3, 3, "surrogate", form, lat.indices):
        res, _, _ = surrogate_device(fk, disc, 8, 3, mode, slab=(lo, hi))
        parts.append(res.to_host())
        res.free()
    ip, ix, d = stitch(parts)
    assert np.array_equal(ip, fip) and np.array_equal(ix, fix)
    assert np.array_equal(d.view(np.int64), fd.view(np.int64))


@pytest.mark.gpu
def test_gpu_concurrent_calls_are_reentrant():
    # studies call the entry points from a ThreadPoolExecutor (studies.py:89-95); ctypes
    # releases the GIL, so calls overlap in the library: results equal the sequential ones bit for bit
    from concurrent.futures import ThreadPoolExecutor

    import paper_1904_06971_b200 as pkg

    jobs = [(pkg.twisted_cube_standin(), 2, (9, 8, 10), "poisson", "full"),
            (pkg.quarter_annulus(1.0, 2.0), 3, (40, 36), "mass", "full"),
            (pkg.twisted_cube_standin(), 3, (28, 29, 27), "poisson", "surrogate"),
            (pkg.sin_map_standin(), 3, (30, 30), "biharmonic", "surrogate"),
            (pkg.quarter_annulus(1.0, 2.0), 2, (50, 44), "poisson", "surrogate")]

    def run(job):
        geo, p, spans, form, path = job
        disc = pkg.make_discretization(geo, p, spans)
        if path == "full":
            return pkg.assemble(pkg.FormKind(form), disc).mat
        return pkg.build_surrogate_matrix(pkg.FormKind(form), disc, pkg.ConstantSampling(8))[0].mat

    seq = [run(j) for j in jobs]
    with ThreadPoolExecutor(max_workers=len(jobs)) as ex:
        par = list(ex.map(run, jobs * 2))
    for k, m in enumerate(par):
        s = seq[k % len(jobs)]
        assert np.array_equal(m.indptr, s.indptr) and np.array_equal(m.indices, s.indices)
        assert np.array_equal(m.data.view(np.int64), s.data.view(np.int64))


@pytest.mark.gpu
@pytest.mark.parametrize("p,gauss", [(5, None), (2, 9)])
def test_gpu_unsupported_degree_or_gauss_is_not_a_value_error(p, gauss):
    # the reference accepts any p >= 1 and any Gauss count (bspline.py:231-234, assembly.py:173); this
    # build instantiates p <= 4, gauss <= 8: outside that it is "unsupported" (NotImplementedError /
    # NativeError), never the ValueError the reference reserves for invalid input
    import paper_1904_06971_b200 as pkg
    from paper_1904_06971_b200._lib import NativeError

    disc = pkg.make_discretization(pkg.quarter_annulus(1.0, 2.0), p, (12, 12), gauss=gauss)
    with pytest.raises(NotImplementedError):
        pkg.assemble(pkg.FormKind.POISSON, disc)
    with pytest.raises(NativeError):
        pkg.assemble(pkg.FormKind.POISSON, disc)


SWEEP2D = [(p, form, geom) for p in (1, 2, 3, 4) for form in ("poisson", "mass", "biharmonic")
           for geom in ("coons_quadratic", "coons_rational")
           if not (form == "biharmonic" and p < 2) and not (geom == "coons_rational" and p < 2)]


@pytest.mark.gpu
@pytest.mark.parametrize("p,form,geom", SWEEP2D)
@pytest.mark.parametrize("run", [None, "3"])
def test_gpu_2d_tiles_every_degree_form_and_map(p, form, geom, run, monkeypatch):
    # the 2D tensor-core kernel (TMA D windows, runs of tiles per CTA) on every degree, form and
    # polynomial / rational map against the oracle; SG_RUN2D=3 forces several tiles per CTA
    # (x-column reuse, the next window streamed during phase 2) on this small mesh
    import paper_1904_06971_b200 as pkg

    if run:
        monkeypatch.setenv("SG_RUN2D", run)
    disc = pkg.make_discretization(pkg.builtin_domain(geom), p, (23, 19))
    A = pkg.assemble(pkg.FormKind(form), disc)
    ip, ix, d, _, _ = O.assemble(O.problem_from_disc(form, disc))
    m = A.mat
    assert np.array_equal(m.indptr, ip) and np.array_equal(m.indices, ix)
    assert O.row_scaled_error(ip, ix, d, m.indptr, m.indices, m.data) <= 1e-12
    assert pkg.is_bitwise_symmetric(A)


@pytest.mark.gpu
def test_gpu_host_generated_columns_equal_device_columns(monkeypatch):
    # full-pattern results hand their column indices to the host in closed form (generated on host
    # threads during the values' D2H); they must equal the device's own indices bit for bit
    import paper_1904_06971_b200 as pkg
    from paper_1904_06971_b200.surrogate import surrogate_device

    disc = pkg.make_discretization(pkg.twisted_cube_standin(), 3, (21, 19, 23))
    ms = tuple(kv.m for kv in disc.space.kvs)
    per = ms[0] * ms[1]
    calls = [lambda: pkg.assemble_device(pkg.FormKind.POISSON, disc)[0],
             lambda: pkg.assemble_device(pkg.FormKind.MASS, disc, slab=(5 * per, 17 * per))[0],
             lambda: surrogate_device(pkg.FormKind.POISSON, disc, 4, 3, "symmetric_kernel_preserving")[0],
             lambda: surrogate_device(pkg.FormKind.MASS, disc, 4, 3, "symmetric", slab=(7 * per, 20 * per))[0]]
    for make in calls:
        res = make()
        ip, ix, d = res.to_host()
        monkeypatch.setenv("SG_COPY_INDICES", "1")
        ip2, ix2, d2 = res.to_host()
        monkeypatch.delenv("SG_COPY_INDICES")
        res.free()
        assert np.array_equal(ip, ip2) and np.array_equal(ix, ix2) and np.array_equal(d.view(np.int64), d2.view(np.int64))
