"""GPU parity at the headline shapes (BASELINE configs 2-4 at full size, config 5's p=3 / q=3 /
M=16 settings at 48^3 and 64^3, config 5 itself at 128^3).

Configs 2-4 and the config-5 ladder are checked against fingerprints of the REAL reference's own
matrices (``tests/golden/headline``, made by ``tests/golden/make_golden_headline.py``): bit-exact
pattern (CRC-32 of int32 indptr / indices), a weighted checksum of every row (block sums, see
``tests/headline_checks.py``), a few hundred sampled rows in full (quadrature and interpolated
rows from every region: boundary band, box edge, lattice neighbours, interior) at 1e-12
row-scaled, and every AssemblyReport field.  Config 5 at 128^3 (741M nnz per matrix; the
reference needs ~580 GB there) is checked on sampled rows against the oracle's sampled-row
surrogate (``surrogate_rows``), which is itself pinned against the reference fingerprints in
``tests/test_oracle_headline.py``.  Calls go through the public drop-in entry points
(``assemble`` / ``build_surrogate_matrix``), as a reference user makes them.
"""
import glob
import json
import os

import numpy as np
import pytest

from headline_checks import block_checksums, check_blocks, crc, rows_segments, sample_rows

TOL = 1e-12
HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "headline")
CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(HERE, "*.npz")))


def load_headline(case):
    z = np.load(os.path.join(HERE, case + ".npz"))
    return json.loads(str(z["meta"])), {k: z[k] for k in z.files if k != "meta"}


def headline_disc(meta):
    import paper_1904_06971_b200 as pkg

    g = {"annulus": lambda: pkg.quarter_annulus(1.0, 2.0), "twisted": pkg.twisted_cube_standin,
         "sinmap": pkg.sin_map_standin}[meta["geometry"]]()
    return pkg.make_discretization(g, meta["p"], tuple(meta["spans"]))


def compare_rows(rows, cnt_ref, cols_ref, vals_ref, ip, ix, d, what):
    ip = np.asarray(ip, dtype=np.int64)
    cnt, cols, vals = rows_segments(ip, ix, d, rows)
    assert np.array_equal(cnt, cnt_ref), f"{what}: row lengths differ"
    assert np.array_equal(cols, cols_ref), f"{what}: columns differ"
    s = 0
    worst = 0.0
    for r, c in zip(rows, cnt):
        ref = vals_ref[s:s + c]
        scale = max(np.max(np.abs(ref)), 1e-300)
        worst = max(worst, float(np.max(np.abs(vals[s:s + c] - ref)) / scale))
        s += c
    assert worst <= TOL, f"{what}: sampled rows differ by {worst:.3e} (row-scaled)"
    return worst


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_gpu_headline_matches_reference_fingerprint(case):
    import paper_1904_06971_b200 as pkg

    meta, arr = load_headline(case)
    disc = headline_disc(meta)
    fk = pkg.FormKind(meta["form"])
    if meta["kind"] == "full":
        A = pkg.assemble(fk, disc)
        rep = None
    else:
        A, rep = pkg.build_surrogate_matrix(fk, disc, pkg.ConstantSampling(meta["M"]), q=meta["q"])
    m = A.mat
    assert m.shape == (meta["N"], meta["N"]) and m.nnz == meta["nnz"]
    assert m.indptr.dtype == np.int32 and m.indices.dtype == np.int32
    assert crc(m.indptr, np.int32) == meta["crc_indptr"], "indptr differs from the reference"
    assert crc(m.indices, np.int32) == meta["crc_indices"], "indices differ from the reference"
    compare_rows(arr["rows"], arr["row_cnt"], arr["row_cols"], arr["row_vals"], m.indptr, m.indices, m.data, case)
    C, W = block_checksums(m.indptr, m.indices, m.data, meta["block"])
    ratio, at = check_blocks(arr["block_C"], arr["block_W"], C, W)
    assert ratio <= 1.0, f"row block {at} (rows {at * meta['block']}..) checksum off by {ratio:.2f}x its 1e-12 bound"
    assert A.symmetric == meta["symmetric"]
    if rep is not None:
        for k, v in meta["report"].items():
            got = getattr(rep, k)
            assert got == v, (k, got, v)
    if A.symmetric:
        assert pkg.is_bitwise_symmetric(A)


@pytest.mark.gpu
@pytest.mark.parametrize("form", ["poisson", "mass"])
def test_gpu_config5_fullsize_surrogate_rows_vs_oracle(form):
    """Config 5 at full size (128^3, p=3, q=3, M=16, default modes): sampled rows of the GPU
    surrogate against the oracle's sampled-row surrogate (interpolated rows at the box corner,
    edges, lattice neighbours and interior; quadrature rows in the boundary band)."""
    import paper_1904_06971_b200 as pkg
    from oracle import surriga_oracle as O
    from paper_1904_06971_b200.configs import CONFIGS
    from paper_1904_06971_b200.surrogate import DEFAULT_MODE, surrogate_device

    cfg = CONFIGS[5]
    disc = pkg.make_discretization(cfg.geom(), cfg.p, cfg.spans)
    prob = O.problem_from_disc(form, disc)
    lat = [O.lattice_indices(cfg.p, m, cfg.M) for m in prob.ms]
    rows = sample_rows(prob.ms, cfg.p, lat, count=120)
    (rr, cnt, cols, vals), cls = O.surrogate_rows(prob, cfg.M, cfg.q, None, rows)
    assert cls["interp"].sum() >= 50
    res, st, _ = surrogate_device(pkg.FormKind(form), disc, cfg.M, cfg.q, DEFAULT_MODE[form].value)
    try:
        ip, ix, d = res.to_host()
    finally:
        res.free()
    assert st.n_zero_dropped == 0
    compare_rows(rr, cnt, cols, vals, ip, ix, d, f"config 5 {form} surrogate")


@pytest.mark.gpu
@pytest.mark.parametrize("form", ["poisson", "mass"])
def test_gpu_config5_fullsize_full_rows_vs_oracle(form):
    """Config 5 full quadrature at full size: the same sampled rows against the oracle."""
    import paper_1904_06971_b200 as pkg
    from oracle import surriga_oracle as O
    from paper_1904_06971_b200.configs import CONFIGS

    cfg = CONFIGS[5]
    disc = pkg.make_discretization(cfg.geom(), cfg.p, cfg.spans)
    prob = O.problem_from_disc(form, disc)
    lat = [O.lattice_indices(cfg.p, m, cfg.M) for m in prob.ms]
    rows = sample_rows(prob.ms, cfg.p, lat, count=120)
    got = O.assemble_rows_grouped(prob, rows)
    cnt = np.array([got[int(r)][0].size for r in rows])
    cols = np.concatenate([got[int(r)][0] for r in rows])
    vals = np.concatenate([got[int(r)][1] for r in rows])
    res, _, _ = pkg.assemble_device(pkg.FormKind(form), disc)
    try:
        ip, ix, d = res.to_host()
    finally:
        res.free()
    compare_rows(rows, cnt, cols, vals, ip, ix, d, f"config 5 {form} full")
