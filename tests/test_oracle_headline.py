"""Pin the oracle's sampled-row paths (``surrogate_rows``, ``assemble_rows_grouped``) -- the
checker used at config 5's full size -- against the whole-matrix oracle at small sizes and
against the REAL reference's fingerprints at the headline shapes (tests/golden/headline)."""
import numpy as np
import pytest

from headline_checks import sample_rows
from oracle import surriga_oracle as O
from test_gpu_headline import CASES, load_headline

TOL = 1e-12


def _problem(meta):
    from paper_1904_06971_b200.configs import CONFIGS  # noqa: F401  (geometry loaders)
    import paper_1904_06971_b200 as pkg

    g = {"annulus": lambda: pkg.quarter_annulus(1.0, 2.0), "twisted": pkg.twisted_cube_standin,
         "sinmap": pkg.sin_map_standin}[meta["geometry"]]()
    disc = pkg.make_discretization(g, meta["p"], tuple(meta["spans"]))
    return O.problem_from_disc(meta["form"], disc)


def _check(rows, cnt, cols, vals, rrows, rcnt, rcols, rvals):
    pos = {int(r): i for i, r in enumerate(rrows)}
    starts = np.concatenate([[0], np.cumsum(rcnt)])
    s = 0
    worst = 0.0
    for r, c in zip(rows, cnt):
        i = pos[int(r)]
        assert c == rcnt[i]
        assert np.array_equal(cols[s:s + c], rcols[starts[i]:starts[i] + c])
        ref = rvals[starts[i]:starts[i] + c]
        worst = max(worst, float(np.max(np.abs(vals[s:s + c] - ref)) / max(np.max(np.abs(ref)), 1e-300)))
        s += c
    return worst


SMALL = [("twisted", 3, (20, 19, 21), "poisson", 4, None), ("twisted", 2, (16, 15, 17), "mass", 3, None),
         ("annulus", 3, (40, 38), "poisson", 8, None), ("annulus", 2, (30, 30), "poisson", 5, "general"),
         ("annulus", 2, (30, 30), "poisson", 5, "symmetric"), ("sinmap", 3, (40, 40), "biharmonic", 8, None)]


@pytest.mark.parametrize("geom,p,spans,form,M,mode", SMALL)
def test_surrogate_rows_equals_whole_oracle(geom, p, spans, form, M, mode):
    meta = dict(geometry=geom, p=p, spans=spans, form=form)
    prob = _problem(meta)
    (ip, ix, d), _, _ = O.surrogate(prob, M, 3, mode)
    lat = [O.lattice_indices(p, m, M) for m in prob.ms]
    rows = sample_rows(prob.ms, p, lat, count=120)
    (rr, cnt, cols, vals), cls = O.surrogate_rows(prob, M, 3, mode, rows)
    assert cls["interp"].sum() >= 20
    whole_cnt = np.diff(ip)[rr]
    whole_cols = np.concatenate([ix[ip[r]:ip[r + 1]] for r in rr])
    whole_vals = np.concatenate([d[ip[r]:ip[r + 1]] for r in rr])
    assert _check(rr, cnt, cols, vals, rr, whole_cnt, whole_cols, whole_vals) <= TOL


# the reference fingerprints: a bounded number of sampled rows per case keeps this suite in minutes
@pytest.mark.parametrize("case", CASES)
def test_oracle_rows_match_reference_headline(case):
    meta, arr = load_headline(case)
    prob = _problem(meta)
    rows_all = arr["rows"]
    cnt_all = arr["row_cnt"]
    ms = prob.ms
    p = meta["p"]
    multi = np.stack(np.unravel_index(rows_all, ms, order="F"), -1)
    inbox = np.all((multi >= 2 * p) & (multi <= np.asarray(ms) - 2 * p - 1), axis=1)
    # every interpolated-looking row plus a few quadrature rows, at most 48
    pick = np.concatenate([np.flatnonzero(inbox)[:36], np.flatnonzero(~inbox)[:12]])
    rows = np.sort(rows_all[pick])
    if meta["kind"] == "full":
        got = O.assemble_rows_grouped(prob, rows)
        cnt = np.array([got[int(r)][0].size for r in rows])
        cols = np.concatenate([got[int(r)][0] for r in rows])
        vals = np.concatenate([got[int(r)][1] for r in rows])
    else:
        (rows, cnt, cols, vals), _ = O.surrogate_rows(prob, meta["M"], meta["q"], None, rows)
    assert _check(rows, cnt, cols, vals, rows_all, cnt_all, arr["row_cols"], arr["row_vals"]) <= TOL
