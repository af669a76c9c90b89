"""Golden vectors from the REAL reference (arXiv 1904.06971 ``surriga``), run in the build container.

Each case stores the inputs exactly as the reference saw them (geometry net,
solution-space weights, degree, spans, Gauss order) and the reference's
output CSR (indptr / indices / data), flags and report, so that the oracle and
the CUDA path can be checked on a machine without /root/reference.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

numpy / scipy versions are recorded in every file.
"""
import json
import os
import sys

import numpy as np
import scipy

from surriga.assembly import FormKind, assemble, make_discretization
from surriga.geometry import builtin_domain, load_geometry, quarter_annulus, unit_cube, unit_square
from surriga.surrogate import ConstantSampling, SurrogateMode, build_surrogate_matrix

HERE = os.path.dirname(os.path.abspath(__file__))
DATA = os.path.join(HERE, "..", "..", "paper_1904_06971_b200", "data")


def geo(name):
    if name == "annulus":
        return quarter_annulus(1.0, 2.0)
    if name == "unit_square":
        return unit_square()
    if name == "unit_cube":
        return unit_cube()
    if name.endswith(".geo"):
        return load_geometry(os.path.join(DATA, name))
    return builtin_domain(name)


# (case, geometry, p, spans, form, kind, extra)
CASES = [
    ("cfg1_full_poisson", "annulus", 2, (32, 32), "poisson", "full", {}),
    ("cfg1_surr_poisson", "annulus", 2, (32, 32), "poisson", "surrogate", {"M": 8}),
    ("annulus_mass_p3", "annulus", 3, (10, 12), "mass", "full", {}),
    ("annulus_biharm_p3", "annulus", 3, (8, 9), "biharmonic", "full", {}),
    ("coons_cubic_biharm", "coons_cubic", 3, (9, 9), "biharmonic", "full", {}),
    ("coons_rational_biharm_p2", "coons_rational", 2, (7, 9), "biharmonic", "full", {}),
    ("coons_quad_poisson_rows", "coons_quadratic", 2, (8, 8), "poisson", "rows", {"rows": [0, 7, 33, 64, 99]}),
    ("coons_quad_stokesvel_coef", "coons_quadratic", 2, (6, 7), "stokes_velocity", "full", {"coefficient": 0.37}),
    ("unit_square_p1_poisson", "unit_square", 1, (4, 4), "poisson", "full", {}),
    ("unit_square_gauss5", "unit_square", 2, (6, 6), "poisson", "full", {"gauss": 5}),
    ("tri3d_poisson_p2", "trivariate_polynomial_3d", 2, (5, 4, 6), "poisson", "full", {}),
    ("tri3d_mass_p3", "trivariate_polynomial_3d", 3, (4, 4, 5), "mass", "full", {}),
    ("tri3d_biharm_p2", "trivariate_polynomial_3d", 2, (4, 4, 4), "biharmonic", "full", {}),
    ("twisted_poisson_p3", "twisted_cube_p3_m12.geo", 3, (5, 5, 6), "poisson", "full", {}),
    ("twisted_mass_p3_rows", "twisted_cube_p3_m12.geo", 3, (6, 6, 6), "mass", "rows", {"rows": [0, 100, 555, 728]}),
    ("sinmap_biharm_p3", "sin_map_p3_m16.geo", 3, (16, 16), "biharmonic", "full", {}),
    ("sinmap_biharm_surr", "sin_map_p3_m16.geo", 3, (24, 24), "biharmonic", "surrogate", {"M": 4}),
    ("annulus_mass_surr_sym", "annulus", 3, (20, 20), "mass", "surrogate", {"M": 4}),
    ("annulus_poisson_surr_general", "annulus", 2, (24, 24), "poisson", "surrogate", {"M": 5, "mode": "general"}),
    ("annulus_poisson_surr_symmetric", "annulus", 2, (24, 24), "poisson", "surrogate", {"M": 5, "mode": "symmetric"}),
    ("annulus_poisson_surr_lowered", "annulus", 2, (12, 12), "poisson", "surrogate", {"M": 8}),
    ("annulus_poisson_surr_disabled", "annulus", 2, (6, 6), "poisson", "surrogate", {"M": 8}),
    ("annulus_poisson_surr_M1", "annulus", 2, (14, 14), "poisson", "surrogate", {"M": 1}),
    ("twisted_poisson_surr_p1", "twisted_cube_p3_m12.geo", 1, (12, 12, 12), "poisson", "surrogate", {"M": 3}),
    ("twisted_mass_surr_nI0", "twisted_cube_p3_m12.geo", 2, (8, 8, 8), "mass", "surrogate", {"M": 2}),
    ("coons_quad_q5_surr", "coons_quadratic", 2, (30, 30), "poisson", "surrogate", {"M": 3, "q": 5}),
    # coefficient 0: every entry is an exact zero, dropped by the CSR add (surrogate.py:670) -> empty pattern
    ("annulus_poisson_surr_zero_general", "annulus", 2, (14, 13), "poisson", "surrogate",
     {"M": 4, "mode": "general", "coefficient": 0.0}),
]


def run_case(case, gname, p, spans, form, kind, extra):
    g = geo(gname)
    disc = make_discretization(g, p, spans, gauss=extra.get("gauss"))
    fk = FormKind(form)
    meta = dict(case=case, geometry=gname, p=p, spans=list(spans), form=form, kind=kind, gauss=disc.gauss,
                geo_p=g.space.p, geo_ms=[kv.m for kv in g.space.kvs], coefficient=extra.get("coefficient", 1.0),
                numpy=np.__version__, scipy=scipy.__version__)
    arrays = dict(sol_w=disc.weights.weights, geo_w=g.weights.weights, geo_ctrl=g.control)
    if kind in ("full", "rows"):
        rows = extra.get("rows")
        A = assemble(fk, disc, rows=None if rows is None else np.asarray(rows), coefficient=meta["coefficient"])
        meta["symmetric"] = A.symmetric
        if rows is not None:
            arrays["rows"] = np.asarray(rows)
            arrays["populated_rows"] = A.populated_rows
    else:
        M = extra["M"]
        mode = extra.get("mode")
        q = extra.get("q", 3)
        A, rep = build_surrogate_matrix(fk, disc, ConstantSampling(M), q=q,
                                        mode=None if mode is None else SurrogateMode(mode),
                                        coefficient=meta["coefficient"])
        meta.update(M=M, q=q, mode=mode, symmetric=A.symmetric,
                    report={k: getattr(rep, k) for k in ("N", "p", "q", "M", "H", "quad_entries", "interp_entries",
                                                         "quad_fraction", "active_elements", "flags")})
    m = A.mat
    arrays.update(indptr=m.indptr, indices=m.indices, data=m.data)
    np.savez_compressed(os.path.join(HERE, f"{case}.npz"), meta=np.array(json.dumps(meta)), **arrays)
    return m.nnz


def main():
    only = set(sys.argv[1:])  # optional case names: regenerate just those
    for c in CASES:
        if only and c[0] not in only:
            continue
        nnz = run_case(*c)
        print(f"{c[0]}: nnz={nnz}", file=sys.stderr)


if __name__ == "__main__":
    main()
