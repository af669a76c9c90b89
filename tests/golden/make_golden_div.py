"""Golden vectors of the mixed divergence pairing from the REAL reference (assembly.py:654-725).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_div.py

Writes tests/golden/div/<case>.npz: geometry net, pressure degree / spans, velocity Gauss order,
the reference's CSR per velocity component (shared indptr/indices, data_c) and, for row-restricted
cases, the rows.  numpy / scipy versions recorded in every file.
"""
import json
import os
import sys

import numpy as np
import scipy

from surriga.assembly import assemble_divergence, stokes_subgrid_spaces
from surriga.surrogate import ConstantSampling, build_surrogate_divergence

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import geo  # noqa: E402

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "div")

# (case, geometry, pressure degree, pressure spans, extra)
CASES = [
    ("div_coons_quad_p2", "coons_quadratic", 2, (6, 6), {}),
    ("div_coons_quad_p2_rows", "coons_quadratic", 2, (6, 6), {"rows": [0, 5, 17, 40]}),
    ("div_unit_square_p1", "unit_square", 1, (3, 4), {}),
    ("div_coons_cubic_gauss5", "coons_cubic", 2, (4, 5), {"gauss": 5}),
    ("div_tri3d_p1", "trivariate_polynomial_3d", 1, (2, 3, 2), {}),
    ("div_twisted_p2", "twisted_cube_p3_m12.geo", 2, (3, 3, 3), {}),
    ("div_twisted_p2_rows", "twisted_cube_p3_m12.geo", 2, (3, 4, 3), {"rows": [0, 11, 30, 74, 149]}),
    ("sdiv_coons_quad_p2", "coons_quadratic", 2, (20, 22), {"M": 4}),
    ("sdiv_coons_quad_p1_lowered", "coons_quadratic", 1, (12, 12), {"M": 5}),
    ("sdiv_unit_square_p1", "unit_square", 1, (14, 12), {"M": 3}),
    ("sdiv_twisted_p1", "twisted_cube_p3_m12.geo", 1, (9, 10, 9), {"M": 3}),
    ("sdiv_coons_quad_disabled", "coons_quadratic", 2, (7, 7), {"M": 2}),
    # rational (NURBS) spaces: both spaces carry the annulus / rational Coons weights
    ("div_annulus_p2", "annulus", 2, (5, 4), {}),
    ("div_annulus_p2_rows", "annulus", 2, (6, 5), {"rows": [0, 9, 20, 41, 55]}),
    ("div_coons_rational_p2", "coons_rational", 2, (4, 5), {}),
    ("sdiv_annulus_p2", "annulus", 2, (20, 18), {"M": 4}),
]


def run_case(case, gname, pp, spans, extra):
    g = geo(gname)
    st = stokes_subgrid_spaces(g, pp, spans, gauss=extra.get("gauss"))
    rows = extra.get("rows")
    meta = dict(case=case, geometry=gname, pp=pp, spans=list(spans), gauss=st.velocity.gauss, geo_p=g.space.p,
                geo_ms=[kv.m for kv in g.space.kvs], n=st.n, numpy=np.__version__, scipy=scipy.__version__)
    if "M" in extra:
        D, rep = build_surrogate_divergence(st, ConstantSampling(extra["M"]), q=extra.get("q", 3))
        meta.update(kind="surrogate", M=extra["M"], q=extra.get("q", 3),
                    report={k: getattr(rep, k) for k in ("N", "p", "q", "M", "H", "quad_entries", "interp_entries",
                                                         "quad_fraction", "active_elements", "flags")})
    else:
        D = assemble_divergence(st, rows=None if rows is None else np.asarray(rows))
        meta.update(kind="full" if rows is None else "rows")
    arrays = dict(geo_w=g.weights.weights, geo_ctrl=g.control, vel_w=st.velocity.weights.weights,
                  prs_w=st.pressure.weights.weights)
    for c, Dc in enumerate(D):
        # surrogate components may differ in pattern (exact zeros dropped by the CSR add)
        arrays[f"indptr_{c}"] = Dc.mat.indptr
        arrays[f"indices_{c}"] = Dc.mat.indices
        arrays[f"data_{c}"] = Dc.mat.data
    if rows is not None:
        arrays["rows"] = np.asarray(rows)
        arrays["populated_rows"] = D[0].populated_rows
    np.savez_compressed(os.path.join(HERE, f"{case}.npz"), meta=np.array(json.dumps(meta)), **arrays)
    return D[0].mat.nnz


def main():
    os.makedirs(HERE, exist_ok=True)
    only = set(sys.argv[1:])  # optional case names: regenerate just those
    for c in CASES:
        if only and c[0] not in only:
            continue
        print(f"{c[0]}: nnz={run_case(*c)}", file=sys.stderr)


if __name__ == "__main__":
    main()
