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
]


def run_case(case, gname, pp, spans, extra):
    g = geo(gname)
    st = stokes_subgrid_spaces(g, pp, spans, gauss=extra.get("gauss"))
    rows = extra.get("rows")
    D = assemble_divergence(st, rows=None if rows is None else np.asarray(rows))
    meta = dict(case=case, geometry=gname, pp=pp, spans=list(spans), gauss=st.velocity.gauss, geo_p=g.space.p,
                geo_ms=[kv.m for kv in g.space.kvs], n=st.n, numpy=np.__version__, scipy=scipy.__version__)
    arrays = dict(geo_w=g.weights.weights, geo_ctrl=g.control, vel_w=st.velocity.weights.weights,
                  prs_w=st.pressure.weights.weights, indptr=D[0].mat.indptr, indices=D[0].mat.indices)
    for c, Dc in enumerate(D):
        assert np.array_equal(Dc.mat.indptr, D[0].mat.indptr) and np.array_equal(Dc.mat.indices, D[0].mat.indices)
        arrays[f"data_{c}"] = Dc.mat.data
    if rows is not None:
        arrays["rows"] = np.asarray(rows)
        arrays["populated_rows"] = D[0].populated_rows
    np.savez_compressed(os.path.join(HERE, f"{case}.npz"), meta=np.array(json.dumps(meta)), **arrays)
    return D[0].mat.nnz


def main():
    os.makedirs(HERE, exist_ok=True)
    for c in CASES:
        print(f"{c[0]}: nnz={run_case(*c)}", file=sys.stderr)


if __name__ == "__main__":
    main()
