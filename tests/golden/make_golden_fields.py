"""Golden quadrature fields from the REAL reference (assembly.py:839-907).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_fields.py
"""
import json
import os
import sys

import numpy as np
import scipy

from surriga.assembly import make_discretization, quadrature_fields

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import geo  # noqa: E402

OUT = os.path.join(HERE, "fields")
# name, geometry, p, spans, nu, gauss
CASES = [
    ("fields_annulus_p2_rational_nu2", "annulus", 2, (5, 6), 2, None),
    ("fields_coons_quad_p2_nu1_g4", "coons_quadratic", 2, (6, 5), 1, 4),
    ("fields_unit_square_p1_nu2", "unit_square", 1, (4, 3), 2, None),
    ("fields_twisted_p3_nu2", "twisted_cube_p3_m12.geo", 3, (4, 5, 4), 2, None),
    ("fields_tri3d_p2_nu1", "trivariate_polynomial_3d", 2, (3, 4, 3), 1, None),
    ("fields_sinmap_p3_nu0", "sin_map_p3_m16.geo", 3, (5, 4), 0, 5),
]


def coefs_for(N):
    k = np.arange(N)
    return np.sin(0.7 * k) + 0.1 * k / N


def main():
    os.makedirs(OUT, exist_ok=True)
    for name, gname, p, spans, nu, gauss in CASES:
        g = geo(gname)
        disc = make_discretization(g, p, spans)
        c = coefs_for(disc.space.N)
        x, w, vals, grads, hesses = quadrature_fields(disc, c, nu=nu, gauss=gauss)
        meta = dict(case=name, geometry=gname, p=p, spans=list(spans), nu=nu, gauss=gauss, geo_p=g.space.p,
                    geo_ms=[kv.m for kv in g.space.kvs], numpy=np.__version__, scipy=scipy.__version__)
        arrs = dict(meta=np.array(json.dumps(meta)), coefs=c, x=x, w=w, vals=vals, sol_w=disc.weights.weights,
                    geo_w=g.weights.weights, geo_ctrl=g.control)
        if grads is not None:
            arrs["grads"] = grads
        if hesses is not None:
            arrs["hesses"] = hesses
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **arrs)
        print(name, vals.size, file=sys.stderr)


if __name__ == "__main__":
    main()
