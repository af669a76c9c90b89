"""Golden load vectors from the REAL reference (assembly.py:728-759).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_load.py

The load callables are named in LOAD_FUNCS (tests/load_funcs.py) so the tests can re-create them.
"""
import json
import os
import sys

import numpy as np
import scipy

from surriga.assembly import assemble_load, make_discretization

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.join(HERE, ".."))
from load_funcs import LOAD_FUNCS  # noqa: E402
from make_golden import geo  # noqa: E402

OUT = os.path.join(HERE, "load")
CASES = [
    ("load_coons_quad_p2", "coons_quadratic", 2, (6, 7), "poly_sin"),
    ("load_annulus_p2_rational", "annulus", 2, (5, 6), "poly_sin"),
    ("load_unit_square_p1_gauss4", "unit_square", 1, (4, 5), "one", {"gauss": 4}),
    ("load_tri3d_p2", "trivariate_polynomial_3d", 2, (3, 4, 3), "prod_cos"),
    ("load_twisted_p3", "twisted_cube_p3_m12.geo", 3, (4, 4, 5), "prod_cos"),
]


def main():
    os.makedirs(OUT, exist_ok=True)
    for case in CASES:
        name, gname, p, spans, fname = case[:5]
        extra = case[5] if len(case) > 5 else {}
        g = geo(gname)
        disc = make_discretization(g, p, spans, gauss=extra.get("gauss"))
        vec = assemble_load(disc, LOAD_FUNCS[fname])
        meta = dict(case=name, geometry=gname, p=p, spans=list(spans), gauss=disc.gauss, func=fname, geo_p=g.space.p,
                    geo_ms=[kv.m for kv in g.space.kvs], numpy=np.__version__, scipy=scipy.__version__)
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), meta=np.array(json.dumps(meta)), vec=vec,
                            sol_w=disc.weights.weights, geo_w=g.weights.weights, geo_ctrl=g.control)
        print(name, vec.size, file=sys.stderr)


if __name__ == "__main__":
    main()
