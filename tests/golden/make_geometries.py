"""Freeze the B-spline stand-ins of BASELINE configs 3-5's analytic maps.

The reference only accepts NURBS control nets (geometry.py:139-182), so the
twisted cube and the sin-perturbed square are interpolated at Greville sites
with the reference's own ``tensor_collocate`` (bspline.py:167-178) and written
with its ``save_geometry`` (geometry.py:512-521).  Run in the build container
(needs /root/reference); the outputs are committed under
``paper_1904_06971_b200/data/`` and are plain inputs afterwards.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_geometries.py
"""
import os
import sys

import numpy as np

from surriga.bspline import NurbsWeights, make_tensor_space, tensor_collocate
from surriga.geometry import GeometryMap, map_grid, save_geometry

OUT = os.path.join(os.path.dirname(__file__), "..", "..", "paper_1904_06971_b200", "data")


def twisted_cube(x, y, z):
    return (x * np.cos(0.5 * z) - y * np.sin(0.5 * z), x * np.sin(0.5 * z) + y * np.cos(0.5 * z), z)


def sin_map(x, y):
    return (x + 0.05 * np.sin(2 * np.pi * x) * np.sin(np.pi * y), y + 0.05 * np.sin(np.pi * x) * np.sin(2 * np.pi * y))


def standin(func, n, pg, mg, name):
    space = make_tensor_space(pg, mg, n)
    sites = [kv.greville() for kv in space.kvs]
    mesh = np.meshgrid(*sites, indexing="ij")
    vals = func(*mesh)
    ctrl = np.empty((space.N, n))
    for c in range(n):
        ctrl[:, c] = tensor_collocate(space.kvs, sites, np.asarray(vals[c], float)).reshape(-1, order="F")
    geom = GeometryMap(space=space, weights=NurbsWeights(np.ones(space.N), polynomial_weight=True), control=ctrl, name=name)
    test = [np.linspace(0, 1, 17)] * n
    err = np.max(np.abs(map_grid(geom, test, 0).phi - np.stack(func(*np.meshgrid(*test, indexing="ij")), -1)))
    return geom, err


def builtins():
    """The reference's builtin domains frozen as fixtures (the product reads them instead of
    rebuilding the nets); the annulus at two outer radii, whose nets span every (r_in, r_out)."""
    from surriga.geometry import builtin_domain, quarter_annulus

    for name in ("unit_square", "unit_cube", "coons_quadratic", "coons_cubic", "coons_rational",
                 "trivariate_polynomial_3d"):
        g = builtin_domain(name)
        save_geometry(g, os.path.join(OUT, f"{name}.geo"))
        print(f"{name}: p={g.space.p} m={g.space.shape} polynomial_weight={g.weights.polynomial_weight}", file=sys.stderr)
    for r_out in (2.0, 3.0):
        g = quarter_annulus(1.0, r_out)
        save_geometry(g, os.path.join(OUT, f"quarter_annulus_1_{int(r_out)}.geo"))
        print(f"quarter_annulus(1,{r_out}): polynomial_weight={g.weights.polynomial_weight}", file=sys.stderr)


def main():
    os.makedirs(OUT, exist_ok=True)
    builtins()
    for func, n, pg, mg, name in ((twisted_cube, 3, 3, 12, "twisted_cube"), (sin_map, 2, 3, 16, "sin_map")):
        geom, err = standin(func, n, pg, mg, name)
        path = os.path.join(OUT, f"{name}_p{pg}_m{mg}.geo")
        save_geometry(geom, path)
        print(f"{path}: max |phi - F| on 17^{n} grid = {err:.2e}", file=sys.stderr)


if __name__ == "__main__":
    main()
