"""Golden CG solves from the REAL reference (solvers.py:74-155, method="conjugate-gradient").

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_solve.py

Each case stores the system (CSR of a reference-assembled matrix, possibly restricted to the
interior dofs), the right-hand side and either the reference's solution or its error message.
"""
import json
import os
import sys

import numpy as np
import scipy

from surriga.assembly import FormKind, assemble, interior_dofs, make_discretization
from surriga.solvers import SolveOptions, solve_spd

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import geo  # noqa: E402

OUT = os.path.join(HERE, "solve")

# name, geometry, p, spans, form, interior-only, negate, tol, maxit, preconditioner
CASES = [
    ("cg_annulus_poisson_p2", "annulus", 2, (12, 10), "poisson", True, False, 1e-10, None, "none"),
    ("cg_annulus_poisson_p2_jacobi", "annulus", 2, (12, 10), "poisson", True, False, 1e-10, None, "diagonal"),
    ("cg_twisted_mass_p2_jacobi", "twisted_cube_p3_m12.geo", 2, (5, 6, 4), "mass", False, False, 1e-12, None, "diagonal"),
    ("cg_coons_poisson_p3", "coons_quadratic", 3, (9, 8), "poisson", True, False, 1e-8, None, "none"),
    ("cg_maxit_fail", "annulus", 2, (12, 10), "poisson", True, False, 1e-12, 5, "none"),
    ("cg_negative_curvature", "annulus", 2, (8, 8), "mass", False, True, 1e-10, None, "none"),
    ("cg_nonpositive_diagonal", "annulus", 2, (8, 8), "mass", False, True, 1e-10, None, "diagonal"),
]


def main():
    os.makedirs(OUT, exist_ok=True)
    for name, gname, p, spans, form, interior, negate, tol, maxit, prec in CASES:
        g = geo(gname)
        disc = make_discretization(g, p, spans)
        A = assemble(FormKind(form), disc).mat
        if interior:
            keep = interior_dofs(disc.space)
            A = A[keep][:, keep].tocsr()
        if negate:
            A = (-A).tocsr()
        A.sort_indices()
        n = A.shape[0]
        b = np.cos(np.arange(n) * 0.37) + 0.5
        opts = SolveOptions(method="conjugate-gradient", tolerance=tol, max_iterations=maxit, preconditioner=prec)
        try:
            x = solve_spd(A, b, opts)
            err = ""
        except RuntimeError as e:
            x = np.zeros(n)
            err = str(e)
        meta = dict(case=name, geometry=gname, p=p, spans=list(spans), form=form, tol=tol, maxit=maxit,
                    preconditioner=prec, error=err, numpy=np.__version__, scipy=scipy.__version__)
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), meta=np.array(json.dumps(meta)),
                            indptr=A.indptr.astype(np.int64), indices=A.indices.astype(np.int32), data=A.data,
                            b=b, x=x)
        print(name, n, A.nnz, err or "ok", file=sys.stderr)


if __name__ == "__main__":
    main()
