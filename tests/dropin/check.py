"""Drop-in check in a fresh process (module rebinding is global): the installed reference
(baseline/_ref) run unpatched, then with the INTEGRATION.md rebinding, on the reference's own
inputs (its make_discretization, FormKind, ConstantSampling, Discretization objects).  Prints one
JSON line of comparisons; tests/test_gpu_dropin.py asserts on it."""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
sys.path.insert(0, HERE)

import surriga.assembly as RA  # noqa: E402
import surriga.studies as RS  # noqa: E402
import surriga.surrogate as RSU  # noqa: E402
from surriga.geometry import load_geometry, quarter_annulus  # noqa: E402

import rebind  # noqa: E402


def scaled_err(A, B):
    a, b = A.mat, B.mat
    if a.shape != b.shape or not (np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)):
        return float("inf")
    cnt = np.diff(a.indptr)
    rows = np.repeat(np.arange(cnt.size), cnt)
    scale = np.zeros(cnt.size)
    np.maximum.at(scale, rows, np.abs(a.data))
    return float(np.max(np.abs(a.data - b.data) / np.where(scale[rows] > 0, scale[rows], 1.0))) if a.nnz else 0.0


def report(rep):
    return {k: getattr(rep, k) for k in ("N", "p", "q", "M", "H", "quad_entries", "interp_entries", "quad_fraction",
                                         "active_elements", "flags")}


cases = {
    "annulus_p3_poisson": (quarter_annulus(1.0, 2.0), 3, (40, 40), RA.FormKind.POISSON, 5),
    "annulus_p3_mass": (quarter_annulus(1.0, 2.0), 3, (40, 40), RA.FormKind.MASS, 5),
    "twisted_p3_poisson": (load_geometry(os.path.join(ROOT, "paper_1904_06971_b200", "data", "twisted_cube_p3_m12.geo")),
                           3, (16, 16, 18), RA.FormKind.POISSON, 4),
}
ref = {}
for name, (g, p, spans, form, M) in cases.items():
    disc = RA.make_discretization(g, p, spans)
    A = RA.assemble(form, disc)
    S, rep = RSU.build_surrogate_matrix(form, disc, RSU.ConstantSampling(M))
    rows = np.array([0, 17, A.mat.shape[0] // 2, A.mat.shape[0] - 1])
    ref[name] = (disc, form, M, A, S, rep, rows, RA.assemble(form, disc, rows=rows))
study_ref = RS.run_poisson_study("coons_rational", p=2, ladder=(12, 20))

out = {}
# 1. the reference's own build_surrogate_matrix with its quadrature rows (surrogate.py:588) on the GPU
rebind.install(only_assemble_in_surrogate=True)
for name, (disc, form, M, A, S, rep, rows, Ar0) in ref.items():
    S1, rep1 = RSU.build_surrogate_matrix(form, disc, RSU.ConstantSampling(M))
    r0, r1 = report(rep), report(rep1)
    out[f"{name}/ref_surrogate_gpu_quadrature"] = {"err": scaled_err(S, S1), "report_equal": r0 == r1,
                                                   "symmetric": S1.symmetric == S.symmetric}
# 2. the whole INTEGRATION.md rebinding: the reference's public names now run the B200 path
rebind.install()
import surriga  # noqa: E402

for name, (disc, form, M, A, S, rep, rows, Ar0) in ref.items():
    A2 = surriga.assembly.assemble(form, disc)
    S2, rep2 = surriga.surrogate.build_surrogate_matrix(form, disc, RSU.ConstantSampling(M))
    out[f"{name}/full"] = {"err": scaled_err(A, A2), "type": type(A2).__module__ + "." + type(A2).__name__,
                           "symmetric": A2.symmetric == A.symmetric, "int32": str(A2.mat.indices.dtype) == "int32"}
    r0, r2 = report(rep), report(rep2)
    out[f"{name}/surrogate"] = {"err": scaled_err(S, S2), "report_equal": r0 == r2, "report": r2,
                                "type": type(rep2).__module__ + "." + type(rep2).__name__}
    Ar = surriga.assembly.assemble(form, disc, rows=rows)
    out[f"{name}/rows"] = {"err": scaled_err(Ar0, Ar),
                           "rows_equal": bool(np.array_equal(Ar.populated_rows, Ar0.populated_rows))}
study = surriga.studies.run_poisson_study("coons_rational", p=2, ladder=(12, 20))
worst = 0.0
same = True
for a, b in zip(study_ref, study):
    for k in ("err_l2_std", "err_l2_surr", "err_h1_std", "err_h1_surr"):
        worst = max(worst, abs(getattr(a, k) - getattr(b, k)) / abs(getattr(a, k)))
    same = same and (a.N, a.M, a.H, a.quad_fraction, a.flags) == (b.N, b.M, b.H, b.quad_fraction, b.flags)
out["studies/run_poisson_study"] = {"rel_err_worst": worst, "rows_equal": same, "levels": len(study)}
print(json.dumps(out))
