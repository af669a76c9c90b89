"""CPU: the oracle's quadrature fields (oracle.quadrature_fields) pinned against the REAL reference's
quadrature_fields goldens (assembly.py:839-907; tests/golden/fields, make_golden_fields.py)."""
import glob
import json
import os

import numpy as np
import pytest

from oracle import surriga_oracle as O

FIELDS = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "fields")
TOL = 1e-12


def field_cases():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(FIELDS, "*.npz")))


def field_golden(case):
    z = np.load(os.path.join(FIELDS, case + ".npz"))
    meta = json.loads(str(z["meta"]))
    return meta, {k: z[k] for k in z.files if k != "meta"}


def gauss_of(meta):
    return meta["gauss"] if meta["gauss"] is not None else meta["p"] + 1


def field_problem(meta, arr):
    p = meta["p"]
    return O.Problem(form="mass", p=p, ms=tuple(s + p for s in meta["spans"]), g=gauss_of(meta), sol_w=arr["sol_w"],
                     geo_p=meta["geo_p"], geo_ms=tuple(meta["geo_ms"]), geo_w=arr["geo_w"], geo_ctrl=arr["geo_ctrl"])


def rel(a, b):
    return np.max(np.abs(a - b)) / max(1e-300, np.max(np.abs(b)))


def check_fields(out, arr, nu, tol=TOL):
    x, w, vals, grads, hesses = out
    assert rel(x, arr["x"]) <= tol and rel(w, arr["w"]) <= tol and rel(vals, arr["vals"]) <= tol
    if nu >= 1:
        assert rel(grads, arr["grads"]) <= tol
    else:
        assert grads is None
    if nu >= 2:
        assert rel(hesses, arr["hesses"]) <= tol
    else:
        assert hesses is None


@pytest.mark.parametrize("case", field_cases())
def test_oracle_fields_match_reference(case):
    meta, arr = field_golden(case)
    out = O.quadrature_fields(field_problem(meta, arr), arr["coefs"], meta["nu"])
    check_fields(out, arr, meta["nu"])
