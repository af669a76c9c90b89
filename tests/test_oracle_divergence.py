"""Pin the divergence restatement of the CPU oracle against the reference's goldens (CPU only).

Fixtures: tests/golden/div/*.npz from tests/golden/make_golden_div.py (assembly.py:654-725); the
properties mirror test_assembly.py:154-178 (constant velocity field -> zero, row restriction bitwise).
"""
import glob
import json
import os

import numpy as np
import pytest

from oracle import surriga_oracle as O

DIV = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "div")
TOL = 1e-12


def div_cases():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(DIV, "*.npz")))


def load_div(case):
    z = np.load(os.path.join(DIV, case + ".npz"))
    meta = json.loads(str(z["meta"]))
    return meta, {k: z[k] for k in z.files if k != "meta"}


def vel_problem(meta, arr):
    pv = meta["pp"] + 1
    return O.Problem(form="stokes_divergence", p=pv, ms=tuple(2 * s + pv for s in meta["spans"]), g=meta["gauss"],
                     sol_w=arr["vel_w"], geo_p=meta["geo_p"], geo_ms=tuple(meta["geo_ms"]), geo_w=arr["geo_w"],
                     geo_ctrl=arr["geo_ctrl"])


def check_component(arr, c, ip, ix, d):
    assert np.array_equal(ip, arr[f"indptr_{c}"].astype(np.int64)), f"indptr differs (component {c})"
    assert np.array_equal(ix, arr[f"indices_{c}"]), f"indices differ (component {c})"
    err = O.row_scaled_error(arr[f"indptr_{c}"], arr[f"indices_{c}"], arr[f"data_{c}"], ip, ix, d)
    assert err <= TOL, (c, err)


@pytest.mark.parametrize("case", [c for c in div_cases() if not c.startswith("sdiv_")])
def test_oracle_divergence_matches_reference(case):
    meta, arr = load_div(case)
    vel = vel_problem(meta, arr)
    ip, ix, data, pop = O.divergence(vel, meta["pp"], rows=arr.get("rows"), prs_w=arr["prs_w"])
    if "rows" in arr:
        assert np.array_equal(pop, arr["populated_rows"])
    for c in range(meta["n"]):
        check_component(arr, c, ip, ix, data[c])


@pytest.mark.parametrize("case", [c for c in div_cases() if c.startswith("sdiv_")])
def test_oracle_surrogate_divergence_matches_reference(case):
    meta, arr = load_div(case)
    mats, rep = O.surrogate_divergence(vel_problem(meta, arr), meta["pp"], meta["M"], meta["q"], prs_w=arr["prs_w"])
    for k, v in meta["report"].items():
        assert rep[k] == v, (k, rep[k], v)
    for c, (ip, ix, d) in enumerate(mats):
        check_component(arr, c, ip, ix, d)


def test_oracle_divergence_constant_field_vanishes():
    meta, arr = load_div("div_coons_quad_p2")
    ip, ix, data, _ = O.divergence(vel_problem(meta, arr), meta["pp"])
    import scipy.sparse as sp

    Nv = int(np.prod([2 * s + meta["pp"] + 1 for s in meta["spans"]]))
    for d in data:
        D = sp.csr_matrix((d, ix, ip), shape=(ip.size - 1, Nv))
        assert np.max(np.abs(D @ np.ones(Nv))) < 1e-13
