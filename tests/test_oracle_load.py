"""Pin the load-vector restatement of the CPU oracle against the reference's goldens (assembly.py:728-759)."""
import glob
import json
import os

import numpy as np
import pytest

from load_funcs import LOAD_FUNCS
from oracle import surriga_oracle as O

LOAD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "load")
TOL = 1e-13


def load_cases():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(LOAD, "*.npz")))


def load_golden(case):
    z = np.load(os.path.join(LOAD, case + ".npz"))
    meta = json.loads(str(z["meta"]))
    return meta, {k: z[k] for k in z.files if k != "meta"}


def problem(meta, arr):
    p = meta["p"]
    return O.Problem(form="mass", p=p, ms=tuple(s + p for s in meta["spans"]), g=meta["gauss"], sol_w=arr["sol_w"],
                     geo_p=meta["geo_p"], geo_ms=tuple(meta["geo_ms"]), geo_w=arr["geo_w"], geo_ctrl=arr["geo_ctrl"])


@pytest.mark.parametrize("case", load_cases())
def test_oracle_load_matches_reference(case):
    meta, arr = load_golden(case)
    vec = O.load_vector(problem(meta, arr), LOAD_FUNCS[meta["func"]])
    ref = arr["vec"]
    assert np.max(np.abs(vec - ref)) <= TOL * max(1.0, np.max(np.abs(ref)))
