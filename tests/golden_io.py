"""Load golden fixtures (made by tests/golden/make_golden.py from the real reference)."""
import glob
import json
import os

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def cases():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(HERE, "*.npz")))


def load(case):
    z = np.load(os.path.join(HERE, case + ".npz"))
    meta = json.loads(str(z["meta"]))
    arr = {k: z[k] for k in z.files if k != "meta"}
    return meta, arr


def oracle_problem(meta, arr):
    from oracle.surriga_oracle import Problem

    p = meta["p"]
    return Problem(form=meta["form"], p=p, ms=tuple(s + p for s in meta["spans"]), g=meta["gauss"],
                   sol_w=arr["sol_w"], geo_p=meta["geo_p"], geo_ms=tuple(meta["geo_ms"]), geo_w=arr["geo_w"],
                   geo_ctrl=arr["geo_ctrl"], coefficient=meta.get("coefficient", 1.0))
