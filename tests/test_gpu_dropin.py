"""The drop-in, exercised through the reference package itself: the installed
reference (baseline/_ref, the unmodified `surriga`) is run unpatched and with the rebinding on its
own Discretization / FormKind / ConstantSampling objects -- (1) its own build_surrogate_matrix with
the quadrature-row call (surrogate.py:588) rebound to the GPU, (2) the whole rebinding, including a
studies cell (studies.py:477-501 via run_poisson_study).  Matrices must agree to 1e-12 row-scaled
with identical patterns, reports equal field by field (seconds excepted), study errors to 1e-9."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref", "surriga")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not installed in baseline/_ref (DESIGN.md §7)")
def test_gpu_dropin_through_reference_package():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "dropin", "check.py")], capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    for k, v in out.items():
        if "err" in v:
            assert v["err"] <= 1e-12, (k, v)
        for flag in ("report_equal", "symmetric", "int32", "rows_equal"):
            if flag in v:
                assert v[flag], (k, flag, v)
        if "type" in v:
            assert v["type"].startswith("surriga."), (k, v["type"])
    assert out["studies/run_poisson_study"]["rel_err_worst"] <= 1e-9
