"""CPU: the oracle's conjugate gradient (oracle.conjugate_gradient) against the REAL reference's
solve_spd golden solves (tests/golden/solve, made by make_golden_solve.py), and the
SolveOptions validation of the drop-in (solvers.py:40-71 messages)."""
import glob
import json
import os

import numpy as np
import pytest

from oracle import surriga_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = sorted(glob.glob(os.path.join(HERE, "golden", "solve", "*.npz")))


def load(path):
    z = np.load(path)
    return json.loads(str(z["meta"])), z


@pytest.mark.parametrize("path", CASES, ids=[os.path.basename(c)[:-4] for c in CASES])
def test_oracle_cg_matches_reference(path):
    meta, z = load(path)
    x, status, it = O.conjugate_gradient(z["indptr"], z["indices"], z["data"], z["b"], meta["tol"], meta["maxit"],
                                         meta["preconditioner"])
    err = meta["error"]
    if not err:
        assert status == "converged"
        assert np.linalg.norm(x - z["x"]) <= 1e-13 * np.linalg.norm(z["x"])
    elif err.startswith("negative curvature"):
        assert status == "negative-curvature" and err.startswith(f"negative curvature at iteration {it};")
    elif err.startswith("non-positive diagonal"):
        assert status == "non-positive-diagonal"
    else:
        assert status == "max-iterations" and f"in {it} iterations" in err


def test_solve_options_validation_messages():
    from paper_1904_06971_b200.solvers import SolveOptions

    assert SolveOptions(method="cg").method == "conjugate-gradient"
    for kw, msg in [({"method": "lu"}, "unknown method 'lu'"), ({"tolerance": 1.0}, "tolerance must lie in (0, 1)"),
                    ({"max_iterations": 0}, "max_iterations must be at least 1"),
                    ({"preconditioner": "ilu"}, "unknown preconditioner 'ilu'")]:
        with pytest.raises(ValueError, match=msg.replace("(", r"\(").replace(")", r"\)")):
            SolveOptions(**kw)


def test_direct_method_is_not_a_silent_fallback():
    from paper_1904_06971_b200.solvers import solve_spd

    with pytest.raises(NotImplementedError):
        solve_spd(np.eye(3), np.ones(3))
