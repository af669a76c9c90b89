"""Device timing of the Stokes divergence pairing (full + surrogate) on a twisted-cube subgrid pair.

    python tools/bench_div.py [pressure spans] [pp] [M]
"""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np

import paper_1904_06971_b200 as pkg
from paper_1904_06971_b200 import _lib

S = int(sys.argv[1]) if len(sys.argv) > 1 else 32
pp = int(sys.argv[2]) if len(sys.argv) > 2 else 2
M = int(sys.argv[3]) if len(sys.argv) > 3 else 8
st = pkg.stokes_subgrid_spaces(pkg.twisted_cube_standin(), pp, (S, S, S))
out = {"pressure_spans": S, "pp": pp, "velocity_N": st.velocity.space.N, "pressure_N": st.pressure.space.N}
for rep in range(3):
    res, _ = pkg.assemble_divergence_device(st)
    ms, nl = _lib.last_timing()
    kt = _lib.last_kernel_times()
    nnz = res[0].sizes()[1]
    for r in res:
        r.free()
out["full"] = {"device_ms": ms, "nnz_per_component": nnz, "nnz_per_s": 3 * nnz / (ms * 1e-3),
               "kernels_ms": {k: round(v, 3) for k, v in kt}, "hbm_floor_ms": 3 * nnz * 12 / 6555.8e9 * 1e3}
t = time.perf_counter()
D, rep_ = pkg.build_surrogate_divergence(st, pkg.ConstantSampling(M))
wall = time.perf_counter() - t
ms, nl = _lib.last_timing()
out["surrogate"] = {"device_ms": ms, "wall_s_incl_d2h": wall, "kernels_ms": {k: round(v, 3) for k, v in _lib.last_kernel_times()},
                    "quad_fraction": rep_.quad_fraction, "nnz_per_component": int(D[0].nnz)}
print(json.dumps(out, indent=1))
