"""Device-resident consumer timing: SpMV and CG iterations on the config-5
mass matrix left in HBM by the assembly.  Prints one JSON line (-> profiles/r01_bench_solve.json)."""
import ctypes as C
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_06971_b200 as pkg  # noqa: E402
from paper_1904_06971_b200 import _lib  # noqa: E402
from paper_1904_06971_b200.configs import CONFIGS  # noqa: E402
from paper_1904_06971_b200.solvers import SolveOptions, solve_spd, spmv  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 5
cfg = CONFIGS[k]
disc = pkg.make_discretization(cfg.geom(), cfg.p, cfg.spans)
res, _, _ = pkg.assemble_device(pkg.FormKind.MASS, disc)
nr, nnz = res.sizes()
x = np.cos(np.arange(nr) * 0.01)
best = 1e9
for _ in range(5):
    spmv(res, x)
    best = min(best, dict(_lib.last_kernel_times())["spmv"])
bytes_spmv = 12 * nnz + 8 * (nr + 1) + 16 * nr  # values + columns, row pointers, x read once, y written
iters = 20
opts = SolveOptions(method="cg", tolerance=1e-14, max_iterations=iters, preconditioner="diagonal")
t0 = time.perf_counter()
try:
    solve_spd(res, np.ones(nr), opts)
except RuntimeError:
    pass  # did not converge in `iters` iterations: expected, only the iteration time is measured
wall = time.perf_counter() - t0
kt = dict(_lib.last_kernel_times())
res.free()
peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
hbm = None
for key in ("hbm_gbs",):
    if key in peaks:
        hbm = peaks[key]
print(json.dumps({"config": f"config{k} mass matrix (device-resident)", "nrows": nr, "nnz": nnz,
                  "spmv_ms": best, "spmv_gbps": bytes_spmv / best / 1e6, "spmv_bytes": bytes_spmv,
                  "hbm_peak_gbps": hbm, "spmv_frac": (bytes_spmv / best / 1e6 / hbm) if hbm else None,
                  "cg_iterations": iters, "cg_ms_per_iteration": kt.get("cg_iterations", float("nan")) / iters,
                  "cg_wall_s": wall}))
