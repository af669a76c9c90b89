"""D2H split on a config-5 matrix: values only, values + host-generated columns, values + copied columns."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_06971_b200 as pkg  # noqa: E402
from paper_1904_06971_b200 import _lib  # noqa: E402
from paper_1904_06971_b200.configs import CONFIGS  # noqa: E402

cfg = CONFIGS[5]
disc = pkg.make_discretization(cfg.geom(), cfg.p, cfg.spans)
_lib.host_staging_init(0)
res, _, _ = pkg.assemble_device(pkg.FormKind.MASS, disc)
nr, nz = res.sizes()
ip = np.empty(nr + 1, np.int64)
ix = np.empty(nz, np.int32)
d = np.empty(nz, np.float64)
for a in (ip, ix, d):
    a.fill(0)
    _lib.check(_lib.lib().sg_host_register(C.c_void_p(a.ctypes.data), C.c_size_t(a.nbytes)))
L = _lib.lib()
def run(label, with_ix, with_d):
    best = 1e9
    for _ in range(3):
        t = time.perf_counter()
        _lib.check(L.sg_result_copy_i64(res.h, ip.ctypes.data_as(_lib._i64), ix.ctypes.data_as(_lib._i32) if with_ix else None,
                                        _lib.dptr(d) if with_d else None))
        best = min(best, time.perf_counter() - t)
    gb = (ip.nbytes + (ix.nbytes if with_ix else 0) + (d.nbytes if with_d else 0)) / 1e9
    print(f"{label:28s} {best * 1e3:7.1f} ms  ({gb:.2f} GB host bytes, {gb / best:.1f} GB/s)", flush=True)
run("values only", False, True)
run("columns only (host gen)", True, False)
run("values + host columns", True, True)
os.environ["SG_COPY_INDICES"] = "1"
run("values + copied columns", True, True)
