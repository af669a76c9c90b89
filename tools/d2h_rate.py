"""to_host() rate on a config-5 matrix (development tool): cold (fresh host buffers) vs warm (pool reuse)."""
import sys
import time

sys.path.insert(0, ".")
import paper_1904_06971_b200 as pkg
from paper_1904_06971_b200 import _lib
from paper_1904_06971_b200.configs import CONFIGS

cfg = CONFIGS[5]
disc = pkg.make_discretization(cfg.geom(), cfg.p, cfg.spans)
_lib.host_staging_init(0)
res, _, _ = pkg.assemble_device(pkg.FormKind("mass"), disc)
nbytes = res.sizes()[1] * 12
keep = []
for it in range(4):
    t = time.perf_counter()
    ip, ix, d = res.to_host()
    dt = time.perf_counter() - t
    print(f"to_host #{it}: {dt:.3f} s  {nbytes / dt / 1e9:.1f} GB/s", flush=True)
    if it == 1:
        keep.append((ip, ix, d))  # hold one set: the next call needs fresh buffers again
    del ip, ix, d
