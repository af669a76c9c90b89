"""Per-matrix wall time of the end-to-end path (device assembly + to_host) over several steps
(development tool for the e2e variance)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_06971_b200 as pkg  # noqa: E402
from paper_1904_06971_b200 import _lib  # noqa: E402
from paper_1904_06971_b200.configs import CONFIGS  # noqa: E402
from paper_1904_06971_b200.surrogate import DEFAULT_MODE, build_sampling_lattice, surrogate_device, tilde_domain  # noqa: E402

cfg = CONFIGS[5]
disc = pkg.make_discretization(cfg.geom(), cfg.p, cfg.spans)
ms = tuple(kv.m for kv in disc.space.kvs)
lat = build_sampling_lattice(disc.space.kvs, cfg.M)
til = tilde_domain(cfg.p, ms)
_lib.host_staging_init(0)
for step in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    row = []
    for f in cfg.forms:
        for path in ("full", "surrogate"):
            t0 = time.perf_counter()
            if path == "full":
                res, _, _ = pkg.assemble_device(pkg.FormKind(f), disc)
            else:
                res, _, _ = surrogate_device(pkg.FormKind(f), disc, cfg.M, cfg.q, DEFAULT_MODE[f].value, lattice=lat, tilde=til)
            t1 = time.perf_counter()
            ip, ix, d = res.to_host()
            t2 = time.perf_counter()
            res.free()
            del ip, ix, d
            row.append(f"{f[:4]}/{path[:4]} {1e3 * (t1 - t0):6.1f}+{1e3 * (t2 - t1):6.1f}")
    print(f"step {step}: " + "  ".join(row), flush=True)
    if step == 1:
        _lib.host_pool_sync()
