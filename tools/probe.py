"""Quick device-time probe of the full assembly per config (not the bench; for development)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1904_06971_b200 as pkg
from paper_1904_06971_b200 import _lib
from paper_1904_06971_b200.configs import CONFIGS

which = [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4, 5]
for k in which:
    cfg = CONFIGS[k]
    t = time.time()
    disc = pkg.make_discretization(cfg.geom(), cfg.p, cfg.spans)
    ts = time.time() - t
    for f in cfg.forms:
        fk = pkg.FormKind(f)
        best = 1e9
        for it in range(3):
            res, sym, _ = pkg.assemble_device(fk, disc)
            ms, nl = _lib.last_timing()
            kt = _lib.last_kernel_times()
            nr, nnz = res.sizes()
            if it == 2:
                cs = res.checksum()
            res.free()
            best = min(best, ms)
        ka = [v for n, v in kt if n.startswith("assemble_")]
        print(f"cfg{k} {f:10s} N={nr} nnz={nnz} total {best:.3f} ms  assemble_tiles {ka[0]:.3f} ms  "
              f"nnz/s {nnz / best * 1e3:.3e}  launches {nl}  setup {ts:.1f}s  checksum {cs[1]:.6e} {cs[4]:.3e}", flush=True)
        print("   ", [(n, round(v, 3)) for n, v in kt], flush=True)
