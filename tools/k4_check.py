"""K4 variant check: full assembly of config-5 forms -> best kernel time and checksum (dev tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_06971_b200 as pkg  # noqa: E402
from paper_1904_06971_b200 import _lib  # noqa: E402
from paper_1904_06971_b200.configs import CONFIGS  # noqa: E402

cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 5]
forms = sys.argv[2:] or cfg.forms
disc = pkg.make_discretization(cfg.geom(), cfg.p, cfg.spans)
for f in forms:
    best = 1e9
    for it in range(3):
        res, _, _ = pkg.assemble_device(pkg.FormKind(f), disc)
        kt = [t for n, t in _lib.last_kernel_times() if n.startswith("assemble_")]
        best = min(best, kt[0])
        if it == 2:
            cs = res.checksum()
        res.free()
    print(f"{f:10s} assemble {best:.3f} ms  checksum {cs[1]:.17e} {cs[2]:.17e} {cs[4]:.17e}", flush=True)
