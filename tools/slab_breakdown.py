"""Per-kernel device times of every slab of a config-5 matrix (strategy B surrogate, full assembly)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from slab_cost import cfg, job_slabs, lat, lattice_owners, ms, run  # noqa: E402
from paper_1904_06971_b200 import _lib  # noqa: E402

N = int(os.environ.get("SG_SLABS", "8"))
for form in cfg.forms:
    for path in ("full", "surrogate"):
        run(form, path, None)
        run(form, path, None)
        print(f"== {form} {path} whole: " + " ".join(f"{k}={v:.2f}" for k, v in _lib.last_kernel_times()))
        sl = job_slabs(ms, cfg.p, N, path, form, lat.indices)
        owner = lattice_owners(ms, lat.indices, sl) if path == "surrogate" else None
        for r, s in enumerate(sl):
            run(form, path, s, "B", owner, r)
            t = run(form, path, s, "B", owner, r)
            kt = {}
            for k, v in _lib.last_kernel_times():
                kt[k] = kt.get(k, 0) + v
            print(f"  slab {r} rows {s[0]}..{s[1]} ({(s[1]-s[0])//(ms[0]*ms[1])} planes) total {t:.2f}: "
                  + " ".join(f"{k}={v:.2f}" for k, v in kt.items() if v > 0.02), flush=True)
