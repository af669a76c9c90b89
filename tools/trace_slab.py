"""SG_TRACE timeline of one config-5 slab call (full and strategy-B surrogate) and the whole calls."""
import os
import sys

os.environ["SG_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from slab_cost import cfg, job_slabs, lat, lattice_owners, ms, run  # noqa: E402

N = 8
for form in ("poisson",):
    for path in ("full", "surrogate"):
        run(form, path, None)
        sl = job_slabs(ms, cfg.p, N, path, form, lat.indices)
        owner = lattice_owners(ms, lat.indices, sl) if path == "surrogate" else None
        run(form, path, sl[2], "B", owner, 2)
        print(f"==== {form} {path} slab 2 (second run)", file=sys.stderr, flush=True)
        run(form, path, sl[2], "B", owner, 2)
