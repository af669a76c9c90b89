"""Row-slab overhead on one GPU: the device time of the N slabs of a config-5 matrix assembled one
after another, against the whole matrix (the multi-GPU step's per-rank work = one slab)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_06971_b200 as pkg  # noqa: E402
from paper_1904_06971_b200 import _lib  # noqa: E402
from paper_1904_06971_b200.configs import CONFIGS  # noqa: E402
from paper_1904_06971_b200.slabs import job_slabs  # noqa: E402
from paper_1904_06971_b200.surrogate import DEFAULT_MODE, build_sampling_lattice, surrogate_device  # noqa: E402

cfg = CONFIGS[5]
disc = pkg.make_discretization(cfg.geom(), cfg.p, cfg.spans)
ms = tuple(kv.m for kv in disc.space.kvs)
lat = build_sampling_lattice(disc.space.kvs, cfg.M)


def run(form, path, slab):
    if path == "full":
        res, _, _ = pkg.assemble_device(pkg.FormKind(form), disc, slab=slab)
    else:
        res, _, _ = surrogate_device(pkg.FormKind(form), disc, cfg.M, cfg.q, DEFAULT_MODE[form].value, slab=slab, lattice=lat)
    t = _lib.last_timing()[0]
    res.free()
    return t


for form in cfg.forms:
    for path in ("full", "surrogate"):
        run(form, path, None)
        whole = min(run(form, path, None) for _ in range(2))
        out = [f"{form:8s} {path:9s} whole {whole:7.2f} ms"]
        for n in (2, 4, 8):
            ts = [min(run(form, path, sl) for _ in range(2)) for sl in job_slabs(ms, cfg.p, n, path, form, lat.indices)]
            out.append(f"N={n}: max {max(ts):6.2f} sum/whole {sum(ts) / whole:5.2f} max*N/whole {max(ts) * n / whole:5.2f}")
        print("  ".join(out), flush=True)
