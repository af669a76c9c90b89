import os, sys
sys.path.insert(0, "/root/repo")
import paper_1904_06971_b200 as pkg
from paper_1904_06971_b200 import _lib
from paper_1904_06971_b200.configs import CONFIGS
from paper_1904_06971_b200.slabs import job_slabs
from paper_1904_06971_b200.surrogate import DEFAULT_MODE, build_sampling_lattice, surrogate_device
cfg = CONFIGS[5]
disc = pkg.make_discretization(cfg.geom(), cfg.p, cfg.spans)
ms = tuple(kv.m for kv in disc.space.kvs)
lat = build_sampling_lattice(disc.space.kvs, cfg.M)
for sl in [None] + job_slabs(ms, cfg.p, 8, "surrogate", "poisson", lat.indices)[::3]:
    for it in range(2):
        res, _, _ = surrogate_device(pkg.FormKind.POISSON, disc, cfg.M, cfg.q, "symmetric_kernel_preserving", slab=sl, lattice=lat)
        t = _lib.last_timing()[0]; kt = _lib.last_kernel_times(); res.free()
    agg = {}
    for n, v in kt: agg[n] = agg.get(n, 0) + v
    print(sl, round(t, 2), {k: round(v, 2) for k, v in agg.items() if v > 0.05})
