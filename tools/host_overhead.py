"""Host-side overhead of one bench step (development tool): wall vs device time per call + cProfile."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_1904_06971_b200 as pkg
from paper_1904_06971_b200 import _lib
from paper_1904_06971_b200.configs import CONFIGS
from paper_1904_06971_b200.surrogate import build_sampling_lattice, surrogate_device, tilde_domain

cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 5]
disc = pkg.make_discretization(cfg.geom(), cfg.p, cfg.spans)
ms = tuple(kv.m for kv in disc.space.kvs)
lattice = build_sampling_lattice(disc.space.kvs, cfg.M)
tilde = tilde_domain(cfg.p, ms)
sptr = torch.cuda.current_stream().cuda_stream


def one(f, path):
    fk = pkg.FormKind(f)
    if path == "full":
        res, _, _ = pkg.assemble_device(fk, disc, stream=sptr)
    else:
        res, _, _ = surrogate_device(fk, disc, cfg.M, cfg.q, pkg.surrogate.DEFAULT_MODE[f].value, stream=sptr,
                                     lattice=lattice, tilde=tilde)
    dev = _lib.last_timing()[0]
    res.free()
    return dev


for f in cfg.forms:
    for path in ("full", "surrogate"):
        one(f, path)
for f in cfg.forms:
    for path in ("full", "surrogate"):
        torch.cuda.synchronize()
        t = time.perf_counter()
        dev = one(f, path)
        torch.cuda.synchronize()
        w = (time.perf_counter() - t) * 1e3
        print(f"{f:8s} {path:9s} wall {w:8.2f} ms  device(sg_last_timing) {dev:8.2f} ms  host {w - dev:7.2f} ms")
pr = cProfile.Profile()
pr.enable()
for f in cfg.forms:
    for path in ("full", "surrogate"):
        one(f, path)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
