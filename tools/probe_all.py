"""Device time of every BASELINE config (full + surrogate, each form): best of 3 calls, nnz/s and
the kernel breakdown (development / DESIGN table tool)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_06971_b200 as pkg  # noqa: E402
from paper_1904_06971_b200 import _lib  # noqa: E402
from paper_1904_06971_b200.configs import CONFIGS  # noqa: E402
from paper_1904_06971_b200.surrogate import DEFAULT_MODE, build_sampling_lattice, surrogate_device, tilde_domain  # noqa: E402

out = []
for k in [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4, 5]:
    cfg = CONFIGS[k]
    disc = pkg.make_discretization(cfg.geom(), cfg.p, cfg.spans)
    ms = tuple(kv.m for kv in disc.space.kvs)
    lat = build_sampling_lattice(disc.space.kvs, cfg.M)
    til = tilde_domain(cfg.p, ms)
    for f in cfg.forms:
        for path in ("full", "surrogate"):
            best, kt = 1e9, None
            for _ in range(3):
                if path == "full":
                    res, _, _ = pkg.assemble_device(pkg.FormKind(f), disc)
                else:
                    res, _, _ = surrogate_device(pkg.FormKind(f), disc, cfg.M, cfg.q, DEFAULT_MODE[f].value, lattice=lat, tilde=til)
                ms_, _ = _lib.last_timing()
                nr, nnz = res.sizes()
                res.free()
                if ms_ < best:
                    best, kt = ms_, _lib.last_kernel_times()
            agg = {}
            for n_, t in kt:
                agg[n_] = agg.get(n_, 0.0) + t
            top = sorted(agg.items(), key=lambda x: -x[1])[:4]
            row = {"config": k, "form": f, "path": path, "ms": round(best, 3), "nnz": nnz, "nnz_per_s": nnz / best * 1e3,
                   "top_kernels_ms": {a: round(b, 3) for a, b in top}}
            print(json.dumps(row), flush=True)
