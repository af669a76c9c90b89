"""Row-slab overhead on one GPU: the device time of the N slabs of a config-5 matrix assembled one
after another, against the whole matrix (the multi-GPU step's per-rank work = one slab).

Surrogate slabs run strategy B: each slab assembles only its own lattice rows; the
exchange that completes the sample table (an NCCL all-gather of <= 2 MB on the real box) is
emulated by a device copy from the whole matrix's table.  ``single`` = a slab call without an
exchange (the other slabs' lattice rows assembled again by row-restricted quadrature)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1904_06971_b200 as pkg  # noqa: E402
from paper_1904_06971_b200 import _lib  # noqa: E402
from paper_1904_06971_b200.configs import CONFIGS  # noqa: E402
from paper_1904_06971_b200.slabs import _device_view, job_slabs, lattice_owners  # noqa: E402
from paper_1904_06971_b200.surrogate import DEFAULT_MODE, build_sampling_lattice, surrogate_device  # noqa: E402

cfg = CONFIGS[int(os.environ.get("SG_SLAB_CONFIG", "5"))]
disc = pkg.make_discretization(cfg.geom(), cfg.p, cfg.spans)
ms = tuple(kv.m for kv in disc.space.kvs)
lat = build_sampling_lattice(disc.space.kvs, cfg.M)
dev = torch.device("cuda", 0)
tables = {}


def keep_table(form):
    def ex(ptr, P, nlat):
        tables[form] = _device_view(ptr, (P, nlat), dev).clone()
    return ex


def fill_table(form, owner, rank):
    def ex(ptr, P, nlat):
        t = _device_view(ptr, (P, nlat), dev)
        other = torch.as_tensor(np.flatnonzero(owner != rank), device=dev)
        t[:, other] = tables[form][:, other]
        torch.cuda.synchronize()
    return ex


def run(form, path, slab, mode="B", owner=None, rank=0):
    if path == "full":
        res, _, _ = pkg.assemble_device(pkg.FormKind(form), disc, slab=slab)
    else:
        ex = None
        if slab is None:
            ex = keep_table(form)
        elif mode == "B":
            ex = fill_table(form, owner, rank)
        res, _, _ = surrogate_device(pkg.FormKind(form), disc, cfg.M, cfg.q, DEFAULT_MODE[form].value, slab=slab,
                                     lattice=lat, exchange=ex)
    t = _lib.last_timing()[0]
    res.free()
    return t


def main():
    for form in cfg.forms:
        for path, mode in (("full", "-"), ("surrogate", "B"), ("surrogate", "single")):
            run(form, path, None)
            whole = min(run(form, path, None) for _ in range(2))
            out = [f"{form:8s} {path:9s} {mode:6s} whole {whole:7.2f} ms"]
            for n in (2, 4, 8):
                sl = job_slabs(ms, cfg.p, n, path, form, lat.indices)
                owner = lattice_owners(ms, lat.indices, sl) if path == "surrogate" else None
                ts = [min(run(form, path, s, mode, owner, r) for _ in range(2)) for r, s in enumerate(sl)]
                out.append(f"N={n}: max {max(ts):6.2f} sum/whole {sum(ts) / whole:5.2f} max*N/whole {max(ts) * n / whole:5.2f}")
            print("  ".join(out), flush=True)


if __name__ == "__main__":
    main()
