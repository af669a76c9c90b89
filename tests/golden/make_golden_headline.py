"""Headline-size golden fingerprints from the REAL reference (run in the build container).

The BASELINE configs 2-4 at full size and config 5's settings at the S=48 step of the survey's
scaled ladder (p=3, q=3, M=16 on the twisted-cube stand-in) are assembled by the
reference itself -- ``build_surrogate_matrix`` in its default mode (Poisson / bi-Laplacian: SKP,
mass: SYMMETRIC) and, for configs 2-4, ``assemble`` -- and each result is reduced to the
fingerprint of ``tests/headline_checks.py`` (pattern CRCs, every row's weighted checksum summed
per row block, a few hundred full sampled rows, the AssemblyReport).  Config 5 at 128^3 is out
of reach of the reference here (~3.2 h / ~580 GB); it is checked against the
oracle's sampled-row surrogate instead (``oracle.surriga_oracle.surrogate_rows``).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_headline.py [case ...]

Writes ``tests/golden/headline/<case>.npz``; numpy / scipy versions are recorded in each file.
"""
import json
import os
import sys
import time

import numpy as np
import scipy

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))  # tests/ (headline_checks)

from headline_checks import block_checksums, crc, rows_segments, sample_rows  # noqa: E402
from surriga.assembly import FormKind, assemble, make_discretization  # noqa: E402
from surriga.geometry import load_geometry, quarter_annulus  # noqa: E402
from surriga.surrogate import ConstantSampling, build_sampling_lattice, build_surrogate_matrix  # noqa: E402

DATA = os.path.join(HERE, "..", "..", "paper_1904_06971_b200", "data")
OUT = os.path.join(HERE, "headline")

GEOMS = {"annulus": lambda: quarter_annulus(1.0, 2.0),
         "twisted": lambda: load_geometry(os.path.join(DATA, "twisted_cube_p3_m12.geo")),
         "sinmap": lambda: load_geometry(os.path.join(DATA, "sin_map_p3_m16.geo"))}

# (case, config, geometry, p, spans, form, kind, M)
CASES = [
    ("c5s48_poisson_surr", 5, "twisted", 3, (48, 48, 48), "poisson", "surrogate", 16),
    ("c5s48_mass_surr", 5, "twisted", 3, (48, 48, 48), "mass", "surrogate", 16),
    ("c2_poisson_surr", 2, "annulus", 3, (512, 512), "poisson", "surrogate", 16),
    ("c2_mass_surr", 2, "annulus", 3, (512, 512), "mass", "surrogate", 16),
    ("c2_poisson_full", 2, "annulus", 3, (512, 512), "poisson", "full", 16),
    ("c4_biharm_surr", 4, "sinmap", 3, (1024, 1024), "biharmonic", "surrogate", 32),
    ("c3_poisson_surr", 3, "twisted", 2, (64, 64, 64), "poisson", "surrogate", 8),
    ("c4_biharm_full", 4, "sinmap", 3, (1024, 1024), "biharmonic", "full", 32),
    ("c3_poisson_full", 3, "twisted", 2, (64, 64, 64), "poisson", "full", 8),
    ("c5s64_poisson_surr", 5, "twisted", 3, (64, 64, 64), "poisson", "surrogate", 16),
    ("c5s48_mass_full", 5, "twisted", 3, (48, 48, 48), "mass", "full", 16),
    ("c5s48_poisson_full", 5, "twisted", 3, (48, 48, 48), "poisson", "full", 16),
]


def block_size(N):
    return max(8, 1 << int(np.ceil(np.log2(max(1, N / 65536)))))  # <= 64k blocks (~1 MB per file)


def run(case, cfg, gname, p, spans, form, kind, M):
    g = GEOMS[gname]()
    disc = make_discretization(g, p, spans)
    fk = FormKind(form)
    meta = dict(case=case, config=cfg, geometry=gname, p=p, spans=list(spans), form=form, kind=kind, M=M, q=3,
                gauss=disc.gauss, numpy=np.__version__, scipy=scipy.__version__)
    t0 = time.perf_counter()
    if kind == "full":
        A = assemble(fk, disc)
    else:
        A, rep = build_surrogate_matrix(fk, disc, ConstantSampling(M), q=3)
        meta["report"] = {k: getattr(rep, k) for k in ("N", "p", "q", "M", "H", "quad_entries", "interp_entries",
                                                        "quad_fraction", "active_elements", "flags")}
    meta["reference_seconds"] = time.perf_counter() - t0
    meta["symmetric"] = bool(A.symmetric)
    m = A.mat
    ip = m.indptr.astype(np.int64)
    ms = tuple(kv.m for kv in disc.space.kvs)
    lat = build_sampling_lattice(disc.space.kvs, M)
    rows = sample_rows(ms, p, lat.indices)
    cnt, cols, vals = rows_segments(ip, m.indices, m.data, rows)
    B = block_size(ip.size - 1)
    C, W = block_checksums(ip, m.indices, m.data, B)
    meta.update(N=int(ip.size - 1), nnz=int(m.nnz), block=B, crc_indptr=crc(m.indptr, np.int32),
                crc_indices=crc(m.indices, np.int32))
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, f"{case}.npz"), meta=np.array(json.dumps(meta)), rows=rows, row_cnt=cnt,
                        row_cols=cols.astype(np.int32), row_vals=vals, block_C=C, block_W=W)
    return meta


def main():
    only = set(sys.argv[1:])
    for c in CASES:
        if only and c[0] not in only:
            continue
        meta = run(*c)
        print(f"{c[0]}: nnz={meta['nnz']} ref {meta['reference_seconds']:.1f} s", file=sys.stderr, flush=True)


if __name__ == "__main__":
    main()
