"""Size-independent CSR fingerprints for headline-size parity (test infrastructure).

A headline matrix (up to 51.5M nnz here) is too large to commit, so the golden files made from
the real reference at those sizes keep
  * the pattern as CRC-32s of the int32 ``indptr`` and ``indices`` bytes (bit-exact check),
  * a few hundred sampled rows in full (cols + values), chosen per row class, and
  * a weighted checksum of every row, summed over blocks of consecutive rows:
      c_i = sum_j a_ij r(j),  r(j) = 1 + frac(j * 0x9E3779B1 / 2^32)      (r in [1, 2))
      C_b = sum_{i in b} c_i,  W_b = sum_{i in b} cnt_i max_j |a_ij|
    Two matrices within 1e-12 row-scaled give |C_b - C'_b| <= 2e-12 W_b (+ the checksum's own
    rounding, ~cnt eps), while any single entry wrong by more than ~1e-11 of its row scale moves
    its block's checksum past that bound.
"""
from __future__ import annotations

import zlib

import numpy as np


def weights(cols):
    c = np.asarray(cols, dtype=np.int64)
    return 1.0 + ((c * 0x9E3779B1) & 0xFFFFFFFF).astype(np.float64) / 4294967296.0


def crc(a, dtype):
    return int(zlib.crc32(np.ascontiguousarray(np.asarray(a).astype(dtype)).tobytes()))


def block_checksums(indptr, indices, data, block):
    """(C_b, W_b) over blocks of ``block`` consecutive rows (last block may be short)."""
    ip = np.asarray(indptr, dtype=np.int64)
    N = ip.size - 1
    prod = np.asarray(data, dtype=np.float64) * weights(indices)
    cnt = np.diff(ip)
    nonempty = cnt > 0
    c = np.zeros(N)
    mx = np.zeros(N)
    if data.size:
        starts = ip[:-1][nonempty]
        c[nonempty] = np.add.reduceat(prod, starts)
        mx[nonempty] = np.maximum.reduceat(np.abs(data), starts)
    w = cnt * mx
    edges = np.arange(0, N, block)
    return np.add.reduceat(c, edges), np.add.reduceat(w, edges)


def check_blocks(ref_C, ref_W, C, W, tol=1e-12):
    """Largest block deviation relative to its bound; <= 1 passes."""
    bound = 2.0 * tol * np.maximum(ref_W, 1e-300) + 4e-16 * np.abs(ref_C)
    ratio = np.abs(C - ref_C) / bound
    return float(ratio.max()), int(ratio.argmax())


def interesting_1d(p, m, lattice):
    """1-D indices covering every row class along one direction: domain boundary, boundary band,
    box edge, lattice sites and their neighbours, box interior, far end."""
    lo, hi = 2 * p, m - 2 * p - 1
    pts = {0, 1, p, 2 * p - 1, lo, lo + 1, hi - 1, hi, hi + 1, m - p - 1, m - 1, (lo + hi) // 2}
    for s in list(lattice)[:3] + list(lattice)[-2:]:
        pts.update({s - 1, s, s + 1})
    return sorted(x for x in pts if 0 <= x < m)


def sample_rows(ms, p, lattices, count=320, seed=7):
    """Deterministic sample of rows whose per-direction indices are all 'interesting': half of
    them interpolated rows (in the box, not on the lattice), half quadrature rows."""
    axes = [interesting_1d(p, m, lat) for m, lat in zip(ms, lattices)]
    grids = np.meshgrid(*axes, indexing="ij")
    multi = np.stack([g.ravel() for g in grids], -1)
    inbox = np.all((multi >= 2 * p) & (multi <= np.asarray(ms) - 2 * p - 1), axis=1)
    onlat = np.all(np.stack([np.isin(multi[:, d], lattices[d]) for d in range(len(ms))], -1), axis=1)
    interp = inbox & ~onlat
    strides = np.cumprod((1,) + tuple(ms[:-1]))
    rng = np.random.default_rng(seed)
    out = []
    for sel, k in ((interp, count // 2), (~interp, count - count // 2)):
        r = np.unique(multi[sel] @ strides)
        out.append(np.sort(rng.choice(r, k, replace=False)) if r.size > k else r)
    return np.unique(np.concatenate(out)).astype(np.int64)


def rows_segments(indptr, indices, data, rows):
    ip = np.asarray(indptr, dtype=np.int64)
    cnt = ip[rows + 1] - ip[rows]
    take = np.concatenate([np.arange(ip[r], ip[r + 1]) for r in rows]) if rows.size else np.zeros(0, np.int64)
    return cnt, np.asarray(indices)[take], np.asarray(data)[take]
