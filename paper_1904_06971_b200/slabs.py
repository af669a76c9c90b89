"""Row-slab partitioning across GPUs.

Each rank assembles a contiguous slab of rows (colex order), cut on planes of the slowest
direction, with the p-layer element halo recomputed locally -- no data-path collective.  The
only collective is an all-reduce of per-slab checksums {nnz, sum a, sum a^2, sum |a|,
sum |row sums|} (NCCL on the GPUs; gloo in the CPU tests).  Because rows are computed
bit-identically whatever the slab (atomics-free, fixed-order accumulation), the stitched matrix
equals the single-GPU matrix bit for bit.
"""
from __future__ import annotations

import numpy as np

__all__ = ["plane_slabs", "weighted_plane_slabs", "csr_checksum", "stitch", "allreduce_checksum"]


def plane_slabs(ms, world: int):
    """Equal slabs of slowest-direction planes: [(row_lo, row_hi)] per rank."""
    ms = tuple(int(m) for m in ms)
    planes = ms[-1]
    per = int(np.prod(ms[:-1]))
    if world < 1 or world > planes:
        raise ValueError(f"cannot cut {planes} planes into {world} slabs")
    cuts = [round(planes * r / world) for r in range(world + 1)]
    return [(cuts[r] * per, cuts[r + 1] * per) for r in range(world)]


def weighted_plane_slabs(plane_cost, per: int, world: int):
    """Slabs balancing a per-plane cost (e.g. quadrature rows per plane for the surrogate)."""
    c = np.cumsum(np.asarray(plane_cost, dtype=float))
    tot = c[-1]
    cuts = [0]
    for r in range(1, world):
        k = int(np.searchsorted(c, tot * r / world)) + 1
        cuts.append(max(cuts[-1] + 1, min(k, len(c) - (world - r))))
    cuts.append(len(c))
    return [(cuts[r] * per, cuts[r + 1] * per) for r in range(world)]


def csr_checksum(indptr, data) -> np.ndarray:
    """Host mirror of sg_result_checksum (values compared with a tolerance, not bitwise)."""
    indptr = np.asarray(indptr, dtype=np.int64)
    data = np.asarray(data, dtype=float)
    cnt = np.diff(indptr)
    rows = np.repeat(np.arange(cnt.size), cnt)
    rs = np.zeros(cnt.size)
    np.add.at(rs, rows, data)
    return np.array([float(data.size), data.sum(), (data * data).sum(), np.abs(data).sum(), np.abs(rs).sum()])


def stitch(parts):
    """Concatenate slab CSRs [(indptr, indices, data)] in rank order into one CSR."""
    ips, ixs, ds = [], [], []
    off = 0
    for k, (ip, ix, d) in enumerate(parts):
        ip = np.asarray(ip, dtype=np.int64)
        ips.append(ip[(0 if k == 0 else 1):] + off)
        off += int(ip[-1])
        ixs.append(np.asarray(ix))
        ds.append(np.asarray(d))
    return np.concatenate(ips), np.concatenate(ixs), np.concatenate(ds)


def allreduce_checksum(cs, dist=None):
    """Sum per-slab checksums over ranks (torch.distributed all-reduce; identity if dist is None)."""
    if dist is None:
        return np.asarray(cs, dtype=float)
    import torch

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor(np.asarray(cs, dtype=np.float64), device=dev)
    dist.all_reduce(t)
    return t.cpu().numpy()
