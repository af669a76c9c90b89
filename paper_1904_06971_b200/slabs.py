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

__all__ = ["plane_slabs", "weighted_plane_slabs", "halo_balanced_plane_slabs", "surrogate_plane_cost", "job_slabs",
           "csr_checksum", "stitch",
           "allreduce_checksum", "lattice_owners", "exchange_samples"]

# Relative device cost per row of the surrogate's parts (measured on one B200 at config 5, p=3,
# DESIGN.md §8): quadrature row (K4 on the quadrature tiles), interpolated row (K7), any row (K3
# geometry of the needed planes, row pointers).  Only the ratios matter.
SURROGATE_ROW_COST = {"poisson": (15.2, 2.25, 0.5), "stokes_velocity": (15.2, 2.25, 0.5),
                      "mass": (3.1, 2.25, 0.4), "biharmonic": (15.2, 2.25, 0.5)}


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
    c = np.r_[0.0, np.cumsum(np.asarray(plane_cost, dtype=float))]  # c[k] = cost of planes [0, k)
    tot = c[-1]
    cuts = [0]
    for r in range(1, world):
        t = tot * r / world
        k = int(np.searchsorted(c, t))  # c[k-1] < t <= c[k]: cut at whichever side is nearer
        if k > 0 and t - c[k - 1] < c[k] - t:
            k -= 1
        cuts.append(max(cuts[-1] + 1, min(k, len(c) - 1 - (world - r))))
    cuts.append(len(c) - 1)
    return [(cuts[r] * per, cuts[r + 1] * per) for r in range(world)]


def halo_balanced_plane_slabs(plane_cost, halo_cost, p: int, per: int, world: int):
    """Slabs minimising the dearest slab when a slab also pays for its p-plane halo on either side
    (the surrogate recomputes the halo's quadrature rows: next to the box's all-quadrature boundary
    planes that halo costs as much as a dozen interior planes, which per-plane balancing ignores).
    cost[a, b) = sum plane_cost[a:b] + sum halo_cost[a-p:a] + sum halo_cost[b:b+p]; exact by dynamic
    programming over the cut positions (planes x planes x world steps)."""
    c = np.r_[0.0, np.cumsum(np.asarray(plane_cost, dtype=float))]
    h = np.r_[0.0, np.cumsum(np.asarray(halo_cost, dtype=float))]
    n = len(c) - 1
    if world < 1 or world > n:
        raise ValueError(f"cannot cut {n} planes into {world} slabs")

    lo_h = h - h[np.maximum(np.arange(n + 1) - p, 0)]           # halo below a cut at plane a
    hi_h = h[np.minimum(np.arange(n + 1) + p, n)] - h             # halo above a cut at plane b
    inf = float("inf")
    best = np.full((world + 1, n + 1), inf)
    arg = np.zeros((world + 1, n + 1), dtype=np.int64)
    best[0, 0] = 0.0
    for r in range(1, world + 1):
        for b in range(r, n - (world - r) + 1):
            a = np.arange(r - 1, b)
            v = np.maximum(best[r - 1, a], c[b] - c[a] + lo_h[a] + hi_h[b])
            k = int(np.argmin(v))
            best[r, b] = v[k]
            arg[r, b] = a[k]
    cuts = [n]
    for r in range(world, 0, -1):
        cuts.append(int(arg[r, cuts[-1]]))
    cuts = cuts[::-1]
    return [(cuts[r] * per, cuts[r + 1] * per) for r in range(world)]


def surrogate_plane_cost(ms, p, lattice_indices, form: str, parts: bool = False):
    """Estimated surrogate cost of every slowest-direction plane (quadrature rows are ~9x dearer
    than interpolated rows for Poisson): the boundary layers of the box make the first and last
    slabs heavy, so equal plane counts do not balance the surrogate."""
    ms = tuple(int(m) for m in ms)
    n = len(ms)
    box, smp = [], []
    for d in range(n):
        b = np.zeros(ms[d], bool)
        b[2 * p:ms[d] - 2 * p] = True
        sm = np.zeros(ms[d], bool)
        sm[np.asarray(lattice_indices[d], dtype=np.int64)] = True
        box.append(b)
        smp.append(sm)
    per = int(np.prod(ms[:-1]))
    inner_box = int(np.prod([box[d].sum() for d in range(n - 1)]))
    inner_smp = int(np.prod([(box[d] & smp[d]).sum() for d in range(n - 1)]))
    interp = np.where(~box[-1], 0, np.where(smp[-1], inner_box - inner_smp, inner_box)).astype(float)
    quad = per - interp
    cq, ci, c0 = SURROGATE_ROW_COST.get(form, SURROGATE_ROW_COST["poisson"])
    total = cq * quad + ci * interp + c0 * per
    # parts: also the cost of a plane as a halo plane (its quadrature rows and their geometry)
    return (total, (cq + c0) * quad) if parts else total


def job_slabs(ms, p, world: int, path: str, form: str, lattice_indices=None):
    """Row slabs of one assembly call: equal planes for the full assembly, cost-weighted planes
    for the surrogate."""
    if world <= 1:
        return [None]
    if path == "full" or lattice_indices is None:
        return plane_slabs(ms, world)
    cost, halo = surrogate_plane_cost(ms, p, lattice_indices, form, parts=True)
    return halo_balanced_plane_slabs(cost, halo, p, int(np.prod(ms[:-1])), world)


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


def lattice_owners(ms, lattice_indices, slabs) -> np.ndarray:
    """Rank owning each lattice row (lattice colex order, direction 0 fastest): the slab holding it."""
    ms = tuple(int(m) for m in ms)
    grids = np.meshgrid(*[np.asarray(ix, dtype=np.int64) for ix in lattice_indices], indexing="ij")
    strides = np.cumprod((1,) + ms[:-1])
    rows = sum(g.ravel(order="F") * s for g, s in zip(grids, strides))
    lo = np.array([a for a, _ in slabs], dtype=np.int64)
    owner = np.searchsorted(lo, rows, side="right") - 1
    hi = np.array([b for _, b in slabs], dtype=np.int64)
    assert np.all(rows < hi[owner]), "slabs do not cover every lattice row"
    return owner


def exchange_samples(owner, dist, device=None):
    """``exchange`` callback of ``surrogate_device`` for strategy B: every rank wrote
    the samples of its own lattice rows into its device table; one all-gather of the owned columns
    (<= 2 MB at config 5) completes every rank's table.  NCCL moves device buffers over NVLink; a
    gloo group (CPU tests) goes through host copies."""
    owner = np.asarray(owner)

    def run(ptr, P, nlat):
        import torch

        rank = dist.get_rank()
        world = dist.get_world_size()
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        table = _device_view(ptr, (P, nlat), dev)
        cols = [np.flatnonzero(owner == k) for k in range(world)]
        width = max(1, max(c.size for c in cols))
        comm_dev = dev if dist.get_backend() == "nccl" else torch.device("cpu")
        mine = torch.zeros((P, width), dtype=torch.float64, device=dev)
        if cols[rank].size:
            mine[:, :cols[rank].size] = table[:, torch.as_tensor(cols[rank], device=dev)]
        mine = mine.to(comm_dev)
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine)
        for k in range(world):
            if k != rank and cols[k].size:
                table[:, torch.as_tensor(cols[k], device=dev)] = parts[k][:, :cols[k].size].to(dev)
        torch.cuda.synchronize(dev)

    return run


def _device_view(ptr, shape, dev):
    """A torch view of a float64 device array owned by the library (``__cuda_array_interface__``)."""
    import torch

    class _Arr:
        __cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f8", "data": (int(ptr), False), "version": 3,
                                    "strides": None}

    return torch.as_tensor(_Arr(), device=dev)
