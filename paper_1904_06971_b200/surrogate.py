"""Drop-in ``build_surrogate_matrix`` (reference: surriga/surrogate.py:538-691) on the B200.

The host keeps the reference's exact-rational bookkeeping (offsets, interior box, sampling
lattice, midpoints, averaged knots; surrogate.py:61-288,386-390), the argument validation and
the ``AssemblyReport``; the quadrature rows, stencil sampling, coefficient solve, interpolant
evaluation, placement, kernel-preserving diagonal and the CSR merge run on the GPU
(``sg_surrogate``, csrc/sg_surrogate.cu).  The only host linear algebra is the inverse of the
per-direction collocation matrix (at most a few dozen lattice sites), computed once per call.
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field
from enum import Enum
from fractions import Fraction

import numpy as np
import scipy.sparse as sp

from . import _lib
from .assembly import (
    FormKind,
    SparseMatrix,
    _elements_for_rows,
    _exec,
    _fname,
    _Keep as _AKeep,
    assemble,
    assemble_divergence,
    form_is_symmetric,
    problem_arrays,
)
from .spaces import make_open_uniform_knots
from .spaces import collocation_matrix

__all__ = [
    "build_surrogate_divergence",
    "SurrogateMode", "DEFAULT_MODE", "OffsetSet", "build_offsets", "TildeDomain", "tilde_domain", "SamplingLattice",
    "build_sampling_lattice", "ConstantSampling", "MeshDependentSampling", "mesh_dependent_M", "AssemblyReport",
    "REPORT_CSV_HEADER", "build_surrogate_matrix", "surrogate_plan", "SurrogatePlan",
]


class SurrogateMode(Enum):
    """surrogate.py:36-41."""

    GENERAL = "general"
    SYMMETRIC = "symmetric"
    SYMMETRIC_KERNEL_PRESERVING = "symmetric_kernel_preserving"


_KERNEL_PRESERVING_FORMS = ("poisson", "biharmonic")
DEFAULT_MODE = {
    "poisson": SurrogateMode.SYMMETRIC_KERNEL_PRESERVING,
    "biharmonic": SurrogateMode.SYMMETRIC_KERNEL_PRESERVING,
    "mass": SurrogateMode.SYMMETRIC,
    "stokes_velocity": SurrogateMode.SYMMETRIC,
    "stokes_divergence": SurrogateMode.GENERAL,
}
_NATIVE_MODE = {"general": 0, "symmetric": 1, "symmetric_kernel_preserving": 2}


@dataclass(frozen=True)
class OffsetSet:
    """Offsets [-p, p]^n in colex order (surrogate.py:61-100)."""

    p: int
    n: int
    shifts: np.ndarray
    mixed: bool = False

    @property
    def count(self) -> int:
        return self.shifts.shape[0]

    @property
    def center(self) -> int:
        if self.mixed:
            raise ValueError("mixed offset sets have no zero offset")
        return (self.count - 1) // 2

    def canonical_half(self) -> np.ndarray:
        if self.mixed:
            raise ValueError("the mixed offset set is not closed under negation")
        return np.arange(self.center, self.count)

    def negated_position(self, pos: int) -> int:
        if self.mixed:
            raise ValueError("the mixed offset set is not closed under negation")
        return self.count - 1 - pos


def build_offsets(p: int, n: int, mixed: bool = False) -> OffsetSet:
    """surrogate.py:103-122."""
    if p < 1:
        raise ValueError("degree must be at least 1")
    if n not in (1, 2, 3):
        raise ValueError("supported dimensions: 1, 2, 3")
    rng = np.arange(-2 * p, p + 3, dtype=np.int64) if mixed else np.arange(-p, p + 1, dtype=np.int64)
    k = rng.size
    grid = np.unravel_index(np.arange(k ** n), (k,) * n, order="F")
    return OffsetSet(p=p, n=n, shifts=np.stack([rng[g] for g in grid], axis=-1), mixed=mixed)


@dataclass(frozen=True)
class TildeDomain:
    """Interior box: in-box 0-based indices [2p, m-2p-1] (surrogate.py:129-179)."""

    p: int
    ms: tuple
    bounds: tuple

    @property
    def n(self) -> int:
        return len(self.ms)

    @property
    def is_empty(self) -> bool:
        return any(lo > hi for lo, hi in self.bounds)

    def index_range(self, d: int) -> tuple:
        return (2 * self.p, self.ms[d] - 2 * self.p - 1)

    def index_count(self, d: int) -> int:
        lo, hi = self.index_range(d)
        return max(0, hi - lo + 1)

    def contains_index(self, multi0) -> bool:
        multi0 = np.atleast_1d(np.asarray(multi0))
        return all(self.index_range(d)[0] <= int(multi0[d]) <= self.index_range(d)[1] for d in range(self.n))

    def offset_domain(self, shift) -> tuple:
        out = []
        for d in range(self.n):
            h = Fraction(1, self.ms[d] - self.p)
            lo0 = Fraction(self.p + 1, 2) * h
            hi0 = 1 - lo0
            s = int(shift[d]) * h
            out.append((max(lo0, lo0 - s), min(hi0, hi0 - s)))
        return tuple(out)


def tilde_domain(p: int, ms) -> TildeDomain:
    """surrogate.py:182-191."""
    if np.isscalar(ms):
        ms = (int(ms),)
    ms = tuple(int(m) for m in ms)
    bounds = []
    for m in ms:
        lo = Fraction(3 * p + 1, 2 * (m - p))
        bounds.append((lo, 1 - lo))
    return TildeDomain(p=p, ms=ms, bounds=tuple(bounds))


@dataclass(frozen=True)
class SamplingLattice:
    """surrogate.py:198-228."""

    M: int
    indices: tuple
    sites: tuple
    h: float

    @property
    def n(self) -> int:
        return len(self.indices)

    @property
    def H(self) -> float:
        return self.M * self.h

    @property
    def shape(self) -> tuple:
        return tuple(ix.size for ix in self.indices)

    @property
    def count(self) -> int:
        return int(np.prod(self.shape))

    def indices_one_based(self, d: int) -> np.ndarray:
        return self.indices[d] + 1


def _midpoints(kv, idx0) -> np.ndarray:
    """((2i+1-p)/2) h, exact then rounded (surrogate.py:231-233)."""
    h = Fraction(1, kv.m - kv.p)
    return np.array([float(Fraction(2 * int(i) + 1 - kv.p, 2) * h) for i in idx0])


def build_sampling_lattice(kvs, M: int, tilde: TildeDomain | None = None) -> SamplingLattice:
    """surrogate.py:236-253."""
    if M < 1:
        raise ValueError("sampling parameter M must be at least 1")
    p = kvs[0].p
    if tilde is None:
        tilde = tilde_domain(p, tuple(kv.m for kv in kvs))
    if tilde.is_empty:
        raise ValueError("interior sampling box is empty; no lattice exists")
    indices, sites = [], []
    for d, kv in enumerate(kvs):
        lo, hi = tilde.index_range(d)
        idx = np.arange(lo, hi + 1, M, dtype=np.int64)
        if idx[-1] != hi:
            idx = np.append(idx, hi)
        indices.append(idx)
        sites.append(_midpoints(kv, idx))
    return SamplingLattice(M=M, indices=tuple(indices), sites=tuple(sites), h=1.0 / (kvs[0].m - kvs[0].p))


@dataclass(frozen=True)
class ConstantSampling:
    M: int


@dataclass(frozen=True)
class MeshDependentSampling:
    c: float
    beta: float = 0.5


def mesh_dependent_M(strategy, h: float, p: int, q: int) -> int:
    """surrogate.py:275-288 (same exceptions)."""
    if isinstance(strategy, ConstantSampling) or type(strategy).__name__ == "ConstantSampling":
        if strategy.M < 1:
            raise ValueError("sampling parameter M must be at least 1")
        return int(strategy.M)
    if isinstance(strategy, MeshDependentSampling) or type(strategy).__name__ == "MeshDependentSampling":
        if strategy.c < 0 or strategy.beta < 0:
            raise ValueError("strategy constants must be nonnegative")
        if q <= p:
            raise ValueError("mesh-dependent sampling requires q > p")
        expo = (p - q + strategy.beta) / (q + 1)
        return max(1, int(np.floor(strategy.c * h ** expo)))
    raise TypeError(f"unknown sampling strategy {strategy!r}")


REPORT_CSV_HEADER = "N,p,q,M,H,quad_entries,interp_entries,quad_fraction,active_elements,assembly_seconds"


@dataclass
class AssemblyReport:
    """surrogate.py:481-502."""

    N: int
    p: int
    q: int
    M: int
    H: float
    quad_entries: int
    interp_entries: int
    quad_fraction: float
    active_elements: int
    assembly_seconds: float
    flags: list = field(default_factory=list)

    def csv_row(self) -> str:
        return (f"{self.N},{self.p},{self.q},{self.M},{self.H!r},{self.quad_entries},{self.interp_entries},"
                f"{self.quad_fraction!r},{self.active_elements},{self.assembly_seconds!r}")


def _averaging_knots(sites: np.ndarray, q: int) -> np.ndarray:
    """surrogate.py:386-390."""
    k = sites.size
    interior = [np.mean(sites[j + 1:j + q + 1]) for j in range(k - q - 1)]
    return np.concatenate([np.full(q + 1, sites[0]), interior, np.full(q + 1, sites[-1])])


def _masks(tilde: TildeDomain, lattice: SamplingLattice):
    inb, smp = [], []
    for d in range(tilde.n):
        m = tilde.ms[d]
        lo, hi = tilde.index_range(d)
        a = np.zeros(m, dtype=bool)
        a[lo:hi + 1] = True
        s = np.zeros(m, dtype=bool)
        s[lattice.indices[d]] = True
        inb.append(a)
        smp.append(s)
    return inb, smp


def _flat(masks) -> np.ndarray:
    acc = np.ones(1, dtype=bool)
    for mk in masks[::-1]:
        acc = (acc[:, None] & mk[None, :]).ravel()
    return acc


def _active_element_count(ms, p, tilde: TildeDomain, lattice: SamplingLattice) -> int:
    """Number of elements supporting a quadrature row, ``_elements_for_rows(quad_rows).size``
    (surrogate.py:590, assembly.py:347-360), without the O(N) row mask.

    Element e supports the rows e..e+p per direction, so it touches no quadrature row iff every
    such row is interpolated: the row box [e, e+p]^n lies inside the tilde box and holds no fully
    sampled row, i.e. not every direction has a lattice index in [e_d, e_d+p].  Both conditions
    factor per direction: inactive = prod_d A_d - prod_d B_d with A_d = #{e_d : [e_d, e_d+p] in the
    box} and B_d = #{those e_d whose window also holds a lattice index}."""
    A = B = 1
    for d, m in enumerate(ms):
        lo, hi = tilde.index_range(d)
        e = np.arange(m - p)
        inside = (e >= lo) & (e + p <= hi)
        lat = np.asarray(lattice.indices[d], dtype=np.int64)
        first = np.searchsorted(lat, e, side="left")
        has = (first < lat.size) & (lat[np.minimum(first, lat.size - 1)] <= e + p)
        A *= int(inside.sum())
        B *= int((inside & has).sum())
    total = int(np.prod([m - p for m in ms]))
    return total - (A - B)


def _pattern_nnz(ms, p) -> int:
    tot = 1
    for m in ms:
        k = np.arange(m)
        tot *= int(np.sum(np.minimum(m - 1, k + p) - np.maximum(0, k - p) + 1))
    return tot


class _Keep:
    def __init__(self):
        self.a = []

    def d(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        self.a.append(x)
        return _lib.dptr(x)

    def i64(self, x):
        x = np.ascontiguousarray(x, dtype=np.int64)
        self.a.append(x)
        return x.ctypes.data_as(_lib._i64)


_FIT_CACHE: dict = {}


def _fit_params(disc, lattice: SamplingLattice, tilde: TildeDomain, q: int, mode_name: str, M: int):
    """Host-side interpolation setup: per-direction degree (lowered if needed), averaged knots,
    inverse collocation matrix at the lattice sites, in-box midpoints (surrogate.py:430-471, 612).

    The arrays depend only on the knot vectors, the lattice and q, so they are built once per such
    key (exact-rational midpoints and collocation inverses cost ~2 ms a call) and reused; the mode
    is set on a copy of the cached parameter block."""
    key = (tuple((int(kv.p), int(kv.m)) for kv in disc.space.kvs), int(M), int(q),
           tuple(tuple(int(i) for i in ix) for ix in lattice.indices),
           tuple(tuple(float(x) for x in st) for st in lattice.sites),
           tuple(tilde.index_range(d) for d in range(len(disc.space.kvs))))
    hit = _FIT_CACHE.get(key)
    if hit is None:
        hit = _fit_params_build(disc, lattice, tilde, q, M)
        if len(_FIT_CACHE) > 16:
            _FIT_CACHE.clear()
        _FIT_CACHE[key] = hit
    base, keep, lowered = hit
    spp = type(base).from_buffer_copy(base)
    spp.mode = _NATIVE_MODE[mode_name]
    return spp, keep, lowered


def _fit_params_build(disc, lattice: SamplingLattice, tilde: TildeDomain, q: int, M: int):
    keep = _Keep()
    spp = _lib.SgSurrogateParams()
    spp.M = int(M)
    spp.q = int(q)
    lowered = False
    for d, kv in enumerate(disc.space.kvs):
        sites = lattice.sites[d]
        qd = min(q, sites.size - 1)
        lowered = lowered or qd < q
        spp.nlat[d] = sites.size
        spp.lat_idx[d] = keep.i64(lattice.indices[d])
        spp.qd[d] = qd
        lo, hi = tilde.index_range(d)
        spp.box_pts[d] = keep.d(_midpoints(kv, np.arange(lo, hi + 1)))
        if qd >= 1:
            kn = _averaging_knots(sites, qd)
            E = collocation_matrix(kn, qd, sites)
            spp.interp_knots[d] = keep.d(kn)
            spp.colloc_inv[d] = keep.d(np.linalg.inv(E))
        else:
            spp.interp_knots[d] = None
            spp.colloc_inv[d] = keep.d(np.ones((1, 1)))
    return spp, keep, lowered


def surrogate_device(form, disc, M: int, q: int, mode_name: str, coefficient=1.0, *, device=None, stream=None,
                     slab=None, lattice=None, tilde=None, exchange=None):
    """Run the native surrogate; returns (Result, stats, lowered).

    ``exchange`` (row slabs on several devices): a callable ``exchange(ptr, P, nlat)``
    that completes the device sample table ``S[o][lattice colex]`` at ``ptr`` (float64, P x nlat)
    with the lattice rows of the other slabs (``slabs.exchange_samples``: an all-gather over the
    process group) and synchronises.  Without it, a slab call assembles the other slabs' lattice
    rows itself (row-restricted quadrature, bitwise the same rows)."""
    pr, keep, fname, N = problem_arrays(form, disc, coefficient)
    space = disc.space
    if tilde is None:
        tilde = tilde_domain(space.kvs[0].p, tuple(kv.m for kv in space.kvs))
    if lattice is None:
        lattice = build_sampling_lattice(space.kvs, M, tilde)
    spp, keep2, lowered = _fit_params(disc, lattice, tilde, q, mode_name, M)
    ex = _exec(device, stream, slab)
    h = C.c_void_p()
    st = _lib.SgSurrogateStats()
    L = _lib.lib()
    if exchange is None:
        _lib.check(L.sg_surrogate(C.byref(pr), C.byref(spp), C.byref(ex), C.byref(h), C.byref(st)))
    else:
        state = C.c_void_p()
        table = C.c_void_p()
        nlat = C.c_int64()
        _lib.check(L.sg_surrogate_begin(C.byref(pr), C.byref(spp), C.byref(ex), C.byref(state), C.byref(table),
                                        C.byref(nlat)))
        try:
            P = (2 * int(space.kvs[0].p) + 1) ** space.n
            exchange(int(table.value), P, int(nlat.value))
        except BaseException:
            L.sg_surrogate_state_free(state)
            raise
        _lib.check(L.sg_surrogate_finish(state, C.byref(spp), C.byref(h), C.byref(st)))
    del keep, keep2
    return _lib.Result(h.value), st, lowered


def build_surrogate_matrix(form, disc, strategy=None, q: int = 3, mode=None, coefficient: float = 1.0):
    """Assemble a square form's matrix with interpolated interior entries (surrogate.py:538-691)."""
    fname = _fname(form)
    if fname == "stokes_divergence":
        raise ValueError("use build_surrogate_divergence for the mixed pairing")
    mode = DEFAULT_MODE[fname] if mode is None else mode
    mode_name = getattr(mode, "value", mode)
    if mode_name == "symmetric_kernel_preserving" and fname not in _KERNEL_PRESERVING_FORMS:
        raise ValueError(f"kernel-preserving mode is not defined for {fname}")
    if strategy is None:
        strategy = ConstantSampling(1)
    t0 = time.perf_counter()
    space = disc.space
    n, p = space.n, space.kvs[0].p
    ms = tuple(kv.m for kv in space.kvs)
    h = 1.0 / (space.kvs[0].m - space.kvs[0].p)
    tilde = tilde_domain(p, ms)
    M = mesh_dependent_M(strategy, h, p, q)
    N = int(np.prod(ms))
    spans = tuple(m - p for m in ms)
    if tilde.is_empty:
        A = assemble(form, disc, coefficient=coefficient)
        dt = time.perf_counter() - t0
        return A, AssemblyReport(N=N, p=p, q=q, M=M, H=M * h, quad_entries=A.nnz, interp_entries=0,
                                 quad_fraction=1.0, active_elements=int(np.prod(spans)), assembly_seconds=dt,
                                 flags=["surrogate=disabled"])
    lattice = build_sampling_lattice(space.kvs, M, tilde)
    # interpolated rows = box minus the lattice's tensor product: counted per direction
    nI = int(np.prod([tilde.index_range(d)[1] - tilde.index_range(d)[0] + 1 for d in range(n)])) - \
        int(np.prod([len(ix) for ix in lattice.indices]))
    active = _active_element_count(ms, p, tilde, lattice)
    if nI == 0:
        A = assemble(form, disc, coefficient=coefficient)  # every row is a quadrature row
        dt = time.perf_counter() - t0
        mat = SparseMatrix(mat=A.mat, symmetric=form_is_symmetric(form), populated_rows=None)
        return mat, AssemblyReport(N=N, p=p, q=q, M=M, H=lattice.H, quad_entries=A.nnz, interp_entries=0,
                                   quad_fraction=1.0, active_elements=active, assembly_seconds=dt, flags=[])
    res, st, lowered = surrogate_device(form, disc, M, q, mode_name, coefficient, lattice=lattice, tilde=tilde)
    indptr, indices, data = res.to_host()
    res.free()
    mat = sp.csr_matrix((data, indices, indptr), shape=(N, N))
    mat.has_sorted_indices = True
    dt = time.perf_counter() - t0
    n_interp = int(st.n_interp_entries)
    quad_entries = _pattern_nnz(ms, p) - n_interp
    flags = ["interpolation-order-lowered"] if lowered else []
    rep = AssemblyReport(N=N, p=p, q=q, M=M, H=lattice.H, quad_entries=int(quad_entries), interp_entries=n_interp,
                         quad_fraction=quad_entries / (quad_entries + n_interp), active_elements=int(active),
                         assembly_seconds=dt, flags=flags)
    sym = mode_name in ("symmetric", "symmetric_kernel_preserving")
    return SparseMatrix(mat=mat, symmetric=sym), rep


@dataclass
class SurrogatePlan:
    """surrogate.py:826-852."""

    N: int
    M: int
    H: float
    quad_rows: int
    interp_rows: int
    quad_entries: int
    interp_entries: int
    active_elements: int
    total_elements: int
    gauss_points_surrogate: int
    gauss_points_full: int

    @property
    def quad_fraction(self) -> float:
        return self.quad_entries / (self.quad_entries + self.interp_entries)

    @property
    def point_fraction(self) -> float:
        return self.gauss_points_surrogate / self.gauss_points_full


def _band_pairs(x, y, p) -> int:
    lo = np.searchsorted(y, x - p, side="left")
    hi = np.searchsorted(y, x + p, side="right")
    return int((hi - lo).sum())


def surrogate_plan(disc, strategy=None, q: int = 3) -> SurrogatePlan:
    """Exact work split without assembling (surrogate.py:862-913); also the slab cost model."""
    if strategy is None:
        strategy = ConstantSampling(1)
    space = disc.space
    n, p = space.n, space.kvs[0].p
    g = disc.gauss
    ms = tuple(kv.m for kv in space.kvs)
    total = int(np.prod([m - p for m in ms]))
    total_entries = 1
    for m in ms:
        total_entries *= _band_pairs(np.arange(m), np.arange(m), p)
    tilde = tilde_domain(p, ms)
    h = 1.0 / (ms[0] - p)
    M = mesh_dependent_M(strategy, h, p, q)
    N = int(np.prod(ms))
    if tilde.is_empty:
        return SurrogatePlan(N=N, M=M, H=M * h, quad_rows=N, interp_rows=0, quad_entries=total_entries,
                             interp_entries=0, active_elements=total, total_elements=total,
                             gauss_points_surrogate=total * g ** n, gauss_points_full=total * g ** n)
    lattice = build_sampling_lattice(space.kvs, M, tilde)
    bb = bl = lb = ll = 1
    for d in range(n):
        lo, hi = tilde.index_range(d)
        box = np.arange(lo, hi + 1)
        lat = np.asarray(lattice.indices[d])
        bb *= _band_pairs(box, box, p)
        bl *= _band_pairs(box, lat, p)
        lb *= _band_pairs(lat, box, p)
        ll *= _band_pairs(lat, lat, p)
    interp_entries = bb - bl - lb + ll
    n_interp = int(np.prod([tilde.index_count(d) for d in range(n)])) - int(np.prod([len(ix) for ix in lattice.indices]))
    active = _active_element_count(ms, p, tilde, lattice)
    return SurrogatePlan(N=N, M=M, H=lattice.H, quad_rows=N - n_interp, interp_rows=n_interp,
                         quad_entries=int(total_entries - interp_entries), interp_entries=int(interp_entries),
                         active_elements=int(active), total_elements=total,
                         gauss_points_surrogate=int(active) * g ** n, gauss_points_full=total * g ** n)


# ---------------------------------------------------------------------------------------
# surrogate divergence pairing (surrogate.py:699-819)
# ---------------------------------------------------------------------------------------

def _div_elements_for_rows(mp, pp, sv, rows) -> int:
    """Count of velocity elements supporting the pressure rows (assembly.py:347-360, ratio 2)."""
    n = len(mp)
    sp_ = tuple(m - pp for m in mp)
    mask = np.zeros(tuple(sv), dtype=bool)
    multi = np.stack(np.unravel_index(np.asarray(rows, dtype=np.int64), tuple(mp), order="F"), axis=-1)
    lo = 2 * np.maximum(0, multi - pp)
    hi = 2 * (np.minimum(np.asarray(sp_) - 1, multi) + 1)
    for a, b in zip(lo, hi):
        mask[tuple(slice(int(a[d]), int(b[d])) for d in range(n))] = True
    return int(mask.sum())


def build_surrogate_divergence(stokes, strategy=None, q: int = 3, mode=None):
    """Surrogate assembly of the divergence pairing, one matrix per component (surrogate.py:702-819).

    Only the general placement applies (the matrix is rectangular); a pressure row is interpolated
    when it lies in the pressure box shrunk by one index and is not on the sampling lattice.
    Returns ``(list of SparseMatrix, AssemblyReport)``.
    """
    mode = SurrogateMode.GENERAL if mode is None else mode
    if getattr(mode, "value", mode) != "general":
        raise ValueError("the divergence pairing only supports the general mode")
    if strategy is None:
        strategy = ConstantSampling(1)
    t0 = time.perf_counter()
    prs, vel = stokes.pressure, stokes.velocity
    n = stokes.n
    pp = int(prs.space.kvs[0].p)
    mp = tuple(int(kv.m) for kv in prs.space.kvs)
    sv = tuple(int(kv.m - kv.p) for kv in vel.space.kvs)
    h = 1.0 / (mp[0] - pp)
    tilde = tilde_domain(pp, mp)
    M = mesh_dependent_M(strategy, h, pp, q)
    Np = int(np.prod(mp))

    if tilde.is_empty:
        D = assemble_divergence(stokes)
        dt = time.perf_counter() - t0
        nnz = sum(Dc.nnz for Dc in D)
        return D, AssemblyReport(N=Np, p=pp, q=q, M=M, H=M * h, quad_entries=nnz, interp_entries=0,
                                 quad_fraction=1.0, active_elements=int(np.prod(sv)), assembly_seconds=dt,
                                 flags=["surrogate=disabled"])
    lattice = build_sampling_lattice(prs.space.kvs, M, tilde)
    inb, smp = _masks(tilde, lattice)
    core = []
    for d in range(n):
        lo, hi = tilde.index_range(d)
        a = np.zeros(mp[d], dtype=bool)
        if lo + 1 <= hi - 1:
            a[lo + 1:hi] = True
        core.append(a)
    core_flat, samp_flat = _flat(core), _flat(smp)
    quad_rows = np.flatnonzero(~core_flat | samp_flat)
    nI = Np - quad_rows.size
    active = _div_elements_for_rows(mp, pp, sv, quad_rows)
    if nI == 0:
        Dq = assemble_divergence(stokes, rows=quad_rows)
        dt = time.perf_counter() - t0
        nnz = sum(Dc.nnz for Dc in Dq)
        return ([SparseMatrix(mat=Dc.mat, symmetric=False) for Dc in Dq],
                AssemblyReport(N=Np, p=pp, q=q, M=M, H=lattice.H, quad_entries=nnz, interp_entries=0,
                               quad_fraction=1.0, active_elements=active, assembly_seconds=dt, flags=[]))
    hs, st, lowered = _surrogate_divergence_call(stokes, lattice, tilde, q, M, quad_rows)
    Nv = int(np.prod([kv.m for kv in vel.space.kvs]))
    out = []
    quad_entries = 0
    for c in range(n):
        r = _lib.Result(hs[c])
        indptr, indices, data = r.to_host()
        r.free()
        mat = sp.csr_matrix((data, indices, indptr), shape=(Np, Nv))
        mat.has_sorted_indices = True
        out.append(SparseMatrix(mat=mat, symmetric=False))
    # quadrature entries = the restricted assembly's pattern size per component (explicit zeros included)
    quad_entries = n * int(_div_pattern_rows_nnz(mp, tuple(int(kv.m) for kv in vel.space.kvs), pp, quad_rows))
    n_interp = int(st.n_interp_entries)
    dt = time.perf_counter() - t0
    flags = ["interpolation-order-lowered"] if lowered else []
    rep = AssemblyReport(N=Np, p=pp, q=q, M=M, H=lattice.H, quad_entries=quad_entries, interp_entries=n_interp,
                         quad_fraction=quad_entries / (quad_entries + n_interp), active_elements=int(active),
                         assembly_seconds=dt, flags=flags)
    return out, rep


def _div_pattern_rows_nnz(mp, mv, pp, rows) -> int:
    multi = np.stack(np.unravel_index(np.asarray(rows, dtype=np.int64), tuple(mp), order="F"), axis=-1)
    lo = np.maximum(2 * multi - 2 * pp, 0)
    hi = np.minimum(2 * multi + pp + 2, np.asarray(mv) - 1)
    return int(np.prod(hi - lo + 1, axis=1).sum())


def _surrogate_divergence_call(stokes, lattice, tilde, q, M, quad_rows, slab=None):
    """The native surrogate divergence call: ``(handles[n], stats, lowered)``."""
    prs, vel = stokes.pressure, stokes.velocity
    n = stokes.n
    pp = int(prs.space.kvs[0].p)
    vpr, vkeep, _, _ = problem_arrays(FormKind.POISSON, vel)
    pkeep = _AKeep()
    ppr = _lib.SgProblem()
    ppr.n = n
    ppr.p = pp
    ppr.g = int(prs.gauss)
    for d, kv in enumerate(prs.space.kvs):
        ppr.m[d] = int(kv.m)
        ppr.knots[d] = pkeep.ptr(make_open_uniform_knots(pp, int(kv.m)).knots)
    pw = np.asarray(prs.weights.weights, dtype=float)
    ppr.sol_w = None if bool(np.all(pw == pw[0])) else pkeep.ptr(pw)
    spp, fkeep, lowered = _fit_params(prs, lattice, tilde, q, "general", M)
    offs = build_offsets(pp, n, mixed=True)
    shifts = np.ascontiguousarray(offs.shifts, dtype=np.int32)
    qr = np.ascontiguousarray(quad_rows, dtype=np.int64)
    hs = (C.c_void_p * 3)()
    st = _lib.SgSurrogateStats()
    ex = _exec(None, None, slab)
    _lib.check(_lib.lib().sg_surrogate_divergence(C.byref(vpr), C.byref(ppr), C.byref(spp),
                                                  shifts.ctypes.data_as(C.POINTER(C.c_int32)),
                                                  qr.ctypes.data_as(_lib._i64), qr.size, C.byref(ex), hs, C.byref(st)))
    del vkeep, pkeep, fkeep
    return hs, st, lowered


def surrogate_divergence_device(stokes, strategy=None, q: int = 3, *, slab=None):
    """Device-resident surrogate divergence pairing (general mode), optionally on a pressure-row slab
    ``(lo, hi)`` (one GPU's share: the slab's quadrature rows plus every lattice row are
    assembled, only the slab's rows interpolated): ``[_lib.Result per component]``.  Needs an active
    surrogate (a non-empty pressure box with interpolated rows)."""
    if strategy is None:
        strategy = ConstantSampling(1)
    prs = stokes.pressure
    n = stokes.n
    pp = int(prs.space.kvs[0].p)
    mp = tuple(int(kv.m) for kv in prs.space.kvs)
    tilde = tilde_domain(pp, mp)
    if tilde.is_empty:
        raise ValueError("the surrogate is disabled for this mesh (empty pressure box)")
    M = mesh_dependent_M(strategy, 1.0 / (mp[0] - pp), pp, q)
    lattice = build_sampling_lattice(prs.space.kvs, M, tilde)
    _, smp = _masks(tilde, lattice)
    core = []
    for d in range(n):
        lo, hi = tilde.index_range(d)
        a = np.zeros(mp[d], dtype=bool)
        if lo + 1 <= hi - 1:
            a[lo + 1:hi] = True
        core.append(a)
    quad_rows = np.flatnonzero(~_flat(core) | _flat(smp))
    hs, _, _ = _surrogate_divergence_call(stokes, lattice, tilde, q, M, quad_rows, slab)
    return [_lib.Result(hs[c]) for c in range(n)]
