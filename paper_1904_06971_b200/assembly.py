"""Drop-in ``assemble`` (reference: surriga/assembly.py:579-651) on the B200.

The host does what the reference does before its element loop -- argument validation with
the reference's messages, exact-rational knots and Gauss points (assembly.py:100-125) -- and
hands plain arrays to ``sg_assemble`` (include/surriga_b200.h).  Basis tables, geometry,
element quadrature and CSR emission all run on the GPU.  Both the reference's own
``FormKind``/``Discretization`` objects and this package's mirrors are accepted.
"""
from __future__ import annotations

import ctypes as C
import functools
import os
import weakref
from dataclasses import dataclass
from enum import Enum

import numpy as np
import scipy.sparse as sp

from . import _lib
from .geometry import GeometryMap, weights_for_space
from .spaces import NurbsWeights, TensorSpace, make_open_uniform_knots, make_tensor_space

__all__ = [
    "FormKind", "Discretization", "SparseMatrix", "gauss_rule", "make_discretization", "assemble", "assemble_device",
    "elements_for_rows", "is_bitwise_symmetric", "matrices_bitwise_equal", "form_is_symmetric", "set_device",
    "problem_arrays", "StokesSpaces", "stokes_subgrid_spaces", "assemble_divergence", "assemble_divergence_device",
    "assemble_load",
]


class FormKind(Enum):
    """assembly.py:51-58."""

    POISSON = "poisson"
    MASS = "mass"
    BIHARMONIC = "biharmonic"
    STOKES_VELOCITY = "stokes_velocity"
    STOKES_DIVERGENCE = "stokes_divergence"


_SYMMETRIC = {"poisson": True, "mass": True, "biharmonic": True, "stokes_velocity": True, "stokes_divergence": False}
_NATIVE_FORM = {"poisson": 0, "stokes_velocity": 0, "mass": 1, "biharmonic": 2}


def _fname(form) -> str:
    v = getattr(form, "value", form)
    if v not in _SYMMETRIC:
        raise ValueError(f"unsupported form {form!r}")
    return v


def form_is_symmetric(form) -> bool:
    return _SYMMETRIC[_fname(form)]


@dataclass(frozen=True)
class QuadratureRule:
    g: int
    nodes: np.ndarray
    weights: np.ndarray


def gauss_rule(g: int) -> QuadratureRule:
    """assembly.py:100-105 (numpy leggauss, same message)."""
    if g < 1:
        raise ValueError(f"need at least one quadrature point, got g={g}")
    x, w = np.polynomial.legendre.leggauss(g)
    return QuadratureRule(g=g, nodes=x, weights=w)


@functools.lru_cache(maxsize=64)
def _axis_1d(p: int, m: int, g: int):
    """One direction of assembly.py:108-117 (pure function of (p, m, g); read-only, cached)."""
    rule = gauss_rule(g)
    h = 1.0 / (m - p)
    offs = (rule.nodes + 1.0) * (0.5 * h)
    br = make_open_uniform_knots(p, m).span_breaks()[:-1]
    ax = np.ascontiguousarray((br[:, None] + offs[None, :]).ravel())
    pw = np.ascontiguousarray(rule.weights * (0.5 * h))
    ax.flags.writeable = False
    pw.flags.writeable = False
    return ax, pw


@functools.lru_cache(maxsize=64)
def _knots_1d(p: int, m: int) -> np.ndarray:
    kn = np.ascontiguousarray(make_open_uniform_knots(p, m).knots, dtype=np.float64)
    kn.flags.writeable = False
    return kn


_UNIT = {}


def _is_unit(w: np.ndarray) -> bool:
    """weights.is_unit (all equal), remembered per weights array (the O(N) scan is ~1 ms at config 5)."""
    hit = _UNIT.get(id(w))
    if hit is not None and hit[0]() is w:
        return hit[1]
    r = bool(np.all(w == w[0]))
    try:
        _UNIT[id(w)] = (weakref.ref(w), r)
    except TypeError:
        pass
    return r


def _quad_axes(kvs, g: int):
    """assembly.py:108-117: points break_k + (x+1) h/2, weights w h/2."""
    axes, pw = [], []
    for kv in kvs:
        a, w = _axis_1d(int(kv.p), int(kv.m), int(g))
        axes.append(a)
        pw.append(w)
    return axes, pw


@dataclass
class Discretization:
    """assembly.py:132-155."""

    geom: GeometryMap
    space: TensorSpace
    weights: NurbsWeights
    gauss: int

    @property
    def n(self) -> int:
        return self.space.n

    @property
    def p(self) -> int:
        return self.space.p

    @property
    def spans(self) -> tuple:
        return tuple(kv.spans for kv in self.space.kvs)

    @property
    def ndof(self) -> int:
        return self.space.N


def make_discretization(geom: GeometryMap, p: int, spans, gauss: int | None = None) -> Discretization:
    """assembly.py:158-176."""
    n = geom.n
    if np.isscalar(spans):
        spans = (int(spans),) * n
    spans = tuple(int(s) for s in spans)
    if len(spans) != n:
        raise ValueError(f"need {n} span counts, got {len(spans)}")
    space = make_tensor_space(p, [s + p for s in spans])
    w = weights_for_space(geom, space)
    g = int(gauss) if gauss is not None else p + 1
    if g < 1:
        raise ValueError("quadrature order must be positive")
    return Discretization(geom=geom, space=space, weights=w, gauss=g)


@dataclass
class SparseMatrix:
    """assembly.py:214-242: CSR (int32 indices, float64 data, sorted) + metadata."""

    mat: sp.csr_matrix
    symmetric: bool = False
    populated_rows: np.ndarray | None = None

    @property
    def shape(self) -> tuple:
        return self.mat.shape

    @property
    def nnz(self) -> int:
        return self.mat.nnz

    def toarray(self) -> np.ndarray:
        return self.mat.toarray()

    def row_sums(self) -> np.ndarray:
        return np.asarray(self.mat.sum(axis=1)).ravel()

    def max_abs(self) -> float:
        return float(np.max(np.abs(self.mat.data))) if self.mat.nnz else 0.0


def is_bitwise_symmetric(A) -> bool:
    M = A.mat.copy()
    M.sort_indices()
    T = A.mat.transpose().tocsr()
    T.sort_indices()
    return (np.array_equal(M.indptr, T.indptr) and np.array_equal(M.indices, T.indices)
            and np.array_equal(M.data.view(np.int64), T.data.view(np.int64)))


def matrices_bitwise_equal(A, B, rows=None) -> bool:
    MA, MB = A.mat, B.mat
    if rows is not None:
        rows = np.asarray(rows)
        MA, MB = MA[rows], MB[rows]
    MA = MA.tocsr().copy()
    MB = MB.tocsr().copy()
    MA.sort_indices()
    MB.sort_indices()
    return (np.array_equal(MA.indptr, MB.indptr) and np.array_equal(MA.indices, MB.indices)
            and np.array_equal(MA.data.view(np.int64), MB.data.view(np.int64)))


def elements_for_rows(disc, rows) -> np.ndarray:
    """Ascending colex ids of elements supporting ``rows`` (assembly.py:347-370); separable dilation."""
    return _elements_for_rows(tuple(kv.m for kv in disc.space.kvs), disc.space.kvs[0].p, rows)


def _elements_for_rows(ms, p, rows) -> np.ndarray:
    ms = tuple(ms)
    spans = tuple(m - p for m in ms)
    R = np.zeros(int(np.prod(ms)), dtype=bool)
    R[np.asarray(rows, dtype=np.int64).reshape(-1)] = True
    R = R.reshape(ms, order="F")
    for d in range(len(ms)):
        R = np.moveaxis(R, d, 0)
        acc = np.zeros((spans[d],) + R.shape[1:], dtype=bool)
        for r in range(p + 1):
            acc |= R[r:r + spans[d]]
        R = np.moveaxis(acc, 0, d)
    return np.flatnonzero(R.ravel(order="F"))


# ---------------------------------------------------------------------------------------
# device selection
# ---------------------------------------------------------------------------------------

_DEVICE = int(os.environ.get("SURRIGA_B200_DEVICE", os.environ.get("LOCAL_RANK", "0")))


def set_device(dev: int) -> None:
    global _DEVICE
    _DEVICE = int(dev)


# ---------------------------------------------------------------------------------------
# problem marshalling
# ---------------------------------------------------------------------------------------

class _Keep:
    """Keeps the numpy arrays referenced by a ctypes struct alive."""

    def __init__(self):
        self.arrays = []

    def ptr(self, a):
        a = np.ascontiguousarray(a, dtype=np.float64)
        self.arrays.append(a)
        return _lib.dptr(a)


def problem_arrays(form, disc, coefficient: float = 1.0):
    """Validate like assembly.py:596-607 and build the C ``sg_problem`` (+ keep-alive)."""
    fname = _fname(form)
    if fname == "stokes_divergence":
        raise ValueError("use assemble_divergence for the mixed pairing")
    space = disc.space
    p = int(space.kvs[0].p)
    if fname == "biharmonic" and p < 2:
        raise ValueError("the fourth-order form needs degree >= 2 for C^1 continuity")
    g = int(disc.gauss)
    axes, pw = _quad_axes(space.kvs, g)
    if coefficient != 1.0 and fname not in ("poisson", "stokes_velocity"):
        raise ValueError("coefficient is only supported for the second-order forms")
    n = len(space.kvs)
    keep = _Keep()
    pr = _lib.SgProblem()
    pr.n = n
    pr.p = p
    pr.form = _NATIVE_FORM[fname]
    pr.g = g
    for d, kv in enumerate(space.kvs):
        pr.m[d] = int(kv.m)
        pr.knots[d] = keep.ptr(_knots_1d(p, int(kv.m)))
        pr.qpts[d] = keep.ptr(axes[d])
        pr.qwts[d] = keep.ptr(pw[d])
    w = np.asarray(disc.weights.weights, dtype=float)
    pr.sol_w = None if _is_unit(w) else keep.ptr(w)     # weights.is_unit (assembly.py:418)
    gs = disc.geom.space
    pg = int(gs.kvs[0].p)
    pr.geo_p = pg
    for d, kv in enumerate(gs.kvs):
        pr.geo_m[d] = int(kv.m)
        pr.geo_knots[d] = keep.ptr(_knots_1d(pg, int(kv.m)))
    gw = np.asarray(disc.geom.weights.weights, dtype=float)
    hom = np.concatenate([np.asarray(disc.geom.control, float) * gw[:, None], gw[:, None]], axis=1)
    pr.geo_hom = keep.ptr(hom)
    pr.coefficient = float(coefficient)
    N = int(np.prod([kv.m for kv in space.kvs]))
    return pr, keep, fname, N


def _exec(device=None, stream=None, slab=None):
    ex = _lib.SgExec()
    ex.device = _DEVICE if device is None else int(device)
    ex.stream = stream
    if slab is not None:
        ex.slab_lo, ex.slab_hi = int(slab[0]), int(slab[1])
    else:
        ex.slab_lo, ex.slab_hi = 0, 0
    return ex


def assemble_device(form, disc, rows=None, coefficient: float = 1.0, *, device=None, stream=None, slab=None):
    """Assemble on the GPU and keep the CSR in HBM; returns ``(_lib.Result, symmetric, rows)``."""
    pr, keep, fname, N = problem_arrays(form, disc, coefficient)
    L = _lib.lib()
    rsel = None
    rptr, nr = None, 0
    if rows is not None:
        rsel = np.unique(np.asarray(rows, dtype=np.int64))
        if rsel.size and (rsel[0] < 0 or rsel[-1] >= N):
            raise ValueError("row index out of range")
        rptr, nr = rsel.ctypes.data_as(_lib._i64), rsel.size
    ex = _exec(device, stream, slab)
    h = C.c_void_p()
    _lib.check(L.sg_assemble(C.byref(pr), rptr, nr, C.byref(ex), C.byref(h)))
    del keep
    return _lib.Result(h.value), _SYMMETRIC[fname] and rows is None, rsel


def assemble(form, disc, rows=None, coefficient: float = 1.0) -> SparseMatrix:
    """Assemble a square Galerkin matrix, fully or for selected rows (assembly.py:579-651)."""
    res, sym, rsel = assemble_device(form, disc, rows=rows, coefficient=coefficient)
    indptr, indices, data = res.to_host()
    res.free()
    N = int(np.prod([kv.m for kv in disc.space.kvs]))
    mat = sp.csr_matrix((data, indices, indptr), shape=(N, N))
    mat.has_sorted_indices = True
    return SparseMatrix(mat=mat, symmetric=sym, populated_rows=None if rows is None else rsel)


# ---------------------------------------------------------------------------------------
# mixed divergence pairing (assembly.py:180-207, 654-725)
# ---------------------------------------------------------------------------------------

@dataclass
class StokesSpaces:
    """assembly.py:180-194: inf-sup stable velocity/pressure pair on nested meshes (velocity degree
    one higher, every pressure element halved)."""

    geom: GeometryMap
    velocity: Discretization
    pressure: Discretization

    @property
    def n(self) -> int:
        return self.geom.n


def stokes_subgrid_spaces(geom: GeometryMap, p_pressure: int, spans, gauss: int | None = None) -> StokesSpaces:
    """assembly.py:197-207; ``spans`` counts pressure elements."""
    if p_pressure < 1:
        raise ValueError("pressure degree must be at least 1")
    n = geom.n
    if np.isscalar(spans):
        spans = (int(spans),) * n
    spans = tuple(int(s) for s in spans)
    pressure = make_discretization(geom, p_pressure, spans)
    velocity = make_discretization(geom, p_pressure + 1, tuple(2 * s for s in spans), gauss=gauss)
    return StokesSpaces(geom=geom, velocity=velocity, pressure=pressure)


def assemble_divergence_device(stokes, rows=None, *, device=None, stream=None, slab=None):
    """Divergence pairing on the GPU, CSRs kept in HBM: ``([_lib.Result per component], rows)``.

    ``slab=(lo, hi)``: only pressure rows [lo, hi) (one GPU's share); the results hold
    those rows, which stitch bitwise into the full matrices (slabs.stitch)."""
    vel, prs = stokes.velocity, stokes.pressure
    n = len(vel.space.kvs)
    vpr, vkeep, _, _ = problem_arrays(FormKind.POISSON, vel)
    pspace = prs.space
    pp = int(pspace.kvs[0].p)
    pkeep = _Keep()
    ppr = _lib.SgProblem()
    ppr.n = n
    ppr.p = pp
    ppr.g = int(prs.gauss)
    for d, kv in enumerate(pspace.kvs):
        ppr.m[d] = int(kv.m)
        ppr.knots[d] = pkeep.ptr(make_open_uniform_knots(pp, int(kv.m)).knots)
    pw = np.asarray(prs.weights.weights, dtype=float)
    ppr.sol_w = None if bool(np.all(pw == pw[0])) else pkeep.ptr(pw)
    Np = int(np.prod([kv.m for kv in pspace.kvs]))
    rsel, rptr, nr = None, None, 0
    if rows is not None:
        rsel = np.unique(np.asarray(rows, dtype=np.int64))
        if rsel.size and (rsel[0] < 0 or rsel[-1] >= Np):
            raise ValueError("pressure row index out of range")
        rptr, nr = rsel.ctypes.data_as(_lib._i64), rsel.size
    ex = _exec(device, stream, slab)
    hs = (C.c_void_p * 3)()
    _lib.check(_lib.lib().sg_assemble_divergence(C.byref(vpr), C.byref(ppr), rptr, nr, C.byref(ex), hs))
    del vkeep, pkeep
    return [_lib.Result(hs[c]) for c in range(n)], rsel


def assemble_divergence(stokes, rows=None) -> list:
    """Pressure/velocity divergence pairing, one matrix per velocity component (assembly.py:654-725)."""
    res, rsel = assemble_divergence_device(stokes, rows=rows)
    Np = int(np.prod([kv.m for kv in stokes.pressure.space.kvs]))
    Nv = int(np.prod([kv.m for kv in stokes.velocity.space.kvs]))
    out = []
    for r in res:
        indptr, indices, data = r.to_host()
        r.free()
        mat = sp.csr_matrix((data, indices, indptr), shape=(Np, Nv))
        mat.has_sorted_indices = True
        out.append(SparseMatrix(mat=mat, symmetric=False, populated_rows=None if rows is None else rsel))
    return out


# ---------------------------------------------------------------------------------------
# load vector (assembly.py:728-759)
# ---------------------------------------------------------------------------------------

def assemble_load(disc, f, *, device=None, stream=None) -> np.ndarray:
    """Load vector of a callable ``f`` of physical coordinates (assembly.py:728-759).

    ``f`` receives the physical quadrature points per element, shape ``(E, Q, n)`` (elements and
    in-element points colex, as the reference passes them) and must return ``(E, Q)``.  The points
    come from the GPU (``sg_map_points``), ``f`` runs on the host, the quadrature sum runs on the GPU
    (``sg_assemble_load``).
    """
    pr, keep, _, N = problem_arrays(FormKind.MASS, disc)
    n = len(disc.space.kvs)
    g = int(disc.gauss)
    E = int(np.prod([kv.m - kv.p for kv in disc.space.kvs]))
    Q = g ** n
    ex = _exec(device, stream, None)
    phi = np.empty((E, Q, n))
    _lib.check(_lib.lib().sg_map_points(C.byref(pr), C.byref(ex), _lib.dptr(phi)))
    fb = np.ascontiguousarray(np.asarray(f(phi), dtype=float))
    if fb.shape != (E, Q):
        raise ValueError("load callable returned a mismatched shape")
    vec = np.empty(N)
    _lib.check(_lib.lib().sg_assemble_load(C.byref(pr), _lib.dptr(fb), C.byref(ex), _lib.dptr(vec)))
    del keep
    return vec


def quadrature_fields(disc, coefs, nu: int = 0, gauss: int | None = None, *, device=None, stream=None):
    """Physical samples of a coefficient field at the element quadrature points (assembly.py:839-907).

    Returns ``(x, w, vals, grads, hesses)``: physical points ``(T, n)``, quadrature weights times
    det J ``(T,)``, values ``(T,)``, physical gradients ``(T, n)`` (nu >= 1, else None) and physical
    Hessians ``(T, n, n)`` (nu >= 2, else None), element-major (``T = E * g**n``), all evaluated on
    the GPU (``sg_quadrature_fields``).
    """
    import dataclasses

    d = disc if gauss is None else dataclasses.replace(disc, gauss=int(gauss))
    pr, keep, _, N = problem_arrays(FormKind.MASS, d)
    n = len(d.space.kvs)
    coefs = np.ascontiguousarray(np.asarray(coefs, dtype=float).ravel())
    if coefs.size != N:
        raise ValueError("coefficient vector does not match the space")
    nu = int(nu)
    if nu not in (0, 1, 2):
        raise ValueError("nu must be 0, 1 or 2")
    E = int(np.prod([kv.m - kv.p for kv in d.space.kvs]))
    T = E * int(d.gauss) ** n
    x = np.empty((T, n))
    w = np.empty(T)
    vals = np.empty(T)
    grads = np.empty((T, n)) if nu >= 1 else None
    hesses = np.empty((T, n, n)) if nu >= 2 else None
    ex = _exec(device, stream, None)
    _lib.check(_lib.lib().sg_quadrature_fields(C.byref(pr), _lib.dptr(coefs), nu, C.byref(ex), _lib.dptr(x), _lib.dptr(w),
                                               _lib.dptr(vals), _lib.dptr(grads) if grads is not None else None,
                                               _lib.dptr(hesses) if hesses is not None else None))
    del keep
    return x, w, vals, grads, hesses


def save_matrix_market(path, A, *, ncols=None, symmetric=None, threads: int = 0) -> None:
    """Write ``A`` in MatrixMarket coordinate format (assembly.py:304-312).

    ``A`` is a ``SparseMatrix`` (host CSR) or a device ``_lib.Result`` (then ``symmetric`` and, for a
    rectangular matrix, ``ncols`` are given by the caller).  Symmetric matrices are tagged
    ``symmetric`` with the lower triangle stored, as the reference's mmwrite call does; values are
    written in the shortest form that reads back bit-exactly (the reference's 16 digits do not
    always).  Formatting runs on ``threads`` native threads (0: all cores).
    """
    L = _lib.lib()
    p = os.fspath(path).encode()
    if isinstance(A, _lib.Result):
        _lib.check(L.sg_write_matrix_market(A.h, int(ncols or 0), p, int(bool(symmetric)), int(threads)))
        return
    mat = A.mat.tocsr()
    mat.sort_indices()
    sym = A.symmetric if symmetric is None else bool(symmetric)
    ip = np.ascontiguousarray(mat.indptr, dtype=np.int64)
    ix = np.ascontiguousarray(mat.indices, dtype=np.int32)
    d = np.ascontiguousarray(mat.data, dtype=np.float64)
    _lib.check(L.sg_write_matrix_market_host(p, mat.shape[0], mat.shape[1], ip.ctypes.data_as(_lib._i64),
                                             ix.ctypes.data_as(_lib._i32), _lib.dptr(d), int(sym), int(threads)))


def load_matrix_market(path) -> "SparseMatrix":
    """Read a MatrixMarket file back into a ``SparseMatrix`` (assembly.py:315-320; host file IO)."""
    from scipy.io import mminfo, mmread

    info = mminfo(str(path))
    try:
        mat = mmread(str(path), spmatrix=True).tocsr()
    except TypeError:  # scipy without the spmatrix switch
        mat = mmread(str(path)).tocsr()
    mat.sort_indices()
    return SparseMatrix(mat=mat, symmetric=(info[5] == "symmetric"))
