"""Host-side geometry maps (setup only): NURBS control nets, builtin domains, geometry files.

Same names, fields and validation as the reference's ``surriga.geometry``
(geometry.py:139-555).  The per-quadrature-point map, Jacobian, adjugate, determinant and
Hessian used by the assembly are evaluated on the GPU inside the assembly kernel
(csrc/sg_assemble.cuh); this module only builds control nets, validates them on a coarse
21^n grid (as the reference does) and reads/writes the ``iga-geo v1`` text format.
"""
from __future__ import annotations

import re
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

from .spaces import (
    NurbsWeights,
    TensorSpace,
    basis_table,
    make_open_uniform_knots,
    make_tensor_space,
    tensor_collocate,
)

__all__ = [
    "GeometryMap", "map_grid", "unit_square", "unit_cube", "quarter_annulus", "coons_2d", "trivariate_polynomial_3d",
    "builtin_domain", "BUILTIN_NAMES", "weights_for_space", "save_geometry", "load_geometry", "twisted_cube_standin",
    "sin_map_standin",
]


def _grid_field(space: TensorSpace, coef: np.ndarray, axes, alpha) -> np.ndarray:
    """Tensor field derivative ``alpha`` on a point grid; coef (N, C) colex -> (G..., C)."""
    t = np.asarray(coef, float).reshape(space.shape + (-1,), order="F")
    for d, kv in enumerate(space.kvs):
        span, tab = basis_table(kv.knots, kv.p, axes[d], max(alpha))
        idx = span[:, None] - kv.p + np.arange(kv.p + 1)[None, :]
        t = np.moveaxis(t, d, 0)
        t = np.einsum("xr,xr...->x...", tab[:, alpha[d], :], t[idx])
        t = np.moveaxis(t, 0, d)
    return t


def map_grid(geom, axes, max_deriv: int = 1) -> dict:
    """Map value and Jacobian on a tensor grid (geometry.py:185-229): dict(phi, W, jac, det)."""
    n = geom.space.n
    axes = tuple(np.asarray(a, float).ravel() for a in axes)
    w = geom.weights.weights
    hom = np.concatenate([geom.control * w[:, None], w[:, None]], axis=1)
    num = _grid_field(geom.space, hom, axes, (0,) * n)
    W = num[..., n]
    phi = num[..., :n] / W[..., None]
    out = {"phi": phi, "W": W}
    if max_deriv >= 1:
        jac = np.empty(W.shape + (n, n))
        for a in range(n):
            dn = _grid_field(geom.space, hom, axes, tuple(1 if d == a else 0 for d in range(n)))
            jac[..., :, a] = (dn[..., :n] - phi * dn[..., n, None]) / W[..., None]
        out["jac"] = jac
        if n == 1:
            out["det"] = jac[..., 0, 0]
        elif n == 2:
            out["det"] = jac[..., 0, 0] * jac[..., 1, 1] - jac[..., 0, 1] * jac[..., 1, 0]
        else:
            out["det"] = np.linalg.det(jac)
    return out


@dataclass
class GeometryMap:
    """Single-patch NURBS map (geometry.py:139-182); validates det J > 0 on a 21^n grid."""

    space: TensorSpace
    weights: NurbsWeights
    control: np.ndarray
    name: str = ""
    is_affine: bool = field(init=False, default=False)
    is_polynomial: bool = field(init=False, default=False)

    def __post_init__(self):
        C = np.asarray(self.control, dtype=float)
        if C.shape != (self.space.N, self.space.n):
            raise ValueError(f"control array must be ({self.space.N}, {self.space.n}), got {C.shape}")
        if self.weights.weights.shape != (self.space.N,):
            raise ValueError("weight count does not match the space dimension")
        self.control = C
        self.is_polynomial = self.weights.is_unit
        grid = map_grid(self, [np.linspace(0.0, 1.0, 21)] * self.space.n, max_deriv=1)
        dets = grid["det"]
        if not np.all(np.isfinite(dets)) or np.min(dets) <= 0.0:
            loc = np.unravel_index(int(np.argmin(dets)), dets.shape)
            pt = tuple(float(np.linspace(0.0, 1.0, 21)[i]) for i in loc)
            raise ValueError(f"Jacobian determinant {np.min(dets):.3e} <= 0 near x_hat={pt}")
        J = grid["jac"].reshape(-1, self.space.n, self.space.n)
        scale = np.max(np.abs(J))
        self.is_affine = bool(self.is_polynomial and np.max(np.abs(J - J[0])) <= 1e-12 * (1.0 + scale))

    @property
    def n(self) -> int:
        return self.space.n

    @property
    def geometry_degree(self) -> int:
        return self.space.p


# ---------------------------------------------------------------------------------------
# builders
# ---------------------------------------------------------------------------------------

def _insert(T, p, coefs, xbar):
    """Boehm knot insertion of one knot (bspline.py:421-446)."""
    nb = len(T) - p - 1
    ell = p
    while ell + 1 < len(T) and T[ell + 1] <= xbar:
        ell += 1
    out = np.empty((nb + 1,) + coefs.shape[1:])
    out[: ell - p + 1] = coefs[: ell - p + 1]
    for i in range(ell - p + 1, ell + 1):
        den = T[i + p] - T[i]
        a = float((xbar - T[i]) / den) if den != 0 else 0.0
        out[i] = a * coefs[i] + (1.0 - a) * coefs[i - 1]
    out[ell + 1:] = coefs[ell:]
    return T[: ell + 1] + [xbar] + T[ell + 1:], out


def _refine_bezier(p, coefs, target_m):
    spans = target_m - p
    T = [Fraction(0)] * (p + 1) + [Fraction(1)] * (p + 1)
    C = np.asarray(coefs, float)
    for k in range(1, spans):
        T, C = _insert(T, p, C, Fraction(k, spans))
    return C


def _poly_weight(space: TensorSpace, w: np.ndarray) -> bool:
    """Is W one global polynomial of coordinate degree p (geometry.py:240-265)?"""
    n, p = space.n, space.p
    if np.all(w == w[0]):
        return True
    cheb = 0.5 * (1.0 - np.cos(np.pi * np.arange(p + 1) / p))
    hom = w[:, None]
    Wc = _grid_field(space, hom, [cheb] * n, (0,) * n)[..., 0]
    bz = np.array([0.0] * (p + 1) + [1.0] * (p + 1))
    coef = Wc
    for d in range(n):
        moved = np.moveaxis(coef, d, 0)
        E = np.zeros((p + 1, p + 1))
        span, t = basis_table(bz, p, cheb, 0)
        for i in range(p + 1):
            E[i, span[i] - p: span[i] + 1] = t[i, 0]
        sol = np.linalg.solve(E, moved.reshape(p + 1, -1))
        coef = np.moveaxis(sol.reshape(moved.shape), 0, d)
    dense = np.linspace(0.0, 1.0, 13)
    Wd = _grid_field(space, hom, [dense] * n, (0,) * n)[..., 0]
    fit = coef
    for d in range(n):
        span, t = basis_table(bz, p, dense, 0)
        E = np.zeros((dense.size, p + 1))
        for i in range(dense.size):
            E[i, span[i] - p: span[i] + 1] = t[i, 0]
        fit = np.moveaxis(np.tensordot(E, np.moveaxis(fit, d, 0), axes=(1, 0)), 0, d)
    return bool(np.max(np.abs(fit - Wd)) <= 1e-10 * np.max(np.abs(Wd)))


def _from_bezier(p: int, n: int, hom_grid: np.ndarray, name: str) -> GeometryMap:
    target = 2 * p + 1
    Cg = hom_grid.astype(float)
    for d in range(n):
        moved = np.moveaxis(Cg, d, 0)
        ref = _refine_bezier(p, moved.reshape(p + 1, -1), target)
        Cg = np.moveaxis(ref.reshape((target,) + moved.shape[1:]), 0, d)
    flat = Cg.reshape(-1, n + 1, order="F")
    w = flat[:, n]
    pts = flat[:, :n] / w[:, None]
    space = make_tensor_space(p, target, n)
    poly = bool(np.all(w == w[0])) or _poly_weight(space, w)
    return GeometryMap(space=space, weights=NurbsWeights(weights=w, polynomial_weight=poly), control=pts, name=name)


def _collocated(p, n, func, name, m=None) -> GeometryMap:
    space = make_tensor_space(p, 2 * p + 1 if m is None else m, n)
    sites = [kv.greville() for kv in space.kvs]
    vals = func(*np.meshgrid(*sites, indexing="ij"))
    ctrl = np.empty((space.N, n))
    for c in range(n):
        ctrl[:, c] = tensor_collocate(space.kvs, sites, np.asarray(vals[c], float)).reshape(-1, order="F")
    return GeometryMap(space=space, weights=NurbsWeights(np.ones(space.N), polynomial_weight=True), control=ctrl, name=name)


def unit_square() -> GeometryMap:
    return _collocated(1, 2, lambda x, y: (x, y), "unit_square")


def unit_cube() -> GeometryMap:
    return _collocated(1, 3, lambda x, y, z: (x, y, z), "unit_cube")


def quarter_annulus(r_in: float = 1.0, r_out: float = 2.0) -> GeometryMap:
    """Exact quarter annulus, radial first / angular second (geometry.py:373-390)."""
    if not 0.0 < r_in < r_out:
        raise ValueError("need 0 < r_in < r_out")
    radii = np.array([r_in, 0.5 * (r_in + r_out), r_out])
    arc = np.array([[1.0, 0.0], [1.0, 1.0], [0.0, 1.0]])
    warc = np.array([1.0, np.sqrt(2.0) / 2.0, 1.0])
    hom = np.empty((3, 3, 3))
    for i in range(3):
        for j in range(3):
            hom[i, j, :2] = warc[j] * radii[i] * arc[j]
            hom[i, j, 2] = warc[j]
    return _from_bezier(2, 2, hom, f"quarter_annulus({r_in:g},{r_out:g})")


def coons_2d(bottom, top, left, right, weights=None, name: str = "coons_2d") -> GeometryMap:
    """Bilinearly blended Coons patch of four degree-p curves (geometry.py:393-431)."""
    curves = [np.asarray(c, dtype=float) for c in (bottom, top, left, right)]
    deg = curves[0].shape[0] - 1
    for c in curves:
        if c.shape != (deg + 1, 2):
            raise ValueError("all four curves need the same number of 2D control points")
    wc = [np.ones(deg + 1) for _ in range(4)] if weights is None else [np.asarray(w, float) for w in weights]
    B, T, L, R = [np.concatenate([c * w[:, None], w[:, None]], axis=1) for c, w in zip(curves, wc)]
    for a, b in [(B[0], L[0]), (B[deg], R[0]), (T[0], L[deg]), (T[deg], R[deg])]:
        if not np.allclose(a, b, rtol=0.0, atol=1e-12):
            raise ValueError("boundary curves do not share corner control points")
    hom = np.empty((deg + 1, deg + 1, 3))
    for k in range(deg + 1):
        for l in range(deg + 1):
            u, v = k / deg, l / deg
            hom[k, l] = ((1 - v) * B[k] + v * T[k] + (1 - u) * L[l] + u * R[l]
                         - ((1 - u) * (1 - v) * B[0] + u * (1 - v) * B[deg] + (1 - u) * v * T[0] + u * v * T[deg]))
    return _from_bezier(deg, 2, hom, name)


def _coons_quadratic():
    return coons_2d([(0.0, 0.0), (0.5, -0.15), (1.0, 0.0)], [(-0.1, 1.0), (0.5, 1.2), (1.1, 1.05)],
                    [(0.0, 0.0), (-0.2, 0.5), (-0.1, 1.0)], [(1.0, 0.0), (1.15, 0.5), (1.1, 1.05)],
                    name="coons_quadratic")


def _coons_cubic():
    return coons_2d([(0.0, 0.0), (0.3, -0.1), (0.7, -0.1), (1.0, 0.0)],
                    [(-0.1, 1.0), (0.3, 1.15), (0.7, 1.15), (1.1, 1.0)],
                    [(0.0, 0.0), (-0.15, 0.3), (-0.15, 0.7), (-0.1, 1.0)],
                    [(1.0, 0.0), (1.1, 0.35), (1.1, 0.65), (1.1, 1.0)], name="coons_cubic")


def _coons_rational():
    return coons_2d([(0.0, 0.0), (0.55, -0.18), (1.0, 0.0)], [(-0.12, 1.0), (0.45, 1.22), (1.08, 1.02)],
                    [(0.0, 0.0), (-0.22, 0.45), (-0.12, 1.0)], [(1.0, 0.0), (1.18, 0.55), (1.08, 1.02)],
                    weights=([1.0, 1.25, 1.0], [1.0, 0.85, 1.0], [1.0, 1.1, 1.0], [1.0, 0.95, 1.0]),
                    name="coons_rational")


def trivariate_polynomial_3d() -> GeometryMap:
    def bump(t):
        return 4.0 * t * (1.0 - t)

    a = 0.05
    return _collocated(2, 3, lambda x, y, z: (x + a * bump(y) * bump(z), y + a * bump(x) * bump(z),
                                               z + a * bump(x) * bump(y)), "trivariate_polynomial_3d")


BUILTIN_NAMES = ("unit_square", "unit_cube", "quarter_annulus", "coons_quadratic", "coons_cubic", "coons_rational",
                 "trivariate_polynomial_3d")


def builtin_domain(name: str, **kwargs) -> GeometryMap:
    table = {"unit_square": unit_square, "unit_cube": unit_cube, "coons_quadratic": _coons_quadratic,
             "coons_cubic": _coons_cubic, "coons_rational": _coons_rational,
             "trivariate_polynomial_3d": trivariate_polynomial_3d}
    if name == "quarter_annulus":
        return quarter_annulus(**kwargs)
    if name in table:
        return table[name]()
    raise ValueError(f"unknown builtin domain {name!r}; choose from {BUILTIN_NAMES}")


# BASELINE configs 3-5: frozen B-spline stand-ins of the analytic maps,
# generated by tests/golden/make_geometries.py with the reference's own collocation.
import os as _os

_DATA = _os.path.join(_os.path.dirname(_os.path.abspath(__file__)), "data")


def twisted_cube_standin() -> GeometryMap:
    return load_geometry(_os.path.join(_DATA, "twisted_cube_p3_m12.geo"))


def sin_map_standin() -> GeometryMap:
    return load_geometry(_os.path.join(_DATA, "sin_map_p3_m16.geo"))


# ---------------------------------------------------------------------------------------
# weight transfer (geometry.py:299-319)
# ---------------------------------------------------------------------------------------

def weights_for_space(geom: GeometryMap, space: TensorSpace) -> NurbsWeights:
    if geom.is_polynomial:
        return NurbsWeights(weights=np.ones(space.N), polynomial_weight=True)
    if space.n != geom.n:
        raise ValueError("dimension mismatch")
    if tuple(kv.m for kv in space.kvs) == geom.space.shape and space.p == geom.space.p:
        return geom.weights
    if not geom.weights.polynomial_weight:
        raise ValueError("weight function is not polynomial; cannot transfer to a finer space")
    if space.p < geom.space.p:
        raise ValueError(f"solution degree {space.p} below geometry degree {geom.space.p}")
    sites = [kv.greville() for kv in space.kvs]
    Wg = _grid_field(geom.space, geom.weights.weights[:, None], sites, (0,) * space.n)[..., 0]
    coef = tensor_collocate(space.kvs, sites, Wg)
    return NurbsWeights(weights=coef.reshape(-1, order="F"), polynomial_weight=True)


# ---------------------------------------------------------------------------------------
# iga-geo v1 text format (geometry.py:509-555)
# ---------------------------------------------------------------------------------------

_HEADER_RE = re.compile(r"^iga-geo v1 n=(\d+) p=(\d+) m=([\d,]+)$")


def save_geometry(geom: GeometryMap, path) -> None:
    ms = ",".join(str(kv.m) for kv in geom.space.kvs)
    lines = [f"iga-geo v1 n={geom.n} p={geom.space.p} m={ms}"]
    w = geom.weights.weights
    for i in range(geom.space.N):
        lines.append(f"{i + 1} {repr(float(w[i]))} " + " ".join(repr(float(v)) for v in geom.control[i]))
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")


def load_geometry(path) -> GeometryMap:
    with open(path) as f:
        raw = [ln.strip() for ln in f if ln.strip()]
    if not raw:
        raise ValueError("empty geometry file")
    mt = _HEADER_RE.match(raw[0])
    if not mt:
        raise ValueError(f"malformed header: {raw[0]!r}")
    n, p = int(mt.group(1)), int(mt.group(2))
    ms = [int(v) for v in mt.group(3).split(",") if v]
    if len(ms) != n:
        raise ValueError(f"header lists {len(ms)} mesh sizes for n={n}")
    space = make_tensor_space(p, ms)
    N = space.N
    if len(raw) - 1 != N:
        raise ValueError(f"expected {N} control point lines, found {len(raw) - 1}")
    w = np.empty(N)
    pts = np.empty((N, n))
    for line in raw[1:]:
        parts = line.split()
        if len(parts) != n + 2:
            raise ValueError(f"bad control point line: {line!r}")
        i = int(parts[0])
        if not 1 <= i <= N:
            raise ValueError(f"index {i} outside 1..{N}")
        w[i - 1] = float(parts[1])
        pts[i - 1] = [float(v) for v in parts[2:]]
    if np.any(w <= 0):
        raise ValueError("nonpositive weight")
    poly = _poly_weight(space, w)
    return GeometryMap(space=space, weights=NurbsWeights(weights=w, polynomial_weight=poly), control=pts, name="file")
