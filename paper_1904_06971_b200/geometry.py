"""Geometry input of the assembly (host, setup only).

The hot path reads a map's tensor space, weights and control net; callers
normally pass the reference's own ``surriga.geometry.GeometryMap`` (duck-typed).  This module only
provides the container for callers without the reference, the check that the map is regular, the
``iga-geo v1`` file format and the benchmark domains -- which are not rebuilt here: their nets were
produced once by the reference itself (``tests/golden/make_geometries.py``) and are read from
``data/*.geo`` (the BASELINE configs 3-5 stand-ins likewise).  The map, Jacobian,
adjugate, determinant and Hessian at the quadrature points are evaluated on the GPU (K3).
"""
from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np

from .spaces import NurbsWeights, TensorSpace, basis_table, make_tensor_space, tensor_collocate

__all__ = [
    "GeometryMap", "map_grid", "unit_square", "unit_cube", "quarter_annulus", "trivariate_polynomial_3d",
    "builtin_domain", "BUILTIN_NAMES", "weights_for_space", "save_geometry", "load_geometry", "twisted_cube_standin",
    "sin_map_standin",
]

_DATA = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data")


def _eval_matrix(space: TensorSpace, axes, orders) -> np.ndarray:
    """Dense (prod G_d) x N matrix of one derivative of the tensor basis on a point grid, rows and
    columns colex (first direction fastest): a Kronecker product of per-direction matrices."""
    K = np.ones((1, 1))
    for kv, x, k in zip(space.kvs, axes, orders):
        span, tab = basis_table(kv.knots, kv.p, x, k)
        E = np.zeros((x.size, kv.m))
        for j in range(kv.p + 1):
            E[np.arange(x.size), span - kv.p + j] = tab[:, k, j]
        K = np.kron(E, K)
    return K


def map_grid(geom, axes, max_deriv: int = 1) -> dict:
    """Map value (and Jacobian ``jac[..., c, a] = d phi_c / d xhat_a``, det) on a tensor point grid
    (the quantities of geometry.py:185-229), arrays shaped (G_0, ..., G_{n-1}, ...)."""
    space = geom.space
    n = space.n
    axes = [np.asarray(a, float).ravel() for a in axes]
    shape = tuple(a.size for a in reversed(axes))        # Kronecker rows: last direction slowest
    w = np.asarray(geom.weights.weights, float)
    hom = np.concatenate([np.asarray(geom.control, float) * w[:, None], w[:, None]], axis=1)

    def field_(orders):
        v = _eval_matrix(space, axes, orders) @ hom
        return np.moveaxis(v.reshape(shape + (n + 1,)), tuple(range(n)), tuple(reversed(range(n))))

    val = field_((0,) * n)
    W = val[..., n]
    phi = val[..., :n] / W[..., None]
    out = {"phi": phi, "W": W}
    if max_deriv >= 1:
        jac = np.empty(W.shape + (n, n))
        for a in range(n):
            dv = field_(tuple(int(d == a) for d in range(n)))
            jac[..., :, a] = (dv[..., :n] - phi * dv[..., n:]) / W[..., None]
        out["jac"] = jac
        out["det"] = np.linalg.det(jac) if n > 1 else jac[..., 0, 0]
    return out


@dataclass
class GeometryMap:
    """Single-patch NURBS map (the fields of geometry.py:139-182): tensor space, weights, control
    net (N x n, colex).  Construction rejects maps whose Jacobian determinant is not positive on a
    21^n grid, as the reference does."""

    space: TensorSpace
    weights: NurbsWeights
    control: np.ndarray
    name: str = ""
    is_affine: bool = field(init=False, default=False)
    is_polynomial: bool = field(init=False, default=False)

    def __post_init__(self):
        ctrl = np.asarray(self.control, dtype=float)
        N, n = self.space.N, self.space.n
        if ctrl.shape != (N, n):
            raise ValueError(f"control array must be ({N}, {n}), got {ctrl.shape}")
        if self.weights.weights.shape != (N,):
            raise ValueError("weight count does not match the space dimension")
        self.control = ctrl
        self.is_polynomial = self.weights.is_unit
        probe = np.linspace(0.0, 1.0, 21)
        g = map_grid(self, [probe] * n)
        det = g["det"]
        worst = int(np.argmin(np.where(np.isfinite(det), det, -np.inf)))
        if not np.all(np.isfinite(det)) or det.flat[worst] <= 0.0:
            where = tuple(float(probe[i]) for i in np.unravel_index(worst, det.shape))
            raise ValueError(f"Jacobian determinant {det.flat[worst]:.3e} <= 0 near x_hat={where}")
        J = g["jac"].reshape(-1, n, n)
        self.is_affine = bool(self.is_polynomial and np.ptp(J, axis=0).max() <= 1e-12 * (1.0 + np.abs(J).max()))

    @property
    def n(self) -> int:
        return self.space.n

    @property
    def geometry_degree(self) -> int:
        return self.space.p


def _weights_polynomial(space: TensorSpace, w: np.ndarray) -> bool:
    """Is the weight spline one global polynomial (geometry.py:240-265's question)?  A C^{p-1}
    spline of degree p is a single polynomial iff its p-th derivative in every direction does not
    jump across any interior knot; the jumps are sampled along each knot line."""
    w = np.asarray(w, float)
    if np.all(w == w[0]):
        return True
    n = space.n
    scale = np.abs(w).max()
    for d, kv in enumerate(space.kvs):
        br = kv.span_breaks()[1:-1]
        if br.size == 0:
            continue
        eps = 0.25 * kv.h
        axes = [np.linspace(0.05, 0.95, 5) for _ in range(n)]
        orders = tuple(kv.p if e == d else 0 for e in range(n))
        lo = list(axes)
        hi = list(axes)
        lo[d] = br - eps
        hi[d] = br + eps
        jump = _eval_matrix(space, hi, orders) @ w - _eval_matrix(space, lo, orders) @ w
        if np.abs(jump).max() > 1e-9 * scale * kv.spans ** kv.p:
            return False
    return True


def _fixture(name) -> "GeometryMap":
    return load_geometry(os.path.join(_DATA, name + ".geo"), name=name)


def unit_square() -> GeometryMap:
    return _fixture("unit_square")


def unit_cube() -> GeometryMap:
    return _fixture("unit_cube")


def trivariate_polynomial_3d() -> GeometryMap:
    return _fixture("trivariate_polynomial_3d")


def quarter_annulus(r_in: float = 1.0, r_out: float = 2.0) -> GeometryMap:
    """The reference's exact quarter annulus (geometry.py:373-390), radial first / angular second.

    Its control points are linear in (r_in, r_out) (the weights are not), so the two frozen nets
    r = (1, 2) and (1, 3) give every other pair; (1, 2) is returned bit for bit as the reference
    builds it."""
    if not 0.0 < r_in < r_out:
        raise ValueError("need 0 < r_in < r_out")
    a = _fixture("quarter_annulus_1_2")
    if (r_in, r_out) == (1.0, 2.0):
        a.name = "quarter_annulus(1,2)"
        return a
    b = _fixture("quarter_annulus_1_3")
    dB = b.control - a.control            # d/d r_out
    dA = a.control - 2.0 * dB             # d/d r_in
    return GeometryMap(space=a.space, weights=a.weights, control=r_in * dA + r_out * dB,
                       name=f"quarter_annulus({r_in:g},{r_out:g})")


BUILTIN_NAMES = ("unit_square", "unit_cube", "quarter_annulus", "coons_quadratic", "coons_cubic", "coons_rational",
                 "trivariate_polynomial_3d")


def builtin_domain(name: str, **kwargs) -> GeometryMap:
    """The reference's benchmark domains by name (geometry.py:486-502), from the frozen nets."""
    if name == "quarter_annulus":
        return quarter_annulus(**kwargs)
    if name in BUILTIN_NAMES:
        return _fixture(name)
    raise ValueError(f"unknown builtin domain {name!r}; choose from {BUILTIN_NAMES}")


def twisted_cube_standin() -> GeometryMap:
    """BASELINE configs 3/5: B-spline stand-in (p=3, 12 functions per direction) of the twisted cube."""
    return load_geometry(os.path.join(_DATA, "twisted_cube_p3_m12.geo"))


def sin_map_standin() -> GeometryMap:
    """BASELINE config 4: B-spline stand-in (p=3, 16 functions per direction) of the sin-perturbed square."""
    return load_geometry(os.path.join(_DATA, "sin_map_p3_m16.geo"))


def weights_for_space(geom, space: TensorSpace) -> NurbsWeights:
    """Weights of the solution space for a map (geometry.py:299-319): unit for polynomial maps, the
    map's own on its own space, else the weight function interpolated at the space's Greville sites
    (possible only when it is one global polynomial of degree <= the space's)."""
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
    W = map_grid(geom, sites, max_deriv=0)["W"]
    return NurbsWeights(weights=tensor_collocate(space.kvs, sites, W).reshape(-1, order="F"), polynomial_weight=True)


# ``iga-geo v1`` text format (geometry.py:509-555): header "iga-geo v1 n=<n> p=<p> m=<m0,m1,..>",
# then one line per control point "<1-based index> <weight> <x> [<y> [<z>]]" (colex order)

def save_geometry(geom, path) -> None:
    N, n = geom.space.N, geom.space.n
    table = np.column_stack([np.arange(1, N + 1), geom.weights.weights, geom.control])
    with open(path, "w") as f:
        f.write(f"iga-geo v1 n={n} p={geom.space.p} m={','.join(str(kv.m) for kv in geom.space.kvs)}\n")
        for row in table:
            f.write(" ".join([str(int(row[0]))] + [repr(float(v)) for v in row[1:]]) + "\n")


def load_geometry(path, name: str = "file") -> GeometryMap:
    with open(path) as f:
        lines = [ln.split() for ln in f if ln.strip()]
    if not lines:
        raise ValueError("empty geometry file")
    head = lines[0]
    try:
        assert head[:2] == ["iga-geo", "v1"] and len(head) == 5
        keys = dict(tok.split("=", 1) for tok in head[2:])
        n, p = int(keys["n"]), int(keys["p"])
        ms = [int(v) for v in keys["m"].split(",") if v]
    except (AssertionError, KeyError, ValueError):
        raise ValueError(f"malformed header: {' '.join(head)!r}") from None
    if len(ms) != n:
        raise ValueError(f"header lists {len(ms)} mesh sizes for n={n}")
    space = make_tensor_space(p, ms)
    N = space.N
    if len(lines) - 1 != N:
        raise ValueError(f"expected {N} control point lines, found {len(lines) - 1}")
    w = np.empty(N)
    pts = np.empty((N, n))
    for parts in lines[1:]:
        if len(parts) != n + 2:
            raise ValueError(f"bad control point line: {' '.join(parts)!r}")
        i = int(parts[0])
        if not 1 <= i <= N:
            raise ValueError(f"index {i} outside 1..{N}")
        w[i - 1] = float(parts[1])
        pts[i - 1] = [float(v) for v in parts[2:]]
    if np.any(w <= 0):
        raise ValueError("nonpositive weight")
    return GeometryMap(space=space, weights=NurbsWeights(weights=w, polynomial_weight=_weights_polynomial(space, w)),
                       control=pts, name=name)
