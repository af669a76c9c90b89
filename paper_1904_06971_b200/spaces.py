"""Host-side spline spaces (setup only): exact open uniform knots, tensor spaces, NURBS weights.

Mirrors the reference types of ``surriga.bspline`` that the hot path reads
(bspline.py:186-414) with the same names, fields and error messages.  Nothing here
runs per matrix entry: the Cox-de Boor tables used by the assembly are evaluated on
the GPU (csrc/sg_common.cuh ``basis_ders``); the host variant below only serves
setup-time collocation (NURBS weight transfer, surrogate interpolation systems, the
geometry constructors).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from fractions import Fraction
from typing import Sequence

import numpy as np

__all__ = [
    "UniformOpenKnotVector", "TensorSpace", "NurbsWeights", "make_open_uniform_knots", "make_tensor_space",
    "unit_weights", "basis_table", "collocation_matrix", "collocation_solve", "tensor_collocate",
]


@dataclass(frozen=True)
class UniformOpenKnotVector:
    """Open uniform knots on [0,1]: p+1 zeros, k/(m-p) interior, p+1 ones (bspline.py:186-222)."""

    p: int
    m: int
    knots_exact: tuple = field(repr=False)

    @property
    def h_exact(self) -> Fraction:
        return Fraction(1, self.m - self.p)

    @property
    def h(self) -> float:
        return 1.0 / (self.m - self.p)

    @property
    def spans(self) -> int:
        return self.m - self.p

    @property
    def knots(self) -> np.ndarray:
        return np.array([float(t) for t in self.knots_exact])

    def span_breaks(self) -> np.ndarray:
        return np.array([float(Fraction(k, self.spans)) for k in range(self.spans + 1)])

    def greville_exact(self) -> list:
        p, T = self.p, self.knots_exact
        return [sum(T[k + 1:k + p + 1], Fraction(0)) / p if p else T[k] for k in range(self.m)]

    def greville(self) -> np.ndarray:
        return np.array([float(g) for g in self.greville_exact()])


def make_open_uniform_knots(p: int, m: int) -> UniformOpenKnotVector:
    """bspline.py:225-238 (same validation messages)."""
    if p < 1:
        raise ValueError(f"degree must be >= 1, got {p}")
    if m < 2 * p + 1:
        raise ValueError(f"basis count m={m} below 2p+1={2 * p + 1}")
    s = m - p
    kn = (Fraction(0),) * (p + 1) + tuple(Fraction(k, s) for k in range(1, s)) + (Fraction(1),) * (p + 1)
    return UniformOpenKnotVector(p=p, m=m, knots_exact=kn)


@dataclass(frozen=True)
class TensorSpace:
    """Equal-degree tensor space, colex flat index (bspline.py:306-339)."""

    kvs: tuple

    @property
    def n(self) -> int:
        return len(self.kvs)

    @property
    def p(self) -> int:
        return self.kvs[0].p

    @property
    def shape(self) -> tuple:
        return tuple(kv.m for kv in self.kvs)

    @property
    def N(self) -> int:
        return int(np.prod(self.shape))

    def ravel(self, multi0) -> np.ndarray:
        multi0 = np.asarray(multi0)
        return np.ravel_multi_index(tuple(multi0[..., d] for d in range(self.n)), self.shape, order="F")

    def unravel(self, flat) -> np.ndarray:
        return np.stack(np.unravel_index(np.asarray(flat), self.shape, order="F"), axis=-1)


def make_tensor_space(p: int, m, n: int | None = None) -> TensorSpace:
    """bspline.py:342-354."""
    if np.isscalar(m):
        if n is None:
            raise ValueError("give n when m is scalar")
        ms = [int(m)] * n
    else:
        ms = [int(v) for v in m]
    if n is not None and len(ms) != n:
        raise ValueError("m length does not match n")
    if len(ms) not in (1, 2, 3):
        raise ValueError("supported dimensions: 1, 2, 3")
    return TensorSpace(kvs=tuple(make_open_uniform_knots(p, mv) for mv in ms))


@dataclass(frozen=True)
class NurbsWeights:
    """Positive per-basis weights, colex (bspline.py:391-414)."""

    weights: np.ndarray
    polynomial_weight: bool = False

    def __post_init__(self):
        w = np.asarray(self.weights, dtype=float)
        if w.ndim != 1:
            raise ValueError("weights must be a flat colex-ordered vector")
        if not np.all(w > 0):
            raise ValueError("nonpositive weight")
        object.__setattr__(self, "weights", w)

    @property
    def is_unit(self) -> bool:
        w = self.weights
        return bool(np.all(w == w[0]))


def unit_weights(space: TensorSpace) -> NurbsWeights:
    return NurbsWeights(weights=np.ones(space.N), polynomial_weight=True)


# ---------------------------------------------------------------------------------------
# setup-time evaluation (vectorised over points; same recurrence as the device kernel)
# ---------------------------------------------------------------------------------------

def basis_table(knots: np.ndarray, p: int, x, nu: int = 0):
    """Spans and (npts, nu+1, p+1) values/derivatives of the nonzero basis at ``x``."""
    x = np.asarray(x, dtype=float).ravel()
    nb = knots.size - p - 1
    span = np.clip(np.searchsorted(knots, x, side="right") - 1, p, nb - 1)
    # inverted triangle of knot differences
    L = np.zeros((p + 1, x.size))
    R = np.zeros((p + 1, x.size))
    ndu = np.zeros((p + 1, p + 1, x.size))
    ndu[0, 0] = 1.0
    for j in range(1, p + 1):
        L[j] = x - knots[span + 1 - j]
        R[j] = knots[span + j] - x
        acc = np.zeros(x.size)
        for r in range(j):
            ndu[j, r] = R[r + 1] + L[j - r]
            t = ndu[r, j - 1] / ndu[j, r]
            ndu[r, j] = acc + R[r + 1] * t
            acc = L[j - r] * t
        ndu[j, j] = acc
    out = np.zeros((x.size, nu + 1, p + 1))
    out[:, 0, :] = ndu[:, p, :].T
    top = min(nu, p)
    for r in range(p + 1):
        prev = np.zeros((p + 1, x.size))
        prev[0] = 1.0
        for k in range(1, top + 1):
            cur = np.zeros((p + 1, x.size))
            d = np.zeros(x.size)
            rk, pk = r - k, p - k
            if r >= k:
                cur[0] = prev[0] / ndu[pk + 1, rk]
                d = cur[0] * ndu[rk, pk]
            lo = 1 if rk >= -1 else -rk
            hi = k - 1 if r - 1 <= pk else p - r
            for j in range(lo, hi + 1):
                cur[j] = (prev[j] - prev[j - 1]) / ndu[pk + 1, rk + j]
                d = d + cur[j] * ndu[rk + j, pk]
            if r <= pk:
                cur[k] = -prev[k - 1] / ndu[pk + 1, r]
                d = d + cur[k] * ndu[r, pk]
            out[:, k, r] = d
            prev = cur
    f = float(p)
    for k in range(1, top + 1):
        out[:, k, :] *= f
        f *= p - k
    return span, out


def collocation_matrix(knots: np.ndarray, p: int, sites) -> np.ndarray:
    """Dense E[i, j] = B_j(sites[i]) (bspline.py:127-135)."""
    sites = np.asarray(sites, dtype=float).ravel()
    nb = knots.size - p - 1
    span, t = basis_table(knots, p, sites, 0)
    E = np.zeros((sites.size, nb))
    cols = span[:, None] - p + np.arange(p + 1)[None, :]
    np.put_along_axis(E, cols, t[:, 0, :], axis=1)
    return E


def collocation_solve(knots: np.ndarray, p: int, sites, rhs) -> np.ndarray:
    """Interpolation solve B_j(sites_i) c_j = rhs_i along the first axis (bspline.py:138-164)."""
    sites = np.asarray(sites, dtype=float).ravel()
    nb = knots.size - p - 1
    if sites.size != nb:
        raise ValueError(f"need {nb} sites, got {sites.size}")
    rhs = np.asarray(rhs, dtype=float)
    if nb == 1:
        return rhs.copy()
    E = collocation_matrix(knots, p, sites)
    from scipy.linalg import solve_banded

    kl = ku = p
    ab = np.zeros((kl + ku + 1, nb))
    for j in range(nb):
        for i in range(max(0, j - ku), min(nb, j + kl + 1)):
            ab[ku + i - j, j] = E[i, j]
    sol = solve_banded((kl, ku), ab, rhs.reshape(nb, -1))
    return sol.reshape(rhs.shape)


def tensor_collocate(kvs: Sequence[UniformOpenKnotVector], sites, values) -> np.ndarray:
    """Direction-by-direction interpolation of tensor-grid data (bspline.py:167-178)."""
    coef = np.asarray(values, dtype=float)
    for d, kv in enumerate(kvs):
        moved = np.moveaxis(coef, d, 0)
        sol = collocation_solve(kv.knots, kv.p, sites[d], moved.reshape(kv.m, -1))
        coef = np.moveaxis(sol.reshape(moved.shape), 0, d)
    return coef
