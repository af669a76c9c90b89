"""CPU oracle (TEST INFRASTRUCTURE ONLY) for the surrogate/full IGA assembly hot path.

This module is a plain-numpy restatement of the reference algorithm of
arXiv 1904.06971's ``surriga`` package (``/root/reference/pkg/src/surriga``),
written independently of the reference's code structure (points are
vectorised, elements are processed in one batch, CSR positions are analytic).
It exists so that the CUDA path can be checked on machines where the
reference is not installed (the GPU box).  It is pinned against golden
vectors produced by the real reference (``tests/golden/make_golden.py``) in
``tests/test_oracle_golden.py``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this module; the product package never does.

Citations (reference file:line) are given per function.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

FORMS = ("poisson", "mass", "biharmonic", "stokes_velocity")
_DERIV = {"poisson": 1, "mass": 0, "biharmonic": 2, "stokes_velocity": 1}


# ---------------------------------------------------------------------------
# problem description (duck-typed from either the reference or the product)
# ---------------------------------------------------------------------------

@dataclass
class Problem:
    form: str
    p: int
    ms: tuple              # basis functions per direction (solution space)
    g: int                 # Gauss points per direction
    sol_w: np.ndarray      # solution-space weights (colex)
    geo_p: int
    geo_ms: tuple
    geo_w: np.ndarray
    geo_ctrl: np.ndarray   # (Ng, n), colex
    coefficient: float = 1.0

    @property
    def n(self):
        return len(self.ms)

    @property
    def N(self):
        return int(np.prod(self.ms))

    @property
    def spans(self):
        return tuple(m - self.p for m in self.ms)

    @property
    def rational(self):
        # assembly.py:418 -- `weights.is_unit` (all weights equal) selects the polynomial path
        w = self.sol_w
        return not bool(np.all(w == w[0]))


def problem_from_disc(form, disc, coefficient=1.0) -> Problem:
    fname = form.value if hasattr(form, "value") else str(form)
    space = disc.space
    gsp = disc.geom.space
    return Problem(
        form=fname,
        p=int(space.kvs[0].p),
        ms=tuple(int(kv.m) for kv in space.kvs),
        g=int(disc.gauss),
        sol_w=np.asarray(disc.weights.weights, dtype=float),
        geo_p=int(gsp.kvs[0].p),
        geo_ms=tuple(int(kv.m) for kv in gsp.kvs),
        geo_w=np.asarray(disc.geom.weights.weights, dtype=float),
        geo_ctrl=np.asarray(disc.geom.control, dtype=float),
        coefficient=float(coefficient),
    )


# ---------------------------------------------------------------------------
# splines (bspline.py:45-124, 186-238)
# ---------------------------------------------------------------------------

def open_uniform_knots(p: int, m: int) -> np.ndarray:
    """bspline.py:225-238: p+1 zeros, k/(m-p) interior, p+1 ones (correctly rounded)."""
    s = m - p
    return np.array([0.0] * (p + 1) + [float(Fraction(k, s)) for k in range(1, s)] + [1.0] * (p + 1))


def span_breaks(p: int, m: int) -> np.ndarray:
    """bspline.py:213-215."""
    s = m - p
    return np.array([float(Fraction(k, s)) for k in range(s + 1)])


def basis_ders(knots: np.ndarray, p: int, x: np.ndarray, nu: int):
    """Cox-de Boor values + derivatives (NURBS book A2.2/A2.3), vectorised over points.

    Follows bspline.py:45-109 (span search with right-clamping, inverted
    knot-difference triangle, derivative recursion).  Returns
    ``(span[npts], ders[npts, nu+1, p+1])``.
    """
    x = np.asarray(x, dtype=float).ravel()
    npts = x.size
    nb = knots.size - p - 1
    span = np.searchsorted(knots, x, side="right") - 1
    span = np.clip(span, p, nb - 1)
    left = np.zeros((npts, p + 1))
    right = np.zeros((npts, p + 1))
    ndu = np.zeros((npts, p + 1, p + 1))
    ndu[:, 0, 0] = 1.0
    for j in range(1, p + 1):
        left[:, j] = x - knots[span + 1 - j]
        right[:, j] = knots[span + j] - x
        saved = np.zeros(npts)
        for r in range(j):
            ndu[:, j, r] = right[:, r + 1] + left[:, j - r]
            tmp = ndu[:, r, j - 1] / ndu[:, j, r]
            ndu[:, r, j] = saved + right[:, r + 1] * tmp
            saved = left[:, j - r] * tmp
        ndu[:, j, j] = saved
    ders = np.zeros((npts, nu + 1, p + 1))
    ders[:, 0, :] = ndu[:, :, p]
    nd = min(nu, p)
    for r in range(p + 1):
        a_prev = np.zeros((npts, p + 1))
        a_prev[:, 0] = 1.0
        for k in range(1, nd + 1):
            a_cur = np.zeros((npts, p + 1))
            d = np.zeros(npts)
            rk, pk = r - k, p - k
            if r >= k:
                a_cur[:, 0] = a_prev[:, 0] / ndu[:, pk + 1, rk]
                d = a_cur[:, 0] * ndu[:, rk, pk]
            j1 = 1 if rk >= -1 else -rk
            j2 = k - 1 if r - 1 <= pk else p - r
            for j in range(j1, j2 + 1):
                a_cur[:, j] = (a_prev[:, j] - a_prev[:, j - 1]) / ndu[:, pk + 1, rk + j]
                d = d + a_cur[:, j] * ndu[:, rk + j, pk]
            if r <= pk:
                a_cur[:, k] = -a_prev[:, k - 1] / ndu[:, pk + 1, r]
                d = d + a_cur[:, k] * ndu[:, r, pk]
            ders[:, k, r] = d
            a_prev = a_cur
    fac = float(p)
    for k in range(1, nd + 1):
        ders[:, k, :] *= fac
        fac *= p - k
    return span, ders


def collocation_matrix(knots, p, sites):
    """Dense B_j(site_i) (bspline.py:127-135)."""
    nb = knots.size - p - 1
    span, t = basis_ders(knots, p, sites, 0)
    E = np.zeros((sites.size, nb))
    for i in range(sites.size):
        E[i, span[i] - p: span[i] + 1] = t[i, 0]
    return E


# ---------------------------------------------------------------------------
# quadrature (assembly.py:100-125)
# ---------------------------------------------------------------------------

def gauss_axes(p, m, g):
    x, w = np.polynomial.legendre.leggauss(g)
    h = 1.0 / (m - p)
    offs = (x + 1.0) * (0.5 * h)
    br = span_breaks(p, m)[:-1]
    return (br[:, None] + offs[None, :]).ravel(), w * (0.5 * h)


# ---------------------------------------------------------------------------
# tensor fields on point grids (geometry.py:185-229, assembly.py:418-437)
# ---------------------------------------------------------------------------

def _multi(n, order):
    """All per-direction derivative multi-indices with total order == ``order``."""
    out = []
    for a in np.ndindex(*([order + 1] * n)):
        if sum(a) == order:
            out.append(tuple(a))
    return out


def field_on_grid(p, ms, coef, axes, nu):
    """Evaluate a tensor spline field with coefficients ``coef`` (N, C) on a grid.

    Returns dict: multi-index alpha -> array (G_0, ..., G_{n-1}, C).
    Contractions run direction by direction over the p+1 nonzero taps.
    """
    n = len(ms)
    coef = np.asarray(coef, dtype=float).reshape(tuple(ms) + (-1,), order="F")
    tabs = []
    for d in range(n):
        kn = open_uniform_knots(p, ms[d])
        tabs.append(basis_ders(kn, p, axes[d], nu))
    out = {}
    for order in range(nu + 1):
        for alpha in _multi(n, order):
            t = coef
            for d in range(n):
                span, ders = tabs[d]
                E = ders[:, alpha[d], :]             # (Gd, p+1)
                idx = span[:, None] - p + np.arange(p + 1)[None, :]
                t = np.moveaxis(t, d, 0)             # (m_d, ...)
                g = t[idx]                           # (Gd, p+1, ...)
                t = np.einsum("xr,xr...->x...", E, g)
                t = np.moveaxis(t, 0, d)
            out[alpha] = t
    return out


def _unit(n, a):
    return tuple(1 if d == a else 0 for d in range(n))


def _pair(n, a, b):
    return tuple((1 if d == a else 0) + (1 if d == b else 0) for d in range(n))


def geometry_on_grid(prob: Problem, axes, nu):
    """Rational map, Jacobian ``jac[...,c,a]``, det, Hessian ``hess[...,c,a,b]`` (geometry.py:185-229)."""
    n = prob.n
    w = prob.geo_w
    hom = np.concatenate([prob.geo_ctrl * w[:, None], w[:, None]], axis=1)
    f = field_on_grid(prob.geo_p, prob.geo_ms, hom, axes, nu)
    num = f[(0,) * n]
    W = num[..., n]
    phi = num[..., :n] / W[..., None]
    res = {"phi": phi, "W": W}
    if nu == 0:
        return res
    jac = np.empty(W.shape + (n, n))
    dW = np.empty(W.shape + (n,))
    for a in range(n):
        dn = f[_unit(n, a)]
        dW[..., a] = dn[..., n]
        jac[..., :, a] = (dn[..., :n] - phi * dn[..., n, None]) / W[..., None]
    res["jac"] = jac
    res["det"] = det(jac)
    if nu == 1:
        return res
    hess = np.empty(W.shape + (n, n, n))
    for a in range(n):
        for b in range(a, n):
            d2 = f[_pair(n, a, b)]
            v = (d2[..., :n] - jac[..., :, a] * dW[..., b, None] - jac[..., :, b] * dW[..., a, None]
                 - phi * d2[..., n, None]) / W[..., None]
            hess[..., :, a, b] = v
            hess[..., :, b, a] = v
    res["hess"] = hess
    return res


def det(J):
    """geometry.py:98-111 (cofactor expansion along the first row)."""
    n = J.shape[-1]
    if n == 1:
        return J[..., 0, 0].copy()
    if n == 2:
        return J[..., 0, 0] * J[..., 1, 1] - J[..., 0, 1] * J[..., 1, 0]
    return (J[..., 0, 0] * (J[..., 1, 1] * J[..., 2, 2] - J[..., 1, 2] * J[..., 2, 1])
            - J[..., 0, 1] * (J[..., 1, 0] * J[..., 2, 2] - J[..., 1, 2] * J[..., 2, 0])
            + J[..., 0, 2] * (J[..., 1, 0] * J[..., 2, 1] - J[..., 1, 1] * J[..., 2, 0]))


def adj(J):
    """geometry.py:114-131: inv = adj / det."""
    n = J.shape[-1]
    A = np.empty_like(J)
    if n == 1:
        A[..., 0, 0] = 1.0
        return A
    if n == 2:
        A[..., 0, 0] = J[..., 1, 1]
        A[..., 0, 1] = -J[..., 0, 1]
        A[..., 1, 0] = -J[..., 1, 0]
        A[..., 1, 1] = J[..., 0, 0]
        return A
    for a in range(3):
        for b in range(3):
            r = [i for i in range(3) if i != b]
            c = [j for j in range(3) if j != a]
            A[..., a, b] = (-1.0) ** (a + b) * (J[..., r[0], c[0]] * J[..., r[1], c[1]]
                                                 - J[..., r[0], c[1]] * J[..., r[1], c[0]])
    return A


# ---------------------------------------------------------------------------
# CSR pattern (analytic; equals csr_from_triplets' pattern, assembly.py:245-270)
# ---------------------------------------------------------------------------

def row_col_range(ms, p, multi):
    lo = np.maximum(multi - p, 0)
    hi = np.minimum(multi + p, np.asarray(ms) - 1)
    return lo, hi


def pattern(ms, p, rows=None):
    """indptr/indices of the basis-overlap pattern, restricted to ``rows`` if given.

    Columns of row i are i + shift(o) for the colex offsets o in [-p,p]^n that
    stay inside the index box; colex offset order is ascending column order
    (surrogate.py:312-322), so no sort is needed.
    """
    ms = tuple(ms)
    n = len(ms)
    N = int(np.prod(ms))
    offs = offsets(p, n)
    strides = np.cumprod((1,) + ms[:-1])
    rsel = np.arange(N) if rows is None else np.asarray(rows, dtype=np.int64)
    multi = np.stack(np.unravel_index(rsel, ms, order="F"), axis=-1)
    jm = multi[:, None, :] + offs[None, :, :]
    ok = np.all((jm >= 0) & (jm < np.asarray(ms)), axis=-1)
    cnt = np.zeros(N, dtype=np.int64)
    cnt[rsel] = ok.sum(1)
    indptr = np.zeros(N + 1, dtype=np.int64)
    np.cumsum(cnt, out=indptr[1:])
    cols = (jm * strides).sum(-1)
    indices = cols[ok].astype(np.int32)
    return indptr, indices


# ---------------------------------------------------------------------------
# element quadrature (assembly.py:402-651)
# ---------------------------------------------------------------------------

def _dir_tables(prob: Problem, nu):
    tabs, axes, pws = [], [], []
    for d in range(prob.n):
        ax, pw = gauss_axes(prob.p, prob.ms[d], prob.g)
        span, ders = basis_ders(open_uniform_knots(prob.p, prob.ms[d]), prob.p, ax, nu)
        S = prob.spans[d]
        assert np.array_equal(span.reshape(S, prob.g), (np.arange(S) + prob.p)[:, None].repeat(prob.g, 1))
        tabs.append(ders.reshape(S, prob.g, nu + 1, prob.p + 1))
        axes.append(ax)
        pws.append(pw)
    return tabs, axes, pws


def _to_elements(arr, spans, g):
    """grid (G_0..G_{n-1}, extra...) -> (E, Q, extra...) with colex element and point order."""
    n = len(spans)
    extra = arr.shape[n:]
    shp = []
    for s in spans:
        shp += [s, g]
    B = arr.reshape(tuple(shp) + extra, order="C")
    # axes (e0, q0, e1, q1, ...) -> element colex (e_{n-1} slowest ... e_0 fastest) etc.
    eax = [2 * d for d in range(n)][::-1]
    qax = [2 * d + 1 for d in range(n)][::-1]
    B = np.transpose(B, eax + qax + list(range(2 * n, 2 * n + len(extra))))
    return B.reshape((int(np.prod(spans)), g ** n) + extra)


def _local_tensor(tabs, et, alpha, p, g):
    """Tensor-product basis derivative ``alpha`` on elements ``et``: (E, Q, L)."""
    n = len(tabs)
    out = None
    for d in range(n):
        v = tabs[d][et[:, d], :, alpha[d], :]          # (E, g, p+1)
        if out is None:
            out = v
        else:
            E = v.shape[0]
            # point index q_d slower, function index l_d slower (colex)
            out = (v[:, :, None, :, None] * out[:, None, :, None, :]).reshape(E, -1, out.shape[-1] * (p + 1))
    return out


def element_matrices(prob: Problem, eids):
    """Local element matrices (E, L, L) for the listed elements (assembly.py:531-551)."""
    n, p, g = prob.n, prob.p, prob.g
    form = prob.form
    nu = _DERIV[form]
    gnu = 2 if form == "biharmonic" else 1
    tabs, axes, pws = _dir_tables(prob, nu)
    wq = pws[0]
    for d in range(1, n):
        wq = (pws[d][:, None] * wq[None, :]).ravel()
    spans = prob.spans
    et = np.stack(np.unravel_index(eids, spans, order="F"), axis=-1)
    # the geometry (and weight function) is evaluated on the sub-grid of the elements' bounding box
    # only: pointwise the same values as the full grid, without the full-grid cost at large meshes
    lo = et.min(axis=0) if et.size else np.zeros(n, np.int64)
    hi = et.max(axis=0) if et.size else np.zeros(n, np.int64)
    sub_spans = tuple(int(h - l + 1) for l, h in zip(lo, hi))
    sub_axes = [axes[d][lo[d] * g:(hi[d] + 1) * g] for d in range(n)]
    sub_eids = np.ravel_multi_index(tuple((et - lo).T), sub_spans, order="F") if et.size else eids
    geo = geometry_on_grid(prob, sub_axes, gnu)
    detE = _to_elements(geo["det"], sub_spans, g)[sub_eids]
    jacE = _to_elements(geo["jac"], sub_spans, g)[sub_eids]
    A = adj(jacE)

    B = _local_tensor(tabs, et, (0,) * n, p, g)
    dB = d2B = None
    if nu >= 1:
        dB = np.stack([_local_tensor(tabs, et, _unit(n, a), p, g) for a in range(n)], axis=-1)
    if nu >= 2:
        d2B = np.empty(B.shape + (n, n))
        for a in range(n):
            for b in range(n):
                d2B[..., a, b] = _local_tensor(tabs, et, _pair(n, a, b), p, g)

    if prob.rational:
        Wf = field_on_grid(p, prob.ms, prob.sol_w[:, None], sub_axes, nu)
        W = _to_elements(Wf[(0,) * n][..., 0], sub_spans, g)[sub_eids][..., None]
        # local weights per element function (colex)
        L = (p + 1) ** n
        Il = np.stack(np.unravel_index(np.arange(L), (p + 1,) * n, order="F"), axis=-1)
        strides = np.cumprod((1,) + tuple(prob.ms[:-1]))
        cols = ((et[:, None, :] + Il[None, :, :]) * strides).sum(-1)
        wl = prob.sol_w[cols][:, None, :]
        N = wl * B / W
        if nu >= 1:
            dW = np.stack([_to_elements(Wf[_unit(n, a)][..., 0], sub_spans, g)[sub_eids] for a in range(n)], axis=-1)
            dN = np.empty_like(dB)
            for a in range(n):
                dN[..., a] = (wl * dB[..., a] - N * dW[..., a][..., None]) / W
        if nu >= 2:
            d2N = np.empty_like(d2B)
            for a in range(n):
                for b in range(n):
                    d2W = _to_elements(Wf[_pair(n, a, b)][..., 0], sub_spans, g)[sub_eids][..., None]
                    d2N[..., a, b] = (wl * d2B[..., a, b] - dN[..., a] * dW[..., b][..., None]
                                      - dN[..., b] * dW[..., a][..., None] - N * d2W) / W
        B = N
        if nu >= 1:
            dB = dN
        if nu >= 2:
            d2B = d2N

    # the (q, derivative) contraction of every element matrix runs as one batched matmul
    # (E, L, Q*k) @ (E, Q*k, L): same sums as the reference's einsums, BLAS speed
    def _gram(X, Y):
        E_, Q_, L_ = X.shape[:3]
        Xf = np.ascontiguousarray(np.moveaxis(X, 2, 1)).reshape(E_, L_, -1)
        Yf = np.ascontiguousarray(np.moveaxis(Y, 2, 1)).reshape(E_, L_, -1)
        return Xf @ np.swapaxes(Yf, 1, 2)

    if form in ("poisson", "stokes_velocity"):
        K = np.einsum("eqab,eqcb->eqac", A, A) / detE[..., None, None]
        K = K * prob.coefficient
        Kw = K * wq[None, :, None, None]
        loc = _gram(np.einsum("eqla,eqab->eqlb", dB, Kw), dB)
    elif form == "mass":
        s = detE * wq[None, :]
        loc = _gram((B * s[..., None])[..., None], B[..., None])
    elif form == "biharmonic":
        hessE = _to_elements(geo["hess"], sub_spans, g)[sub_eids]
        C = np.einsum("eqac,eqbc->eqab", A, A) / (detE ** 2)[..., None, None]
        pg = np.einsum("eqla,eqac->eqlc", dB, A) / detE[..., None, None]
        T = d2B - np.einsum("eqlc,eqcab->eqlab", pg, hessE)
        lap = np.einsum("eqlab,eqab->eql", T, C)
        s = detE * wq[None, :]
        loc = _gram((lap * s[..., None])[..., None], lap[..., None])
    else:
        raise ValueError(f"unsupported square form {form}")
    # upper triangle mirrored (assembly.py:524-528)
    Lr = loc.shape[1]
    up = np.arange(Lr)[:, None] <= np.arange(Lr)[None, :]
    return np.where(up[None], loc, np.swapaxes(loc, 1, 2)), et


def elements_for_rows(ms, p, rows):
    """Ascending colex ids of elements supporting any of ``rows`` (assembly.py:347-360).

    Computed as a separable box dilation of the row mask instead of a loop.
    """
    ms = tuple(ms)
    n = len(ms)
    spans = tuple(m - p for m in ms)
    rmask = np.zeros(int(np.prod(ms)), dtype=bool)
    rmask[np.asarray(rows, dtype=np.int64)] = True
    R = rmask.reshape(ms, order="F")
    # element e touches rows e..e+p per direction
    for d in range(n):
        R = np.moveaxis(R, d, 0)
        acc = np.zeros((spans[d],) + R.shape[1:], dtype=bool)
        for r in range(p + 1):
            acc |= R[r:r + spans[d]]
        R = np.moveaxis(acc, 0, d)
    return np.flatnonzero(R.ravel(order="F"))


def assemble(prob: Problem, rows=None, chunk=4096):
    """Full or row-restricted Galerkin matrix (assembly.py:579-651).

    Returns ``(indptr, indices, data, symmetric, populated_rows)``.
    """
    if prob.form == "biharmonic" and prob.p < 2:
        raise ValueError("the fourth-order form needs degree >= 2 for C^1 continuity")
    if prob.coefficient != 1.0 and prob.form not in ("poisson", "stokes_velocity"):
        raise ValueError("coefficient is only supported for the second-order forms")
    n, p = prob.n, prob.p
    ms = prob.ms
    N = prob.N
    if rows is None:
        eids = np.arange(int(np.prod(prob.spans)))
        rowsel = None
    else:
        rowsel = np.unique(np.asarray(rows, dtype=np.int64))
        if rowsel.size and (rowsel[0] < 0 or rowsel[-1] >= N):
            raise ValueError("row index out of range")
        eids = elements_for_rows(ms, p, rowsel) if rowsel.size else np.zeros(0, np.int64)
    indptr, indices = pattern(ms, p, rowsel)
    data = np.zeros(indices.size)
    if rowsel is not None:
        keep = np.zeros(N, dtype=bool)
        keep[rowsel] = True
    L = (p + 1) ** n
    Il = np.stack(np.unravel_index(np.arange(L), (p + 1,) * n, order="F"), axis=-1)
    strides = np.cumprod((1,) + tuple(ms[:-1]))
    for s in range(0, eids.size, chunk):
        ce = eids[s:s + chunk]
        loc, et = element_matrices(prob, ce)
        gm = et[:, None, :] + Il[None, :, :]                 # (E, L, n) global multi
        cols = (gm * strides).sum(-1)                         # (E, L)
        # position of (row=gm_l, col=gm_k) inside the CSR row of gm_l
        lo = np.maximum(gm - p, 0)
        hi = np.minimum(gm + p, np.asarray(ms) - 1)
        cnt = hi - lo + 1
        rel = gm[:, None, :, :] - lo[:, :, None, :]          # (E, Lrow, Lcol, n)
        cstr = np.concatenate([np.ones(cnt.shape[:2] + (1,), np.int64), np.cumprod(cnt[..., :-1], -1)], -1)
        colpos = (rel * cstr[:, :, None, :]).sum(-1)
        rr = np.broadcast_to(cols[:, :, None], colpos.shape)
        if rowsel is not None:
            sel = keep[rr]
        else:
            sel = np.ones(rr.shape, dtype=bool)
        pos = indptr[rr[sel]] + colpos[sel]
        data += np.bincount(pos, weights=loc[sel], minlength=data.size)
    sym = prob.form in FORMS
    return indptr, indices, data, (sym and rows is None), (None if rows is None else rowsel)


# ---------------------------------------------------------------------------
# load vector (assembly.py:728-759)
# ---------------------------------------------------------------------------

def load_vector(prob: Problem, f):
    """vec_i = sum_e sum_q f(phi(x_q)) det J(x_q) w_q N_i(x_q), N rational when the weights are not unit.

    ``f`` receives the physical points per element, shape (E, Q, n), and returns (E, Q).
    """
    n, p, g = prob.n, prob.p, prob.g
    tabs, axes, pws = _dir_tables(prob, 0)
    wq = pws[0]
    for d in range(1, n):
        wq = (pws[d][:, None] * wq[None, :]).ravel()
    spans = prob.spans
    geo = geometry_on_grid(prob, axes, 1)
    phiE = _to_elements(geo["phi"], spans, g)
    detE = _to_elements(geo["det"], spans, g)
    fb = np.asarray(f(phiE), dtype=float)
    if fb.shape != detE.shape:
        raise ValueError("load callable returned a mismatched shape")
    E = int(np.prod(spans))
    et = np.stack(np.unravel_index(np.arange(E), spans, order="F"), axis=-1)
    B = _local_tensor(tabs, et, (0,) * n, p, g)
    L = (p + 1) ** n
    Il = np.stack(np.unravel_index(np.arange(L), (p + 1,) * n, order="F"), axis=-1)
    strides = np.cumprod((1,) + tuple(prob.ms[:-1]))
    cols = ((et[:, None, :] + Il[None, :, :]) * strides).sum(-1)
    if prob.rational:
        Wf = field_on_grid(p, prob.ms, prob.sol_w[:, None], axes, 0)
        W = _to_elements(Wf[(0,) * n][..., 0], spans, g)[..., None]
        B = prob.sol_w[cols][:, None, :] * B / W
    lv = np.einsum("eq,eql->el", fb * detE * wq[None, :], B)
    vec = np.zeros(prob.N)
    np.add.at(vec, cols.ravel(), lv.ravel())
    return vec


# ---------------------------------------------------------------------------
# mixed divergence pairing (assembly.py:180-207, 654-725)
# ---------------------------------------------------------------------------

def div_col_range(mv, pp, multi):
    """Velocity columns of pressure row(s) ``multi``: j_d in [2 i_d - 2pp, 2 i_d + pp + 2] (clipped)."""
    lo = np.maximum(2 * multi - 2 * pp, 0)
    hi = np.minimum(2 * multi + pp + 2, np.asarray(mv) - 1)
    return lo, hi


def div_pattern(mp, mv, pp, rows=None):
    """indptr/indices of the pressure x velocity overlap pattern (rows restricted if given)."""
    mp, mv = tuple(mp), tuple(mv)
    Np = int(np.prod(mp))
    rsel = np.arange(Np) if rows is None else np.asarray(rows, dtype=np.int64)
    multi = np.stack(np.unravel_index(rsel, mp, order="F"), axis=-1)
    lo, hi = div_col_range(mv, pp, multi)
    cnt = np.zeros(Np, dtype=np.int64)
    cnt[rsel] = np.prod(hi - lo + 1, axis=1)
    indptr = np.zeros(Np + 1, dtype=np.int64)
    np.cumsum(cnt, out=indptr[1:])
    vstr = np.cumprod((1,) + mv[:-1])
    cols = []
    for r in range(rsel.size):
        axes = [np.arange(lo[r, d], hi[r, d] + 1) for d in range(len(mv))]
        grid = np.stack(np.meshgrid(*axes, indexing="ij"), axis=-1).reshape(-1, len(mv), order="F")
        cols.append((grid * vstr).sum(-1))
    indices = (np.concatenate(cols) if cols else np.zeros(0, np.int64)).astype(np.int32)
    return indptr, indices


def div_elements_for_rows(mp, pp, sv, rows):
    """assembly.py:347-360 with ratio 2: velocity elements [2 max(0, i-pp), 2 min(Sp-1, i) + 1] per direction."""
    mp = tuple(mp)
    n = len(mp)
    sp_ = tuple(m - pp for m in mp)
    mask = np.zeros(tuple(sv), dtype=bool)
    multi = np.stack(np.unravel_index(np.asarray(rows, dtype=np.int64), mp, order="F"), axis=-1)
    for mi in multi:
        sl = tuple(slice(2 * max(0, int(mi[d]) - pp), 2 * (min(sp_[d] - 1, int(mi[d])) + 1)) for d in range(n))
        mask[sl] = True
    return np.flatnonzero(mask.ravel(order="F"))


def divergence(vel: Problem, pp: int, rows=None, chunk=1024, prs_w=None):
    """Pressure/velocity divergence pairing, one CSR per component c (assembly.py:654-725).

    ``vel`` describes the velocity discretisation (degree pp+1 on the halved mesh, Gauss order,
    geometry); the pressure space has degree ``pp`` and half the velocity spans.  Entry (i, j) of
    component c is  sum_q w_q P_i(x_q) sum_a d_a V_j(x_q) adj(J)[a, c]  (no determinant: the
    adjugate folds it).  Rational spaces (``vel.sol_w`` / ``prs_w`` not all equal) use the NURBS
    basis R = w N / W and its quotient-rule gradient, as the reference's _SpaceBinding
    (assembly.py:400-430, 689-691) binds both spaces with their own weights.
    Returns ``(indptr, indices, [data_c for c < n], populated_rows)``.
    """
    n, pv, g = vel.n, vel.p, vel.g
    if pv != pp + 1:
        raise ValueError("velocity degree must be pressure degree + 1")
    sv = vel.spans
    if any(s % 2 for s in sv):
        raise ValueError("velocity spans must be twice the pressure spans")
    spn = tuple(s // 2 for s in sv)
    mp = tuple(s + pp for s in spn)
    mv = vel.ms
    Np = int(np.prod(mp))
    tabs_v, axes, pws = _dir_tables(vel, 1)
    tabs_p = []
    for d in range(n):
        span, ders = basis_ders(open_uniform_knots(pp, mp[d]), pp, axes[d], 0)
        assert np.array_equal(span.reshape(sv[d], g), (np.arange(sv[d]) // 2 + pp)[:, None].repeat(g, 1))
        tabs_p.append(ders.reshape(sv[d], g, 1, pp + 1))
    wq = pws[0]
    for d in range(1, n):
        wq = (pws[d][:, None] * wq[None, :]).ravel()
    geo = geometry_on_grid(vel, axes, 1)
    jacE = _to_elements(geo["jac"], sv, g)
    vrat = vel.rational
    prs_w = None if prs_w is None else np.asarray(prs_w, dtype=float)
    prat = prs_w is not None and not bool(np.all(prs_w == prs_w[0]))
    if vrat:
        Wvf = field_on_grid(pv, mv, vel.sol_w[:, None], axes, 1)
        WvE = _to_elements(Wvf[(0,) * n][..., 0], sv, g)
        dWvE = np.stack([_to_elements(Wvf[_unit(n, a)][..., 0], sv, g) for a in range(n)], axis=-1)
    if prat:
        WpE = _to_elements(field_on_grid(pp, mp, prs_w[:, None], axes, 0)[(0,) * n][..., 0], sv, g)
    if rows is None:
        eids = np.arange(int(np.prod(sv)))
        rowsel = None
    else:
        rowsel = np.unique(np.asarray(rows, dtype=np.int64))
        if rowsel.size and (rowsel[0] < 0 or rowsel[-1] >= Np):
            raise ValueError("pressure row index out of range")
        eids = div_elements_for_rows(mp, pp, sv, rowsel) if rowsel.size else np.zeros(0, np.int64)
        keep = np.zeros(Np, dtype=bool)
        keep[rowsel] = True
    indptr, indices = div_pattern(mp, mv, pp, rowsel)
    data = [np.zeros(indices.size) for _ in range(n)]
    Lp, Lv = (pp + 1) ** n, (pv + 1) ** n
    Ip = np.stack(np.unravel_index(np.arange(Lp), (pp + 1,) * n, order="F"), axis=-1)
    Iv = np.stack(np.unravel_index(np.arange(Lv), (pv + 1,) * n, order="F"), axis=-1)
    pstr = np.cumprod((1,) + mp[:-1])
    for s0 in range(0, eids.size, chunk):
        ce = eids[s0:s0 + chunk]
        et = np.stack(np.unravel_index(ce, sv, order="F"), axis=-1)
        A = adj(jacE[ce])                                    # (E, Q, a, c)
        Bp = _local_tensor(tabs_p, et, (0,) * n, pp, g)      # (E, Q, Lp)
        dV = np.stack([_local_tensor(tabs_v, et, _unit(n, a), pv, g) for a in range(n)], axis=-1)  # (E,Q,Lv,a)
        Pw = Bp * wq[None, :, None]
        gp = et[:, None, :] // 2 + Ip[None, :, :]           # pressure multi (E, Lp, n)
        gv = et[:, None, :] + Iv[None, :, :]                # velocity multi (E, Lv, n)
        rflat = (gp * pstr).sum(-1)
        if prat:  # R_l = w_l N_l / W_p
            Pw = prs_w[rflat][:, None, :] * Bp / WpE[ce][..., None] * wq[None, :, None]
        if vrat:  # d_a R_k = (w_k d_a N_k - R_k d_a W_v) / W_v
            wlv = vel.sol_w[(gv * np.cumprod((1,) + tuple(mv[:-1]))).sum(-1)][:, None, :]
            Wv = WvE[ce][..., None]
            Rv = wlv * _local_tensor(tabs_v, et, (0,) * n, pv, g) / Wv
            dV = np.stack([(wlv * dV[..., a] - Rv * dWvE[ce][..., a][..., None]) / Wv for a in range(n)], axis=-1)
        lo, hi = div_col_range(mv, pp, gp)
        cnt = hi - lo + 1
        rel = gv[:, None, :, :] - lo[:, :, None, :]          # (E, Lp, Lv, n)
        cstr = np.concatenate([np.ones(cnt.shape[:2] + (1,), np.int64), np.cumprod(cnt[..., :-1], -1)], -1)
        colpos = (rel * cstr[:, :, None, :]).sum(-1)
        rr = np.broadcast_to(rflat[:, :, None], colpos.shape)
        sel = keep[rr] if rowsel is not None else np.ones(rr.shape, dtype=bool)
        pos = indptr[rr[sel]] + colpos[sel]
        for c in range(n):
            t = np.einsum("eqka,eqa->eqk", dV, A[..., :, c])
            loc = np.einsum("eql,eqk->elk", Pw, t)
            data[c] += np.bincount(pos, weights=loc[sel], minlength=indices.size)
    return indptr, indices, data, rowsel


# ---------------------------------------------------------------------------
# surrogate (surrogate.py:36-691)
# ---------------------------------------------------------------------------

DEFAULT_MODE = {"poisson": "symmetric_kernel_preserving", "biharmonic": "symmetric_kernel_preserving",
                "mass": "symmetric", "stokes_velocity": "symmetric"}


def offsets(p, n):
    """[-p, p]^n colex (surrogate.py:103-122)."""
    rng = np.arange(-p, p + 1)
    k = rng.size
    grid = np.unravel_index(np.arange(k ** n), (k,) * n, order="F")
    return np.stack([rng[g] for g in grid], axis=-1)


def box_range(p, m):
    """In-box 0-based indices [2p, m-2p-1] (surrogate.py:150-152)."""
    return 2 * p, m - 2 * p - 1


def lattice_indices(p, m, M):
    """surrogate.py:236-253."""
    lo, hi = box_range(p, m)
    idx = np.arange(lo, hi + 1, M)
    if idx[-1] != hi:
        idx = np.append(idx, hi)
    return idx


def midpoints(p, m, idx):
    """surrogate.py:231-233: ((2i+1-p)/2) h exactly, then rounded."""
    h = Fraction(1, m - p)
    return np.array([float(Fraction(2 * int(i) + 1 - p, 2) * h) for i in idx])


def averaging_knots(sites, q):
    """surrogate.py:386-390."""
    k = sites.size
    interior = [np.mean(sites[j + 1:j + q + 1]) for j in range(k - q - 1)]
    return np.concatenate([np.full(q + 1, sites[0]), interior, np.full(q + 1, sites[-1])])


def surrogate(prob: Problem, M: int, q: int = 3, mode=None):
    """Surrogate matrix + report dict (surrogate.py:538-691)."""
    from scipy.linalg import solve

    n, p, ms = prob.n, prob.p, prob.ms
    N = prob.N
    mode = DEFAULT_MODE[prob.form] if mode is None else mode
    if mode == "symmetric_kernel_preserving" and prob.form not in ("poisson", "biharmonic"):
        raise ValueError(f"kernel-preserving mode is not defined for {prob.form}")
    h0 = 1.0 / (ms[0] - p)
    empty = any(m <= 4 * p for m in ms)
    if empty:
        ip, ix, dt, _, _ = assemble(prob)
        rep = dict(N=N, p=p, q=q, M=M, H=M * h0, quad_entries=ix.size, interp_entries=0,
                   quad_fraction=1.0, active_elements=int(np.prod(prob.spans)), flags=["surrogate=disabled"])
        return (ip, ix, dt), True, rep

    lat = [lattice_indices(p, m, M) for m in ms]
    inb = []
    smp = []
    for d, m in enumerate(ms):
        lo, hi = box_range(p, m)
        a = np.zeros(m, bool)
        a[lo:hi + 1] = True
        s = np.zeros(m, bool)
        s[lat[d]] = True
        inb.append(a)
        smp.append(s)

    def flat(masks):
        acc = np.ones(1, bool)
        for mk in masks[::-1]:
            acc = (acc[:, None] & mk[None, :]).ravel()
        return acc

    in_flat = flat(inb)
    samp_flat = flat(smp)
    quad_rows = np.flatnonzero(~in_flat | samp_flat)
    interp_rows = np.flatnonzero(in_flat & ~samp_flat)
    ipq, ixq, dq, _, _ = assemble(prob, rows=quad_rows)
    active = elements_for_rows(ms, p, quad_rows).size
    H = M * h0
    nI = interp_rows.size
    if nI == 0:
        rep = dict(N=N, p=p, q=q, M=M, H=H, quad_entries=ixq.size, interp_entries=0,
                   quad_fraction=1.0, active_elements=active, flags=[])
        return (ipq, ixq, dq), prob.form in FORMS, rep

    offs = offsets(p, n)
    P = offs.shape[0]
    center = (P - 1) // 2
    strides = np.cumprod((1,) + tuple(ms[:-1]))
    # samples: row positions o in each lattice row (surrogate.py:336-379)
    lat_grid = np.stack([g.ravel(order="F") for g in np.meshgrid(*lat, indexing="ij")], -1)
    lat_rows = lat_grid @ strides
    assert np.all(np.diff(ipq)[lat_rows] == P)
    S = dq[ipq[lat_rows][:, None] + np.arange(P)[None, :]]           # (nlat, P)
    lat_shape = tuple(x.size for x in lat)
    coef = S.T.reshape((P,) + lat_shape, order="F")                 # (P, l0, l1, ...)

    flags = []
    qd, kn = [], []
    for d in range(n):
        sites = midpoints(p, ms[d], lat[d])
        qq = min(q, sites.size - 1)
        if qq < q and "interpolation-order-lowered" not in flags:
            flags.append("interpolation-order-lowered")
        qd.append(qq)
        kn.append(averaging_knots(sites, qq) if qq >= 1 else None)
        if qq >= 1:
            C = collocation_matrix(kn[d], qq, sites)
            moved = np.moveaxis(coef, 1 + d, 0)
            sol = solve(C, moved.reshape(sites.size, -1))
            coef = np.moveaxis(sol.reshape(moved.shape), 0, 1 + d)
    # evaluate on all in-box midpoints
    V = coef
    box_n = []
    for d in range(n):
        lo, hi = box_range(p, ms[d])
        pts = midpoints(p, ms[d], np.arange(lo, hi + 1))
        box_n.append(pts.size)
        E = np.ones((pts.size, 1)) if kn[d] is None else collocation_matrix(kn[d], qd[d], pts)
        V = np.moveaxis(np.tensordot(E, np.moveaxis(V, 1 + d, 0), axes=(1, 0)), 0, 1 + d)
    VF = V.reshape(P, -1, order="F")
    box_str = np.cumprod((1,) + tuple(box_n[:-1]))
    Im = np.stack(np.unravel_index(interp_rows, ms, order="F"), -1)
    Ib = (Im - 2 * p) @ box_str

    # final matrix = quad rows from Aq, interp rows filled per offset
    indptr, indices = pattern(ms, p)
    data = np.zeros(indices.size)
    rowid = np.repeat(np.arange(N), np.diff(indptr))
    isq = np.zeros(N, dtype=bool)
    isq[quad_rows] = True
    data[isq[rowid]] = dq
    canonical_from = center
    offd = np.zeros(nI, np.int64)
    n_interp = 0
    for o in range(P):
        sh = offs[o]
        jm = Im + sh[None, :]
        jflat = jm @ strides
        jin = np.ones(nI, bool)
        jsm = np.ones(nI, bool)
        for d in range(n):
            jin &= inb[d][jm[:, d]]
            jsm &= smp[d][jm[:, d]]
        jint = jin & ~jsm
        vals = np.empty(nI)
        t = ~jint
        vals[t] = dq[ipq[jflat[t]] + (P - 1 - o)]
        if mode == "general" or o >= canonical_from:
            vals[jint] = VF[o, Ib[jint]]
        else:
            jb = (jm[jint] - 2 * p) @ box_str
            vals[jint] = VF[P - 1 - o, jb]
        if o != center:
            offd[jint] += 1
        n_interp += int(jint.sum())
        data[indptr[interp_rows] + o] = vals
    # merge drops exact zeros (scipy csr add, surrogate.py:670)
    nz = data != 0.0
    if not np.all(nz):
        keep_cnt = np.add.reduceat(nz.astype(np.int64), indptr[:-1]) * (np.diff(indptr) > 0)
        new_ip = np.zeros_like(indptr)
        np.cumsum(keep_cnt, out=new_ip[1:])
        indices, data, indptr = indices[nz], data[nz], new_ip
    if mode == "symmetric_kernel_preserving":
        reset = interp_rows[offd > 0]
        if reset.size:
            take = indptr[reset][:, None] + np.arange(P)[None, :]
            rv = data[take]
            data[indptr[reset] + center] = rv[:, center] - rv.sum(axis=1)
    quad_entries = int(ixq.size + nI * P - n_interp)
    rep = dict(N=N, p=p, q=q, M=M, H=H, quad_entries=quad_entries, interp_entries=n_interp,
               quad_fraction=quad_entries / (quad_entries + n_interp), active_elements=int(active), flags=flags)
    return (indptr, indices, data), mode in ("symmetric", "symmetric_kernel_preserving"), rep


# ---------------------------------------------------------------------------
# sampled-row surrogate: selected rows of the surrogate matrix at sizes where the whole
# matrix is out of reach of a CPU oracle (config 5: 741M nnz)
# ---------------------------------------------------------------------------

def _assemble_rows_local(prob: Problem, rows):
    """Full-quadrature rows ``rows`` (sorted, unique) as (cnt, cols, vals), without any O(N) array.

    Same element sums as ``assemble(prob, rows=rows)`` (assembly.py:579-651): every element
    supporting a row contributes its local row, in ascending element order.
    """
    n, p, ms = prob.n, prob.p, prob.ms
    spans = np.asarray(prob.spans)
    rows = np.asarray(rows, dtype=np.int64)
    strides = np.cumprod((1,) + tuple(ms[:-1]))
    multi = np.stack(np.unravel_index(rows, ms, order="F"), axis=-1)
    lo, hi = row_col_range(ms, p, multi)
    cnt = np.prod(hi - lo + 1, axis=1)
    start = np.zeros(rows.size + 1, np.int64)
    np.cumsum(cnt, out=start[1:])
    L = (p + 1) ** n
    Il = np.stack(np.unravel_index(np.arange(L), (p + 1,) * n, order="F"), axis=-1)
    em = multi[:, None, :] - Il[None, :, :]
    ok = np.all((em >= 0) & (em < spans), axis=-1)
    eids = np.unique((em[ok] * np.cumprod((1,) + tuple(spans[:-1]))).sum(-1))
    vals = np.zeros(start[-1])
    loc, et = element_matrices(prob, eids)
    gm = et[:, None, :] + Il[None, :, :]                       # (E, L, n)
    grow = (gm * strides).sum(-1)                               # (E, L) global row of local l
    k = np.searchsorted(rows, grow)
    k = np.minimum(k, rows.size - 1)
    hit = rows[k] == grow                                       # local row l of element e is requested
    ee, ll = np.nonzero(hit)
    rr = k[ee, ll]
    # position of column gm[e, kc] inside row rr's segment
    rel = gm[ee][:, :, :] - lo[rr][:, None, :]                  # (H, L, n)
    cs = np.concatenate([np.ones((rr.size, 1), np.int64), np.cumprod((hi - lo + 1)[rr][:, :-1], -1)], -1)
    pos = start[rr][:, None] + (rel * cs[:, None, :]).sum(-1)
    vals += np.bincount(pos.ravel(), weights=loc[ee, ll].ravel(), minlength=vals.size)
    cols = []
    offs = offsets(p, n)
    for r in range(rows.size):
        jm = multi[r] + offs
        inside = np.all((jm >= 0) & (jm < np.asarray(ms)), axis=-1)
        cols.append((jm[inside] * strides).sum(-1))
    return cnt, (np.concatenate(cols) if cols else np.zeros(0, np.int64)), vals


def assemble_rows_grouped(prob: Problem, rows, lines_per_group=8):
    """``_assemble_rows_local`` over spatially local groups of rows (rows sharing their slower
    indices up to blocks of ``lines_per_group``), so the geometry of each batch stays on a small
    sub-grid.  Returns a dict row -> (cols, vals)."""
    rows = np.unique(np.asarray(rows, dtype=np.int64))
    ms = prob.ms
    multi = np.stack(np.unravel_index(rows, ms, order="F"), axis=-1)
    key = multi[:, 1:] // lines_per_group if prob.n > 1 else np.zeros((rows.size, 1), np.int64)
    out = {}
    _, inv = np.unique(key, axis=0, return_inverse=True)
    for gidx in np.unique(inv):
        grp = rows[inv.ravel() == gidx]
        cnt, cols, vals = _assemble_rows_local(prob, grp)
        s = 0
        for r, c in zip(grp, cnt):
            out[int(r)] = (cols[s:s + c], vals[s:s + c])
            s += c
    return out


def surrogate_rows(prob: Problem, M: int, q: int = 3, mode=None, rows=None):
    """Rows ``rows`` of ``surrogate(prob, M, q, mode)`` without building the whole matrix.

    Follows surrogate.py:538-691 for the requested rows only: the lattice rows and the
    quadrature neighbours of the requested interpolated rows are assembled by quadrature
    (``assemble_rows_grouped``), the stencil interpolant is fitted exactly as in ``surrogate``
    (same collocation solves), evaluated only at the box points the rows need, and the placement
    (quadrature transposes / canonical / symmetric copies, surrogate.py:611-667) and the
    kernel-preserving diagonal reset (surrogate.py:673-680) are applied per row.  Exact-zero drop
    (surrogate.py:670) is not modelled: a requested row that would drop a zero raises.

    Returns ``(rows, cnt, cols, vals)`` (rows sorted) and the row classes ``{"interp": mask}``.
    """
    from scipy.linalg import solve

    n, p, ms = prob.n, prob.p, prob.ms
    mode = DEFAULT_MODE[prob.form] if mode is None else mode
    rows = np.unique(np.asarray(rows, dtype=np.int64))
    if any(m <= 4 * p for m in ms):
        got = assemble_rows_grouped(prob, rows)
        cnt = np.array([got[int(r)][0].size for r in rows])
        return (rows, cnt, np.concatenate([got[int(r)][0] for r in rows]),
                np.concatenate([got[int(r)][1] for r in rows])), {"interp": np.zeros(rows.size, bool)}
    lat = [lattice_indices(p, m, M) for m in ms]
    inb, smp = [], []
    for d, m in enumerate(ms):
        lo, hi = box_range(p, m)
        a = np.zeros(m, bool)
        a[lo:hi + 1] = True
        s = np.zeros(m, bool)
        s[lat[d]] = True
        inb.append(a)
        smp.append(s)

    def is_interp(mult):
        jin = np.ones(mult.shape[0], bool)
        jsm = np.ones(mult.shape[0], bool)
        for d in range(n):
            jin &= inb[d][mult[:, d]]
            jsm &= smp[d][mult[:, d]]
        return jin & ~jsm

    offs = offsets(p, n)
    P = offs.shape[0]
    center = (P - 1) // 2
    strides = np.cumprod((1,) + tuple(ms[:-1]))
    multi = np.stack(np.unravel_index(rows, ms, order="F"), axis=-1)
    interp = is_interp(multi)
    Im = multi[interp]
    # quadrature rows needed: every lattice row (the samples), the requested quadrature rows and the
    # quadrature neighbours of the requested interpolated rows (their transposed entries)
    lat_grid = np.stack([g.ravel(order="F") for g in np.meshgrid(*lat, indexing="ij")], -1)
    lat_rows = lat_grid @ strides
    need = [lat_rows, rows[~interp]]
    jm_all = Im[:, None, :] + offs[None, :, :]                  # (nI, P, n)
    jint_all = is_interp(jm_all.reshape(-1, n)).reshape(Im.shape[0], P)
    need.append((jm_all[~jint_all] * strides).sum(-1))
    qv = assemble_rows_grouped(prob, np.concatenate(need))

    S = np.stack([qv[int(r)][1] for r in lat_rows])             # (nlat, P): lattice rows are full
    assert S.shape[1] == P
    lat_shape = tuple(x.size for x in lat)
    coef = S.T.reshape((P,) + lat_shape, order="F")
    qd, kn = [], []
    for d in range(n):
        sites = midpoints(p, ms[d], lat[d])
        qq = min(q, sites.size - 1)
        qd.append(qq)
        kn.append(averaging_knots(sites, qq) if qq >= 1 else None)
        if qq >= 1:
            C = collocation_matrix(kn[d], qq, sites)
            moved = np.moveaxis(coef, 1 + d, 0)
            sol = solve(C, moved.reshape(sites.size, -1))
            coef = np.moveaxis(sol.reshape(moved.shape), 0, 1 + d)
    Ed = []
    for d in range(n):
        lo, hi = box_range(p, ms[d])
        pts = midpoints(p, ms[d], np.arange(lo, hi + 1))
        Ed.append(np.ones((pts.size, 1)) if kn[d] is None else collocation_matrix(kn[d], qd[d], pts))

    def V(o, bm):
        """Interpolant of offset o at box multi-indices bm (k, n): directions contracted in order."""
        t = np.broadcast_to(coef[o], (bm.shape[0],) + coef.shape[1:])
        for d in range(n):
            t = np.einsum("kr,kr...->k...", Ed[d][bm[:, d]], t)
        return t

    out_cnt, out_cols, out_vals = [], [], []
    ii = 0
    for r, mlt, isi in zip(rows, multi, interp):
        if not isi:
            c, v = qv[int(r)]
            out_cnt.append(c.size)
            out_cols.append(c)
            out_vals.append(v)
            continue
        jm = jm_all[ii]
        jint = jint_all[ii]
        ii += 1
        vals = np.empty(P)
        for o in np.flatnonzero(~jint):
            vals[o] = qv[int(jm[o] @ strides)][1][P - 1 - o]
        bi = (mlt - 2 * p)[None, :]
        for o in np.flatnonzero(jint):
            if mode == "general" or o >= center:
                vals[o] = V(o, bi)[0]
            else:
                vals[o] = V(P - 1 - o, (jm[o] - 2 * p)[None, :])[0]
        if np.any(vals == 0.0):
            raise ValueError(f"row {r}: exact zero (the merge would drop it); not modelled here")
        offd = int(jint.sum()) - int(jint[center])
        if mode == "symmetric_kernel_preserving" and offd > 0:
            vals[center] = vals[center] - vals.sum()
        out_cnt.append(P)
        out_cols.append((jm * strides).sum(-1))
        out_vals.append(vals)
    return (rows, np.array(out_cnt, np.int64), np.concatenate(out_cols), np.concatenate(out_vals)), \
        {"interp": interp}


def surrogate_divergence(vel: Problem, pp: int, M: int, q: int = 3, prs_w=None):
    """Surrogate divergence pairing, general mode only (surrogate.py:702-819).

    Returns ``([(indptr, indices, data) per component], report dict)``.
    """
    from scipy.linalg import solve

    n, pv = vel.n, vel.p
    sv = vel.spans
    mp = tuple(s // 2 + pp for s in sv)
    mv = vel.ms
    Np = int(np.prod(mp))
    h0 = 1.0 / (mp[0] - pp)
    if any(m <= 4 * pp for m in mp):
        ip, ix, data, _ = divergence(vel, pp, prs_w=prs_w)
        rep = dict(N=Np, p=pp, q=q, M=M, H=M * h0, quad_entries=ix.size * n, interp_entries=0, quad_fraction=1.0,
                   active_elements=int(np.prod(sv)), flags=["surrogate=disabled"])
        return [(ip, ix, d) for d in data], rep
    lat = [lattice_indices(pp, m, M) for m in mp]
    core, smp = [], []
    for d, m in enumerate(mp):
        lo, hi = box_range(pp, m)
        a = np.zeros(m, bool)
        if lo + 1 <= hi - 1:
            a[lo + 1:hi] = True
        sm_ = np.zeros(m, bool)
        sm_[lat[d]] = True
        core.append(a)
        smp.append(sm_)

    def flat(masks):
        acc = np.ones(1, bool)
        for mk in masks[::-1]:
            acc = (acc[:, None] & mk[None, :]).ravel()
        return acc

    core_flat, samp_flat = flat(core), flat(smp)
    quad_rows = np.flatnonzero(~core_flat | samp_flat)
    interp_rows = np.flatnonzero(core_flat & ~samp_flat)
    ipq, ixq, dq, _ = divergence(vel, pp, rows=quad_rows, prs_w=prs_w)
    active = div_elements_for_rows(mp, pp, sv, quad_rows).size
    H = M * h0
    nI = interp_rows.size
    if nI == 0:
        rep = dict(N=Np, p=pp, q=q, M=M, H=H, quad_entries=ixq.size * n, interp_entries=0, quad_fraction=1.0,
                   active_elements=int(active), flags=[])
        return [(ipq, ixq, d) for d in dq], rep
    rng = np.arange(-2 * pp, pp + 3)
    k = rng.size
    offs = np.stack([rng[g] for g in np.unravel_index(np.arange(k ** n), (k,) * n, order="F")], -1)
    P = offs.shape[0]
    pstr = np.cumprod((1,) + mp[:-1])
    vstr = np.cumprod((1,) + tuple(mv[:-1]))
    lat_grid = np.stack([g.ravel(order="F") for g in np.meshgrid(*lat, indexing="ij")], -1)
    lat_rows = lat_grid @ pstr
    assert np.all(np.diff(ipq)[lat_rows] == P)
    lat_shape = tuple(x.size for x in lat)
    flags = []
    qd, kn, Es = [], [], []
    box_n = []
    for d in range(n):
        sites = midpoints(pp, mp[d], lat[d])
        qq = min(q, sites.size - 1)
        if qq < q and "interpolation-order-lowered" not in flags:
            flags.append("interpolation-order-lowered")
        qd.append(qq)
        kn.append(averaging_knots(sites, qq) if qq >= 1 else None)
        lo, hi = box_range(pp, mp[d])
        pts = midpoints(pp, mp[d], np.arange(lo, hi + 1))
        box_n.append(pts.size)
        Es.append(np.ones((pts.size, 1)) if kn[d] is None else collocation_matrix(kn[d], qq, pts))
    box_str = np.cumprod((1,) + tuple(box_n[:-1]))
    Im = np.stack(np.unravel_index(interp_rows, mp, order="F"), -1)
    Ib = (Im - 2 * pp) @ box_str
    indptr, indices = div_pattern(mp, mv, pp)
    rowid = np.repeat(np.arange(Np), np.diff(indptr))
    isq = np.zeros(Np, dtype=bool)
    isq[quad_rows] = True
    out = []
    for c in range(n):
        coef = dq[c][ipq[lat_rows][:, None] + np.arange(P)[None, :]].T.reshape((P,) + lat_shape, order="F")
        for d in range(n):
            if qd[d] >= 1:
                sites = midpoints(pp, mp[d], lat[d])
                C = collocation_matrix(kn[d], qd[d], sites)
                moved = np.moveaxis(coef, 1 + d, 0)
                coef = np.moveaxis(solve(C, moved.reshape(sites.size, -1)).reshape(moved.shape), 0, 1 + d)
        V = coef
        for d in range(n):
            V = np.moveaxis(np.tensordot(Es[d], np.moveaxis(V, 1 + d, 0), axes=(1, 0)), 0, 1 + d)
        VF = V.reshape(P, -1, order="F")
        data = np.zeros(indices.size)
        data[isq[rowid]] = dq[c]
        data[indptr[interp_rows][:, None] + np.arange(P)[None, :]] = VF[:, Ib].T
        ip_c, ix_c = indptr, indices
        nz = data != 0.0                       # scipy CSR add drops exact zeros (surrogate.py:810)
        if not np.all(nz):
            cnt = np.add.reduceat(nz.astype(np.int64), indptr[:-1]) * (np.diff(indptr) > 0)
            ip_c = np.zeros_like(indptr)
            np.cumsum(cnt, out=ip_c[1:])
            ix_c, data = indices[nz], data[nz]
        out.append((ip_c, ix_c, data))
    quad_entries = int(ixq.size * n)
    n_interp = int(nI * P * n)
    rep = dict(N=Np, p=pp, q=q, M=M, H=H, quad_entries=quad_entries, interp_entries=n_interp,
               quad_fraction=quad_entries / (quad_entries + n_interp), active_elements=int(active), flags=flags)
    return out, rep


# ---------------------------------------------------------------------------
# comparisons
# ---------------------------------------------------------------------------

def row_scaled_error(ipA, ixA, dA, ipB, ixB, dB):
    """max_ij |A_ij - B_ij| / max_k |A_ik| (patterns must already agree)."""
    if not (np.array_equal(ipA, ipB) and np.array_equal(ixA, ixB)):
        return np.inf
    if dA.size == 0:
        return 0.0
    cnt = np.diff(ipA)
    rows = np.repeat(np.arange(cnt.size), cnt)
    scale = np.zeros(cnt.size)
    np.maximum.at(scale, rows, np.abs(dA))
    err = np.abs(dA - dB) / np.where(scale[rows] > 0, scale[rows], 1.0)
    return float(err.max())


# ---------------------------------------------------------------------------
# conjugate gradient (the device-resident consumer of the CSR)
# ---------------------------------------------------------------------------

def conjugate_gradient(indptr, indices, data, rhs, tol, maxit=None, preconditioner="none"):
    """solvers.py:118-155 restated: x0 = 0, stop when |r| <= tol |b|.

    Returns ``(x, status, iterations)`` with status "converged", "negative-curvature" (at
    ``iterations``), "non-positive-diagonal" or "max-iterations" instead of raising, so the GPU
    tests can compare the outcome as well as the iterate.
    """
    import scipy.sparse as sp

    n = rhs.size
    mat = sp.csr_matrix((data, indices, indptr), shape=(n, n))
    maxit = 10 * n if maxit is None else maxit
    if preconditioner == "diagonal":
        diag = mat.diagonal()
        if np.any(diag <= 0.0):
            return np.zeros(n), "non-positive-diagonal", 0
        prec = lambda r: r / diag  # noqa: E731
    else:
        prec = lambda r: r  # noqa: E731
    target = tol * np.linalg.norm(rhs)
    x = np.zeros(n)
    r = rhs.copy()
    z = prec(r)
    d = z.copy()
    rz = r @ z
    for it in range(1, maxit + 1):
        Ad = mat @ d
        curv = d @ Ad
        if curv <= 0.0:
            return x, "negative-curvature", it
        alpha = rz / curv
        x += alpha * d
        r -= alpha * Ad
        if np.linalg.norm(r) <= target:
            return x, "converged", it
        z = prec(r)
        rz_new = r @ z
        d = z + (rz_new / rz) * d
        rz = rz_new
    return x, "max-iterations", maxit


# ---------------------------------------------------------------------------
# quadrature fields (assembly.py:839-907)
# ---------------------------------------------------------------------------

def quadrature_fields(prob: Problem, coefs, nu=0):
    """(x, w, vals, grads, hesses) element-major, as assembly.py:839-907 returns them.

    The field is evaluated as the weighted numerator over the weight function (the reference's
    rational basis contracted with the coefficients, assembly.py:496-517, 891-903).
    """
    n, p, g = prob.n, prob.p, prob.g
    _, axes, pws = _dir_tables(prob, 0)
    wq = pws[0]
    for d in range(1, n):
        wq = (pws[d][:, None] * wq[None, :]).ravel()
    spans = prob.spans
    geo = geometry_on_grid(prob, axes, 2 if nu >= 2 else 1)
    coefs = np.asarray(coefs, dtype=float).ravel()
    w = prob.sol_w if prob.rational else np.ones(prob.N)
    f = field_on_grid(p, prob.ms, np.stack([coefs * w, w], axis=1), axes, nu)
    z = (0,) * n
    U, W = f[z][..., 0], f[z][..., 1]
    u = U / W
    E = lambda a: _to_elements(a, spans, g)  # noqa: E731
    detg = geo["det"]
    x = E(geo["phi"]).reshape(-1, n)
    wts = (wq[None, :] * E(detg)).ravel()
    vals = E(u).ravel()
    grads = hesses = None
    if nu >= 1:
        du = np.stack([(f[_unit(n, a)][..., 0] - u * f[_unit(n, a)][..., 1]) / W for a in range(n)], axis=-1)
        A = adj(geo["jac"])
        gph = np.einsum("...a,...ac->...c", du, A) / detg[..., None]
        grads = E(gph).reshape(-1, n)
    if nu >= 2:
        d2u = np.empty(u.shape + (n, n))
        for a in range(n):
            for b in range(n):
                fab = f[_pair(n, a, b)]
                d2u[..., a, b] = (fab[..., 0] - du[..., a] * f[_unit(n, b)][..., 1] - du[..., b] * f[_unit(n, a)][..., 1]
                                  - u * fab[..., 1]) / W
        T = d2u - np.einsum("...c,...cab->...ab", gph, geo["hess"])
        H = np.einsum("...ac,...ab,...bd->...cd", A, T, A) / (detg ** 2)[..., None, None]
        hesses = E(H).reshape(-1, n, n)
    return x, wts, vals, grads, hesses
