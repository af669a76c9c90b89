// Mixed divergence pairing (reference: surriga/assembly.py:180-207 StokesSpaces /
// stokes_subgrid_spaces, :654-725 assemble_divergence), one CSR per velocity component c:
//
//     D^c[i, j] = sum_q  w_q P_i(x_q)  sum_a d_a V_j(x_q) adj(J)(x_q)[a, c]
//
// rows i: pressure functions (degree pp, spans S), columns j: velocity functions (degree pp+1 on
// the halved mesh, spans 2S), quadrature on the velocity elements (velocity Gauss order).
//
//   KD1 div_geom    : adjugate of the map Jacobian times the point weight, once per Gauss point
//   KD2 div_local   : element matrices loc[e][c][l][k] (one CTA per element, the reference's
//                     per-element einsum, assembly.py:700-706)
//   KD3 div_counts  : row lengts prod_d (hi_d - lo_d + 1), j_d in [2 i_d - 2pp, 2 i_d + pp + 2]
//   KD4 div_gather  : one warp per pressure row, lanes on its columns; every entry sums its
//                     elements' contributions in ascending element order (atomics-free: a
//                     row-restricted assembly equals the full one bit for bit, test_assembly.py:173-178)
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "../../include/surriga_b200.h"
#include "sg_common.cuh"
#include "sg_internal.h"

namespace sg {

struct DivParams {
    int n, pp, pv, pg, g;
    int Sv[3], Sp[3], mp[3], mv[3], mg[3];
    int G[3];                      // velocity Gauss points per direction (Sv * g)
    const double* V[3];            // velocity tables [G][2][pv+1]
    const double* Pt[3];           // pressure tables at the velocity points [G][pp+1]
    const double* Gt[3];           // geometry tables [G][2][pg+1]
    const int* gspan[3];
    const double* qw[3];
    const double* hom;             // [Ng][n+1] homogeneous control points (colex)
    double* Dg;                    // [npts][na][n]: w_q adj[a][c] (rational: see div_geom_kernel)
    int na;                        // a-terms per point: n, or n + 1 for a rational velocity space
    const double* wv;              // velocity weights (colex, device) or nullptr (B-spline space)
    const double* wp;              // pressure weights (colex, device) or nullptr
    const int64_t* elems;          // element ids (colex over velocity elements), ascending
    int64_t nelem;
    const int* eslot;              // element id -> slot (-1: not computed); nullptr = identity
    double* eloc;                  // [slot][c][Lp][Lv]
    const uint8_t* rowmask;        // pressure rows to assemble (nullptr = all)
    const uint8_t* countmask;      // rows present in the CSR pattern (nullptr = all)
    const int64_t* rowstart;
    int* indices[3];
    double* data[3];
    int64_t Np;
};

template <int NDIM>
__global__ void div_geom_kernel(DivParams s) {
    const int64_t npts = (int64_t)s.G[0] * (NDIM >= 2 ? s.G[1] : 1) * (NDIM >= 3 ? s.G[2] : 1);
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= npts) return;
    int x[3] = {0, 0, 0};
    x[0] = (int)(t % s.G[0]);
    if (NDIM >= 2) x[1] = (int)((t / s.G[0]) % s.G[1]);
    if (NDIM >= 3) x[2] = (int)(t / ((int64_t)s.G[0] * s.G[1]));
    const int pg = s.pg;
    // homogeneous field and its first derivatives: num[comp][code], code 0 = value, 1 + a = d_a
    double num[NDIM + 1][NDIM + 1];
#pragma unroll
    for (int c = 0; c <= NDIM; ++c)
#pragma unroll
        for (int k = 0; k <= NDIM; ++k) num[c][k] = 0.0;
    const int s0 = s.gspan[0][x[0]], s1 = NDIM >= 2 ? s.gspan[1][x[1]] : 0, s2 = NDIM >= 3 ? s.gspan[2][x[2]] : 0;
    const double* g0 = s.Gt[0] + (int64_t)x[0] * 2 * (pg + 1);
    const double* g1 = NDIM >= 2 ? s.Gt[1] + (int64_t)x[1] * 2 * (pg + 1) : nullptr;
    const double* g2 = NDIM >= 3 ? s.Gt[2] + (int64_t)x[2] * 2 * (pg + 1) : nullptr;
    for (int t2 = 0; t2 <= (NDIM >= 3 ? pg : 0); ++t2)
        for (int t1 = 0; t1 <= (NDIM >= 2 ? pg : 0); ++t1)
            for (int t0 = 0; t0 <= pg; ++t0) {
                const int64_t ci = (int64_t)(s0 - pg + t0) +
                                   (int64_t)s.mg[0] * ((NDIM >= 2 ? (int64_t)(s1 - pg + t1) : 0) +
                                                       (int64_t)s.mg[1] * (NDIM >= 3 ? (int64_t)(s2 - pg + t2) : 0));
                double b[NDIM + 1];
                const double v0 = g0[t0], d0 = g0[pg + 1 + t0];
                const double v1 = NDIM >= 2 ? g1[t1] : 1.0, d1 = NDIM >= 2 ? g1[pg + 1 + t1] : 0.0;
                const double v2 = NDIM >= 3 ? g2[t2] : 1.0, d2 = NDIM >= 3 ? g2[pg + 1 + t2] : 0.0;
                b[0] = v0 * v1 * v2;
                b[1] = d0 * v1 * v2;
                if (NDIM >= 2) b[2] = v0 * d1 * v2;
                if (NDIM >= 3) b[3] = v0 * v1 * d2;
#pragma unroll
                for (int c = 0; c <= NDIM; ++c) {
                    const double h = s.hom[ci * (NDIM + 1) + c];
#pragma unroll
                    for (int k = 0; k <= NDIM; ++k) num[c][k] = fma(b[k], h, num[c][k]);
                }
            }
    const double W = num[NDIM][0], iW = 1.0 / W;
    double phi[NDIM], jac[NDIM][NDIM];
#pragma unroll
    for (int c = 0; c < NDIM; ++c) phi[c] = num[c][0] * iW;
#pragma unroll
    for (int a = 0; a < NDIM; ++a)
#pragma unroll
        for (int c = 0; c < NDIM; ++c) jac[c][a] = (num[c][1 + a] - phi[c] * num[NDIM][1 + a]) * iW;
    double adj[NDIM][NDIM];
    if constexpr (NDIM == 1) {
        adj[0][0] = 1.0;
    } else if constexpr (NDIM == 2) {
        adj[0][0] = jac[1][1];
        adj[0][1] = -jac[0][1];
        adj[1][0] = -jac[1][0];
        adj[1][1] = jac[0][0];
    } else {
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) {
                const int r0 = b == 0 ? 1 : 0, r1 = b == 2 ? 1 : 2;
                const int c0 = a == 0 ? 1 : 0, c1 = a == 2 ? 1 : 2;
                const double minor = jac[r0][c0] * jac[r1][c1] - jac[r0][c1] * jac[r1][c0];
                adj[a][b] = ((a + b) & 1) ? -minor : minor;
            }
    }
    double wq = s.qw[0][x[0] % s.g];
    if (NDIM >= 2) wq *= s.qw[1][x[1] % s.g];
    if (NDIM >= 3) wq *= s.qw[2][x[2] % s.g];
    if (!s.wv && !s.wp) {
        double* out = s.Dg + t * NDIM * NDIM;
#pragma unroll
        for (int a = 0; a < NDIM; ++a)
#pragma unroll
            for (int c = 0; c < NDIM; ++c) out[a * NDIM + c] = wq * adj[a][c];
        return;
    }
    // NURBS spaces (assembly.py:400-430 via _SpaceBinding): R_l = w_l N_l / W_p for the pressure,
    // d_a R_k = w_k (d_a N_k / W_v - N_k d_a W_v / W_v^2) for the velocity.  The global weights
    // w_l w_k are applied at the gather; here the point factors: a < n carries
    // w_q adj[a][c] / (W_p W_v) against d_a N_k, the extra term a = n carries
    // -w_q sum_b d_b W_v adj[b][c] / (W_p W_v^2) against N_k.
    double Wv = 1.0, dWv[NDIM], Wp = 1.0;
#pragma unroll
    for (int a = 0; a < NDIM; ++a) dWv[a] = 0.0;
    int ev[3] = {0, 0, 0};
    for (int d = 0; d < NDIM; ++d) ev[d] = x[d] / s.g;  // velocity element = first local function
    if (s.wv) {
        const int pv = s.pv;
        Wv = 0.0;
        for (int t2 = 0; t2 <= (NDIM >= 3 ? pv : 0); ++t2)
            for (int t1 = 0; t1 <= (NDIM >= 2 ? pv : 0); ++t1)
                for (int t0 = 0; t0 <= pv; ++t0) {
                    const int tt[3] = {t0, t1, t2};
                    const int64_t ci = (int64_t)(ev[0] + t0) +
                                       (int64_t)s.mv[0] * ((NDIM >= 2 ? (int64_t)(ev[1] + t1) : 0) +
                                                           (int64_t)s.mv[1] * (NDIM >= 3 ? (int64_t)(ev[2] + t2) : 0));
                    const double w = s.wv[ci];
                    double val[NDIM], der[NDIM];
#pragma unroll
                    for (int d = 0; d < NDIM; ++d) {
                        const double* vt = s.V[d] + (int64_t)x[d] * 2 * (pv + 1);
                        val[d] = vt[tt[d]];
                        der[d] = vt[pv + 1 + tt[d]];
                    }
                    double b = w;
#pragma unroll
                    for (int d = 0; d < NDIM; ++d) b *= val[d];
                    Wv += b;
#pragma unroll
                    for (int a = 0; a < NDIM; ++a) {
                        double db = w;
#pragma unroll
                        for (int d = 0; d < NDIM; ++d) db *= d == a ? der[d] : val[d];
                        dWv[a] += db;
                    }
                }
    }
    if (s.wp) {
        const int pp = s.pp;
        Wp = 0.0;
        for (int t2 = 0; t2 <= (NDIM >= 3 ? pp : 0); ++t2)
            for (int t1 = 0; t1 <= (NDIM >= 2 ? pp : 0); ++t1)
                for (int t0 = 0; t0 <= pp; ++t0) {
                    const int tt[3] = {t0, t1, t2};
                    const int64_t ci = (int64_t)(ev[0] / 2 + t0) +
                                       (int64_t)s.mp[0] * ((NDIM >= 2 ? (int64_t)(ev[1] / 2 + t1) : 0) +
                                                           (int64_t)s.mp[1] * (NDIM >= 3 ? (int64_t)(ev[2] / 2 + t2) : 0));
                    double b = s.wp[ci];
#pragma unroll
                    for (int d = 0; d < NDIM; ++d) b *= s.Pt[d][(int64_t)x[d] * (pp + 1) + tt[d]];
                    Wp += b;
                }
    }
    const double f = wq / (Wp * Wv);
    double* out = s.Dg + t * s.na * NDIM;
#pragma unroll
    for (int a = 0; a < NDIM; ++a)
#pragma unroll
        for (int c = 0; c < NDIM; ++c) out[a * NDIM + c] = f * adj[a][c];
    if (s.na > NDIM) {
#pragma unroll
        for (int c = 0; c < NDIM; ++c) {
            double g = 0.0;
#pragma unroll
            for (int b = 0; b < NDIM; ++b) g = fma(dWv[b], adj[b][c], g);
            out[NDIM * NDIM + c] = -f * g / Wv;
        }
    }
}

// one CTA per element: loc[c][l][k] = sum_q P_l(q) sum_a dV_k^a(q) Dg(q)[a][c]
template <int NDIM>
__global__ void __launch_bounds__(256) div_local_kernel(DivParams s) {
    extern __shared__ double sm[];
    const int pp = s.pp, pv = s.pv, g = s.g;
    const int Q = NDIM == 1 ? g : (NDIM == 2 ? g * g : g * g * g);
    double* Pt = sm;                                  // [d][g][pp+1]
    double* Vt = Pt + NDIM * g * (pp + 1);            // [d][g][2][pv+1]
    double* Dq = Vt + NDIM * g * 2 * (pv + 1);        // [Q][na][NDIM]
    const int NA = s.na, NAN_ = NA * NDIM;
    const int64_t eid = s.elems[blockIdx.x];
    int e[3] = {0, 0, 0};
    e[0] = (int)(eid % s.Sv[0]);
    if (NDIM >= 2) e[1] = (int)((eid / s.Sv[0]) % s.Sv[1]);
    if (NDIM >= 3) e[2] = (int)(eid / ((int64_t)s.Sv[0] * s.Sv[1]));
    for (int it = threadIdx.x; it < NDIM * g * (pp + 1); it += blockDim.x) {
        const int d = it / (g * (pp + 1)), r = it % (g * (pp + 1));
        Pt[it] = s.Pt[d][(int64_t)e[d] * g * (pp + 1) + r];
    }
    for (int it = threadIdx.x; it < NDIM * g * 2 * (pv + 1); it += blockDim.x) {
        const int d = it / (g * 2 * (pv + 1)), r = it % (g * 2 * (pv + 1));
        Vt[it] = s.V[d][(int64_t)e[d] * g * 2 * (pv + 1) + r];
    }
    for (int it = threadIdx.x; it < Q * NAN_; it += blockDim.x) {
        const int q = it / NAN_, u = it % NAN_;
        const int q0 = q % g, q1 = (q / g) % g, q2 = q / (g * g);
        int64_t pt = (int64_t)e[0] * g + q0;
        if (NDIM >= 2) pt += (int64_t)s.G[0] * ((int64_t)e[1] * g + q1);
        if (NDIM >= 3) pt += (int64_t)s.G[0] * s.G[1] * ((int64_t)e[2] * g + q2);
        Dq[it] = s.Dg[pt * NAN_ + u];
    }
    __syncthreads();
    int Lp = pp + 1, Lv = pv + 1;
    if (NDIM >= 2) { Lp *= pp + 1; Lv *= pv + 1; }
    if (NDIM >= 3) { Lp *= pp + 1; Lv *= pv + 1; }
    const int64_t slot = s.eslot ? s.eslot[eid] : eid;
    double* out = s.eloc + slot * NDIM * Lp * Lv;
    for (int it = threadIdx.x; it < Lp * Lv; it += blockDim.x) {
        const int l = it / Lv, k = it % Lv;
        int l_[3] = {0, 0, 0}, k_[3] = {0, 0, 0};
        l_[0] = l % (pp + 1);
        k_[0] = k % (pv + 1);
        if (NDIM >= 2) { l_[1] = (l / (pp + 1)) % (pp + 1); k_[1] = (k / (pv + 1)) % (pv + 1); }
        if (NDIM >= 3) { l_[2] = l / ((pp + 1) * (pp + 1)); k_[2] = k / ((pv + 1) * (pv + 1)); }
        double acc[NDIM];
#pragma unroll
        for (int c = 0; c < NDIM; ++c) acc[c] = 0.0;
        for (int q = 0; q < Q; ++q) {
            int qd[3] = {q % g, (q / g) % g, q / (g * g)};
            double pval = 1.0, val[NDIM], der[NDIM];
#pragma unroll
            for (int d = 0; d < NDIM; ++d) {
                pval *= Pt[(d * g + qd[d]) * (pp + 1) + l_[d]];
                const double* vt = Vt + ((d * g + qd[d]) * 2) * (pv + 1);
                val[d] = vt[k_[d]];
                der[d] = vt[pv + 1 + k_[d]];
            }
            const double* Dp = Dq + q * NAN_;
#pragma unroll
            for (int c = 0; c < NDIM; ++c) {
                double t = 0.0;
#pragma unroll
                for (int a = 0; a < NDIM + 1; ++a) {
                    if (a == NA) break;  // a = NDIM: the rational value term (N_k against its factor)
                    double dv = 1.0;
#pragma unroll
                    for (int d = 0; d < NDIM; ++d) dv *= (d == a) ? der[d] : val[d];
                    t = fma(dv, Dp[a * NDIM + c], t);
                }
                acc[c] = fma(pval, t, acc[c]);
            }
        }
#pragma unroll
        for (int c = 0; c < NDIM; ++c) out[(int64_t)c * Lp * Lv + it] = acc[c];
    }
}

// Sum-factorised element matrices (2D / 3D): per (c, a) the element tensor
//   T[l][k] = sum_q prod_d W_d^{a}[l_d k_d][q_d] Dg(q)[a][c],  W_d^{a}[l k][q] = P_d[l](q) V_d^{(d == a)}[k](q)
// is contracted direction by direction (q0, q1, q2) in shared memory: ~30x fewer flops than the
// per-point triple product of div_local_kernel; each thread accumulates its (l, k) entries over a.
template <int NDIM>
__global__ void __launch_bounds__(256) div_local_sf_kernel(DivParams s) {
    static_assert(NDIM == 2 || NDIM == 3, "2D / 3D");
    extern __shared__ double sm[];
    const int NA = s.na, NAC = NA * NDIM;              // (a, c) pairs (a = NDIM: rational value term)
    const int pp = s.pp, pv = s.pv, g = s.g;
    const int LK = (pp + 1) * (pv + 1);               // 1D (l, k) pairs
    const int Q = NDIM == 2 ? g * g : g * g * g;
    const int R = Q / g;
    double* Dq = sm;                                   // [Q][na][NDIM]
    double* W = Dq + Q * NAC;                          // [d][alpha][LK][g]
    double* A1 = W + NDIM * 2 * LK * g;                // [ac][LK][R]
    double* A2 = A1 + NAC * LK * R;                    // [ac][LK][LK][g] (3D)
    const int64_t eid = s.elems[blockIdx.x];
    int e[3] = {0, 0, 0};
    e[0] = (int)(eid % s.Sv[0]);
    e[1] = (int)((eid / s.Sv[0]) % s.Sv[1]);
    if (NDIM >= 3) e[2] = (int)(eid / ((int64_t)s.Sv[0] * s.Sv[1]));
    for (int it = threadIdx.x; it < Q * NAC; it += blockDim.x) {
        const int q = it / NAC, u = it % NAC;
        const int q0 = q % g, q1 = (q / g) % g, q2 = q / (g * g);
        int64_t pt = (int64_t)e[0] * g + q0 + (int64_t)s.G[0] * ((int64_t)e[1] * g + q1);
        if (NDIM >= 3) pt += (int64_t)s.G[0] * s.G[1] * ((int64_t)e[2] * g + q2);
        Dq[it] = s.Dg[pt * NAC + u];
    }
    for (int it = threadIdx.x; it < NDIM * 2 * LK * g; it += blockDim.x) {
        const int q = it % g, lk = (it / g) % LK, al = (it / (g * LK)) % 2, d = it / (g * LK * 2);
        const int l = lk / (pv + 1), k = lk % (pv + 1);
        const int x = e[d] * g + q;  // velocity Gauss point of direction d
        W[it] = s.Pt[d][(int64_t)x * (pp + 1) + l] * s.V[d][((int64_t)x * 2 + al) * (pv + 1) + k];
    }
    __syncthreads();
    // stage 1 (all a, c): A1[ac][lk0][r] = sum_q0 W0^{a==0}[lk0][q0] D[(q0, r)][a][c]
    for (int it = threadIdx.x; it < NAC * LK * R; it += blockDim.x) {
        const int r = it % R, lk0 = (it / R) % LK, ac = it / (R * LK);
        const int a = ac / NDIM;
        const double* w0 = W + ((0 * 2 + (a == 0)) * LK + lk0) * g;
        double v = 0.0;
        for (int q0 = 0; q0 < g; ++q0) v = fma(w0[q0], Dq[(r * g + q0) * NAC + ac], v);
        A1[it] = v;
    }
    __syncthreads();
    if constexpr (NDIM == 3) {
        // stage 2: A2[ac][lk0][lk1][q2] = sum_q1 W1^{a==1}[lk1][q1] A1[ac][lk0][q1 + g q2]
        for (int it = threadIdx.x; it < NAC * LK * LK * g; it += blockDim.x) {
            const int q2 = it % g, lk1 = (it / g) % LK, lk0 = (it / (g * LK)) % LK, ac = it / (g * LK * LK);
            const int a = ac / NDIM;
            const double* w1 = W + ((1 * 2 + (a == 1)) * LK + lk1) * g;
            const double* a1 = A1 + (ac * LK + lk0) * R + g * q2;
            double v = 0.0;
            for (int q1 = 0; q1 < g; ++q1) v = fma(w1[q1], a1[q1], v);
            A2[it] = v;
        }
        __syncthreads();
    }
    int Lp = (pp + 1) * (pp + 1), Lv = (pv + 1) * (pv + 1);
    if (NDIM >= 3) { Lp *= pp + 1; Lv *= pv + 1; }
    const int64_t slot = s.eslot ? s.eslot[eid] : eid;
    double* out = s.eloc + slot * NDIM * Lp * Lv;
    // last stage: entry (l, k) of component c = sum_a (...) in ascending a
    for (int it = threadIdx.x; it < Lp * Lv; it += blockDim.x) {
        const int l = it / Lv, k = it % Lv;
        const int l0 = l % (pp + 1), k0 = k % (pv + 1);
        const int l1 = (l / (pp + 1)) % (pp + 1), k1 = (k / (pv + 1)) % (pv + 1);
        const int lk0 = l0 * (pv + 1) + k0, lk1 = l1 * (pv + 1) + k1;
#pragma unroll
        for (int c = 0; c < NDIM; ++c) {
            double acc = 0.0;
#pragma unroll
            for (int a = 0; a < NDIM + 1; ++a) {
                if (a == NA) break;
                const int ac = a * NDIM + c;
                double v = 0.0;
                if constexpr (NDIM == 2) {
                    const double* w1 = W + ((1 * 2 + (a == 1)) * LK + lk1) * g;
                    const double* a1 = A1 + (ac * LK + lk0) * R;
                    for (int q1 = 0; q1 < g; ++q1) v = fma(w1[q1], a1[q1], v);
                } else {
                    const int l2 = l / ((pp + 1) * (pp + 1)), k2 = k / ((pv + 1) * (pv + 1));
                    const int lk2 = l2 * (pv + 1) + k2;
                    const double* w2 = W + ((2 * 2 + (a == 2)) * LK + lk2) * g;
                    const double* a2 = A2 + ((ac * LK + lk0) * LK + lk1) * g;
                    for (int q2 = 0; q2 < g; ++q2) v = fma(w2[q2], a2[q2], v);
                }
                acc += v;
            }
            out[(int64_t)c * Lp * Lv + it] = acc;
        }
    }
}

__device__ __forceinline__ void div_cols(const DivParams& s, int d, int i, int& lo, int& hi) {
    lo = max(2 * i - 2 * s.pp, 0);
    hi = min(2 * i + s.pp + 2, s.mv[d] - 1);
}

template <int NDIM>
__global__ void div_counts_kernel(DivParams s, int64_t* counts) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r > s.Np) return;
    if (r == s.Np || (s.countmask && !s.countmask[r])) {
        counts[r] = 0;
        return;
    }
    int64_t rem = r, c = 1;
    for (int d = 0; d < NDIM; ++d) {
        const int i = (int)(rem % s.mp[d]);
        rem /= s.mp[d];
        int lo, hi;
        div_cols(s, d, i, lo, hi);
        c *= hi - lo + 1;
    }
    counts[r] = c;
}

template <int NDIM>
__global__ void div_gather_kernel(DivParams s) {
    const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= s.Np || (s.rowmask && !s.rowmask[r])) return;
    int i[3] = {0, 0, 0}, lo[3] = {0, 0, 0}, cnt[3] = {1, 1, 1};
    int64_t rem = r;
    for (int d = 0; d < NDIM; ++d) {
        i[d] = (int)(rem % s.mp[d]);
        rem /= s.mp[d];
        int hi;
        div_cols(s, d, i[d], lo[d], hi);
        cnt[d] = hi - lo[d] + 1;
    }
    const int pp = s.pp, pv = s.pv;
    int Lp = pp + 1, Lv = pv + 1;
    if (NDIM >= 2) { Lp *= pp + 1; Lv *= pv + 1; }
    if (NDIM >= 3) { Lp *= pp + 1; Lv *= pv + 1; }
    const int64_t base = s.rowstart[r];
    const int ncol = cnt[0] * cnt[1] * cnt[2];
    // element window of the row per direction: [2 max(0, i - pp), 2 min(Sp - 1, i) + 1]
    int elo[3] = {0, 0, 0}, ehi[3] = {0, 0, 0};
    for (int d = 0; d < NDIM; ++d) {
        elo[d] = 2 * max(0, i[d] - pp);
        ehi[d] = min(2 * min(s.Sp[d] - 1, i[d]) + 1, s.Sv[d] - 1);
    }
    for (int t = lane; t < ncol; t += 32) {
        int j[3] = {0, 0, 0};
        j[0] = lo[0] + t % cnt[0];
        if (NDIM >= 2) j[1] = lo[1] + (t / cnt[0]) % cnt[1];
        if (NDIM >= 3) j[2] = lo[2] + t / (cnt[0] * cnt[1]);
        int a[3] = {0, 0, 0}, b[3] = {0, 0, 0};
        for (int d = 0; d < NDIM; ++d) {
            a[d] = max(elo[d], j[d] - pv);
            b[d] = min(ehi[d], j[d]);
        }
        double acc[NDIM];
#pragma unroll
        for (int c = 0; c < NDIM; ++c) acc[c] = 0.0;
        for (int e2 = a[2]; e2 <= b[2]; ++e2)
            for (int e1 = a[1]; e1 <= b[1]; ++e1)
                for (int e0 = a[0]; e0 <= b[0]; ++e0) {
                    const int64_t eid = (int64_t)e0 + (int64_t)s.Sv[0] * ((int64_t)e1 + (int64_t)s.Sv[1] * e2);
                    const int64_t slot = s.eslot ? s.eslot[eid] : eid;
                    int l = i[0] - e0 / 2, k = j[0] - e0;
                    if (NDIM >= 2) { l += (pp + 1) * (i[1] - e1 / 2); k += (pv + 1) * (j[1] - e1); }
                    if (NDIM >= 3) { l += (pp + 1) * (pp + 1) * (i[2] - e2 / 2); k += (pv + 1) * (pv + 1) * (j[2] - e2); }
                    const double* lp = s.eloc + slot * NDIM * Lp * Lv + (int64_t)l * Lv + k;
#pragma unroll
                    for (int c = 0; c < NDIM; ++c) acc[c] += lp[(int64_t)c * Lp * Lv];
                }
        const int64_t col = (int64_t)j[0] + (int64_t)s.mv[0] * ((int64_t)j[1] + (int64_t)s.mv[1] * j[2]);
        if (s.wv || s.wp) {  // global NURBS weights w_l w_k of the pair
            const double wlk = (s.wp ? s.wp[r] : 1.0) * (s.wv ? s.wv[col] : 1.0);
#pragma unroll
            for (int c = 0; c < NDIM; ++c) acc[c] *= wlk;
        }
#pragma unroll
        for (int c = 0; c < NDIM; ++c) {
            s.data[c][base + t] = acc[c];
            s.indices[c][base + t] = (int)col;
        }
    }
}

__global__ void div_mask_kernel(const int64_t* rows, int64_t n, uint8_t* mask) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) mask[rows[k]] = 1;
}

template <int NDIM>
static int run_divergence(Call& c, DivParams& s, int64_t npts, size_t local_smem) {
    c.kbegin("div_geom");
    div_geom_kernel<NDIM><<<(unsigned)((npts + 127) / 128), 128, 0, c.stream>>>(s);
    c.kend();
    if (s.nelem > 0) {
        int LpLv = 1;
        for (int d = 0; d < NDIM; ++d) LpLv *= (s.pp + 1) * (s.pv + 1);
        const int LK = (s.pp + 1) * (s.pv + 1);
        int Q = 1;
        for (int d = 0; d < NDIM; ++d) Q *= s.g;
        const size_t nac = (size_t)s.na * NDIM;
        const size_t sf_smem = sizeof(double) * ((size_t)Q * nac + (size_t)NDIM * 2 * LK * s.g + nac * LK * (Q / s.g) +
                                                 (NDIM == 3 ? nac * LK * LK * s.g : 0));
        if constexpr (NDIM >= 2) {
            if (sf_smem <= 227 * 1024 && !getenv("SG_DIV_DIRECT")) {
                if (sf_smem > 48 * 1024)
                    cudaFuncSetAttribute(div_local_sf_kernel<NDIM>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemOptinMax);
                c.kbegin("div_local");
                div_local_sf_kernel<NDIM><<<(unsigned)s.nelem, 256, sf_smem, c.stream>>>(s);
                c.kend();
                goto gathered;
            }
        }
        if (local_smem > 48 * 1024)
            cudaFuncSetAttribute(div_local_kernel<NDIM>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemOptinMax);
        c.kbegin("div_local");
        div_local_kernel<NDIM><<<(unsigned)s.nelem, 256, local_smem, c.stream>>>(s);
        c.kend();
    }
gathered:
    c.kbegin("div_gather");
    div_gather_kernel<NDIM><<<(unsigned)((s.Np * 32 + 255) / 256), 256, 0, c.stream>>>(s);
    c.kend();
    return 0;
}


// ---- surrogate pieces (surrogate.py:702-819): samples, coefficient solve, interpolant evaluation
__global__ void div_samples_kernel(const int64_t* __restrict__ rowstart, const double* __restrict__ data,
                                   const int64_t* __restrict__ latrows, int64_t nlat, int P, double* __restrict__ S) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nlat * P) return;
    const int64_t t = k / P;
    const int o = (int)(k % P);
    S[(int64_t)o * nlat + t] = data[rowstart[latrows[t]] + o];
}

// out[a][s][b] = sum_t Cinv[s][t] in[a][t][b]  (one direction of the tensor collocation solve)
__global__ void div_apply_dir_kernel(const double* __restrict__ in, double* __restrict__ out, const double* __restrict__ Cinv,
                                     int64_t outer, int len, int64_t inner) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= outer * len * inner) return;
    const int64_t a = k / (len * inner), rem = k % (len * inner);
    const int sidx = (int)(rem / inner);
    const int64_t b = rem % inner;
    double acc = 0.0;
    for (int t = 0; t < len; ++t) acc = fma(Cinv[(int64_t)sidx * len + t], in[(a * len + t) * inner + b], acc);
    out[k] = acc;
}

struct DivInterp {
    int n, P, pp;
    int mp[3], mv[3], blo[3], nl[3], qd[3];
    const uint8_t* core[3];        // pressure index in the shrunk box (one index of margin)
    const uint8_t* smp[3];         // pressure index on the lattice
    const int* esp[3];             // interpolant spans at the box points
    const double* etab[3];         // interpolant basis values at the box points [nbox][qd+1]
    const double* coef[3];         // per component [P][nl2][nl1][nl0]
    const int* shifts;             // [P][3] mixed offsets
    const int64_t* rowstart;
    int* indices[3];
    double* data[3];
    int64_t Np;
    int64_t row_lo, row_hi;  // rows interpolated by this call (row slab)
    unsigned long long* counters;  // 0 interp rows, 1 zeros
};

// one warp per interpolated pressure row, lanes on offsets: the row's P columns 2 i + shift(o)
template <int NDIM>
__global__ void div_interp_kernel(DivInterp s) {
    const int64_t r = s.row_lo + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (r >= s.row_hi) return;
    int i[3] = {0, 0, 0};
    int64_t rem = r;
    bool core = true, samp = true;
    for (int d = 0; d < NDIM; ++d) {
        i[d] = (int)(rem % s.mp[d]);
        rem /= s.mp[d];
        core = core && s.core[d][i[d]];
        samp = samp && s.smp[d][i[d]];
    }
    if (!core || samp) return;
    if (lane == 0) atomicAdd(&s.counters[0], 1ull);
    const double* e[3];
    int lo[3] = {0, 0, 0}, q[3] = {0, 0, 0};
    for (int d = 0; d < 3; ++d) {
        if (d < NDIM) {
            const int b = i[d] - s.blo[d];
            q[d] = s.qd[d];
            e[d] = s.etab[d] + (int64_t)b * (q[d] + 1);
            lo[d] = s.esp[d][b] - q[d];
        } else {
            e[d] = nullptr;
        }
    }
    const int64_t base = s.rowstart[r];
    unsigned long long zeros = 0;
    for (int o = lane; o < s.P; o += 32) {
        int j[3] = {0, 0, 0};
        for (int d = 0; d < NDIM; ++d) j[d] = 2 * i[d] + s.shifts[o * 3 + d];
        const int64_t col = (int64_t)j[0] + (int64_t)s.mv[0] * ((int64_t)j[1] + (int64_t)s.mv[1] * j[2]);
        for (int c = 0; c < NDIM; ++c) {
            const double* cf = s.coef[c] + (int64_t)o * s.nl[0] * s.nl[1] * s.nl[2];
            double v = 0.0;
            for (int r2 = 0; r2 <= (NDIM >= 3 ? q[2] : 0); ++r2) {
                const double w2 = NDIM >= 3 ? e[2][r2] : 1.0;
                const int64_t c2 = NDIM >= 3 ? (int64_t)(lo[2] + r2) * s.nl[1] * s.nl[0] : 0;
                double v1 = 0.0;
                for (int r1 = 0; r1 <= (NDIM >= 2 ? q[1] : 0); ++r1) {
                    const double w1 = NDIM >= 2 ? e[1][r1] : 1.0;
                    const double* row = cf + c2 + (NDIM >= 2 ? (int64_t)(lo[1] + r1) * s.nl[0] : 0) + lo[0];
                    double v0 = 0.0;
                    for (int r0 = 0; r0 <= q[0]; ++r0) v0 = fma(e[0][r0], row[r0], v0);
                    v1 = fma(w1, v0, v1);
                }
                v = fma(w2, v1, v);
            }
            s.data[c][base + o] = v;
            s.indices[c][base + o] = (int)col;
            zeros += (v == 0.0);
        }
    }
    if (zeros) atomicAdd(&s.counters[1], zeros);
}

__global__ void div_nz_count_kernel(const int64_t* __restrict__ rowstart, const double* __restrict__ data, int64_t N,
                                    int64_t* __restrict__ cnt) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > N) return;
    if (i == N) {
        cnt[i] = 0;
        return;
    }
    int64_t c = 0;
    for (int64_t k = rowstart[i]; k < rowstart[i + 1]; ++k) c += (data[k] != 0.0);
    cnt[i] = c;
}

__global__ void div_compact_kernel(const int64_t* __restrict__ rowstart, const double* __restrict__ data,
                                   const int* __restrict__ indices, int64_t N, const int64_t* __restrict__ newptr,
                                   double* __restrict__ ndata, int* __restrict__ nind) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    int64_t w = newptr[i];
    for (int64_t k = rowstart[i]; k < rowstart[i + 1]; ++k)
        if (data[k] != 0.0) {
            ndata[w] = data[k];
            nind[w] = indices[k];
            ++w;
        }
}

// shared set-up of both entry points: validation, velocity tables + geometry, pressure tables
static int div_setup(Call& c, const sg_problem* vel, const sg_problem* prs, DevProblem& dp, DivParams& s, int64_t& npts,
                     int64_t& Ev) {
    const int n = vel->n;
    if (prs->n != n || n < 1 || n > 3) return fail(-1, "velocity/pressure dimension mismatch");
    if (vel->p != prs->p + 1) return fail(-1, "velocity degree must be the pressure degree + 1");
    for (int d = 0; d < n; ++d)
        if (vel->m[d] - vel->p != 2 * (prs->m[d] - prs->p))
            return fail(-1, "velocity mesh must halve every pressure element (subgrid pair)");
    sg_problem vp = *vel;
    vp.form = POISSON;  // velocity tables with first derivatives, geometry with first derivatives
    int rc = prepare_problem(c, &vp, dp);
    if (rc) return rc;
    s = DivParams{};
    s.n = n;
    s.pv = vel->p;
    s.pp = prs->p;
    s.pg = vel->geo_p;
    s.g = vel->g;
    int64_t Np = 1;
    Ev = 1;
    npts = 1;
    for (int d = 0; d < 3; ++d) {
        if (d < n) {
            s.Sv[d] = dp.S[d];
            s.Sp[d] = prs->m[d] - prs->p;
            s.mp[d] = prs->m[d];
            s.mv[d] = vel->m[d];
            s.mg[d] = vel->geo_m[d];
            s.G[d] = dp.S[d] * dp.g;
            s.V[d] = dp.B[d];
            s.Gt[d] = dp.G[d];
            s.gspan[d] = dp.gspan[d];
            s.qw[d] = dp.qw[d];
        } else {
            s.Sv[d] = s.Sp[d] = s.mp[d] = s.mv[d] = s.mg[d] = s.G[d] = 1;
        }
        Np *= s.mp[d];
        Ev *= s.Sv[d];
        npts *= s.G[d];
    }
    s.Np = Np;
    s.hom = dp.hom;
    // pressure basis at the velocity Gauss points (bspline.py:112-124 with ratio 2, assembly.py:410-412)
    for (int d = 0; d < n; ++d) {
        const int np_ = s.G[d];
        double* kn = (double*)c.upload(prs->knots[d], sizeof(double) * (prs->m[d] + prs->p + 1));
        double* qp = (double*)c.upload(vel->qpts[d], sizeof(double) * np_);
        double* tab = (double*)c.alloc(sizeof(double) * np_ * (prs->p + 1), true);
        int* sp = (int*)c.alloc(sizeof(int) * np_, true);
        tabulate(c, kn, prs->m[d] + prs->p + 1, prs->p, qp, np_, 0, sp, tab);
        s.Pt[d] = tab;
    }
    // NURBS spaces: weights of both spaces on the device (K4 keeps the velocity ones in dp.sol_w)
    s.wv = vel->sol_w ? dp.sol_w : nullptr;
    s.wp = prs->sol_w ? (const double*)c.upload(prs->sol_w, sizeof(double) * Np) : nullptr;
    s.na = s.wv ? n + 1 : n;
    s.Dg = (double*)c.alloc(sizeof(double) * npts * s.na * n, true);
    return s.Dg && (!vel->sol_w || s.wv) ? 0 : fail(-4, "device allocation failed");
}

// elements supporting the listed pressure rows (assembly.py:347-360, ratio 2) + gather row mask
static int div_elements(Call& c, DivParams& s, const int64_t* rows, int64_t nrows, int64_t Ev, std::vector<int64_t>& elist) {
    const int n = s.n;
    if (rows) {
        for (int64_t k = 0; k < nrows; ++k) {
            if (rows[k] < 0 || rows[k] >= s.Np) return fail(-1, "pressure row index out of range");
            if (k && rows[k] <= rows[k - 1]) return fail(-1, "rows must be sorted and unique");
        }
        std::vector<uint8_t> emask(Ev, 0);
        for (int64_t k = 0; k < nrows; ++k) {
            int64_t rem = rows[k];
            int elo[3] = {0, 0, 0}, ehi[3] = {0, 0, 0};
            for (int d = 0; d < n; ++d) {
                const int i = (int)(rem % s.mp[d]);
                rem /= s.mp[d];
                elo[d] = 2 * std::max(0, i - s.pp);
                ehi[d] = std::min(2 * std::min(s.Sp[d] - 1, i) + 1, s.Sv[d] - 1);
            }
            for (int e2 = elo[2]; e2 <= ehi[2]; ++e2)
                for (int e1 = elo[1]; e1 <= ehi[1]; ++e1)
                    for (int e0 = elo[0]; e0 <= ehi[0]; ++e0) emask[e0 + (int64_t)s.Sv[0] * (e1 + (int64_t)s.Sv[1] * e2)] = 1;
        }
        std::vector<int> slot(Ev, -1);
        for (int64_t e = 0; e < Ev; ++e)
            if (emask[e]) {
                slot[e] = (int)elist.size();
                elist.push_back(e);
            }
        s.eslot = (const int*)c.upload(slot.data(), sizeof(int) * Ev);
        uint8_t* rowmask = (uint8_t*)c.alloc(s.Np + 1, true);
        cudaMemsetAsync(rowmask, 0, s.Np + 1, c.stream);
        if (nrows > 0) {
            int64_t* dr = (int64_t*)c.upload(rows, sizeof(int64_t) * nrows);
            div_mask_kernel<<<(unsigned)((nrows + 255) / 256), 256, 0, c.stream>>>(dr, nrows, rowmask);
        }
        s.rowmask = rowmask;
    } else {
        elist.resize(Ev);
        for (int64_t e = 0; e < Ev; ++e) elist[e] = e;
        s.eslot = nullptr;
        s.rowmask = nullptr;
    }
    s.nelem = (int64_t)elist.size();
    s.elems = s.nelem ? (const int64_t*)c.upload(elist.data(), sizeof(int64_t) * elist.size()) : nullptr;
    int64_t Lp = 1, Lv = 1;
    for (int d = 0; d < n; ++d) {
        Lp *= s.pp + 1;
        Lv *= s.pv + 1;
    }
    const double loc_bytes = (double)s.nelem * n * Lp * Lv * sizeof(double);
    if (loc_bytes > 32e9) return fail(-4, "divergence element matrices need %.1f GB of device memory", loc_bytes / 1e9);
    s.eloc = (double*)c.alloc(std::max<size_t>((size_t)loc_bytes, 8), true);
    return s.eloc ? 0 : fail(-4, "device allocation failed");
}

static int div_rowstart(Call& c, DivParams& s, int64_t*& rowstart, int64_t& nnz) {
    const int64_t Np = s.Np;
    int64_t* counts = (int64_t*)c.alloc(sizeof(int64_t) * (Np + 1), true);
    rowstart = (int64_t*)c.alloc(sizeof(int64_t) * (Np + 1), true);
    c.kbegin("div_counts");
    if (s.n == 1) div_counts_kernel<1><<<(unsigned)((Np + 256) / 256), 256, 0, c.stream>>>(s, counts);
    if (s.n == 2) div_counts_kernel<2><<<(unsigned)((Np + 256) / 256), 256, 0, c.stream>>>(s, counts);
    if (s.n == 3) div_counts_kernel<3><<<(unsigned)((Np + 256) / 256), 256, 0, c.stream>>>(s, counts);
    c.kend();
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, counts, rowstart, Np + 1, c.stream);
    void* tmp = c.alloc(tb, true);
    cub::DeviceScan::ExclusiveSum(tmp, tb, counts, rowstart, Np + 1, c.stream);
    nnz = 0;
    cudaMemcpyAsync(&nnz, rowstart + Np, sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream);
    cudaStreamSynchronize(c.stream);
    s.rowstart = rowstart;
    return 0;
}

static size_t div_local_smem(const DivParams& s) {
    int Q = 1;
    for (int d = 0; d < s.n; ++d) Q *= s.g;
    return sizeof(double) * ((size_t)s.n * s.g * (s.pp + 1) + (size_t)s.n * s.g * 2 * (s.pv + 1) + (size_t)Q * s.na * s.n);
}

static int div_run(Call& c, DivParams& s, int64_t npts) {
    const size_t local_smem = div_local_smem(s);
    if (local_smem > 227 * 1024) return fail(-2, "divergence element tables do not fit shared memory");
    if (s.n == 1) return run_divergence<1>(c, s, npts, local_smem);
    if (s.n == 2) return run_divergence<2>(c, s, npts, local_smem);
    return run_divergence<3>(c, s, npts, local_smem);
}

static sg_result* new_result(Call& c, int64_t Np, int64_t nnz, bool with_arrays) {
    sg_result* r = new sg_result();
    r->dev = c.dev;
    r->nrows = Np;
    r->nrows_global = Np;
    r->row_lo = 0;
    r->nnz = nnz;
    r->indptr = (int64_t*)c.alloc(sizeof(int64_t) * (Np + 1), false);
    if (with_arrays) {
        r->indices = (int*)c.alloc(sizeof(int) * std::max<int64_t>(nnz, 1), false);
        r->data = (double*)c.alloc(sizeof(double) * std::max<int64_t>(nnz, 1), false);
    }
    return r;
}

static int div_finish(Call& c, sg_result** res, int n, sg_result** out) {
    int rc = c.finish();
    if (!rc) {
        cudaStreamSynchronize(c.stream);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) rc = fail(-3, "CUDA error in the divergence assembly: %s", cudaGetErrorString(e));
    }
    if (rc) {
        for (int q = 0; q < n; ++q)
            if (res[q]) sg_result_free(res[q]);
        return rc;
    }
    c.record_timing();
    for (int k = 0; k < n; ++k) out[k] = res[k];
    return 0;
}

}  // namespace sg

using namespace sg;

extern "C" int sg_assemble_divergence(const sg_problem* vel, const sg_problem* prs, const int64_t* rows, int64_t nrows,
                                      const sg_exec* ex, sg_result** out) {
    if (!out) return fail(-1, "null output handles");
    if (!vel || !prs) return fail(-1, "null problem");
    for (int k = 0; k < 3 && k < vel->n; ++k) out[k] = nullptr;
    const bool slab = ex && (ex->slab_lo != 0 || ex->slab_hi != 0);
    if (slab && rows) return fail(-1, "rows= cannot be combined with a row slab");
    Call c(ex);
    DevProblem dp;
    DivParams s;
    int64_t npts = 0, Ev = 0;
    int rc = div_setup(c, vel, prs, dp, s, npts, Ev);
    if (rc) return rc;
    std::vector<int64_t> elist;
    int64_t lo = 0, hi = s.Np;
    if (slab) {
        // a contiguous block of pressure rows per GPU; the velocity element layers under it
        // (halo included) are recomputed, no exchange.  Element superset: every element whose slowest
        // index lies in the window of the slab's first / last slowest-direction plane.
        lo = ex->slab_lo;
        hi = ex->slab_hi;
        if (lo < 0 || hi > s.Np || lo >= hi) return fail(-1, "row slab [%lld, %lld) outside [0, %lld)", (long long)lo, (long long)hi, (long long)s.Np);
        const int ls = s.n - 1;
        int64_t pstride = 1, estride = 1;
        for (int d = 0; d < ls; ++d) {
            pstride *= s.mp[d];
            estride *= s.Sv[d];
        }
        const int ilo = (int)(lo / pstride), ihi = (int)((hi - 1) / pstride);
        const int64_t elo = 2 * std::max(0, ilo - s.pp), ehi = std::min<int64_t>(2 * std::min(s.Sp[ls] - 1, ihi) + 1, s.Sv[ls] - 1);
        for (int64_t e = elo * estride; e < (ehi + 1) * estride; ++e) elist.push_back(e);
        std::vector<int> slot(Ev, -1);
        for (size_t k = 0; k < elist.size(); ++k) slot[elist[k]] = (int)k;
        s.eslot = (const int*)c.upload(slot.data(), sizeof(int) * Ev);
        uint8_t* rowmask = (uint8_t*)c.alloc(s.Np + 1, true);
        cudaMemsetAsync(rowmask, 0, s.Np + 1, c.stream);
        cudaMemsetAsync(rowmask + lo, 1, hi - lo, c.stream);
        s.rowmask = rowmask;
        s.nelem = (int64_t)elist.size();
        s.elems = (const int64_t*)c.upload(elist.data(), sizeof(int64_t) * elist.size());
        int64_t Lp = 1, Lv = 1;
        for (int d = 0; d < s.n; ++d) {
            Lp *= s.pp + 1;
            Lv *= s.pv + 1;
        }
        s.eloc = (double*)c.alloc(std::max<size_t>((size_t)s.nelem * s.n * Lp * Lv * sizeof(double), 8), true);
        if (!s.eloc || !s.eslot || !s.elems) return fail(-4, "device allocation failed");
    } else if ((rc = div_elements(c, s, rows, nrows, Ev, elist))) {
        return rc;
    }
    s.countmask = s.rowmask;  // restricted rows / slab: only those rows are present
    int64_t* rowstart = nullptr;
    int64_t nnz = 0;
    div_rowstart(c, s, rowstart, nnz);
    const int n = s.n;
    sg_result* res[3] = {nullptr, nullptr, nullptr};
    for (int k = 0; k < n; ++k) {
        res[k] = new_result(c, hi - lo, nnz, true);
        if (!res[k]->indptr || !res[k]->indices || !res[k]->data) {
            for (int q = 0; q <= k; ++q) sg_result_free(res[q]);
            return fail(-4, "device allocation failed (nnz=%lld)", (long long)nnz);
        }
        res[k]->nrows_global = s.Np;
        res[k]->row_lo = lo;
        // rows before the slab hold no entries, so rowstart[lo] = 0: the slab's indptr is a plain slice
        cudaMemcpyAsync(res[k]->indptr, rowstart + lo, sizeof(int64_t) * (hi - lo + 1), cudaMemcpyDeviceToDevice, c.stream);
        s.indices[k] = res[k]->indices;
        s.data[k] = res[k]->data;
    }
    rc = div_run(c, s, npts);
    if (rc) {
        for (int q = 0; q < n; ++q) sg_result_free(res[q]);
        return rc;
    }
    return div_finish(c, res, n, out);
}

extern "C" int sg_surrogate_divergence(const sg_problem* vel, const sg_problem* prs, const sg_surrogate_params* sp,
                                       const int32_t* shifts, const int64_t* quad_rows, int64_t nquad, const sg_exec* ex,
                                       sg_result** out, sg_surrogate_stats* stats) {
    if (!out || !vel || !prs || !sp || !shifts) return fail(-1, "null argument");
    for (int k = 0; k < 3 && k < vel->n; ++k) out[k] = nullptr;
    if (sp->mode != SG_GENERAL) return fail(-1, "the divergence pairing only supports the general mode");
    const bool slab = ex && (ex->slab_lo != 0 || ex->slab_hi != 0);
    Call c(ex);
    DevProblem dp;
    DivParams s;
    int64_t npts = 0, Ev = 0;
    int rc = div_setup(c, vel, prs, dp, s, npts, Ev);
    if (rc) return rc;
    const int n = s.n, pp = s.pp;
    int64_t lo = 0, hi = s.Np;
    if (slab) {
        lo = ex->slab_lo;
        hi = ex->slab_hi;
        if (lo < 0 || hi > s.Np || lo >= hi) return fail(-1, "row slab [%lld, %lld) outside [0, %lld)", (long long)lo, (long long)hi, (long long)s.Np);
    }
    // lattice rows (colex) -- sampled rows, assembled by every slab
    int64_t nlat = 1;
    for (int d = 0; d < n; ++d) nlat *= sp->nlat[d];
    std::vector<int64_t> latrows(nlat);
    for (int64_t t = 0; t < nlat; ++t) {
        int64_t rem = t, row = 0, str = 1;
        for (int d = 0; d < n; ++d) {
            const int a = (int)(rem % sp->nlat[d]);
            rem /= sp->nlat[d];
            row += sp->lat_idx[d][a] * str;
            str *= s.mp[d];
        }
        latrows[t] = row;
    }
    // quadrature rows by quadrature (elements supporting them); every row present in the pattern.
    // Row slab: the slab's quadrature rows plus every lattice row (the samples of the
    // coefficient solve), so each slab interpolates exactly as the whole-matrix call does
    std::vector<int64_t> qsel;
    if (slab) {
        std::vector<int64_t> ls(latrows);
        std::sort(ls.begin(), ls.end());
        for (int64_t k = 0; k < nquad; ++k) {
            const int64_t q = quad_rows[k];
            if ((q >= lo && q < hi) || std::binary_search(ls.begin(), ls.end(), q)) qsel.push_back(q);
        }
    }
    std::vector<int64_t> elist;
    if ((rc = div_elements(c, s, slab ? qsel.data() : quad_rows, slab ? (int64_t)qsel.size() : nquad, Ev, elist))) return rc;
    s.countmask = nullptr;
    int64_t* rowstart = nullptr;
    int64_t nnz = 0;
    div_rowstart(c, s, rowstart, nnz);
    int* wind[3] = {nullptr, nullptr, nullptr};
    double* wdat[3] = {nullptr, nullptr, nullptr};
    for (int k = 0; k < n; ++k) {
        wind[k] = (int*)c.alloc(sizeof(int) * std::max<int64_t>(nnz, 1), true);
        wdat[k] = (double*)c.alloc(sizeof(double) * std::max<int64_t>(nnz, 1), true);
        if (!wind[k] || !wdat[k]) return fail(-4, "device allocation failed (nnz=%lld)", (long long)nnz);
        s.indices[k] = wind[k];
        s.data[k] = wdat[k];
    }
    if ((rc = div_run(c, s, npts))) return rc;
    // samples S[o][lattice colex] from the quadrature rows (surrogate.py:336-379), per component
    int P = 1;
    for (int d = 0; d < n; ++d) P *= 3 * pp + 3;
    const int64_t* dlat = (const int64_t*)c.upload(latrows.data(), sizeof(int64_t) * nlat);
    DivInterp I{};
    I.n = n;
    I.P = P;
    I.pp = pp;
    I.Np = s.Np;
    I.row_lo = lo;
    I.row_hi = hi;
    I.rowstart = rowstart;
    for (int d = 0; d < 3; ++d) {
        I.mp[d] = s.mp[d];
        I.mv[d] = s.mv[d];
        I.nl[d] = d < n ? sp->nlat[d] : 1;
        I.qd[d] = d < n ? sp->qd[d] : 0;
        I.blo[d] = 2 * pp;
    }
    const double* cinv[3];
    for (int d = 0; d < n; ++d) cinv[d] = (const double*)c.upload(sp->colloc_inv[d], sizeof(double) * sp->nlat[d] * sp->nlat[d]);
    for (int k = 0; k < n; ++k) {
        double* S0 = (double*)c.alloc(sizeof(double) * P * nlat, true);
        double* S1 = (double*)c.alloc(sizeof(double) * P * nlat, true);
        c.kbegin("div_samples");
        div_samples_kernel<<<(unsigned)((nlat * P + 255) / 256), 256, 0, c.stream>>>(rowstart, wdat[k], dlat, nlat, P, S0);
        c.kend();
        // coefficient solve per direction (surrogate.py:430-471): S[P][l2][l1][l0]
        for (int d = 0; d < n; ++d) {
            if (sp->qd[d] < 1) continue;
            int64_t inner = 1, outer = P;
            for (int e = 0; e < d; ++e) inner *= sp->nlat[e];
            for (int e = d + 1; e < n; ++e) outer *= sp->nlat[e];
            c.kbegin("div_coef_solve");
            div_apply_dir_kernel<<<(unsigned)((P * nlat + 255) / 256), 256, 0, c.stream>>>(S0, S1, cinv[d], outer, sp->nlat[d], inner);
            c.kend();
            std::swap(S0, S1);
        }
        I.coef[k] = S0;
        I.indices[k] = wind[k];
        I.data[k] = wdat[k];
    }
    // interpolant tables at the box points, masks
    for (int d = 0; d < n; ++d) {
        const int nbox = s.mp[d] - 4 * pp;
        int* esp = (int*)c.alloc(sizeof(int) * std::max(nbox, 1), true);
        double* et = (double*)c.alloc(sizeof(double) * std::max(nbox, 1) * (sp->qd[d] + 1), true);
        if (sp->qd[d] >= 1) {
            double* kn = (double*)c.upload(sp->interp_knots[d], sizeof(double) * (sp->nlat[d] + sp->qd[d] + 1));
            double* bp = (double*)c.upload(sp->box_pts[d], sizeof(double) * nbox);
            tabulate(c, kn, sp->nlat[d] + sp->qd[d] + 1, sp->qd[d], bp, nbox, 0, esp, et);
        } else {
            std::vector<int> z(nbox, 0);
            std::vector<double> one(nbox, 1.0);
            cudaMemcpyAsync(esp, z.data(), sizeof(int) * nbox, cudaMemcpyHostToDevice, c.stream);
            cudaMemcpyAsync(et, one.data(), sizeof(double) * nbox, cudaMemcpyHostToDevice, c.stream);
            cudaStreamSynchronize(c.stream);
        }
        I.esp[d] = esp;
        I.etab[d] = et;
        std::vector<uint8_t> core(s.mp[d], 0), smp(s.mp[d], 0);
        const int lo = 2 * pp, hi = s.mp[d] - 2 * pp - 1;
        for (int i = lo + 1; i <= hi - 1; ++i) core[i] = 1;
        for (int a = 0; a < sp->nlat[d]; ++a) smp[sp->lat_idx[d][a]] = 1;
        I.core[d] = (const uint8_t*)c.upload(core.data(), s.mp[d]);
        I.smp[d] = (const uint8_t*)c.upload(smp.data(), s.mp[d]);
    }
    std::vector<int> sh3((size_t)P * 3, 0);
    for (int o = 0; o < P; ++o)
        for (int d = 0; d < n; ++d) sh3[(size_t)o * 3 + d] = shifts[(size_t)o * n + d];
    I.shifts = (const int*)c.upload(sh3.data(), sizeof(int) * P * 3);
    unsigned long long* counters = (unsigned long long*)c.alloc(sizeof(unsigned long long) * 2, true);
    cudaMemsetAsync(counters, 0, sizeof(unsigned long long) * 2, c.stream);
    I.counters = counters;
    c.kbegin("div_interp");
    const unsigned nb = (unsigned)(((hi - lo) * 32 + 255) / 256);
    if (n == 1) div_interp_kernel<1><<<nb, 256, 0, c.stream>>>(I);
    if (n == 2) div_interp_kernel<2><<<nb, 256, 0, c.stream>>>(I);
    if (n == 3) div_interp_kernel<3><<<nb, 256, 0, c.stream>>>(I);
    c.kend();
    unsigned long long hc[2] = {0, 0};
    cudaMemcpyAsync(hc, counters, sizeof(hc), cudaMemcpyDeviceToHost, c.stream);
    cudaStreamSynchronize(c.stream);
    // merge: exact zeros dropped (scipy CSR add, surrogate.py:810), per component
    sg_result* res[3] = {nullptr, nullptr, nullptr};
    int64_t dropped = 0;
    // slab: rows [lo, hi) of the work CSR (rowstart + lo keeps absolute offsets into the work arrays)
    const int64_t nr = hi - lo;
    int64_t slab_nnz = nnz;
    if (slab) {
        int64_t b[2] = {0, 0};
        cudaMemcpyAsync(&b[0], rowstart + lo, sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream);
        cudaMemcpyAsync(&b[1], rowstart + hi, sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream);
        cudaStreamSynchronize(c.stream);
        slab_nnz = b[1] - b[0];
    }
    for (int k = 0; k < n; ++k) {
        int64_t* cnt = (int64_t*)c.alloc(sizeof(int64_t) * (nr + 1), true);
        c.kbegin("div_nz_count");
        div_nz_count_kernel<<<(unsigned)((nr + 256) / 256), 256, 0, c.stream>>>(rowstart + lo, wdat[k], nr, cnt);
        c.kend();
        sg_result* r = new_result(c, nr, 0, false);
        r->nrows_global = s.Np;
        r->row_lo = lo;
        size_t tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, r->indptr, nr + 1, c.stream);
        void* tmp = c.alloc(tb, true);
        cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, r->indptr, nr + 1, c.stream);
        int64_t nz = 0;
        cudaMemcpyAsync(&nz, r->indptr + nr, sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream);
        cudaStreamSynchronize(c.stream);
        r->nnz = nz;
        dropped += slab_nnz - nz;
        if (!slab && nz == nnz) {
            c.release(wind[k]);
            c.release(wdat[k]);
            r->indices = wind[k];
            r->data = wdat[k];
        } else {
            r->indices = (int*)c.alloc(sizeof(int) * std::max<int64_t>(nz, 1), false);
            r->data = (double*)c.alloc(sizeof(double) * std::max<int64_t>(nz, 1), false);
            c.kbegin("div_compact");
            div_compact_kernel<<<(unsigned)((nr + 255) / 256), 256, 0, c.stream>>>(rowstart + lo, wdat[k], wind[k], nr, r->indptr,
                                                                                   r->data, r->indices);
            c.kend();
        }
        res[k] = r;
    }
    if (stats) {
        stats->n_interp_rows = (int64_t)hc[0];
        stats->n_quad_rows = nquad;
        stats->n_interp_entries = (int64_t)hc[0] * P * n;
        stats->n_zero_dropped = dropped;
        stats->n_reset_rows = 0;
    }
    return div_finish(c, res, n, out);
}
