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
    double* Dg;                    // [npts][n][n]: w_q adj[a][c]
    const int64_t* elems;          // element ids (colex over velocity elements), ascending
    int64_t nelem;
    const int* eslot;              // element id -> slot (-1: not computed); nullptr = identity
    double* eloc;                  // [slot][c][Lp][Lv]
    const uint8_t* rowmask;        // pressure rows to assemble (nullptr = all)
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
    double* out = s.Dg + t * NDIM * NDIM;
#pragma unroll
    for (int a = 0; a < NDIM; ++a)
#pragma unroll
        for (int c = 0; c < NDIM; ++c) out[a * NDIM + c] = wq * adj[a][c];
}

// one CTA per element: loc[c][l][k] = sum_q P_l(q) sum_a dV_k^a(q) Dg(q)[a][c]
template <int NDIM>
__global__ void __launch_bounds__(256) div_local_kernel(DivParams s) {
    extern __shared__ double sm[];
    const int pp = s.pp, pv = s.pv, g = s.g;
    const int Q = NDIM == 1 ? g : (NDIM == 2 ? g * g : g * g * g);
    double* Pt = sm;                                  // [d][g][pp+1]
    double* Vt = Pt + NDIM * g * (pp + 1);            // [d][g][2][pv+1]
    double* Dq = Vt + NDIM * g * 2 * (pv + 1);        // [Q][NDIM][NDIM]
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
    for (int it = threadIdx.x; it < Q * NDIM * NDIM; it += blockDim.x) {
        const int q = it / (NDIM * NDIM), u = it % (NDIM * NDIM);
        const int q0 = q % g, q1 = (q / g) % g, q2 = q / (g * g);
        int64_t pt = (int64_t)e[0] * g + q0;
        if (NDIM >= 2) pt += (int64_t)s.G[0] * ((int64_t)e[1] * g + q1);
        if (NDIM >= 3) pt += (int64_t)s.G[0] * s.G[1] * ((int64_t)e[2] * g + q2);
        Dq[it] = s.Dg[pt * NDIM * NDIM + u];
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
            const double* Dp = Dq + q * NDIM * NDIM;
#pragma unroll
            for (int c = 0; c < NDIM; ++c) {
                double t = 0.0;
#pragma unroll
                for (int a = 0; a < NDIM; ++a) {
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

__device__ __forceinline__ void div_cols(const DivParams& s, int d, int i, int& lo, int& hi) {
    lo = max(2 * i - 2 * s.pp, 0);
    hi = min(2 * i + s.pp + 2, s.mv[d] - 1);
}

template <int NDIM>
__global__ void div_counts_kernel(DivParams s, int64_t* counts) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r > s.Np) return;
    if (r == s.Np || (s.rowmask && !s.rowmask[r])) {
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
        if (local_smem > 48 * 1024)
            cudaFuncSetAttribute(div_local_kernel<NDIM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)local_smem);
        c.kbegin("div_local");
        div_local_kernel<NDIM><<<(unsigned)s.nelem, 256, local_smem, c.stream>>>(s);
        c.kend();
    }
    c.kbegin("div_gather");
    div_gather_kernel<NDIM><<<(unsigned)((s.Np * 32 + 255) / 256), 256, 0, c.stream>>>(s);
    c.kend();
    return 0;
}

}  // namespace sg

using namespace sg;

extern "C" int sg_assemble_divergence(const sg_problem* vel, const sg_problem* prs, const int64_t* rows, int64_t nrows,
                                      const sg_exec* ex, sg_result** out) {
    if (!out) return fail(-1, "null output handles");
    if (!vel || !prs) return fail(-1, "null problem");
    const int n = vel->n;
    for (int c = 0; c < n && c < 3; ++c) out[c] = nullptr;
    if (prs->n != n || n < 1 || n > 3) return fail(-1, "velocity/pressure dimension mismatch");
    if (vel->p != prs->p + 1) return fail(-1, "velocity degree must be the pressure degree + 1");
    for (int d = 0; d < n; ++d)
        if (vel->m[d] - vel->p != 2 * (prs->m[d] - prs->p))
            return fail(-1, "velocity mesh must halve every pressure element (subgrid pair)");
    if (vel->sol_w || prs->sol_w) return fail(-2, "rational (NURBS) Stokes spaces are not supported by the divergence kernels");
    if (ex && (ex->slab_lo != 0 || ex->slab_hi != 0)) return fail(-2, "row slabs are not supported for the divergence pairing");
    Call c(ex);
    sg_problem vp = *vel;
    vp.form = POISSON;  // velocity tables with first derivatives, geometry with first derivatives
    DevProblem dp;
    int rc = prepare_problem(c, &vp, dp);
    if (rc) return rc;
    DivParams s{};
    s.n = n;
    s.pv = vel->p;
    s.pp = prs->p;
    s.pg = vel->geo_p;
    s.g = vel->g;
    int64_t Np = 1, Ev = 1, npts = 1;
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
    s.Dg = (double*)c.alloc(sizeof(double) * npts * n * n, true);
    // elements and rows
    std::vector<int64_t> elist;
    uint8_t* rowmask = nullptr;
    if (rows) {
        for (int64_t k = 0; k < nrows; ++k) {
            if (rows[k] < 0 || rows[k] >= Np) return fail(-1, "pressure row index out of range");
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
                    for (int e0 = elo[0]; e0 <= ehi[0]; ++e0)
                        emask[e0 + (int64_t)s.Sv[0] * (e1 + (int64_t)s.Sv[1] * e2)] = 1;
        }
        std::vector<int> slot(Ev, -1);
        for (int64_t e = 0; e < Ev; ++e)
            if (emask[e]) {
                slot[e] = (int)elist.size();
                elist.push_back(e);
            }
        s.eslot = (const int*)c.upload(slot.data(), sizeof(int) * Ev);
        rowmask = (uint8_t*)c.alloc(Np + 1, true);
        cudaMemsetAsync(rowmask, 0, Np + 1, c.stream);
        if (nrows > 0) {
            int64_t* dr = (int64_t*)c.upload(rows, sizeof(int64_t) * nrows);
            div_mask_kernel<<<(unsigned)((nrows + 255) / 256), 256, 0, c.stream>>>(dr, nrows, rowmask);
        }
    } else {
        elist.resize(Ev);
        for (int64_t e = 0; e < Ev; ++e) elist[e] = e;
        s.eslot = nullptr;
    }
    s.rowmask = rowmask;
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
    if (!s.eloc || !s.Dg) return fail(-4, "device allocation failed");
    // row pointers
    int64_t* counts = (int64_t*)c.alloc(sizeof(int64_t) * (Np + 1), true);
    int64_t* rowstart = (int64_t*)c.alloc(sizeof(int64_t) * (Np + 1), true);
    c.kbegin("div_counts");
    if (n == 1) div_counts_kernel<1><<<(unsigned)((Np + 256) / 256), 256, 0, c.stream>>>(s, counts);
    if (n == 2) div_counts_kernel<2><<<(unsigned)((Np + 256) / 256), 256, 0, c.stream>>>(s, counts);
    if (n == 3) div_counts_kernel<3><<<(unsigned)((Np + 256) / 256), 256, 0, c.stream>>>(s, counts);
    c.kend();
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, counts, rowstart, Np + 1, c.stream);
    void* tmp = c.alloc(tb, true);
    cub::DeviceScan::ExclusiveSum(tmp, tb, counts, rowstart, Np + 1, c.stream);
    int64_t nnz = 0;
    cudaMemcpyAsync(&nnz, rowstart + Np, sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream);
    cudaStreamSynchronize(c.stream);
    s.rowstart = rowstart;
    sg_result* res[3] = {nullptr, nullptr, nullptr};
    for (int k = 0; k < n; ++k) {
        sg_result* r = new sg_result();
        r->dev = c.dev;
        r->nrows = Np;
        r->nrows_global = Np;
        r->row_lo = 0;
        r->nnz = nnz;
        r->indptr = (int64_t*)c.alloc(sizeof(int64_t) * (Np + 1), false);
        r->indices = (int*)c.alloc(sizeof(int) * std::max<int64_t>(nnz, 1), false);
        r->data = (double*)c.alloc(sizeof(double) * std::max<int64_t>(nnz, 1), false);
        res[k] = r;
        if (!r->indptr || !r->indices || !r->data) {
            for (int q = 0; q <= k; ++q) sg_result_free(res[q]);
            return fail(-4, "device allocation failed (nnz=%lld)", (long long)nnz);
        }
        cudaMemcpyAsync(r->indptr, rowstart, sizeof(int64_t) * (Np + 1), cudaMemcpyDeviceToDevice, c.stream);
        s.indices[k] = r->indices;
        s.data[k] = r->data;
    }
    // local kernel shared memory: tables + the element's point tensors
    int Q = 1;
    for (int d = 0; d < n; ++d) Q *= s.g;
    const size_t local_smem = sizeof(double) * ((size_t)n * s.g * (s.pp + 1) + (size_t)n * s.g * 2 * (s.pv + 1) + (size_t)Q * n * n);
    if (local_smem > 227 * 1024) {
        for (int q = 0; q < n; ++q) sg_result_free(res[q]);
        return fail(-2, "divergence element tables do not fit shared memory");
    }
    if (n == 1) rc = run_divergence<1>(c, s, npts, local_smem);
    if (n == 2) rc = run_divergence<2>(c, s, npts, local_smem);
    if (n == 3) rc = run_divergence<3>(c, s, npts, local_smem);
    if (!rc) rc = c.finish();
    if (!rc) {
        cudaStreamSynchronize(c.stream);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) rc = fail(-3, "CUDA error in the divergence assembly: %s", cudaGetErrorString(e));
    }
    if (rc) {
        for (int q = 0; q < n; ++q) sg_result_free(res[q]);
        return rc;
    }
    c.record_timing();
    for (int k = 0; k < n; ++k) out[k] = res[k];
    return 0;
}
