// Quadrature fields (reference: surriga/assembly.py:839-907 quadrature_fields): physical samples
// of a coefficient field at every element quadrature point, the step after assembly in the
// studies (error norms, right-hand sides).
//
// One thread per tensor Gauss point.  The geometry map is evaluated from its homogeneous control
// net with up to second derivatives (geometry.py:185-229 quotient rule), the field as the weighted
// numerator U = sum_l c_l w_l B_l over the weight function W = sum_l w_l B_l (the reference's
// rational basis N_l = w_l B_l / W, assembly.py:496-517, contracted with the coefficients), then
//   grad u = adj(J)^T du / det,   Hess u = adj^T (d2u - grad u . hess phi) adj / det^2
// (assembly.py:891-903).  Outputs are element-major (element colex, point colex inside it), as the
// reference returns them.
#include <algorithm>

#include "../../include/surriga_b200.h"
#include "sg_common.cuh"
#include "sg_internal.h"

namespace sg {

struct FieldParams {
    int p, pg, g;
    int S[3], m[3], mg[3], G[3];
    const double* B[3];   // solution tables [G][nu+1][p+1]
    const int* bspan[3];
    const double* Gt[3];  // geometry tables [G][nug+1][pg+1]
    const int* gspan[3];
    const double* qw[3];
    const double* hom;    // [Ng][n+1]
    const double* sol_w;  // rational weights or nullptr
    const double* coef;   // [N]
    double* x;            // [T][n]
    double* w;            // [T]
    double* val;          // [T]
    double* grad;         // [T][n] or nullptr
    double* hess;         // [T][n][n] or nullptr
};

// derivative components: 0 value, 1..n first derivatives, then the upper-triangle (a <= b) seconds
template <int NDIM>
struct DerivIdx {
    static constexpr int NC2 = 1 + NDIM + NDIM * (NDIM + 1) / 2;
};
__host__ __device__ constexpr int d2idx(int ndim, int a, int b) {
    // position of (min, max) in the upper-triangle list after 1 + ndim entries
    const int lo = a < b ? a : b, hi = a < b ? b : a;
    int k = 1 + ndim;
    for (int i = 0; i < lo; ++i) k += ndim - i;
    return k + (hi - lo);
}

template <int NDIM, int NU>
__global__ void __launch_bounds__(128) fields_kernel(FieldParams s) {
    constexpr int NUG = NU >= 2 ? 2 : 1;                        // geometry derivatives needed
    constexpr int NCG = NUG >= 2 ? DerivIdx<NDIM>::NC2 : 1 + NDIM;
    constexpr int NCF = NU >= 2 ? DerivIdx<NDIM>::NC2 : (NU >= 1 ? 1 + NDIM : 1);
    const int64_t npts = (int64_t)s.G[0] * s.G[1] * s.G[2];
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= npts) return;
    const int x[3] = {(int)(t % s.G[0]), (int)((t / s.G[0]) % s.G[1]), (int)(t / ((int64_t)s.G[0] * s.G[1]))};
    // derivative orders per direction of every component
    int ord[NCG > NCF ? NCG : NCF][3];
    {
        constexpr int NCX = NCG > NCF ? NCG : NCF;
        for (int k = 0; k < NCX; ++k) ord[k][0] = ord[k][1] = ord[k][2] = 0;
        for (int a = 0; a < NDIM && 1 + a < NCX; ++a) ord[1 + a][a] = 1;
        if (NCX > 1 + NDIM)
            for (int a = 0; a < NDIM; ++a)
                for (int b = a; b < NDIM; ++b) {
                    const int k = d2idx(NDIM, a, b);
                    ord[k][a] += 1;
                    ord[k][b] += 1;
                }
    }
    // ---- geometry: homogeneous numerators num[c][k] (c < NDIM: P_c, c = NDIM: W)
    double num[NDIM + 1][NCG];
#pragma unroll
    for (int c = 0; c <= NDIM; ++c)
#pragma unroll
        for (int k = 0; k < NCG; ++k) num[c][k] = 0.0;
    {
        const int pg = s.pg;
        const int sp0 = s.gspan[0][x[0]], sp1 = NDIM >= 2 ? s.gspan[1][x[1]] : 0, sp2 = NDIM >= 3 ? s.gspan[2][x[2]] : 0;
        for (int t2 = 0; t2 <= (NDIM >= 3 ? pg : 0); ++t2)
            for (int t1 = 0; t1 <= (NDIM >= 2 ? pg : 0); ++t1)
                for (int t0 = 0; t0 <= pg; ++t0) {
                    const int64_t ci = (int64_t)(sp0 - pg + t0) +
                                       (int64_t)s.mg[0] * ((NDIM >= 2 ? (int64_t)(sp1 - pg + t1) : 0) +
                                                           (int64_t)s.mg[1] * (NDIM >= 3 ? (int64_t)(sp2 - pg + t2) : 0));
                    const int tt[3] = {t0, t1, t2};
                    double b[NCG];
#pragma unroll
                    for (int k = 0; k < NCG; ++k) {
                        double v = 1.0;
#pragma unroll
                        for (int d = 0; d < NDIM; ++d)
                            v *= s.Gt[d][((int64_t)x[d] * (NUG + 1) + ord[k][d]) * (pg + 1) + tt[d]];
                        b[k] = v;
                    }
#pragma unroll
                    for (int c = 0; c <= NDIM; ++c) {
                        const double h = s.hom[ci * (NDIM + 1) + c];
#pragma unroll
                        for (int k = 0; k < NCG; ++k) num[c][k] = fma(b[k], h, num[c][k]);
                    }
                }
    }
    const double W = num[NDIM][0], iW = 1.0 / W;
    double phi[NDIM], jac[NDIM][NDIM], hs[NDIM][NDIM][NDIM];
#pragma unroll
    for (int c = 0; c < NDIM; ++c) phi[c] = num[c][0] * iW;
#pragma unroll
    for (int c = 0; c < NDIM; ++c)
#pragma unroll
        for (int a = 0; a < NDIM; ++a) jac[c][a] = (num[c][1 + a] - phi[c] * num[NDIM][1 + a]) * iW;
    if constexpr (NU >= 2) {
#pragma unroll
        for (int c = 0; c < NDIM; ++c)
#pragma unroll
            for (int a = 0; a < NDIM; ++a)
#pragma unroll
                for (int b = 0; b < NDIM; ++b) {
                    const int k = d2idx(NDIM, a, b);
                    hs[c][a][b] = (num[c][k] - jac[c][a] * num[NDIM][1 + b] - jac[c][b] * num[NDIM][1 + a] - phi[c] * num[NDIM][k]) * iW;
                }
    }
    // det and adjugate (geometry.py:98-131): adj = det * J^{-1}, adj[a][c]
    double det, adj[NDIM][NDIM];
    if constexpr (NDIM == 1) {
        det = jac[0][0];
        adj[0][0] = 1.0;
    } else if constexpr (NDIM == 2) {
        det = jac[0][0] * jac[1][1] - jac[0][1] * jac[1][0];
        adj[0][0] = jac[1][1];
        adj[0][1] = -jac[0][1];
        adj[1][0] = -jac[1][0];
        adj[1][1] = jac[0][0];
    } else {
        adj[0][0] = jac[1][1] * jac[2][2] - jac[1][2] * jac[2][1];
        adj[0][1] = jac[0][2] * jac[2][1] - jac[0][1] * jac[2][2];
        adj[0][2] = jac[0][1] * jac[1][2] - jac[0][2] * jac[1][1];
        adj[1][0] = jac[1][2] * jac[2][0] - jac[1][0] * jac[2][2];
        adj[1][1] = jac[0][0] * jac[2][2] - jac[0][2] * jac[2][0];
        adj[1][2] = jac[0][2] * jac[1][0] - jac[0][0] * jac[1][2];
        adj[2][0] = jac[1][0] * jac[2][1] - jac[1][1] * jac[2][0];
        adj[2][1] = jac[0][1] * jac[2][0] - jac[0][0] * jac[2][1];
        adj[2][2] = jac[0][0] * jac[1][1] - jac[0][1] * jac[1][0];
        det = jac[0][0] * adj[0][0] + jac[0][1] * adj[1][0] + jac[0][2] * adj[2][0];
    }
    // ---- field: weighted numerator and weight function with their derivatives
    double U[NCF], Ws[NCF];
#pragma unroll
    for (int k = 0; k < NCF; ++k) U[k] = Ws[k] = 0.0;
    {
        const int p = s.p;
        const int b0 = s.bspan[0][x[0]], b1 = NDIM >= 2 ? s.bspan[1][x[1]] : 0, b2 = NDIM >= 3 ? s.bspan[2][x[2]] : 0;
        for (int t2 = 0; t2 <= (NDIM >= 3 ? p : 0); ++t2)
            for (int t1 = 0; t1 <= (NDIM >= 2 ? p : 0); ++t1)
                for (int t0 = 0; t0 <= p; ++t0) {
                    const int64_t j = (int64_t)(b0 - p + t0) +
                                      (int64_t)s.m[0] * ((NDIM >= 2 ? (int64_t)(b1 - p + t1) : 0) +
                                                         (int64_t)s.m[1] * (NDIM >= 3 ? (int64_t)(b2 - p + t2) : 0));
                    const int tt[3] = {t0, t1, t2};
                    const double wj = s.sol_w ? s.sol_w[j] : 1.0;
                    const double cw = s.coef[j] * wj;
#pragma unroll
                    for (int k = 0; k < NCF; ++k) {
                        double v = 1.0;
#pragma unroll
                        for (int d = 0; d < NDIM; ++d) v *= s.B[d][((int64_t)x[d] * (NU + 1) + ord[k][d]) * (p + 1) + tt[d]];
                        U[k] = fma(cw, v, U[k]);
                        if (s.sol_w) Ws[k] = fma(wj, v, Ws[k]);
                    }
                }
    }
    double u, du[NDIM], d2u[NDIM][NDIM];
    if (s.sol_w) {
        const double iWs = 1.0 / Ws[0];
        u = U[0] * iWs;
        if constexpr (NU >= 1) {
#pragma unroll
            for (int a = 0; a < NDIM; ++a) du[a] = (U[1 + a] - u * Ws[1 + a]) * iWs;
        }
        if constexpr (NU >= 2) {
#pragma unroll
            for (int a = 0; a < NDIM; ++a)
#pragma unroll
                for (int b = 0; b < NDIM; ++b) {
                    const int k = d2idx(NDIM, a, b);
                    d2u[a][b] = (U[k] - du[a] * Ws[1 + b] - du[b] * Ws[1 + a] - u * Ws[k]) * iWs;
                }
        }
    } else {
        u = U[0];
        if constexpr (NU >= 1) {
#pragma unroll
            for (int a = 0; a < NDIM; ++a) du[a] = U[1 + a];
        }
        if constexpr (NU >= 2) {
#pragma unroll
            for (int a = 0; a < NDIM; ++a)
#pragma unroll
                for (int b = 0; b < NDIM; ++b) d2u[a][b] = U[d2idx(NDIM, a, b)];
        }
    }
    // ---- element-major output
    const int g = s.g;
    const int64_t e = (int64_t)(x[0] / g) + (int64_t)s.S[0] * ((int64_t)(x[1] / g) + (int64_t)s.S[1] * (x[2] / g));
    int Q = g;
    if (NDIM >= 2) Q *= g;
    if (NDIM >= 3) Q *= g;
    const int q = x[0] % g + g * (x[1] % g + g * (x[2] % g));
    const int64_t idx = e * Q + q;
    double wq = s.qw[0][x[0] % g];
    if (NDIM >= 2) wq *= s.qw[1][x[1] % g];
    if (NDIM >= 3) wq *= s.qw[2][x[2] % g];
#pragma unroll
    for (int c = 0; c < NDIM; ++c) s.x[idx * NDIM + c] = phi[c];
    s.w[idx] = wq * det;
    s.val[idx] = u;
    if constexpr (NU >= 1) {
        double gph[NDIM];
        const double idet = 1.0 / det;
#pragma unroll
        for (int c = 0; c < NDIM; ++c) {
            double v = 0.0;
#pragma unroll
            for (int a = 0; a < NDIM; ++a) v = fma(du[a], adj[a][c], v);
            gph[c] = v * idet;
            s.grad[idx * NDIM + c] = gph[c];
        }
        if constexpr (NU >= 2) {
            double T[NDIM][NDIM];
#pragma unroll
            for (int a = 0; a < NDIM; ++a)
#pragma unroll
                for (int b = 0; b < NDIM; ++b) {
                    double v = d2u[a][b];
#pragma unroll
                    for (int c = 0; c < NDIM; ++c) v = fma(-gph[c], hs[c][a][b], v);
                    T[a][b] = v;
                }
            const double idet2 = idet * idet;
#pragma unroll
            for (int c = 0; c < NDIM; ++c)
#pragma unroll
                for (int d = 0; d < NDIM; ++d) {
                    double v = 0.0;
#pragma unroll
                    for (int a = 0; a < NDIM; ++a) {
                        double r = 0.0;
#pragma unroll
                        for (int b = 0; b < NDIM; ++b) r = fma(T[a][b], adj[b][d], r);
                        v = fma(adj[a][c], r, v);
                    }
                    s.hess[(idx * NDIM + c) * NDIM + d] = v * idet2;
                }
        }
    }
}

template <int NDIM>
static void* fields_fn(int nu) {
    return nu == 0 ? (void*)fields_kernel<NDIM, 0> : (nu == 1 ? (void*)fields_kernel<NDIM, 1> : (void*)fields_kernel<NDIM, 2>);
}

}  // namespace sg

using namespace sg;

extern "C" int sg_quadrature_fields(const sg_problem* prob, const double* coefs, int32_t nu, const sg_exec* ex, double* x_out,
                                    double* w_out, double* val_out, double* grad_out, double* hess_out) {
    if (!prob || !coefs || !x_out || !w_out || !val_out) return fail(-1, "null argument");
    if (nu < 0 || nu > 2) return fail(-1, "nu must be 0, 1 or 2");
    if ((nu >= 1 && !grad_out) || (nu >= 2 && !hess_out)) return fail(-1, "null derivative output");
    Call c(ex);
    DevProblem dp;
    sg_problem pr = *prob;
    pr.form = MASS;  // validation + uploads; the tables are re-tabulated below with the needed orders
    int rc = prepare_problem(c, &pr, dp);
    if (rc) return rc;
    const int n = dp.n, nug = nu >= 2 ? 2 : 1;
    FieldParams s{};
    s.p = dp.p;
    s.pg = pr.geo_p;
    s.g = dp.g;
    int64_t E = 1;
    int Q = 1;
    for (int d = 0; d < 3; ++d) {
        s.S[d] = dp.S[d];
        s.m[d] = dp.m[d];
        s.mg[d] = dp.mg[d];
        s.G[d] = d < n ? dp.S[d] * dp.g : 1;
        s.qw[d] = dp.qw[d];
        E *= dp.S[d];
        if (d < n) {
            Q *= dp.g;
            const int npts = dp.S[d] * dp.g;
            double* kn = (double*)c.upload(pr.knots[d], sizeof(double) * (dp.m[d] + dp.p + 1));
            double* qp = (double*)c.upload(pr.qpts[d], sizeof(double) * npts);
            double* Bt = (double*)c.alloc(sizeof(double) * npts * (nu + 1) * (dp.p + 1), true);
            int* bs = (int*)c.alloc(sizeof(int) * npts, true);
            tabulate(c, kn, dp.m[d] + dp.p + 1, dp.p, qp, npts, nu, bs, Bt);
            double* gk = (double*)c.upload(pr.geo_knots[d], sizeof(double) * (dp.mg[d] + pr.geo_p + 1));
            double* Gt = (double*)c.alloc(sizeof(double) * npts * (nug + 1) * (pr.geo_p + 1), true);
            int* gs = (int*)c.alloc(sizeof(int) * npts, true);
            tabulate(c, gk, dp.mg[d] + pr.geo_p + 1, pr.geo_p, qp, npts, nug, gs, Gt);
            s.B[d] = Bt;
            s.bspan[d] = bs;
            s.Gt[d] = Gt;
            s.gspan[d] = gs;
        }
    }
    s.hom = dp.hom;
    s.sol_w = dp.sol_w;
    const int64_t T = E * Q;
    s.coef = (const double*)c.upload(coefs, sizeof(double) * dp.N);
    s.x = (double*)c.alloc(sizeof(double) * T * n, true);
    s.w = (double*)c.alloc(sizeof(double) * T, true);
    s.val = (double*)c.alloc(sizeof(double) * T, true);
    s.grad = nu >= 1 ? (double*)c.alloc(sizeof(double) * T * n, true) : nullptr;
    s.hess = nu >= 2 ? (double*)c.alloc(sizeof(double) * T * n * n, true) : nullptr;
    if (!s.coef || !s.x || !s.w || !s.val || (nu >= 1 && !s.grad) || (nu >= 2 && !s.hess)) return fail(-4, "device allocation failed");
    void* fn = n == 1 ? fields_fn<1>(nu) : (n == 2 ? fields_fn<2>(nu) : fields_fn<3>(nu));
    void* args[] = {&s};
    c.kbegin("quadrature_fields");
    cudaError_t e = cudaLaunchKernel(fn, dim3((unsigned)((T + 127) / 128)), dim3(128), args, 0, c.stream);
    c.kend();
    if (e != cudaSuccess) return fail(-3, "fields launch failed: %s", cudaGetErrorString(e));
    cudaMemcpyAsync(x_out, s.x, sizeof(double) * T * n, cudaMemcpyDeviceToHost, c.stream);
    cudaMemcpyAsync(w_out, s.w, sizeof(double) * T, cudaMemcpyDeviceToHost, c.stream);
    cudaMemcpyAsync(val_out, s.val, sizeof(double) * T, cudaMemcpyDeviceToHost, c.stream);
    if (nu >= 1) cudaMemcpyAsync(grad_out, s.grad, sizeof(double) * T * n, cudaMemcpyDeviceToHost, c.stream);
    if (nu >= 2) cudaMemcpyAsync(hess_out, s.hess, sizeof(double) * T * n * n, cudaMemcpyDeviceToHost, c.stream);
    if ((rc = c.finish())) return rc;
    cudaStreamSynchronize(c.stream);
    e = cudaGetLastError();
    if (e != cudaSuccess) return fail(-3, "CUDA error in sg_quadrature_fields: %s", cudaGetErrorString(e));
    c.record_timing();
    return 0;
}
