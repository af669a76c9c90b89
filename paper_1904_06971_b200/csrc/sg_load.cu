// Load vector (reference: surriga/assembly.py:728-759 assemble_load):
//     vec_i = sum_e sum_q f(phi(x_q)) det J(x_q) w_q N_i(x_q)
// f is the caller's Python callable of physical coordinates, so the call is split at the host:
//   sg_map_points   : physical quadrature points phi(x_q), element-major (E, Q, n) -> host (f runs there)
//   sg_assemble_load: f values (E, Q) -> device; det * w_q (and the NURBS weight W for rational spaces)
//                     per point, then one thread per basis function sums its elements' points in
//                     ascending element order (no atomics: deterministic, like np.add.at's order).
#include <algorithm>
#include <vector>

#include "../../include/surriga_b200.h"
#include "sg_common.cuh"
#include "sg_internal.h"

namespace sg {

struct LoadParams {
    int n, p, pg, g;
    int S[3], m[3], mg[3], G[3];
    const double* B[3];        // solution tables [G][p+1] (values)
    const int* bspan[3];
    const double* Gt[3];       // geometry tables [G][2][pg+1]
    const int* gspan[3];
    const double* qw[3];
    const double* hom;         // [Ng][n+1]
    const double* sol_w;       // rational weights or nullptr
    double* phi;               // [E*Q][n] element-major
    double* wdet;              // [E*Q] det * w_q
    double* Wq;                // [E*Q] NURBS weight (rational) or nullptr
    const double* f;           // [E*Q]
    double* vec;               // [N]
};

template <int NDIM>
__global__ void load_geom_kernel(LoadParams s) {
    const int64_t npts = (int64_t)s.G[0] * s.G[1] * s.G[2];
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= npts) return;
    int x[3] = {(int)(t % s.G[0]), (int)((t / s.G[0]) % s.G[1]), (int)(t / ((int64_t)s.G[0] * s.G[1]))};
    const int pg = s.pg, g = s.g;
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
    double det;
    if constexpr (NDIM == 1) det = jac[0][0];
    else if constexpr (NDIM == 2) det = jac[0][0] * jac[1][1] - jac[0][1] * jac[1][0];
    else
        det = jac[0][0] * (jac[1][1] * jac[2][2] - jac[1][2] * jac[2][1]) -
              jac[0][1] * (jac[1][0] * jac[2][2] - jac[1][2] * jac[2][0]) +
              jac[0][2] * (jac[1][0] * jac[2][1] - jac[1][1] * jac[2][0]);
    double wq = s.qw[0][x[0] % g];
    if (NDIM >= 2) wq *= s.qw[1][x[1] % g];
    if (NDIM >= 3) wq *= s.qw[2][x[2] % g];
    // element-major index: element colex, point colex inside the element
    const int64_t e = (int64_t)(x[0] / g) + (int64_t)s.S[0] * ((int64_t)(x[1] / g) + (int64_t)s.S[1] * (x[2] / g));
    int Q = g;
    if (NDIM >= 2) Q *= g;
    if (NDIM >= 3) Q *= g;
    const int q = x[0] % g + g * (x[1] % g + g * (x[2] % g));
    const int64_t idx = e * Q + q;
    if (s.phi)
#pragma unroll
        for (int c = 0; c < NDIM; ++c) s.phi[idx * NDIM + c] = phi[c];
    if (s.wdet) s.wdet[idx] = det * wq;
    if (s.Wq) {
        // NURBS weight of the solution space: sum_j w_j B_j(x_q)
        const int p = s.p;
        const int b0 = s.bspan[0][x[0]], b1 = NDIM >= 2 ? s.bspan[1][x[1]] : 0, b2 = NDIM >= 3 ? s.bspan[2][x[2]] : 0;
        double Wv = 0.0;
        for (int t2 = 0; t2 <= (NDIM >= 3 ? p : 0); ++t2)
            for (int t1 = 0; t1 <= (NDIM >= 2 ? p : 0); ++t1)
                for (int t0 = 0; t0 <= p; ++t0) {
                    const int64_t j = (int64_t)(b0 - p + t0) +
                                      (int64_t)s.m[0] * ((NDIM >= 2 ? (int64_t)(b1 - p + t1) : 0) +
                                                         (int64_t)s.m[1] * (NDIM >= 3 ? (int64_t)(b2 - p + t2) : 0));
                    double bv = s.B[0][(int64_t)x[0] * (p + 1) + t0];
                    if (NDIM >= 2) bv *= s.B[1][(int64_t)x[1] * (p + 1) + t1];
                    if (NDIM >= 3) bv *= s.B[2][(int64_t)x[2] * (p + 1) + t2];
                    Wv = fma(s.sol_w[j], bv, Wv);
                }
        s.Wq[idx] = Wv;
    }
}

template <int NDIM>
__global__ void load_gather_kernel(LoadParams s) {
    const int64_t N = (int64_t)s.m[0] * s.m[1] * s.m[2];
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const int p = s.p, g = s.g;
    int id[3] = {(int)(i % s.m[0]), (int)((i / s.m[0]) % s.m[1]), (int)(i / ((int64_t)s.m[0] * s.m[1]))};
    int elo[3] = {0, 0, 0}, ehi[3] = {0, 0, 0};
    for (int d = 0; d < NDIM; ++d) {
        elo[d] = max(0, id[d] - p);
        ehi[d] = min(s.S[d] - 1, id[d]);
    }
    int Q = g;
    if (NDIM >= 2) Q *= g;
    if (NDIM >= 3) Q *= g;
    const double wi = s.sol_w ? s.sol_w[i] : 1.0;
    double acc = 0.0;
    for (int e2 = elo[2]; e2 <= ehi[2]; ++e2)
        for (int e1 = elo[1]; e1 <= ehi[1]; ++e1)
            for (int e0 = elo[0]; e0 <= ehi[0]; ++e0) {
                const int64_t e = (int64_t)e0 + (int64_t)s.S[0] * ((int64_t)e1 + (int64_t)s.S[1] * e2);
                const int l0 = id[0] - e0, l1 = id[1] - e1, l2 = id[2] - e2;
                double lv = 0.0;
                for (int q = 0; q < Q; ++q) {
                    const int q0 = q % g, q1 = (q / g) % g, q2 = q / (g * g);
                    double b = s.B[0][((int64_t)e0 * g + q0) * (p + 1) + l0];
                    if (NDIM >= 2) b *= s.B[1][((int64_t)e1 * g + q1) * (p + 1) + l1];
                    if (NDIM >= 3) b *= s.B[2][((int64_t)e2 * g + q2) * (p + 1) + l2];
                    const int64_t idx = e * Q + q;
                    if (s.Wq) b = wi * b / s.Wq[idx];
                    lv = fma(s.f[idx] * s.wdet[idx], b, lv);
                }
                acc += lv;
            }
    s.vec[i] = acc;
}

static int load_setup(Call& c, const sg_problem* prob, DevProblem& dp, LoadParams& s, int64_t& E, int& Q) {
    sg_problem pr = *prob;
    pr.form = MASS;  // solution tables (values), geometry tables with first derivatives
    int rc = prepare_problem(c, &pr, dp);
    if (rc) return rc;
    s = LoadParams{};
    s.n = dp.n;
    s.p = dp.p;
    s.pg = pr.geo_p;
    s.g = dp.g;
    E = 1;
    Q = 1;
    for (int d = 0; d < 3; ++d) {
        s.S[d] = dp.S[d];
        s.m[d] = dp.m[d];
        s.mg[d] = dp.mg[d];
        s.G[d] = d < dp.n ? dp.S[d] * dp.g : 1;
        s.B[d] = dp.B[d];
        s.bspan[d] = dp.bspan[d];
        s.Gt[d] = dp.G[d];
        s.gspan[d] = dp.gspan[d];
        s.qw[d] = dp.qw[d];
        E *= dp.S[d];
        if (d < dp.n) Q *= dp.g;
    }
    s.hom = dp.hom;
    s.sol_w = dp.sol_w;
    return 0;
}

template <int NDIM>
static void launch_load_geom(Call& c, const LoadParams& s, int64_t npts) {
    c.kbegin("load_geom");
    load_geom_kernel<NDIM><<<(unsigned)((npts + 127) / 128), 128, 0, c.stream>>>(s);
    c.kend();
}

}  // namespace sg

using namespace sg;

extern "C" int sg_map_points(const sg_problem* prob, const sg_exec* ex, double* phi_out) {
    if (!prob || !phi_out) return fail(-1, "null argument");
    Call c(ex);
    DevProblem dp;
    LoadParams s;
    int64_t E = 0;
    int Q = 0;
    int rc = load_setup(c, prob, dp, s, E, Q);
    if (rc) return rc;
    const int64_t npts = E * Q;
    s.phi = (double*)c.alloc(sizeof(double) * npts * s.n, true);
    if (!s.phi) return fail(-4, "device allocation failed");
    if (s.n == 1) launch_load_geom<1>(c, s, npts);
    if (s.n == 2) launch_load_geom<2>(c, s, npts);
    if (s.n == 3) launch_load_geom<3>(c, s, npts);
    cudaMemcpyAsync(phi_out, s.phi, sizeof(double) * npts * s.n, cudaMemcpyDeviceToHost, c.stream);
    if ((rc = c.finish())) return rc;
    cudaStreamSynchronize(c.stream);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(-3, "CUDA error in sg_map_points: %s", cudaGetErrorString(e));
    c.record_timing();
    return 0;
}

extern "C" int sg_assemble_load(const sg_problem* prob, const double* fvals, const sg_exec* ex, double* vec_out) {
    if (!prob || !fvals || !vec_out) return fail(-1, "null argument");
    Call c(ex);
    DevProblem dp;
    LoadParams s;
    int64_t E = 0;
    int Q = 0;
    int rc = load_setup(c, prob, dp, s, E, Q);
    if (rc) return rc;
    const int64_t npts = E * Q;
    int64_t N = 1;
    for (int d = 0; d < 3; ++d) N *= s.m[d];
    s.wdet = (double*)c.alloc(sizeof(double) * npts, true);
    s.Wq = s.sol_w ? (double*)c.alloc(sizeof(double) * npts, true) : nullptr;
    s.f = (const double*)c.upload(fvals, sizeof(double) * npts);
    s.vec = (double*)c.alloc(sizeof(double) * N, true);
    if (!s.wdet || !s.f || !s.vec || (s.sol_w && !s.Wq)) return fail(-4, "device allocation failed");
    if (s.n == 1) launch_load_geom<1>(c, s, npts);
    if (s.n == 2) launch_load_geom<2>(c, s, npts);
    if (s.n == 3) launch_load_geom<3>(c, s, npts);
    c.kbegin("load_gather");
    if (s.n == 1) load_gather_kernel<1><<<(unsigned)((N + 127) / 128), 128, 0, c.stream>>>(s);
    if (s.n == 2) load_gather_kernel<2><<<(unsigned)((N + 127) / 128), 128, 0, c.stream>>>(s);
    if (s.n == 3) load_gather_kernel<3><<<(unsigned)((N + 127) / 128), 128, 0, c.stream>>>(s);
    c.kend();
    cudaMemcpyAsync(vec_out, s.vec, sizeof(double) * N, cudaMemcpyDeviceToHost, c.stream);
    if ((rc = c.finish())) return rc;
    cudaStreamSynchronize(c.stream);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(-3, "CUDA error in sg_assemble_load: %s", cudaGetErrorString(e));
    c.record_timing();
    return 0;
}
