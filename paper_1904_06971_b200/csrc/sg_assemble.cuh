// Tiled, sum-factorised Galerkin assembly kernel (full quadrature and row-restricted).
//
// Replaces the reference's element loop (assembly.py:579-651: _local_square :531-551,
// _SpaceBinding.local_basis :468-517, _geometry_blocks :558-576, csr_from_triplets :245-270).
//
// One CTA owns a box of rows T0 x T1 x T2 (colex multi-indices).  The entry A_ij is the
// global tensor contraction
//     A_ij = s_i s_j sum_{z} B2 B2 sum_{y} B1 B1 sum_{x} B0 B0  D_{mu nu}(x,y,z)
// over the Gauss points of the elements shared by i and j; the CTA evaluates it plane by
// plane (direction 2), contracting direction 0 (phase 1) and direction 1 (phase 2) in shared
// memory and direction 2 (phase 3) in registers, layer by layer.  The geometry (NURBS map,
// Jacobian, adjugate, determinant, Hessian) and the rational weight function are evaluated on
// each plane by sum factorisation from the coarse control nets, never materialised in HBM.
// Values are accumulated deterministically (fixed order, no atomics); each (i,j) and (j,i)
// are computed by the mirror-image sequence of IEEE operations, so the matrix is bitwise
// symmetric and any row subset / row slab is bitwise equal to the full assembly.
#pragma once
#include "sg_common.cuh"

namespace sg {

template <int NDIM>
__device__ __forceinline__ int c12(int a1, int a2) {
    if constexpr (NDIM == 3) return (a1 + a2) * (a1 + a2 + 1) / 2 + a2;
    else return a1;
}
template <int NDIM, int NU>
struct NC12 { static constexpr int v = NDIM == 3 ? (NU + 1) * (NU + 2) / 2 : NU + 1; };

// ---------------------------------------------------------------------------------------------
// plane preparation of a tensor field sum_{i} c_i B_i(x) (geometry or weight function):
//   3D: Hz[i1][i0][c][a2] = sum_r2 tz[a2][r2] coef[i0, i1, sz-deg+r2]
//       Hy[y][i0][c][c12(a1,a2)] = sum_r1 t1[y][a1][r1] Hz[s1(y)-deg+r1][i0][c][a2]
//   2D: Hy[y][i0][c][a1]        = sum_r1 t1[y][a1][r1] coef[i0, s1(y)-deg+r1]
// ---------------------------------------------------------------------------------------------
template <int NDIM, int NU, int C>
__device__ void field_plane_prep(const double* __restrict__ coef, int deg, const int* md, const double* t1,
                                 const int* s1, int Y, const double* tz, int sz, int lo0, int n0, int lo1, int n1,
                                 double* Hz, double* Hy) {
    const int tid = threadIdx.x, nt = blockDim.x;
    constexpr int NC = NC12<NDIM, NU>::v;
    if constexpr (NDIM == 3) {
        const int items = n0 * n1 * C;
        for (int it = tid; it < items; it += nt) {
            const int c = it % C;
            const int i0 = (it / C) % n0;
            const int i1 = it / (C * n0);
            const int g0 = lo0 + i0, g1 = lo1 + i1;
            double acc[NU + 1];
#pragma unroll
            for (int a = 0; a <= NU; ++a) acc[a] = 0.0;
            if (g0 < md[0] && g1 < md[1]) {
                for (int r = 0; r <= deg; ++r) {
                    const double v = coef[((long long)g0 + (long long)md[0] * (g1 + (long long)md[1] * (sz - deg + r))) * C + c];
#pragma unroll
                    for (int a = 0; a <= NU; ++a) acc[a] = fma(tz[a * (deg + 1) + r], v, acc[a]);
                }
            }
#pragma unroll
            for (int a = 0; a <= NU; ++a) Hz[((i1 * n0 + i0) * C + c) * (NU + 1) + a] = acc[a];
        }
        __syncthreads();
    }
    if constexpr (NDIM >= 2) {
        const int items = Y * n0 * C;
        for (int it = tid; it < items; it += nt) {
            const int c = it % C;
            const int i0 = (it / C) % n0;
            const int y = it / (C * n0);
            const int sy = s1[y];
            double acc[NC];
#pragma unroll
            for (int k = 0; k < NC; ++k) acc[k] = 0.0;
            for (int r = 0; r <= deg; ++r) {
                if constexpr (NDIM == 3) {
                    const double* hz = Hz + (((sy - deg + r - lo1) * n0 + i0) * C + c) * (NU + 1);
#pragma unroll
                    for (int a1 = 0; a1 <= NU; ++a1) {
                        const double b = t1[(y * (NU + 1) + a1) * (deg + 1) + r];
#pragma unroll
                        for (int a2 = 0; a2 + a1 <= NU; ++a2) acc[c12<3>(a1, a2)] = fma(b, hz[a2], acc[c12<3>(a1, a2)]);
                    }
                } else {
                    const int g0 = lo0 + i0;
                    const double v = (g0 < md[0]) ? coef[((long long)g0 + (long long)md[0] * (sy - deg + r)) * C + c] : 0.0;
#pragma unroll
                    for (int a1 = 0; a1 <= NU; ++a1) acc[a1] = fma(t1[(y * (NU + 1) + a1) * (deg + 1) + r], v, acc[a1]);
                }
            }
#pragma unroll
            for (int k = 0; k < NC; ++k) Hy[((y * n0 + i0) * C + c) * NC + k] = acc[k];
        }
    }
}

// point evaluation: out[c][code] for all multi-indices with |alpha| <= NU (code = a0+3a1+9a2)
template <int NDIM, int NU, int C>
__device__ __forceinline__ void field_point(const double* __restrict__ coef, int deg, const double* t0, int sx,
                                            const double* Hy, int y, int lo0, int n0, double (&out)[C][27]) {
    constexpr int NC = NC12<NDIM, NU>::v;
#pragma unroll
    for (int c = 0; c < C; ++c)
#pragma unroll
        for (int k = 0; k < 27; ++k) out[c][k] = 0.0;
    for (int r = 0; r <= deg; ++r) {
        const int i0 = sx - deg + r;
#pragma unroll
        for (int c = 0; c < C; ++c) {
            if constexpr (NDIM == 1) {
                const double v = coef[(long long)i0 * C + c];
#pragma unroll
                for (int a0 = 0; a0 <= NU; ++a0) out[c][a0] = fma(t0[a0 * (deg + 1) + r], v, out[c][a0]);
            } else {
                const double* hy = Hy + ((y * n0 + (i0 - lo0)) * C + c) * NC;
#pragma unroll
                for (int a0 = 0; a0 <= NU; ++a0) {
                    const double b = t0[a0 * (deg + 1) + r];
#pragma unroll
                    for (int a1 = 0; a1 + a0 <= NU; ++a1) {
                        if constexpr (NDIM == 3) {
#pragma unroll
                            for (int a2 = 0; a2 + a1 + a0 <= NU; ++a2)
                                out[c][a0 + 3 * a1 + 9 * a2] = fma(b, hy[c12<3>(a1, a2)], out[c][a0 + 3 * a1 + 9 * a2]);
                        } else {
                            out[c][a0 + 3 * a1] = fma(b, hy[a1], out[c][a0 + 3 * a1]);
                        }
                    }
                }
            }
        }
    }
}

__device__ __forceinline__ constexpr int ucode(int a) { return a == 0 ? 1 : (a == 1 ? 3 : 9); }

// ---------------------------------------------------------------------------------------------
// per-point physics: D_{mu nu} (packed upper triangle over Mset) from geometry numerators,
// weight-function values and the tensor Gauss weight.  Reference: geometry.py:185-229 (map,
// quotient rule), :98-131 (det, adj), assembly.py:558-576 (K, C, hess), :531-548 (integrands),
// :496-517 (rational basis).
// ---------------------------------------------------------------------------------------------
template <int NDIM, int FORM, bool RAT>
__device__ __forceinline__ void point_D(const double (&num)[NDIM + 1][27], const double (&wf)[1][27], double wq,
                                        double coefv, double* Dout) {
    constexpr Tables TT = TermTables<NDIM, FORM, RAT>::T;
    constexpr int MS = TT.MS;
    constexpr int NUG = geo_deriv(FORM);
    const double W = num[NDIM][0];
    double phi[NDIM], jac[NDIM][NDIM], dW[NDIM];
#pragma unroll
    for (int c = 0; c < NDIM; ++c) phi[c] = num[c][0] / W;
#pragma unroll
    for (int a = 0; a < NDIM; ++a) {
        dW[a] = num[NDIM][ucode(a)];
#pragma unroll
        for (int c = 0; c < NDIM; ++c) jac[c][a] = (num[c][ucode(a)] - phi[c] * num[NDIM][ucode(a)]) / W;
    }
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
        det = jac[0][0] * (jac[1][1] * jac[2][2] - jac[1][2] * jac[2][1]) -
              jac[0][1] * (jac[1][0] * jac[2][2] - jac[1][2] * jac[2][0]) +
              jac[0][2] * (jac[1][0] * jac[2][1] - jac[1][1] * jac[2][0]);
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
    // functional coefficient vectors over Mset: f[k][mu], D = sum_k f_k Core_k f_k^T
    double Dl[MS * (MS + 1) / 2];
    if constexpr (FORM == POISSON) {
        double Kw[NDIM][NDIM];
#pragma unroll
        for (int a = 0; a < NDIM; ++a)
#pragma unroll
            for (int c = 0; c < NDIM; ++c) {
                double s = 0.0;
#pragma unroll
                for (int b = 0; b < NDIM; ++b) s = fma(adj[a][b], adj[c][b], s);
                Kw[a][c] = (s / det) * coefv * wq;
            }
        if constexpr (!RAT) {
            // Mset = {e_a} in code order e0 (1), e1 (3), e2 (9)
#pragma unroll
            for (int mu = 0; mu < MS; ++mu)
#pragma unroll
                for (int nu = mu; nu < MS; ++nu) Dl[tri_index(mu, nu, MS)] = Kw[mu][nu];
        } else {
            const double Ws = wf[0][0];
            // d_a N = w (d_a B / W - B d_a W / W^2): R[a][mu]
            double R[NDIM][MS];
            static_for<0, MS>([&](auto MU) {
                constexpr int mu = decltype(MU)::value;
                constexpr int code = TT.mcode[mu];
#pragma unroll
                for (int a = 0; a < NDIM; ++a)
                    R[a][mu] = (code == 0) ? -wf[0][ucode(a)] / (Ws * Ws) : (code == ucode(a) ? 1.0 / Ws : 0.0);
            });
#pragma unroll
            for (int mu = 0; mu < MS; ++mu)
#pragma unroll
                for (int nu = mu; nu < MS; ++nu) {
                    double s = 0.0;
#pragma unroll
                    for (int a = 0; a < NDIM; ++a)
#pragma unroll
                        for (int b = 0; b < NDIM; ++b) s = fma(R[a][mu] * Kw[a][b], R[b][nu], s);
                    Dl[tri_index(mu, nu, MS)] = s;
                }
        }
    } else if constexpr (FORM == MASS) {
        if constexpr (!RAT) Dl[0] = det * wq;
        else Dl[0] = det * wq / (wf[0][0] * wf[0][0]);
    } else {
        // biharmonic: lap N = sum_ab C_ab d_ab N - sum_a g_a d_a N
        double hess[NDIM][NDIM][NDIM];
#pragma unroll
        for (int a = 0; a < NDIM; ++a)
#pragma unroll
            for (int b = a; b < NDIM; ++b) {
                const int cd = ucode(a) + ucode(b);
#pragma unroll
                for (int c = 0; c < NDIM; ++c) {
                    const double v = (num[c][cd] - jac[c][a] * dW[b] - jac[c][b] * dW[a] - phi[c] * num[NDIM][cd]) / W;
                    hess[c][a][b] = v;
                    hess[c][b][a] = v;
                }
            }
        double Cm[NDIM][NDIM];
        const double det2 = det * det;
#pragma unroll
        for (int a = 0; a < NDIM; ++a)
#pragma unroll
            for (int b = 0; b < NDIM; ++b) {
                double s = 0.0;
#pragma unroll
                for (int c = 0; c < NDIM; ++c) s = fma(adj[a][c], adj[b][c], s);
                Cm[a][b] = s / det2;
            }
        double h[NDIM], gv[NDIM];
#pragma unroll
        for (int c = 0; c < NDIM; ++c) {
            double s = 0.0;
#pragma unroll
            for (int a = 0; a < NDIM; ++a)
#pragma unroll
                for (int b = 0; b < NDIM; ++b) s = fma(hess[c][a][b], Cm[a][b], s);
            h[c] = s;
        }
#pragma unroll
        for (int a = 0; a < NDIM; ++a) {
            double s = 0.0;
#pragma unroll
            for (int c = 0; c < NDIM; ++c) s = fma(adj[a][c], h[c], s);
            gv[a] = s / det;
        }
        double f[MS];
        if constexpr (!RAT) {
            static_for<0, MS>([&](auto MU) {
                constexpr int mu = decltype(MU)::value;
                constexpr int code = TT.mcode[mu];
                double v = 0.0;
#pragma unroll
                for (int a = 0; a < NDIM; ++a) {
                    if (code == ucode(a)) v = -gv[a];
#pragma unroll
                    for (int b = a; b < NDIM; ++b)
                        if (code == ucode(a) + ucode(b)) v = (a == b) ? Cm[a][a] : 2.0 * Cm[a][b];
                }
                f[mu] = v;
            });
        } else {
            const double Ws = wf[0][0];
            double dWs[NDIM], d2Ws[NDIM][NDIM];
#pragma unroll
            for (int a = 0; a < NDIM; ++a) {
                dWs[a] = wf[0][ucode(a)];
#pragma unroll
                for (int b = 0; b < NDIM; ++b) d2Ws[a][b] = wf[0][ucode(a) + ucode(b)];
            }
            const double iW = 1.0 / Ws, iW2 = iW * iW, iW3 = iW2 * iW;
            double cC2W = 0.0, dWCdW = 0.0, gdW = 0.0;
#pragma unroll
            for (int a = 0; a < NDIM; ++a) {
                gdW = fma(gv[a], dWs[a], gdW);
#pragma unroll
                for (int c = 0; c < NDIM; ++c) {
                    cC2W = fma(Cm[a][c], d2Ws[a][c], cC2W);
                    dWCdW = fma(dWs[a] * Cm[a][c], dWs[c], dWCdW);
                }
            }
            static_for<0, MS>([&](auto MU) {
                constexpr int mu = decltype(MU)::value;
                constexpr int code = TT.mcode[mu];
                double v = 0.0;
                if (code == 0) v = -cC2W * iW2 + 2.0 * dWCdW * iW3 + gdW * iW2;
#pragma unroll
                for (int a = 0; a < NDIM; ++a) {
                    if (code == ucode(a)) {
                        double s = 0.0;
#pragma unroll
                        for (int c = 0; c < NDIM; ++c) s = fma(Cm[a][c] + Cm[c][a], dWs[c], s);
                        v = -s * iW2 - gv[a] * iW;
                    }
#pragma unroll
                    for (int b = a; b < NDIM; ++b)
                        if (code == ucode(a) + ucode(b)) v = ((a == b) ? Cm[a][a] : 2.0 * Cm[a][b]) * iW;
                }
                f[mu] = v;
            });
        }
        const double sw = det * wq;
#pragma unroll
        for (int mu = 0; mu < MS; ++mu)
#pragma unroll
            for (int nu = mu; nu < MS; ++nu) Dl[tri_index(mu, nu, MS)] = (f[mu] * f[nu]) * sw;
    }
#pragma unroll
    for (int k = 0; k < MS * (MS + 1) / 2; ++k) Dout[k] = Dl[k];
}

// ---------------------------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------------------------
template <int NDIM, int P, int FORM, bool RAT, int KMAX>
__global__ void __launch_bounds__(512, 1) assemble_tiles(const AsmParams prm) {
    constexpr Tables TT = TermTables<NDIM, FORM, RAT>::T;
    constexpr int MS = TT.MS;
    constexpr int U = MS * (MS + 1) / 2;
    constexpr int NU = form_deriv(FORM);
    constexpr int NUG = geo_deriv(FORM);
    constexpr int NB = (NU + 1) * (P + 1);       // solution table entries per point
    constexpr int W2P = 2 * P + 1;
    extern __shared__ double smem[];
    const int tid = threadIdx.x, nt = blockDim.x;
    const int g = prm.g;
    const int pg = prm.pg;
    const int NBG = (NUG + 1) * (pg + 1);

    // ---- tile geometry
    const int tile = prm.tiles ? prm.tiles[blockIdx.x] : (int)blockIdx.x;
    int tcoord[3];
    tcoord[0] = tile % prm.tgrid[0];
    tcoord[1] = (tile / prm.tgrid[0]) % prm.tgrid[1];
    tcoord[2] = tile / (prm.tgrid[0] * prm.tgrid[1]);
    int b[3], elo[3], ehi[3], NE[3], X[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        b[d] = tcoord[d] * prm.T[d];
        elo[d] = max(0, b[d] - P);
        ehi[d] = min(prm.S[d] - 1, b[d] + prm.T[d] - 1);
        NE[d] = ehi[d] - elo[d] + 1;
        X[d] = NE[d] * g;
    }
    if (NDIM < 2) { X[1] = 1; }
    const int T0 = prm.T[0], T1n = prm.T[1];
    const int Y = X[1];
    const int ypad = prm.ypad;

    double* B0s = smem + prm.off_B0;
    double* B1s = smem + prm.off_B1;
    double* G0s = smem + prm.off_G0;
    double* G1s = smem + prm.off_G1;
    int* gs0 = reinterpret_cast<int*>(smem + prm.off_gs0);
    int* gs1 = reinterpret_cast<int*>(smem + prm.off_gs1);
    double* Hz = smem + prm.off_Hz;
    double* Hy = smem + prm.off_Hy;
    double* Wz = smem + prm.off_Wz;
    double* Wy = smem + prm.off_Wy;
    double* Ds = smem + prm.off_D;
    double* T1s = smem + prm.off_T1;
    double* T2s = smem + prm.off_T2;
    double* misc = smem + prm.off_misc;
    // misc layout: qw[3][8] | B2 plane [NB] | G2 plane [(NUG+1)(pg+1)] | ws span ints
    double* qws = misc;
    double* B2p = misc + 24;
    double* G2p = B2p + NB;
    int* ws0 = reinterpret_cast<int*>(G2p + NBG);  // solution-field spans for window points (dir 0)
    int* ws1 = ws0 + X[0];

    // ---- window tables
    for (int it = tid; it < X[0] * NB; it += nt) {
        const int x = it / NB, k = it % NB;
        B0s[it] = prm.B[0][((long long)(elo[0] * g + x)) * NB + k];
    }
    for (int it = tid; it < X[0] * NBG; it += nt) {
        const int x = it / NBG, k = it % NBG;
        G0s[it] = prm.G[0][((long long)(elo[0] * g + x)) * NBG + k];
    }
    for (int x = tid; x < X[0]; x += nt) {
        gs0[x] = prm.gspan[0][elo[0] * g + x];
        ws0[x] = elo[0] + x / g + P;
    }
    if constexpr (NDIM >= 2) {
        for (int it = tid; it < X[1] * NB; it += nt) {
            const int y = it / NB, k = it % NB;
            B1s[it] = prm.B[1][((long long)(elo[1] * g + y)) * NB + k];
        }
        for (int it = tid; it < X[1] * NBG; it += nt) {
            const int y = it / NBG, k = it % NBG;
            G1s[it] = prm.G[1][((long long)(elo[1] * g + y)) * NBG + k];
        }
        for (int y = tid; y < X[1]; y += nt) {
            gs1[y] = prm.gspan[1][elo[1] * g + y];
            ws1[y] = elo[1] + y / g + P;
        }
    }
    for (int it = tid; it < 3 * g; it += nt) {
        const int d = it / g, q = it % g;
        qws[d * 8 + q] = (d < NDIM) ? prm.qw[d][q] : 1.0;
    }
    __syncthreads();
    // geometry function ranges on this window
    const int glo0 = gs0[0] - pg, gn0 = gs0[X[0] - 1] - gs0[0] + pg + 1;
    int glo1 = 0, gn1 = 1;
    if constexpr (NDIM >= 2) { glo1 = gs1[0] - pg; gn1 = gs1[X[1] - 1] - gs1[0] + pg + 1; }
    const int wlo0 = elo[0], wn0 = NE[0] + P;
    const int wlo1 = elo[1], wn1 = NE[1] + P;

    const int nlayer = (NDIM == 3) ? NE[2] : 1;
    const int gz = (NDIM == 3) ? g : 1;
    const int ncombo = T0 * W2P * T1n * W2P;
    double acc3[KMAX][P + 1];
    (void)acc3;

    for (int layer = 0; layer < nlayer; ++layer) {
        const int e2 = elo[2] + layer;
        if constexpr (NDIM == 3) {
#pragma unroll
            for (int k = 0; k < KMAX; ++k)
#pragma unroll
                for (int r = 0; r <= P; ++r) acc3[k][r] = 0.0;
        }
        for (int q2 = 0; q2 < gz; ++q2) {
            // ---------------- geometry + D on the plane
            int sz = 0, szw = 0;
            const int qz = e2 * g + q2;
            if constexpr (NDIM == 3) {
                __syncthreads();
                for (int k = tid; k < NB; k += nt) B2p[k] = prm.B[2][(long long)qz * NB + k];
                for (int k = tid; k < NBG; k += nt) G2p[k] = prm.G[2][(long long)qz * NBG + k];
                sz = prm.gspan[2][qz];
                szw = e2 + P;
                __syncthreads();
            }
            field_plane_prep<NDIM, NUG, NDIM + 1>(prm.hom, pg, prm.mg, G1s, gs1, Y, G2p, sz, glo0, gn0, glo1, gn1, Hz, Hy);
            if constexpr (RAT)
                field_plane_prep<NDIM, NU, 1>(prm.sol_w, P, prm.m, B1s, ws1, Y, B2p, szw, wlo0, wn0, wlo1, wn1, Wz, Wy);
            __syncthreads();
            const double wz = qws[2 * 8 + q2];
            for (int it = tid; it < X[0] * Y; it += nt) {
                const int y = it % Y, x = it / Y;
                double num[NDIM + 1][27];
                field_point<NDIM, NUG, NDIM + 1>(prm.hom, pg, G0s + x * NBG, gs0[x], Hy, y, glo0, gn0, num);
                double wf[1][27];
                if constexpr (RAT) field_point<NDIM, NU, 1>(prm.sol_w, P, B0s + x * NB, ws0[x], Wy, y, wlo0, wn0, wf);
                else wf[0][0] = 1.0;
                // tensor weight, reference order: wq = pw2 * (pw1 * pw0)  (assembly.py:120-125)
                double wq = qws[x % g];
                if constexpr (NDIM >= 2) wq = qws[8 + y % g] * wq;
                if constexpr (NDIM == 3) wq = wz * wq;
                double Dp[U];
                point_D<NDIM, FORM, RAT>(num, wf, wq, prm.coef, Dp);
#pragma unroll
                for (int u = 0; u < U; ++u) Ds[(u * X[0] + x) * ypad + y] = Dp[u];
            }
            __syncthreads();

            // ---------------- phase 1: contract direction 0 -> T1[G][i0l][d0][y]
            {
                const int items = TT.NG1 * T0 * Y;
                for (int it = tid; it < items; it += nt) {
                    const int y = it % Y;
                    const int i0l = (it / Y) % T0;
                    const int G = it / (Y * T0);
                    const int i0 = b[0] + i0l;
                    double acc[W2P];
#pragma unroll
                    for (int k = 0; k < W2P; ++k) acc[k] = 0.0;
                    if (i0 < prm.m[0]) {
                        static_for<0, TT.NG1>([&](auto GI) {
                            constexpr int Gc = decltype(GI)::value;
                            if (G != Gc) return;
#pragma unroll
                            for (int ri = P; ri >= 0; --ri) {
                                const int e0 = i0 - ri;
                                if (e0 < 0 || e0 >= prm.S[0]) continue;
                                const int le = e0 - elo[0];
                                for (int q = 0; q < g; ++q) {
                                    const int x = le * g + q;
                                    const double* bx = B0s + x * NB;
                                    static_for<0, TT.g1n[Gc]>([&](auto UI) {
                                        constexpr int Uc = decltype(UI)::value;
                                        constexpr int mu = TT.g1mu[Gc][Uc], nu = TT.g1nu[Gc][Uc];
                                        constexpr int am = acode(TT.mcode[mu], 0), an = acode(TT.mcode[nu], 0);
                                        constexpr bool pair = TT.g1pair[Gc][Uc] != 0;
                                        const double Dv = Ds[(tri_index(mu, nu, MS) * X[0] + x) * ypad + y];
                                        const double bim = bx[am * (P + 1) + ri];
                                        const double bin = bx[an * (P + 1) + ri];
#pragma unroll
                                        for (int rj = 0; rj <= P; ++rj) {
                                            double Q = __dmul_rn(bim, bx[an * (P + 1) + rj]);
                                            if constexpr (pair) Q = __dadd_rn(Q, __dmul_rn(bin, bx[am * (P + 1) + rj]));
                                            acc[rj - ri + P] = fma(Q, Dv, acc[rj - ri + P]);
                                        }
                                    });
                                }
                            }
                        });
                    }
                    if constexpr (NDIM == 1) {
                        // final: row i0, columns i0 + d0
                        const int64_t row = i0;
                        if (i0 < prm.m[0] && row >= prm.slab_lo && row < prm.slab_hi && (!prm.rowmask || prm.rowmask[row])) {
                            const int lo = max(0, i0 - P);
                            const int64_t base = prm.rowstart[row];
                            const double si = RAT ? prm.sol_w[i0] : 1.0;
#pragma unroll
                            for (int d0 = -P; d0 <= P; ++d0) {
                                const int j0 = i0 + d0;
                                if (j0 < 0 || j0 >= prm.m[0]) continue;
                                double v = acc[d0 + P];
                                if constexpr (RAT) v = v * (si * prm.sol_w[j0]);
                                prm.data[base + (j0 - lo)] = v;
                                prm.indices[base + (j0 - lo)] = j0;
                                if (prm.zeros && v == 0.0) atomicAdd(prm.zeros, 1ull);
                            }
                        }
                    } else {
#pragma unroll
                        for (int k = 0; k < W2P; ++k) T1s[((G * T0 + i0l) * W2P + k) * ypad + y] = acc[k];
                    }
                }
            }
            if constexpr (NDIM >= 2) {
                __syncthreads();
                // ---------------- phase 2: contract direction 1
                const int NG2x = (NDIM == 3) ? TT.NG2 : 1;
                const int items = NG2x * T0 * W2P * T1n;
                for (int it = tid; it < items; it += nt) {
                    const int i1l = it % T1n;
                    const int d0i = (it / T1n) % W2P;
                    const int i0l = (it / (T1n * W2P)) % T0;
                    const int G2 = it / (T1n * W2P * T0);
                    const int i0 = b[0] + i0l, i1 = b[1] + i1l;
                    double acc[W2P];
#pragma unroll
                    for (int k = 0; k < W2P; ++k) acc[k] = 0.0;
                    const bool valid = (i0 < prm.m[0]) && (i1 < prm.m[1]);
                    if (valid) {
#pragma unroll
                        for (int ri = P; ri >= 0; --ri) {
                            const int e1 = i1 - ri;
                            if (e1 < 0 || e1 >= prm.S[1]) continue;
                            const int le = e1 - elo[1];
                            for (int q = 0; q < g; ++q) {
                                const int y = le * g + q;
                                const double* by = B1s + y * NB;
                                const double* t1b = T1s + (i0l * W2P + d0i) * ypad + y;
                                auto unit = [&](auto GA, auto GB, auto PAIR) {
                                    constexpr int ga = decltype(GA)::value, gb = decltype(GB)::value;
                                    constexpr bool pr = decltype(PAIR)::value != 0;
                                    constexpr int k1 = TT.g1key[ga];
                                    constexpr int a1 = k1 % 3, b1 = (k1 / 3) % 3;
                                    const double t = t1b[ga * T0 * W2P * ypad];
                                    const double bia = by[a1 * (P + 1) + ri];
                                    if constexpr (!pr) {
#pragma unroll
                                        for (int rj = 0; rj <= P; ++rj)
                                            acc[rj - ri + P] = fma(__dmul_rn(bia, by[b1 * (P + 1) + rj]), t, acc[rj - ri + P]);
                                    } else {
                                        const double tT = t1b[gb * T0 * W2P * ypad];
                                        const double bib = by[b1 * (P + 1) + ri];
#pragma unroll
                                        for (int rj = 0; rj <= P; ++rj) {
                                            const double uu = __dmul_rn(__dmul_rn(bia, by[b1 * (P + 1) + rj]), t);
                                            const double vv = __dmul_rn(__dmul_rn(bib, by[a1 * (P + 1) + rj]), tT);
                                            acc[rj - ri + P] = __dadd_rn(acc[rj - ri + P], __dadd_rn(uu, vv));
                                        }
                                    }
                                };
                                if constexpr (NDIM == 2) {
                                    static_for<0, TT.NF>([&](auto FI) {
                                        constexpr int f = decltype(FI)::value;
                                        constexpr int ga = TT.fu[f];
                                        unit(std::integral_constant<int, ga>{}, std::integral_constant<int, TT.g1T[ga]>{},
                                             std::integral_constant<int, TT.fpair[f]>{});
                                    });
                                } else {
                                    static_for<0, TT.NG2>([&](auto GI) {
                                        constexpr int Gc = decltype(GI)::value;
                                        if (G2 != Gc) return;
                                        static_for<0, TT.g2n[Gc]>([&](auto UI) {
                                            constexpr int Uc = decltype(UI)::value;
                                            constexpr int ga = TT.g2u[Gc][Uc];
                                            unit(std::integral_constant<int, ga>{}, std::integral_constant<int, TT.g1T[ga]>{},
                                                 std::integral_constant<int, TT.g2pair[Gc][Uc]>{});
                                        });
                                    });
                                }
                            }
                        }
                    }
                    if constexpr (NDIM == 2) {
                        const int64_t row = (int64_t)i0 + (int64_t)prm.m[0] * i1;
                        if (valid && row >= prm.slab_lo && row < prm.slab_hi && (!prm.rowmask || prm.rowmask[row])) {
                            const int d0 = d0i - P;
                            const int j0 = i0 + d0;
                            if (j0 >= 0 && j0 < prm.m[0]) {
                                const int lo0 = max(0, i0 - P), lo1 = max(0, i1 - P);
                                const int cnt0 = min(prm.m[0] - 1, i0 + P) - lo0 + 1;
                                const int64_t base = prm.rowstart[row];
                                const double si = RAT ? prm.sol_w[row] : 1.0;
#pragma unroll
                                for (int d1 = -P; d1 <= P; ++d1) {
                                    const int j1 = i1 + d1;
                                    if (j1 < 0 || j1 >= prm.m[1]) continue;
                                    double v = acc[d1 + P];
                                    const int64_t col = (int64_t)j0 + (int64_t)prm.m[0] * j1;
                                    if constexpr (RAT) v = v * (si * prm.sol_w[col]);
                                    const int64_t pos = base + (j0 - lo0) + (int64_t)cnt0 * (j1 - lo1);
                                    prm.data[pos] = v;
                                    prm.indices[pos] = (int)col;
                                    if (prm.zeros && v == 0.0) atomicAdd(prm.zeros, 1ull);
                                }
                            }
                        }
                    } else {
                        const int combo = ((i0l * W2P + d0i) * T1n + i1l) * W2P;
#pragma unroll
                        for (int k = 0; k < W2P; ++k) T2s[G2 * ncombo + combo + k] = acc[k];
                    }
                }
            }
            if constexpr (NDIM == 3) {
                __syncthreads();
                // ---------------- phase 3: contract direction 2 within the layer (registers)
                const double* bz = B2p;
#pragma unroll
                for (int k = 0; k < KMAX; ++k) {
                    const int it = tid + k * nt;
                    if (it >= ncombo * (P + 1)) break;
                    const int combo = it % ncombo;
                    const int ri2 = it / ncombo;
                    static_for<0, TT.NF>([&](auto FI) {
                        constexpr int f = decltype(FI)::value;
                        constexpr int ga = TT.fu[f];
                        constexpr int gb = TT.g2T[ga];
                        constexpr bool pr = TT.fpair[f] != 0;
                        constexpr int k2 = TT.g2key[ga];
                        constexpr int a2 = k2 % 3, b2 = k2 / 3;
                        const double t = T2s[ga * ncombo + combo];
                        const double bia = bz[a2 * (P + 1) + ri2];
                        if constexpr (!pr) {
#pragma unroll
                            for (int rj = 0; rj <= P; ++rj)
                                acc3[k][rj] = fma(__dmul_rn(bia, bz[b2 * (P + 1) + rj]), t, acc3[k][rj]);
                        } else {
                            const double tT = T2s[gb * ncombo + combo];
                            const double bib = bz[b2 * (P + 1) + ri2];
#pragma unroll
                            for (int rj = 0; rj <= P; ++rj) {
                                const double uu = __dmul_rn(__dmul_rn(bia, bz[b2 * (P + 1) + rj]), t);
                                const double vv = __dmul_rn(__dmul_rn(bib, bz[a2 * (P + 1) + rj]), tT);
                                acc3[k][rj] = __dadd_rn(acc3[k][rj], __dadd_rn(uu, vv));
                            }
                        }
                    });
                }
            }
        }  // q2
        if constexpr (NDIM == 3) {
            // ---------------- layer end: accumulate into the CSR (rows owned by this CTA only)
#pragma unroll
            for (int k = 0; k < KMAX; ++k) {
                const int it = tid + k * nt;
                if (it >= ncombo * (P + 1)) break;
                const int combo = it % ncombo;
                const int ri2 = it / ncombo;
                const int d1 = combo % W2P - P;
                const int i1l = (combo / W2P) % T1n;
                const int d0 = (combo / (W2P * T1n)) % W2P - P;
                const int i0l = combo / (W2P * T1n * W2P);
                const int i0 = b[0] + i0l, i1 = b[1] + i1l, i2 = e2 + ri2;
                const int j0 = i0 + d0, j1 = i1 + d1;
                if (i0 >= prm.m[0] || i1 >= prm.m[1] || i2 < b[2] || i2 >= b[2] + prm.T[2] || i2 >= prm.m[2]) continue;
                if (j0 < 0 || j0 >= prm.m[0] || j1 < 0 || j1 >= prm.m[1]) continue;
                const int64_t row = (int64_t)i0 + (int64_t)prm.m[0] * ((int64_t)i1 + (int64_t)prm.m[1] * i2);
                if (row < prm.slab_lo || row >= prm.slab_hi) continue;
                if (prm.rowmask && !prm.rowmask[row]) continue;
                const int lo0 = max(0, i0 - P), lo1 = max(0, i1 - P), lo2 = max(0, i2 - P);
                const int cnt0 = min(prm.m[0] - 1, i0 + P) - lo0 + 1;
                const int cnt1 = min(prm.m[1] - 1, i1 + P) - lo1 + 1;
                const int64_t base = prm.rowstart[row] + (j0 - lo0) + (int64_t)cnt0 * (j1 - lo1);
                const double si = RAT ? prm.sol_w[row] : 1.0;
#pragma unroll
                for (int rj = 0; rj <= P; ++rj) {
                    const int j2 = e2 + rj;
                    const int64_t pos = base + (int64_t)cnt0 * cnt1 * (j2 - lo2);
                    const int first = max(0, max(i2, j2) - P);
                    const int last = min(min(i2, j2), prm.S[2] - 1);
                    double v = acc3[k][rj];
                    if (e2 != first) v = prm.data[pos] + v;
                    const int64_t col = (int64_t)j0 + (int64_t)prm.m[0] * ((int64_t)j1 + (int64_t)prm.m[1] * j2);
                    if (e2 == last) {
                        if constexpr (RAT) v = v * (si * prm.sol_w[col]);
                        if (prm.zeros && v == 0.0) atomicAdd(prm.zeros, 1ull);
                    }
                    if (e2 == first) prm.indices[pos] = (int)col;
                    prm.data[pos] = v;
                }
            }
            __syncthreads();
        }
    }
}

}  // namespace sg
