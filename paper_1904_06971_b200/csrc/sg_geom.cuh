// K3: geometry at the Gauss points -> per-point form tensor D_{mu nu}(x, y, z).
//
// Replaces the reference's full-grid geometry evaluation (geometry.py:185-229 map_grid,
// :98-131 det/adj; assembly.py:558-576 _geometry_blocks, :402-438 weight function of a rational
// space) and folds the integrand algebra of assembly.py:531-548 / :496-517 into D, so that
//     A_ij = s_i s_j sum_q sum_{mu,nu} D_{mu nu}(q) d^mu B_i(q) d^nu B_j(q).
// Each CTA evaluates one block of points of one z-plane by sum factorisation over the coarse
// control net (contract z, then y, then x), so every Gauss point is evaluated exactly once.
// D is stored plane-major, [z][u][x][y] (y fastest), the layout the tile kernel streams.
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
// plane preparation of a tensor field sum_i c_i B_i (geometry map or NURBS weight function) on a
// block of points of one z-plane (x fastest-changing per warp is avoided: a warp shares x):
//   3D: Hz[i1][i0][c][a2]           = sum_r2 tz[a2][r2] coef[i0, i1, sz-deg+r2]
//       Hx[x][i1][c][k(a0,a2)]      = sum_r0 t0[x][a0][r0] Hz[i1][s0(x)-deg+r0][c][a2]
//   2D: Hx[x][i1][c][a0]            = sum_r0 t0[x][a0][r0] coef[s0(x)-deg+r0, i1]
// then per point (x, y): out[c][a0+3a1+9a2] = sum_r1 t1[y][a1][r1] Hx[x][s1(y)-deg+r1][c][k(a0,a2)]
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ constexpr int k02(int a0, int a2) { return (a0 + a2) * (a0 + a2 + 1) / 2 + a2; }
template <int NDIM, int NU>
struct NCx { static constexpr int v = NDIM == 3 ? (NU + 1) * (NU + 2) / 2 : NU + 1; };

// C components of the field are read from coefficient rows of stride CS (a polynomial geometry map
// skips the weight column of its homogeneous net)
template <int NDIM, int NU, int C, int CS = C>
__device__ void field_plane_prep(const double* __restrict__ coef, int deg, const int* md, const double* t0, int ts0,
                                 const int* s0, int X, const double* tz, int sz, int lo0, int n0, int lo1, int n1,
                                 double* Hz, double* Hx, int hxs) {
    const int tid = threadIdx.x, nt = blockDim.x;
    constexpr int NC = NCx<NDIM, NU>::v;
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
                    const double v = coef[((long long)g0 + (long long)md[0] * (g1 + (long long)md[1] * (sz - deg + r))) * CS + c];
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
        const int items = X * n1 * C;
        for (int it = tid; it < items; it += nt) {
            const int c = it % C;
            const int i1 = (it / C) % n1;
            const int x = it / (C * n1);
            const int sx = s0[x];
            double acc[NC];
#pragma unroll
            for (int k = 0; k < NC; ++k) acc[k] = 0.0;
            for (int r = 0; r <= deg; ++r) {
                if constexpr (NDIM == 3) {
                    const double* hz = Hz + ((i1 * n0 + (sx - deg + r - lo0)) * C + c) * (NU + 1);
#pragma unroll
                    for (int a0 = 0; a0 <= NU; ++a0) {
                        const double b = t0[x * ts0 + a0 * (deg + 1) + r];
#pragma unroll
                        for (int a2 = 0; a2 + a0 <= NU; ++a2) acc[k02(a0, a2)] = fma(b, hz[a2], acc[k02(a0, a2)]);
                    }
                } else {
                    const int g1 = lo1 + i1;
                    const double v = (g1 < md[1]) ? coef[((long long)(sx - deg + r) + (long long)md[0] * g1) * CS + c] : 0.0;
#pragma unroll
                    for (int a0 = 0; a0 <= NU; ++a0) acc[a0] = fma(t0[x * ts0 + a0 * (deg + 1) + r], v, acc[a0]);
                }
            }
#pragma unroll
            for (int k = 0; k < NC; ++k) Hx[x * hxs + (i1 * C + c) * NC + k] = acc[k];
        }
    }
}

// point evaluation: out[c][code] for all multi-indices with |alpha| <= NU (code = a0+3a1+9a2).
// 2D/3D: t = y table of this point, s = its span, H = Hx + x*hxs.  1D: t = x table, s = x span.
// DEG >= 0: the degree as a compile-time constant (the r loop unrolls and its shared-memory loads are
// scheduled ahead of the FMAs: the runtime-degree loop issued each load right before its FMA and
// stalled on it, geom_D ran at ~32% of the fp64 pipe); DEG < 0: runtime degree `deg`
template <int NDIM, int NU, int C, int DEG = -1, int CS = C>
__device__ __forceinline__ void field_point(const double* __restrict__ coef, int deg_rt, const double* t, int s,
                                            const double* H, int lo1, double (&out)[C][27]) {
    if constexpr (DEG < 0 && NDIM >= 2) {
        if (deg_rt == 2) return field_point<NDIM, NU, C, 2, CS>(coef, 2, t, s, H, lo1, out);
        if (deg_rt == 3) return field_point<NDIM, NU, C, 3, CS>(coef, 3, t, s, H, lo1, out);
    }
    const int deg = DEG >= 0 ? DEG : deg_rt;
    constexpr int NC = NCx<NDIM, NU>::v;
#pragma unroll
    for (int c = 0; c < C; ++c)
#pragma unroll
        for (int k = 0; k < 27; ++k) out[c][k] = 0.0;
#pragma unroll
    for (int r = 0; r <= deg; ++r) {
        const int i = s - deg + r;
#pragma unroll
        for (int c = 0; c < C; ++c) {
            if constexpr (NDIM == 1) {
                const double v = coef[(long long)i * CS + c];
#pragma unroll
                for (int a0 = 0; a0 <= NU; ++a0) out[c][a0] = fma(t[a0 * (deg + 1) + r], v, out[c][a0]);
            } else {
                const double* h = H + ((i - lo1) * C + c) * NC;
#pragma unroll
                for (int a1 = 0; a1 <= NU; ++a1) {
                    const double b = t[a1 * (deg + 1) + r];
#pragma unroll
                    for (int a0 = 0; a0 + a1 <= NU; ++a0) {
                        if constexpr (NDIM == 3) {
#pragma unroll
                            for (int a2 = 0; a2 + a1 + a0 <= NU; ++a2)
                                out[c][a0 + 3 * a1 + 9 * a2] = fma(b, h[k02(a0, a2)], out[c][a0 + 3 * a1 + 9 * a2]);
                        } else {
                            out[c][a0 + 3 * a1] = fma(b, h[a0], out[c][a0 + 3 * a1]);
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
// GPOLY: the geometry map is polynomial (unit weights, the reference's GeometryMap.is_polynomial,
// geometry.py:167): W = 1 and its derivatives vanish, so the quotient rule of map_grid
// (geometry.py:196-227) reduces to the numerators (num[NDIM] is not read)
template <int NDIM, int FORM, bool RAT, bool GPOLY = false>
__device__ __forceinline__ void point_D(const double (&num)[NDIM + 1][27], const double (&wf)[1][27], double wq,
                                        double coefv, double* Dout) {
    constexpr Tables TT = TermTables<NDIM, FORM, RAT>::T;
    constexpr int MS = TT.MS;
    constexpr int NUG = geo_deriv(FORM);
    const double iW = GPOLY ? 1.0 : 1.0 / num[NDIM][0];
    double phi[NDIM], jac[NDIM][NDIM], dW[NDIM];
#pragma unroll
    for (int c = 0; c < NDIM; ++c) phi[c] = GPOLY ? num[c][0] : num[c][0] * iW;
#pragma unroll
    for (int a = 0; a < NDIM; ++a) {
        dW[a] = GPOLY ? 0.0 : num[NDIM][ucode(a)];
#pragma unroll
        for (int c = 0; c < NDIM; ++c)
            jac[c][a] = GPOLY ? num[c][ucode(a)] : (num[c][ucode(a)] - phi[c] * num[NDIM][ucode(a)]) * iW;
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
    const double idet = 1.0 / det;
    if constexpr (FORM == POISSON) {
        double Kw[NDIM][NDIM];
#pragma unroll
        for (int a = 0; a < NDIM; ++a)
#pragma unroll
            for (int c = 0; c < NDIM; ++c) {
                double s = 0.0;
#pragma unroll
                for (int b = 0; b < NDIM; ++b) s = fma(adj[a][b], adj[c][b], s);
                Kw[a][c] = (s * idet) * coefv * wq;
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
                    const double v = GPOLY ? num[c][cd] : (num[c][cd] - jac[c][a] * dW[b] - jac[c][b] * dW[a] - phi[c] * num[NDIM][cd]) * iW;
                    hess[c][a][b] = v;
                    hess[c][b][a] = v;
                }
            }
        double Cm[NDIM][NDIM];
        const double idet2 = idet * idet;
#pragma unroll
        for (int a = 0; a < NDIM; ++a)
#pragma unroll
            for (int b = 0; b < NDIM; ++b) {
                double s = 0.0;
#pragma unroll
                for (int c = 0; c < NDIM; ++c) s = fma(adj[a][c], adj[b][c], s);
                Cm[a][b] = s * idet2;
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
            gv[a] = s * idet;
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


struct GeomParams {
    int p, g, pg;
    int m[3], mg[3];
    const double* B[3];      // solution tables [S*g][nu+1][p+1]
    const double* qw[3];
    const double* sol_w;
    const int* gspan[3];
    const double* G[3];      // geometry tables [S*g][nug+1][pg+1]
    const double* hom;
    double coef;
    int Gp[3];               // global Gauss points per direction (1 for unused directions)
    int BX, BY;              // points per block (x, y)
    int nbx, nby;            // blocks per plane
    const int* blocks;       // block ids (bx + nbx*(by + nby*z)) or nullptr = all
    const uint8_t* blockmask; // restricted plans: blocks to compute (others exit), or nullptr
    int GN0, GN1, WN0, WN1;  // smem bounds of function ranges
    int off_G0, off_G1, off_gs0, off_gs1, off_B0, off_B1, off_ws0, off_ws1, off_Hz, off_Hy, off_Wz, off_Wy, off_misc;
    int U;
    int ZB;                  // z-planes per block (3D): the x/y tables are loaded once per block
    int Dys;                 // y stride of D (Gp1 rounded up to even: 16-byte rows for TMA)
    double* D;               // [Gp2][U][Gp0][Dys]
};

template <int NDIM, int FORM, bool RAT, bool GPOLY>
__global__ void __launch_bounds__(256) geom_D_kernel(const GeomParams prm) {
    constexpr Tables TT = TermTables<NDIM, FORM, RAT>::T;
    constexpr int MS = TT.MS;
    constexpr int U = MS * (MS + 1) / 2;
    constexpr int NU = form_deriv(FORM);
    constexpr int NUG = geo_deriv(FORM);
    extern __shared__ double smem[];
    const int tid = threadIdx.x, nt = blockDim.x;
    const int g = prm.g, pg = prm.pg, p = prm.p;
    const int NB = (NU + 1) * (p + 1), NBG = (NUG + 1) * (pg + 1);
    const int NBp = NB | 1, NBGp = NBG | 1;  // odd per-point strides: per-lane y tables conflict free
    // block = (bx, by, z-batch of ZB planes); a plane whose (bx, by, z) block is not marked in a
    // restricted plan is skipped
    const int blk = (int)blockIdx.x;
    const int bx = blk % prm.nbx, by = (blk / prm.nbx) % prm.nby, zb = blk / (prm.nbx * prm.nby);
    const int z0 = zb * prm.ZB, z1 = min(prm.Gp[2], z0 + prm.ZB);
    if (prm.blockmask) {
        bool any = false;
        for (int z = z0; z < z1; ++z) any = any || prm.blockmask[bx + prm.nbx * (by + prm.nby * z)];
        if (!any) return;
    }
    const int x0 = bx * prm.BX, y0 = by * prm.BY;
    const int X = min(prm.BX, prm.Gp[0] - x0);
    const int Y = NDIM >= 2 ? min(prm.BY, prm.Gp[1] - y0) : 1;
    double* G0s = smem + prm.off_G0;
    double* G1s = smem + prm.off_G1;
    int* gs0 = reinterpret_cast<int*>(smem + prm.off_gs0);
    int* gs1 = reinterpret_cast<int*>(smem + prm.off_gs1);
    double* B0s = smem + prm.off_B0;
    double* B1s = smem + prm.off_B1;
    int* ws0 = reinterpret_cast<int*>(smem + prm.off_ws0);
    int* ws1 = reinterpret_cast<int*>(smem + prm.off_ws1);
    double* Hz = smem + prm.off_Hz;
    double* Hx = smem + prm.off_Hy;
    double* Wz = smem + prm.off_Wz;
    double* Wx = smem + prm.off_Wy;
    double* misc = smem + prm.off_misc;
    double* G2p = misc;
    double* B2p = misc + 32;
    double* qwx = misc + 64;
    double* qwy = qwx + prm.BX;
    for (int it = tid; it < X * NBG; it += nt) G0s[it] = prm.G[0][(long long)x0 * NBG + it];
    for (int x = tid; x < X; x += nt) {
        gs0[x] = prm.gspan[0][x0 + x];
        qwx[x] = prm.qw[0][(x0 + x) % g];
    }
    if constexpr (RAT) {
        for (int it = tid; it < X * NB; it += nt) B0s[it] = prm.B[0][(long long)x0 * NB + it];
        for (int x = tid; x < X; x += nt) ws0[x] = (x0 + x) / g + p;
    }
    if constexpr (NDIM >= 2) {
        for (int it = tid; it < Y * NBG; it += nt) G1s[(it / NBG) * NBGp + it % NBG] = prm.G[1][(long long)y0 * NBG + it];
        for (int y = tid; y < Y; y += nt) {
            gs1[y] = prm.gspan[1][y0 + y];
            qwy[y] = prm.qw[1][(y0 + y) % g];
        }
        if constexpr (RAT) {
            for (int it = tid; it < Y * NB; it += nt) B1s[(it / NB) * NBp + it % NB] = prm.B[1][(long long)y0 * NB + it];
            for (int y = tid; y < Y; y += nt) ws1[y] = (y0 + y) / g + p;
        }
    }
    for (int z = z0; z < z1; ++z) {
    if (prm.blockmask && !prm.blockmask[bx + prm.nbx * (by + prm.nby * z)]) continue;  // uniform over the block
    __syncthreads();  // the previous plane's Hz / Hx / z tables are no longer read
    int sz = 0, szw = 0;
    if constexpr (NDIM == 3) {
        for (int k = tid; k < NBG; k += nt) G2p[k] = prm.G[2][(long long)z * NBG + k];
        if constexpr (RAT)
            for (int k = tid; k < NB; k += nt) B2p[k] = prm.B[2][(long long)z * NB + k];
        sz = prm.gspan[2][z];
        szw = z / g + p;
    }
    __syncthreads();
    const int glo0 = gs0[0] - pg, gn0 = gs0[X - 1] - gs0[0] + pg + 1;
    int glo1 = 0, gn1 = 1;
    if constexpr (NDIM >= 2) { glo1 = gs1[0] - pg; gn1 = gs1[Y - 1] - gs1[0] + pg + 1; }
    const int wlo0 = x0 / g, wn0 = (x0 + X - 1) / g - x0 / g + 1 + p;
    int wlo1 = 0, wn1 = 1;
    if constexpr (NDIM >= 2) { wlo1 = y0 / g; wn1 = (y0 + Y - 1) / g - y0 / g + 1 + p; }
    constexpr int C = GPOLY ? NDIM : NDIM + 1;  // field components evaluated (polynomial map: no weight)
    constexpr int CS = NDIM + 1;                 // row stride of the homogeneous net
    const int hxs = gn1 * C * NCx<NDIM, NUG>::v;
    const int wxs = wn1 * NCx<NDIM, NU>::v;
    field_plane_prep<NDIM, NUG, C, CS>(prm.hom, pg, prm.mg, G0s, NBG, gs0, X, G2p, sz, glo0, gn0, glo1, gn1, Hz, Hx, hxs);
    if constexpr (RAT)
        field_plane_prep<NDIM, NU, 1>(prm.sol_w, p, prm.m, B0s, NB, ws0, X, B2p, szw, wlo0, wn0, wlo1, wn1, Wz, Wx, wxs);
    __syncthreads();
    const double wz = NDIM == 3 ? prm.qw[2][z % g] : 1.0;
    for (int it = tid; it < X * Y; it += nt) {
        const int y = it % Y, x = it / Y;  // a warp shares x: Hx reads broadcast, y tables per lane
        double num[NDIM + 1][27];
        double wf[1][27];
        auto& numc = *reinterpret_cast<double(*)[C][27]>(&num);
        if constexpr (NDIM == 1) {
            field_point<1, NUG, C, -1, CS>(prm.hom, pg, G0s + x * NBG, gs0[x], nullptr, 0, numc);
            if constexpr (RAT) field_point<1, NU, 1>(prm.sol_w, p, B0s + x * NB, ws0[x], nullptr, 0, wf);
        } else {
            field_point<NDIM, NUG, C, -1, CS>(prm.hom, pg, G1s + y * NBGp, gs1[y], Hx + x * hxs, glo1, numc);
            if constexpr (RAT) field_point<NDIM, NU, 1>(prm.sol_w, p, B1s + y * NBp, ws1[y], Wx + x * wxs, wlo1, wf);
        }
        if constexpr (!RAT) wf[0][0] = 1.0;
        // tensor weight in the reference order wq = pw2 * (pw1 * pw0)  (assembly.py:120-125)
        double wq = qwx[x];
        if constexpr (NDIM >= 2) wq = qwy[y] * wq;
        if constexpr (NDIM == 3) wq = wz * wq;
        double Dp[U];
        point_D<NDIM, FORM, RAT, GPOLY>(num, wf, wq, prm.coef, Dp);
        const long long plane = (long long)z * U;
#pragma unroll
        for (int u = 0; u < U; ++u)
            prm.D[((plane + u) * prm.Gp[0] + x0 + x) * (long long)prm.Dys + y0 + y] = Dp[u];
    }
    }  // z planes of the block
}

}  // namespace sg
