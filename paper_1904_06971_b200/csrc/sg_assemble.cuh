// K4: tiled, sum-factorised Galerkin assembly (full quadrature and row-restricted).
//
// Replaces the reference's element loop (assembly.py:579-651: _local_square :531-551,
// _SpaceBinding.local_basis :468-517, csr_from_triplets :245-270).
//
// One CTA owns a box of rows T0 x T1 x T2 (colex multi-indices).  The entry A_ij is the
// global tensor contraction
//     A_ij = s_i s_j sum_{z} B2 B2 sum_{y} B1 B1 sum_{x} B0 B0  D_{mu nu}(x,y,z)
// over the Gauss points of the elements shared by i and j (D from K3, sg_geom.cuh); the CTA
// streams the D window plane by plane (direction 2), contracts direction 0 (phase 1) and
// direction 1 (phase 2) in shared memory and direction 2 (phase 3) in registers, layer by layer.
// Values are accumulated deterministically (fixed order, no atomics); each (i,j) and (j,i)
// are computed by the mirror-image sequence of IEEE operations, so the matrix is bitwise
// symmetric and any row subset / row slab is bitwise equal to the full assembly.
#pragma once
#include "sg_common.cuh"

namespace sg {

// ---------------------------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------------------------
template <int NDIM, int P, int FORM, bool RAT, int KMAX>
__global__ void __launch_bounds__(512, 1) assemble_tiles(const AsmParams prm) {
    constexpr Tables TT = TermTables<NDIM, FORM, RAT>::T;
    constexpr int MS = TT.MS;
    constexpr int U = MS * (MS + 1) / 2;
    constexpr int NU = form_deriv(FORM);
    constexpr int NB = (NU + 1) * (P + 1);       // solution table entries per point
    constexpr int W2P = 2 * P + 1;
    extern __shared__ double smem[];
    const int tid = threadIdx.x, nt = blockDim.x;
    const int g = prm.g;

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
    double* Ds = smem + prm.off_D;
    double* T1s = smem + prm.off_T1;
    double* T2s = smem + prm.off_T2;
    double* B2p = smem + prm.off_misc;

    // ---- window basis tables
    for (int it = tid; it < X[0] * NB; it += nt) B0s[it] = prm.B[0][(long long)elo[0] * g * NB + it];
    if constexpr (NDIM >= 2)
        for (int it = tid; it < X[1] * NB; it += nt) B1s[it] = prm.B[1][(long long)elo[1] * g * NB + it];
    const long long xw0 = (long long)elo[0] * g, yw0 = (long long)elo[1] * g;
    const long long G0 = prm.Gp[0], G1 = prm.Dys;

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
            // ---------------- stream the D window of this plane (from K3)
            const int qz = e2 * g + q2;
            if constexpr (NDIM == 3) {
                __syncthreads();
                for (int k = tid; k < NB; k += nt) B2p[k] = prm.B[2][(long long)qz * NB + k];
            }
            {
                const long long zoff = (long long)qz * U;
                const int rows = U * X[0];
                for (int it = tid; it < rows * Y; it += nt) {
                    const int y = it % Y, r = it / Y;
                    const int u = r / X[0], x = r % X[0];
                    Ds[r * ypad + y] = prm.D[((zoff + u) * G0 + xw0 + x) * G1 + yw0 + y];
                }
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
