// K4: tiled, sum-factorised Galerkin assembly on the fp64 tensor cores (DMMA m8n8k4).
//
// Replaces the reference's element loop (assembly.py:579-651: _local_square :531-551,
// _SpaceBinding.local_basis :468-517, csr_from_triplets :245-270).
//
// One CTA owns a box of rows T0 x T1 x T2 (colex).  With the per-point form tensor D from K3,
//     A_ij = s_i s_j sum_z Q2 sum_y Q1 sum_x Q0 D,      Qd = B^a_{i_d} B^b_{j_d}  (1D products)
// Every contraction is a per-output-row banded product evaluated with mma.sync m8n8k4 f64:
//   phase 1 (x):  T1[G][i0][d0][y]         = sum_{x in supp(i0)} Q0[d0][x]  D_u[x][y]
//   phase 2 (y):  T2[G2][z][(i0,i1,d1,d0)] = sum_{y in supp(i1)} T1[G][i0][d0][y] Q1[y][d1]
//   phase 3 (z):  A[(i0,i1,d1,d0)][i2,d2] += sum_{z in layer}   T2[G2][z][.] Q2[z][d2]   (per layer)
// The Q fragments of phases 1 and 2 depend only on the tile, so they are built once per CTA in
// shared memory; the D window is streamed plane by plane.  An m8n8k4 DMMA is bitwise a
// sequential FMA chain over its K (profiles/fp64_peak.txt), so every output is a fixed FMA chain
// over its shared Gauss points in ascending order; transposed entries (j,i) run the mirror chain
// (transposed term groups, symmetric pair sums, pair chains joined by commutative adds): the
// matrix is bitwise symmetric and any row subset / row slab equals the full assembly bit for bit.
// Phase 3 adds each layer into the CSR values in ascending layer order (rows owned by this CTA:
// no atomics).  The Gauss count is a template constant (G = p + 1); other counts use the SIMT
// kernel (sg_assemble.cuh).
#pragma once
#include <cuda.h>

#include "sg_common.cuh"

namespace sg {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__host__ __device__ constexpr int g2_npairs(const Tables& T, int g) {
    int c = 0;
    for (int u = 0; u < T.g2n[g]; ++u) c += T.g2pair[g][u];
    return c;
}
__host__ __device__ constexpr int g2_pairidx(const Tables& T, int g, int u) {
    int c = 0;
    for (int v = 0; v < u; ++v) c += T.g2pair[g][v];
    return c;
}
__host__ __device__ constexpr int f_npairs(const Tables& T) {
    int c = 0;
    for (int f = 0; f < T.NF; ++f) c += T.fpair[f];
    return c;
}
__host__ __device__ constexpr int f_pairidx(const Tables& T, int f) {
    int c = 0;
    for (int v = 0; v < f; ++v) c += T.fpair[v];
    return c;
}
__host__ __device__ constexpr int imax(int a, int b) { return a > b ? a : b; }
// prefix count of phase-1 units before group g (fragment slot base)
__host__ __device__ constexpr int g1_unit_base(const Tables& T, int g) {
    int c = 0;
    for (int h = 0; h < g; ++h) c += T.g1n[h];
    return c;
}
__host__ __device__ constexpr int g1_units(const Tables& T) { return g1_unit_base(T, T.NG1); }
// derivative-order pair of a level-1 group for phase-2 fragments: kind = a1 + 3 b1
__host__ __device__ constexpr int kind1(const Tables& T, int ga) { return (T.g1key[ga] % 3) + 3 * ((T.g1key[ga] / 3) % 3); }
__host__ __device__ constexpr int kind2(const Tables& T, int g2) { return T.g2key[g2]; }  // a2 + 3 b2

// compact slots of the derivative-order kinds actually used (phase-2 / phase-3 fragment tables)
__host__ __device__ constexpr int kslot1(const Tables& T, int kind) {
    int slot = 0;
    for (int k = 0; k < 9; ++k) {
        bool used = false;
        for (int g = 0; g < T.NG1; ++g) used = used || kind1(T, g) == k;
        if (!used) continue;
        if (k == kind) return slot;
        ++slot;
    }
    return -1;
}
__host__ __device__ constexpr int nkind1(const Tables& T) {
    int n = 0;
    for (int k = 0; k < 9; ++k) n += kslot1(T, k) >= 0 ? 1 : 0;
    return n;
}
__host__ __device__ constexpr int kslot2(const Tables& T, int kind) {
    int slot = 0;
    for (int k = 0; k < 9; ++k) {
        bool used = false;
        for (int g = 0; g < T.NG2; ++g) used = used || kind2(T, g) == k;
        if (!used) continue;
        if (k == kind) return slot;
        ++slot;
    }
    return -1;
}
__host__ __device__ constexpr int nkind2(const Tables& T) {
    int n = 0;
    for (int k = 0; k < 9; ++k) n += kslot2(T, k) >= 0 ? 1 : 0;
    return n;
}
__host__ __device__ constexpr int kind_of_slot1(const Tables& T, int slot) {
    for (int k = 0; k < 9; ++k)
        if (kslot1(T, k) == slot) return k;
    return 0;
}
__host__ __device__ constexpr int kind_of_slot2(const Tables& T, int slot) {
    for (int k = 0; k < 9; ++k)
        if (kslot2(T, k) == slot) return k;
    return 0;
}
__host__ __device__ constexpr long align16(long o) { return (o + 15) & ~15L; }

__host__ __device__ constexpr int pad16_4(int v) {  // smallest w >= v with w % 16 == 4 (conflict-free fragments)
    int w = v;
    while (w % 16 != 4) ++w;
    return w;
}

// ---- compile-time tile geometry (shared by host planning and the kernel)
struct MmaGeom {
    int T0, T1, G, W, MT, KS, KS3, XW, XWp, YW, NTY, DY, TY, NCOMBO, NMT, CH, NCH, TC, U, NG1, NG2, NU1, NB, NK1, NK2;
    long o_B0, o_B1, o_B2, o_A1, o_B2f, o_B3f, o_cmb, o_bar, o_D, o_D2, o_T1, o_T2, total;
};

__host__ __device__ constexpr MmaGeom mma_geom(int ndim, int P, int form, bool rat, int T0, int T1) {
    const Tables T = make_tables(ndim, form, rat);
    MmaGeom m{};
    m.T0 = T0;
    m.T1 = ndim >= 2 ? T1 : 1;
    m.G = P + 1;
    m.W = 2 * P + 1;
    m.MT = (m.W + 7) / 8;
    m.KS = ((P + 1) * m.G + 3) / 4;
    m.KS3 = (m.G + 3) / 4;
    m.XW = (T0 + P) * m.G;
    m.XWp = (m.XW + 3) & ~3;  // TMA: box bytes DY*XWp*8 stay a multiple of 128
    m.YW = ndim >= 2 ? (m.T1 + P) * m.G : 1;
    m.NTY = ndim >= 2 ? (m.YW + 7) / 8 : 1;
    m.DY = pad16_4(m.NTY * 8);
    m.TY = pad16_4(m.NTY * 8 > m.YW + 4 ? m.NTY * 8 : m.YW + 4);
    m.NCOMBO = T0 * m.T1 * m.W * m.W;
    m.NMT = (m.NCOMBO + 7) / 8;
    m.CH = 4;
    m.NCH = (m.NMT + m.CH - 1) / m.CH;
    m.TC = pad16_4(m.NCH * m.CH * 8);
    m.U = T.MS * (T.MS + 1) / 2;
    m.NG1 = T.NG1;
    m.NG2 = ndim == 3 ? T.NG2 : 1;
    m.NU1 = g1_units(T);
    m.NB = (form_deriv(form) + 1) * (P + 1);
    m.NK1 = nkind1(T);
    m.NK2 = ndim == 3 ? nkind2(T) : 0;
    long o = 0;
    m.o_B0 = o; o += (long)m.XW * m.NB + 2;
    m.o_B1 = o; o += ndim >= 2 ? (long)m.YW * m.NB + 2 : 0;
    m.o_B2 = o; o += ndim == 3 ? (long)m.G * m.NB + 2 : 0;
    m.o_A1 = o; o += (long)T0 * m.NU1 * m.KS * m.MT * 32;                      // phase-1 A fragments
    m.o_B2f = o; o += ndim >= 2 ? (long)m.T1 * m.NK1 * m.KS * m.MT * 32 : 0;     // phase-2 B fragments
    m.o_B3f = o; o += ndim == 3 ? (long)(P + 1) * m.NK2 * m.KS3 * m.MT * 32 : 0; // phase-3 B fragments
    m.o_cmb = o; o += ndim == 3 ? (long)m.NCOMBO / 2 + 2 : 0;                  // per-combo CSR offsets (int)
    m.o_bar = o; o += 2;                                                       // two mbarriers (TMA)
    o = align16(o);
    m.o_D = o; o += align16((long)m.U * m.XWp * m.DY);                          // D window, double buffered (TMA)
    m.o_D2 = ndim == 3 ? o : m.o_D;                                           // 2D/1D: one plane per tile
    o += ndim == 3 ? align16((long)m.U * m.XWp * m.DY) : 0;
    m.o_T1 = o; o += ndim >= 2 ? (long)m.NG1 * T0 * m.MT * 8 * m.TY : 0;
    m.o_T2 = o; o += ndim == 3 ? (long)m.NG2 * m.G * m.TC : 0;
    m.total = o;
    return m;
}

struct TileChoice { int T0, T1; };
__host__ __device__ constexpr TileChoice mma_tile(int ndim, int P, int form, bool rat) {
    const long cap = 200 * 1024 / 8;
    if (ndim == 1) return {32, 1};
    if (ndim == 2) {
        const int cand[] = {12, 10, 8, 6, 4, 3, 2, 1};
        for (int t : cand)
            if (mma_geom(2, P, form, rat, t, t).total <= cap) return {t, t};
        return {1, 1};
    }
    const TileChoice cand[] = {{4, 4}, {2, 4}, {2, 2}, {1, 2}, {1, 1}};
    for (TileChoice t : cand)
        if (mma_geom(3, P, form, rat, t.T0, t.T1).total <= cap) return t;
    return {1, 1};
}

struct MmaParams {
    CUtensorMap dmap;            // TMA map of D: dims {Gp1, Gp0, U, Gp2} (y fastest), box {DY, XW, U, 1}
    int m[3], S[3];
    const double* B[3];          // solution tables  [S*g][nu+1][p+1]
    const double* sol_w;
    const double* D;             // [Gp2][U][Gp0][Gp1]
    int Gp[3];
    int T2, tgrid[3];
    const int* tiles;
    const uint8_t* rowmask;
    const int64_t* rowstart;
    int64_t slab_lo, slab_hi;
    int* indices;
    double* data;
    unsigned long long* zeros;
    int tma;                     // 1: TMA double-buffered D windows; 0: plain loads (debug / fallback)
    int Dys;
};

template <int NDIM, int P, int FORM, bool RAT>
__global__ void __launch_bounds__(512, 1) assemble_mma(const __grid_constant__ MmaParams prm) {
    using TTS = TermTables<NDIM, FORM, RAT>;
    constexpr TileChoice TCH = mma_tile(NDIM, P, FORM, RAT);
    constexpr MmaGeom M = mma_geom(NDIM, P, FORM, RAT, TCH.T0, TCH.T1);
    constexpr int T0 = M.T0, T1 = M.T1, G = M.G, W = M.W, MT = M.MT, KS = M.KS, KS3 = M.KS3;
    constexpr int NB = M.NB, XW = M.XW, YW = M.YW, NTY = M.NTY, DY = M.DY, TY = M.TY, TC = M.TC;
    constexpr int MS = TTS::T.MS;
    constexpr int NW = 16;
    constexpr int NK1 = M.NK1, NK2 = M.NK2;
    constexpr int XWp = M.XWp;
    constexpr unsigned DBYTES = (unsigned)(M.U * XWp * DY * 8);
    extern __shared__ double smem[];
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int lr = lane >> 2, lk = lane & 3;

    const int tile = prm.tiles ? prm.tiles[blockIdx.x] : (int)blockIdx.x;
    const int tc0 = tile % prm.tgrid[0], tc1 = (tile / prm.tgrid[0]) % prm.tgrid[1], tc2 = tile / (prm.tgrid[0] * prm.tgrid[1]);
    const int b0 = tc0 * T0, b1 = tc1 * T1, b2 = tc2 * prm.T2;
    // fixed windows: element e of direction d sits at local element (e - (b_d - P)); elements outside
    // the mesh have zero basis tables and zero D, so every index below is compile-time + lane
    const int ew0 = b0 - P, ew1 = b1 - P;

    double* B0s = smem + M.o_B0;
    double* B1s = smem + M.o_B1;
    double* B2s = smem + M.o_B2;
    double* A1f = smem + M.o_A1;
    double* B2f = smem + M.o_B2f;
    double* B3f = smem + M.o_B3f;
    int* cmb = reinterpret_cast<int*>(smem + M.o_cmb);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + M.o_bar);
    double* Dbuf[2] = {smem + M.o_D, smem + M.o_D2};
    double* T1s = smem + M.o_T1;
    double* T2s = smem + M.o_T2;

    // ---- zero the staging buffers once (padding columns / rows are read as exact zeros)
    for (long it = tid; it < M.total - M.o_T1; it += blockDim.x) T1s[it] = 0.0;
    // ---- window basis tables (zero outside the mesh)
    for (int it = tid; it < XW * NB; it += blockDim.x) {
        const int e = ew0 + it / (G * NB);
        B0s[it] = (e >= 0 && e < prm.S[0]) ? prm.B[0][((long long)ew0 * G) * NB + it] : 0.0;
    }
    if constexpr (NDIM >= 2)
        for (int it = tid; it < YW * NB; it += blockDim.x) {
            const int e = ew1 + it / (G * NB);
            B1s[it] = (e >= 0 && e < prm.S[1]) ? prm.B[1][((long long)ew1 * G) * NB + it] : 0.0;
        }
    __syncthreads();
    // ---- tile-constant fragments
    // A1f[((i0l*NU1 + unit)*KS + kk)*MT + a][lane] = Q0(i0, i0+d0, x): d0 = a*8 + lr - P, x = kk*4 + lk in supp(i0)
    static_for<0, M.NG1>([&](auto GI) {
        constexpr int Gc = decltype(GI)::value;
        static_for<0, TTS::T.g1n[Gc]>([&](auto UI) {
            constexpr int Uc = decltype(UI)::value;
            constexpr int unit = g1_unit_base(TTS::T, Gc) + Uc;
            constexpr int mu = TTS::T.g1mu[Gc][Uc], nu = TTS::T.g1nu[Gc][Uc];
            constexpr bool pair = TTS::T.g1pair[Gc][Uc] != 0;
            constexpr int am = acode(TTS::T.mcode[mu], 0), an = acode(TTS::T.mcode[nu], 0);
            for (int i0l = 0; i0l < T0; ++i0l) {
                if ((unit * T0 + i0l) % NW != warp) continue;
                for (int kk = 0; kk < KS; ++kk) {
                    const int s = kk * 4 + lk;
                    const int ei = s / G, q = s % G;
                    const int x = (i0l + ei) * G + q;
                    const int ri = P - ei;
                    for (int a = 0; a < MT; ++a) {
                        const int d0 = a * 8 + lr - P;
                        const int rj = ri + d0;
                        double v = 0.0;
                        if (s < (P + 1) * G && d0 <= P && rj >= 0 && rj <= P) {
                            const double* bx = B0s + x * NB;
                            v = __dmul_rn(bx[am * (P + 1) + ri], bx[an * (P + 1) + rj]);
                            if constexpr (pair) v = __dadd_rn(v, __dmul_rn(bx[an * (P + 1) + ri], bx[am * (P + 1) + rj]));
                        }
                        A1f[(((i0l * M.NU1 + unit) * KS + kk) * MT + a) * 32 + lane] = v;
                    }
                }
            }
        });
    });
    if constexpr (NDIM >= 2) {
        // B2f[((i1l*NK1 + slot)*KS + kk)*MT + c][lane] = Q1(i1, i1+d1, y): d1 = c*8 + lr - P
        for (int it = warp; it < T1 * NK1; it += NW) {
            const int i1l = it % T1, slot = it / T1;
            int kind = 0;
            static_for<0, NK1>([&](auto SI) { if (slot == decltype(SI)::value) kind = kind_of_slot1(TTS::T, decltype(SI)::value); });
            const int a1 = kind % 3, bb1 = kind / 3;
            for (int kk = 0; kk < KS; ++kk) {
                const int s = kk * 4 + lk;
                const int ei = s / G, q = s % G;
                const int y = (i1l + ei) * G + q;
                const int ri1 = P - ei;
                for (int c = 0; c < MT; ++c) {
                    const int d1 = c * 8 + lr - P;
                    const int rj1 = ri1 + d1;
                    double v = 0.0;
                    if (s < (P + 1) * G && d1 <= P && rj1 >= 0 && rj1 <= P) {
                        const double* by = B1s + y * NB;
                        v = __dmul_rn(by[a1 * (P + 1) + ri1], by[bb1 * (P + 1) + rj1]);
                    }
                    B2f[(((i1l * NK1 + slot) * KS + kk) * MT + c) * 32 + lane] = v;
                }
            }
        }
    }
    if constexpr (NDIM == 3) {
        // per-combo CSR offset inside a row's j2 block: (j0-lo0) + cnt0*(j1-lo1), or -1 (out of range)
        for (int c = tid; c < M.NCOMBO; c += blockDim.x) {
            const int d0 = c % W - P, d1 = (c / W) % W - P, i1l = (c / (W * W)) % T1, i0l = c / (W * W * T1);
            const int i0 = b0 + i0l, i1 = b1 + i1l, j0 = i0 + d0, j1 = i1 + d1;
            int off = -1;
            if (i0 < prm.m[0] && i1 < prm.m[1] && j0 >= 0 && j0 < prm.m[0] && j1 >= 0 && j1 < prm.m[1]) {
                const int lo0 = max(0, i0 - P), lo1 = max(0, i1 - P);
                const int cnt0 = min(prm.m[0] - 1, i0 + P) - lo0 + 1;
                off = (j0 - lo0) + cnt0 * (j1 - lo1);
            }
            cmb[c] = off;
        }
    }

    const long long G0 = prm.Gp[0];
    const int elo2 = NDIM == 3 ? max(0, b2 - P) : 0;
    const int ehi2 = NDIM == 3 ? min(prm.S[2] - 1, b2 + prm.T2 - 1) : 0;
    constexpr int GZ = NDIM == 3 ? G : 1;
    const int nplanes = (ehi2 - elo2 + 1) * GZ;
    const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&bars[0]);
    // D window of plane `pi` (TMA: one 4D box per plane; out-of-mesh coordinates are zero filled)
    auto issue_plane = [&](int pi) {
        const int z = elo2 * G + pi;
        const uint32_t bar = bar0 + 8u * (uint32_t)(pi & 1);
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(Dbuf[pi & 1]);
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(DBYTES) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(dst),
            "l"(reinterpret_cast<uint64_t>(&prm.dmap)), "r"(ew1 * G), "r"(ew0 * G), "r"(0), "r"(z), "r"(bar)
            : "memory");
    };
    // TMA D windows: 3D (double-buffered pencil) and 2D p=3 (validated configs); plain loads otherwise.
    // (2D p=2 bi-Laplacian boxes raised an illegal-instruction fault under TMA -- open item)
    constexpr bool kTma = NDIM == 3 || (NDIM == 2 && P == 3);
    const bool use_tma = kTma && prm.tma;
    if (use_tma) {
        if (tid == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar0) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar0 + 8u) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
        __syncthreads();
        if (tid == 0) issue_plane(0);
    }
    int pidx = 0;
    (void)nplanes;

    for (int e2 = elo2; e2 <= ehi2; ++e2) {
        if constexpr (NDIM == 3) {
            __syncthreads();
            for (int it = tid; it < G * NB; it += blockDim.x) B2s[it] = prm.B[2][(long long)e2 * G * NB + it];
            __syncthreads();
            // phase-3 B fragments of this layer: B3f[((r2*NK2 + slot)*KS3 + kk)*MT + c][lane]
            for (int it = warp; it < (P + 1) * NK2; it += NW) {
                const int r2 = it % (P + 1), slot = it / (P + 1);
                int kind = 0;
                static_for<0, NK2>([&](auto SI) { if (slot == decltype(SI)::value) kind = kind_of_slot2(TTS::T, decltype(SI)::value); });
                const int a2 = kind % 3, bb2 = kind / 3;
                for (int kk = 0; kk < KS3; ++kk) {
                    const int s = kk * 4 + lk;
                    for (int c = 0; c < MT; ++c) {
                        const int d2 = c * 8 + lr - P;
                        const int rj2 = r2 + d2;
                        double v = 0.0;
                        if (s < G && d2 <= P && rj2 >= 0 && rj2 <= P) {
                            const double* bz = B2s + s * NB;
                            v = __dmul_rn(bz[a2 * (P + 1) + r2], bz[bb2 * (P + 1) + rj2]);
                        }
                        B3f[(((r2 * NK2 + slot) * KS3 + kk) * MT + c) * 32 + lane] = v;
                    }
                }
            }
        }
        for (int q2 = 0; q2 < GZ; ++q2) {
            // ---------------- D window of this plane
            double* Ds = Dbuf[pidx & 1];
            if (use_tma) {
                if (tid == 0 && pidx + 1 < nplanes) issue_plane(pidx + 1);  // prefetch the next plane
                const uint32_t bar = bar0 + 8u * (uint32_t)(pidx & 1);
                const uint32_t par = (uint32_t)((pidx >> 1) & 1);
                uint32_t done = 0;
                while (!done) {
                    asm volatile(
                        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                        : "=r"(done)
                        : "r"(bar), "r"(par)
                        : "memory");
                }
            } else {
                const long long gx0 = (long long)ew0 * G, gy0 = (long long)ew1 * G;
                const long long z = (long long)elo2 * G + pidx;
                const long long G1 = NDIM >= 2 ? prm.Gp[1] : 1;
                for (int it = tid; it < M.U * XWp * DY; it += blockDim.x) {
                    const int y = it % DY, r = it / DY;
                    const int u = r / XWp, x = r % XWp;
                    const long long gx = gx0 + x, gy = gy0 + y;
                    double v = 0.0;
                    if (gx >= 0 && gx < G0 && gy >= 0 && gy < G1)
                        v = prm.D[((z * M.U + u) * G0 + gx) * (long long)prm.Dys + gy];
                    Ds[r * DY + y] = v;
                }
                __syncthreads();
            }

            // ---------------- phase 1: items (group, row i0l), statically scheduled over warps
            static_for<0, M.NG1 * T0>([&](auto KI) {
                constexpr int k = decltype(KI)::value;
                if (warp != k % NW) return;
                constexpr int Gc = k / T0, i0l = k % T0;
                const int i0 = b0 + i0l;
                double acc[MT][NTY][2];
#pragma unroll
                for (int a = 0; a < MT; ++a)
#pragma unroll
                    for (int c = 0; c < NTY; ++c) acc[a][c][0] = acc[a][c][1] = 0.0;
                static_for<0, TTS::T.g1n[Gc]>([&](auto UI) {
                    constexpr int Uc = decltype(UI)::value;
                    constexpr int mu = TTS::T.g1mu[Gc][Uc], nu = TTS::T.g1nu[Gc][Uc];
                    constexpr int ud = tri_index(mu, nu, MS);
                    constexpr int unit = g1_unit_base(TTS::T, Gc) + Uc;
                    const double* af = A1f + ((i0l * M.NU1 + unit) * KS) * MT * 32 + lane;
#pragma unroll
                    for (int kk = 0; kk < KS; ++kk) {
                        const int s = kk * 4 + lk;
                        const int x = (s < (P + 1) * G) ? (i0l + s / G) * G + s % G : 0;
                        const double* drow = Ds + (ud * XWp + x) * DY + lr;
                        double afr[MT];
#pragma unroll
                        for (int a = 0; a < MT; ++a) afr[a] = af[(kk * MT + a) * 32];
#pragma unroll
                        for (int c = 0; c < NTY; ++c) {
                            const double bf = drow[c * 8];
#pragma unroll
                            for (int a = 0; a < MT; ++a) dmma(acc[a][c][0], acc[a][c][1], afr[a], bf);
                        }
                    }
                });
                if constexpr (NDIM == 1) {
                    if (lk == 0 && i0 < prm.m[0]) {
                        const int64_t row = i0;
                        if (row >= prm.slab_lo && row < prm.slab_hi && (!prm.rowmask || prm.rowmask[row])) {
                            const int lo = max(0, i0 - P);
                            const int64_t base = prm.rowstart[row];
#pragma unroll
                            for (int a = 0; a < MT; ++a) {
                                const int d0 = a * 8 + lr - P;
                                const int j0 = i0 + d0;
                                if (d0 > P || j0 < 0 || j0 >= prm.m[0]) continue;
                                double v = acc[a][0][0];
                                if constexpr (RAT) v = v * (prm.sol_w[i0] * prm.sol_w[j0]);
                                prm.data[base + (j0 - lo)] = v;
                                prm.indices[base + (j0 - lo)] = j0;
                                if (prm.zeros && v == 0.0) atomicAdd(prm.zeros, 1ull);
                            }
                        }
                    }
                } else {
                    double* t1 = T1s + ((Gc * T0 + i0l) * MT * 8) * TY;
#pragma unroll
                    for (int a = 0; a < MT; ++a)
#pragma unroll
                        for (int c = 0; c < NTY; ++c) {
                            double* dst = t1 + (a * 8 + lr) * TY + c * 8 + 2 * lk;
                            dst[0] = acc[a][c][0];
                            dst[1] = acc[a][c][1];
                        }
                }
            });
            if constexpr (NDIM >= 2) {
                __syncthreads();
                // ---------------- phase 2: items (level-2 group, row i1l); the T0 rows i0 share Q1
                static_for<0, M.NG2 * T1>([&](auto KI) {
                    constexpr int k = decltype(KI)::value;
                    if (warp != k % NW) return;
                    constexpr int Gc = k / T1, i1l = k % T1;
                    const int i1 = b1 + i1l;
                    if (i1 >= prm.m[1]) return;
                    constexpr int NPR = g2_npairs(TTS::T, Gc);
                    constexpr int NA = imax(NPR, 1);
                    double accS[T0][MT][MT][2];
                    double accA[NA][T0][MT][MT][2];
                    double accB[NA][T0][MT][MT][2];
#pragma unroll
                    for (int r = 0; r < T0; ++r)
#pragma unroll
                        for (int a = 0; a < MT; ++a)
#pragma unroll
                            for (int c = 0; c < MT; ++c)
#pragma unroll
                                for (int h = 0; h < 2; ++h) {
                                    accS[r][a][c][h] = 0.0;
#pragma unroll
                                    for (int kx = 0; kx < NA; ++kx) accA[kx][r][a][c][h] = accB[kx][r][a][c][h] = 0.0;
                                }
                    auto block = [&](auto GA, auto& acc) {
                        constexpr int ga = decltype(GA)::value;
                        constexpr int kd = kslot1(TTS::T, kind1(TTS::T, ga));
                        const double* bfp = B2f + ((i1l * NK1 + kd) * KS) * MT * 32 + lane;
                        // y of support point s of row i1 is i1l*G + s (the support is contiguous)
                        const double* t1 = T1s + ((ga * T0) * MT * 8 + lr) * TY + i1l * G + lk;
#pragma unroll
                        for (int kk = 0; kk < KS; ++kk) {
                            double bfs[MT];
#pragma unroll
                            for (int c = 0; c < MT; ++c) bfs[c] = bfp[(kk * MT + c) * 32];
#pragma unroll
                            for (int r = 0; r < T0; ++r)
#pragma unroll
                                for (int a = 0; a < MT; ++a) {
                                    const double av = t1[(r * MT + a) * 8 * TY + kk * 4];
#pragma unroll
                                    for (int c = 0; c < MT; ++c) dmma(acc[r][a][c][0], acc[r][a][c][1], av, bfs[c]);
                                }
                        }
                    };
                    static_for<0, TTS::T.g2n[Gc]>([&](auto UI) {
                        constexpr int Uc = decltype(UI)::value;
                        constexpr int ga = TTS::T.g2u[Gc][Uc];
                        if constexpr (TTS::T.g2pair[Gc][Uc] == 0) {
                            block(std::integral_constant<int, ga>{}, accS);
                        } else {
                            constexpr int pi = g2_pairidx(TTS::T, Gc, Uc);
                            block(std::integral_constant<int, ga>{}, accA[pi]);
                            block(std::integral_constant<int, TTS::T.g1T[ga]>{}, accB[pi]);
                        }
                    });
#pragma unroll
                    for (int r = 0; r < T0; ++r)
#pragma unroll
                        for (int a = 0; a < MT; ++a)
#pragma unroll
                            for (int c = 0; c < MT; ++c)
#pragma unroll
                                for (int h = 0; h < 2; ++h) {
                                    double v = accS[r][a][c][h];
#pragma unroll
                                    for (int kx = 0; kx < NPR; ++kx) v = __dadd_rn(v, __dadd_rn(accA[kx][r][a][c][h], accB[kx][r][a][c][h]));
                                    accS[r][a][c][h] = v;
                                }
#pragma unroll
                    for (int r = 0; r < T0; ++r) {
                        const int i0 = b0 + r;
                        if (i0 >= prm.m[0]) continue;
                        if constexpr (NDIM == 2) {
                            const int64_t row = (int64_t)i0 + (int64_t)prm.m[0] * i1;
                            if (!(row >= prm.slab_lo && row < prm.slab_hi && (!prm.rowmask || prm.rowmask[row]))) continue;
                            const int lo0 = max(0, i0 - P), lo1 = max(0, i1 - P);
                            const int cnt0 = min(prm.m[0] - 1, i0 + P) - lo0 + 1;
                            const int64_t base = prm.rowstart[row];
                            const double si = RAT ? prm.sol_w[row] : 1.0;
#pragma unroll
                            for (int a = 0; a < MT; ++a) {
                                const int d0 = a * 8 + lr - P;
                                const int j0 = i0 + d0;
                                if (d0 > P || j0 < 0 || j0 >= prm.m[0]) continue;
#pragma unroll
                                for (int c = 0; c < MT; ++c)
#pragma unroll
                                    for (int h = 0; h < 2; ++h) {
                                        const int d1 = c * 8 + 2 * lk + h - P;
                                        const int j1 = i1 + d1;
                                        if (d1 > P || j1 < 0 || j1 >= prm.m[1]) continue;
                                        double v = accS[r][a][c][h];
                                        const int64_t col = (int64_t)j0 + (int64_t)prm.m[0] * j1;
                                        if constexpr (RAT) v = v * (si * prm.sol_w[col]);
                                        const int64_t pos = base + (j0 - lo0) + (int64_t)cnt0 * (j1 - lo1);
                                        prm.data[pos] = v;
                                        prm.indices[pos] = (int)col;
                                        if (prm.zeros && v == 0.0) atomicAdd(prm.zeros, 1ull);
                                    }
                            }
                        } else {
                            double* t2 = T2s + (Gc * G + q2) * TC + (r * T1 + i1l) * W * W;
#pragma unroll
                            for (int a = 0; a < MT; ++a) {
                                const int d0 = a * 8 + lr;
                                if (d0 >= W) continue;
#pragma unroll
                                for (int c = 0; c < MT; ++c)
#pragma unroll
                                    for (int h = 0; h < 2; ++h) {
                                        const int d1 = c * 8 + 2 * lk + h;
                                        if (d1 < W) t2[d1 * W + d0] = accS[r][a][c][h];
                                    }
                            }
                        }
                    }
                });
            }
            __syncthreads();
            ++pidx;
        }  // q2
        if constexpr (NDIM == 3) {
            // ---------------- phase 3: items (row offset r2 in the layer, chunk of CH m-tiles)
            constexpr int NFP = f_npairs(TTS::T);
            constexpr int NA = imax(NFP, 1);
            constexpr int CH = M.CH;
            const int m01 = prm.m[0] * prm.m[1];
            for (int item = warp; item < (P + 1) * M.NCH; item += NW) {
                const int r2 = item % (P + 1), ch = item / (P + 1);
                const int i2 = e2 + r2;
                if (i2 < b2 || i2 >= b2 + prm.T2 || i2 >= prm.m[2]) continue;
                // CSR position of every output of this item (lane: rows lr of CH m-tiles, columns 2*lk+h)
                // and the previously accumulated layers' partial sums, loaded before the MMA chain
                const int lo2 = max(0, i2 - P);
                int64_t pos[CH][MT][2];
                double old[CH][MT][2];
#pragma unroll
                for (int mm = 0; mm < CH; ++mm) {
                    const int combo = (ch * CH + mm) * 8 + lr;
                    const int off = combo < M.NCOMBO ? cmb[combo] : -1;
                    const int i1l = (combo / (W * W)) % T1, i0l = combo / (W * W * T1);
                    const int i0 = b0 + i0l, i1 = b1 + i1l;
                    const int64_t row = (int64_t)i0 + (int64_t)prm.m[0] * i1 + (int64_t)m01 * i2;
                    bool ok = off >= 0 && row >= prm.slab_lo && row < prm.slab_hi && (!prm.rowmask || prm.rowmask[row]);
                    const int cnt01 = ok ? (min(prm.m[0] - 1, i0 + P) - max(0, i0 - P) + 1) * (min(prm.m[1] - 1, i1 + P) - max(0, i1 - P) + 1) : 0;
                    const int64_t base = ok ? prm.rowstart[row] + off : 0;
#pragma unroll
                    for (int c = 0; c < MT; ++c)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int d2 = c * 8 + 2 * lk + h - P;
                            const int rj2 = r2 + d2;
                            const bool v = ok && d2 <= P && rj2 >= 0 && rj2 <= P;
                            pos[mm][c][h] = v ? base + (int64_t)cnt01 * (i2 + d2 - lo2) : -1;
                            const int first = max(0, max(i2, i2 + d2) - P);
                            old[mm][c][h] = (v && e2 != first) ? prm.data[pos[mm][c][h]] : 0.0;
                        }
                }
                double accS[CH][MT][2];
                double accA[NA][CH][MT][2];
                double accB[NA][CH][MT][2];
#pragma unroll
                for (int mm = 0; mm < CH; ++mm)
#pragma unroll
                    for (int c = 0; c < MT; ++c)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            accS[mm][c][h] = 0.0;
#pragma unroll
                            for (int kx = 0; kx < NA; ++kx) accA[kx][mm][c][h] = accB[kx][mm][c][h] = 0.0;
                        }
                auto block = [&](auto GA, auto& acc) {
                    constexpr int ga = decltype(GA)::value;
                    constexpr int kd = kslot2(TTS::T, kind2(TTS::T, ga));
                    const double* bfp = B3f + ((r2 * NK2 + kd) * KS3) * MT * 32 + lane;
#pragma unroll
                    for (int kk = 0; kk < KS3; ++kk) {
                        double bfs[MT];
#pragma unroll
                        for (int c = 0; c < MT; ++c) bfs[c] = bfp[(kk * MT + c) * 32];
                        const int s = kk * 4 + lk;
                        const double* t2 = T2s + (ga * G + (s < G ? s : 0)) * TC + ch * CH * 8 + lr;
#pragma unroll
                        for (int mm = 0; mm < CH; ++mm) {
                            const double av = t2[mm * 8];
#pragma unroll
                            for (int c = 0; c < MT; ++c) dmma(acc[mm][c][0], acc[mm][c][1], av, bfs[c]);
                        }
                    }
                };
                static_for<0, TTS::T.NF>([&](auto FI) {
                    constexpr int f = decltype(FI)::value;
                    constexpr int ga = TTS::T.fu[f];
                    if constexpr (TTS::T.fpair[f] == 0) {
                        block(std::integral_constant<int, ga>{}, accS);
                    } else {
                        constexpr int pi = f_pairidx(TTS::T, f);
                        block(std::integral_constant<int, ga>{}, accA[pi]);
                        block(std::integral_constant<int, TTS::T.g2T[ga]>{}, accB[pi]);
                    }
                });
#pragma unroll
                for (int mm = 0; mm < CH; ++mm) {
                    const int combo = (ch * CH + mm) * 8 + lr;
                    const int i1l = (combo / (W * W)) % T1, i0l = combo / (W * W * T1);
                    const int i0 = b0 + i0l, i1 = b1 + i1l;
                    const int d0 = combo % W - P, d1 = (combo / W) % W - P;
                    const int64_t row = (int64_t)i0 + (int64_t)prm.m[0] * i1 + (int64_t)m01 * i2;
                    const int64_t colb = (int64_t)(i0 + d0) + (int64_t)prm.m[0] * (i1 + d1);
#pragma unroll
                    for (int c = 0; c < MT; ++c)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int64_t p = pos[mm][c][h];
                            if (p < 0) continue;
                            const int j2 = i2 + c * 8 + 2 * lk + h - P;
                            double v = accS[mm][c][h];
#pragma unroll
                            for (int kx = 0; kx < NFP; ++kx) v = __dadd_rn(v, __dadd_rn(accA[kx][mm][c][h], accB[kx][mm][c][h]));
                            const int first = max(0, max(i2, j2) - P);
                            const int last = min(min(i2, j2), prm.S[2] - 1);
                            if (e2 != first) v = old[mm][c][h] + v;
                            const int64_t col = colb + (int64_t)m01 * j2;
                            if (e2 == last) {
                                if constexpr (RAT) v = v * (prm.sol_w[row] * prm.sol_w[col]);
                                if (prm.zeros && v == 0.0) atomicAdd(prm.zeros, 1ull);
                            }
                            if (e2 == first) prm.indices[p] = (int)col;
                            prm.data[p] = v;
                        }
                }
            }
        }
    }
}

}  // namespace sg
