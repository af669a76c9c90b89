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

#include <climits>

#include "sg_common.cuh"

namespace sg {


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
// 3D with single-unit level-1 groups (Poisson, mass): a phase-1 item covers two groups, two
// independent DMMA chains interleaved (fewer, fatter items: the interval's warps each take one)
__host__ __device__ constexpr bool p1_pair(const Tables& T, int ndim) {
    if (ndim != 3 || T.NG1 < 2) return false;
    for (int g = 0; g < T.NG1; ++g)
        if (T.g1n[g] != 1) return false;
    return true;
}
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

// D window row length: w >= v with w % 16 in {4, 12}.  Phase 1's B fragment takes four consecutive x rows
// (lane bits 0-1) and eight consecutive y per row: the rows must start in distinct quarter-bank groups
// (w = 8 mod 16 left rows 0/2 and 1/3 on the same banks: 2-way, 13% of the 3D Poisson kernel's shared
// wavefronts, profiles/r02_assemble_mma_poisson128_ncu.txt)
__host__ __device__ constexpr int pad_dy(int v) {
    int w = v;
    while (w % 8 != 4) ++w;
    return w;
}
__host__ __device__ constexpr int pad8_4(int v) {  // smallest w >= v with w % 8 == 4 (conflict-free fragment rows)
    int w = v;
    while (w % 8 != 4) ++w;
    return w;
}

#ifndef SG_CH_MASS
#define SG_CH_MASS 1
#endif
#ifndef SG_CH_POIS
#define SG_CH_POIS 1
#endif
// unit descriptors of the phase 1-3 items as compile-time constants (static_for over the groups)
#ifndef SG_STATIC_UNITS
#define SG_STATIC_UNITS 1
#endif
// non-pair units of a phase-2 / phase-3 item in two interleaved DMMA chains (see phase2)
#ifndef SG_P2_ILP
#define SG_P2_ILP 0
#endif
#ifndef SG_P3_ILP
#define SG_P3_ILP 0
#endif
#ifndef SG_P12_EPI
#define SG_P12_EPI 0
#endif
#ifndef SG_P3_EPI
#define SG_P3_EPI 3
#endif
// 3D Poisson: 20 warps = 16 (phases 1-2) + 4 (phase 3).  Sweep at config 5 (ms): 16+4: 23.1 | 15+5: 23.9 |
// 15+4: 23.9 | 18+6: 24.1 | 14+6: 24.9 | 20+4: 25.0 | 12+4: 25.1 | 17+4: 25.7 | 16+5: 26.0 | 16+6: 26.1 |
// 21+7: 25.3 | 24+8: 27.0.  Warp w runs on sub-partition w mod 4: group sizes that are multiples of 4 give
// every sub-partition the same mix (one phase-3 warp each), and 640 threads leave 96 registers per thread.
#ifndef SG_3D_NW
#define SG_3D_NW 20
#endif
#ifndef SG_MASS_NW
#define SG_MASS_NW 16
#endif
// 2D: 20 warps (16: config 2 Poisson 0.407 / mass 0.145 / config 4 3.23 ms; 20: 0.384 / 0.134 / 3.23; 12: 0.403 / 0.173 / 3.16)
#ifndef SG_2D_NW
#define SG_2D_NW 20
#endif
#ifndef SG_MASS_MINB
#define SG_MASS_MINB 2
#endif
#ifndef SG_MASS_T0
#define SG_MASS_T0 2
#endif
#ifndef SG_MASS_T1
#define SG_MASS_T1 4
#endif
// warps per CTA (items are scheduled against it at compile time)
__host__ __device__ constexpr int mma_warps(int ndim, int P, int form, bool rat) {
#ifdef SG_MMA_NW
    return SG_MMA_NW;
#else
    // 3D Poisson: 20 warps (16 + 4) at p = 3, 24 (18 + 6) otherwise: see SG_3D_NW above (round 1's
    // unspecialised kernel wanted 24: 52.4 -> 48.2 ms against 16).
    // 3D mass: two CTAs of SG_MASS_NW warps per SM on half-size tiles (the barrier waits of one CTA
    // overlap the other's work)
    return ndim == 3 ? (form == 1 ? SG_MASS_NW : (P == 3 ? SG_3D_NW : 24)) : SG_2D_NW;
#endif
}
// CTAs per SM the kernel is compiled for (register budget of __launch_bounds__)
__host__ __device__ constexpr int mma_minb(int ndim, int P, int form, bool rat) {
    return ndim == 3 && form == 1 ? SG_MASS_MINB : 1;
}

// ---- warp specialisation of the 3D pipeline (Poisson / Stokes velocity, mass): warps [0, NW - NB) run
// phases 1-2 plane by plane (group A), warps [NW - NB, NW) run phase 3 layer by layer (group B); the
// groups hand T2 planes over through mbarriers instead of one CTA barrier per plane, so the phase-3
// burst of every G-th plane no longer stalls phases 1-2 (and B's barrier waits overlap A's work)
#ifndef SG_SPEC_NB
#define SG_SPEC_NB 4
#endif
__host__ __device__ constexpr bool mma_spec(int ndim, int form) {
#ifdef SG_NO_SPEC
    return false;
#else
    // mass too (two CTAs of 10 + 6 warps per SM; config 5 mass full 5.99 -> 4.71 ms, quadrature rows
    // 1.92 -> 1.62; SG_NO_SPEC_MASS keeps one barrier interval per plane)
#ifdef SG_NO_SPEC_MASS
    return ndim == 3 && form == 0;
#else
    return ndim == 3 && (form == 0 || form == 1);
#endif
#endif
}
#ifndef SG_SPEC_NB_MASS
#define SG_SPEC_NB_MASS 6
#endif
__host__ __device__ constexpr int mma_spec_nb(int ndim, int form, int P) {
    // (p = 3 Poisson: 16 + 4 of 20 warps; other degrees keep 18 + 6 of 24: config 3, p = 2, 1.68 vs 1.74 ms)
    return mma_spec(ndim, form) ? (form == 1 ? SG_SPEC_NB_MASS : (P == 3 ? SG_SPEC_NB : 6)) : 0;
}
// T2 ring: G + 1 planes (phase 3 of a layer while phase 2 writes the next plane); + 1 under
// specialisation (group A may run two planes ahead of the layer group B is consuming)
// phase 3 contracts a row plane i2 over the whole z support of its rows (layers i2-P .. i2, (P+1) G
// planes): the ring holds those planes plus the one phase 2 writes meanwhile; under specialisation one
// more layer, so group A can run a layer ahead of group B
__host__ __device__ constexpr int mma_ns(int ndim, int P, int form) {
    return (P + 1) * (P + 1) + 1 + (mma_spec(ndim, form) ? P + 1 : 0);
}

// ---- compile-time tile geometry (shared by host planning and the kernel)
// (136: the 131 row planes of config 5 in ONE z tile instead of two of 66: no second start-up and no
// re-streamed halo layers, Poisson 23.05 -> 22.27 ms; the row-start table grows by 1.5-4 KB, every 3D tile
// choice stays the same and the p = 3 mass kernel still fits two CTAs per SM at 112 KB)
#ifndef SG_MMA_T2
#define SG_MMA_T2 136
#endif
constexpr int kMmaT2 = SG_MMA_T2;  // max rows per CTA in z (3D); the plan picks the depth T2 <= kMmaT2 per call

struct MmaGeom {
    int NC1, NCP, T0, T1, G, W, MT, KS, KS3, XW, XWp, YW, NTY, DY, TY, T1SW, NCOMBO, NMT, CH, NCH, TC, T2PS, U, NG1, NG2, NU1, NB, NK1, NK2;
    int NTAB;
    long o_B0, o_B1, o_B2, o_A1, o_B2f, o_B3f, o_cmb, o_rb, o_tab, o_bar, o_D, o_D2, o_T1, o_T2, o_O, total;
};

// doubles of one T1 plane (NG1 T0 MT 8 rows; see T1SW) and the offset of its row r
__host__ __device__ constexpr long mma_t1_plane(const MmaGeom& m) {
    const long rows = (long)m.NG1 * m.T0 * m.MT * 8;
    return m.T1SW ? rows / 4 * (4L * m.TY + 8) : rows * m.TY;
}
__host__ __device__ constexpr int mma_t1_row(const MmaGeom& m, int r) {
    return m.T1SW ? (r >> 2) * (4 * m.TY + 8) + (r & 3) * m.TY + 4 * ((r >> 1) & 1) : r * m.TY;
}

__host__ __device__ constexpr MmaGeom mma_geom(int ndim, int P, int form, bool rat, int T0, int T1) {
    const Tables T = make_tables(ndim, form, rat);
    MmaGeom m{};
    m.T0 = T0;
    m.T1 = ndim >= 2 ? T1 : 1;
    m.G = P + 1;
    m.W = 2 * P + 1;
    m.MT = (m.W + 7) / 8;
    m.KS = ((P + 1) * m.G + 3) / 4;
    m.KS3 = ((P + 1) * m.G + 3) / 4;  // phase 3: the whole z support of a row (P+1 layers)
    m.XW = (T0 + P) * m.G;
    m.XWp = (m.XW + 3) & ~3;  // TMA: box bytes DY*XWp*8 stay a multiple of 128
    m.YW = ndim >= 2 ? (m.T1 + P) * m.G : 1;
    m.NTY = ndim >= 2 ? (m.YW + 7) / 8 : 1;
    // phase-1 items may be split by y n-tile (NC1 > 1); measured slower for Poisson and mass (the
    // A fragments are then reloaded per n-tile), so one item covers all n-tiles unless forced
#ifdef SG_NC1_FORCE
    m.NC1 = ndim >= 2 ? SG_NC1_FORCE : 1;
#else
    m.NC1 = 1;
#endif
    m.DY = pad_dy(m.NTY * 8);
    // (3D p = 4 mass keeps its 2 x 4 tile: the conflict-free row would push it past the shared-memory cap)
    if (ndim == 3 && form == 1 && P == 4 && T0 == 2 && m.T1 == 4) m.DY = m.NTY * 8;
    m.TY = pad8_4(m.NTY * 8 > m.YW + 4 ? m.NTY * 8 : m.YW + 4);
    // T1SW: T1 rows r placed at t1_row(r) = (r / 4) (4 TY + 8) + (r % 4) TY + 4 ((r >> 1) & 1) with
    // TY = 8 (mod 16): rows 0..3 of a half-warp start in distinct quarter-bank groups (phase 2's
    // A-fragment loads: 4 consecutive y per row) and rows r, r+1 of a 128-bit store wavefront in
    // opposite halves (phase 1's row stores; 2-way with the plain TY = 4 (mod 8) rows)
    // (used where it takes no more shared memory than the plain rows: not for config 4's 2 x 5 tiles)
    {
        const int need = m.NTY * 8 > (m.T1 - 1) * m.G + m.KS * 4 ? m.NTY * 8 : (m.T1 - 1) * m.G + m.KS * 4;
        int tys = need;
        while (tys % 16 != 8) ++tys;
        m.T1SW = 4 * tys + 8 <= 4 * m.TY ? 1 : 0;
        if (m.T1SW) m.TY = tys;
    }
    m.NCOMBO = T0 * m.T1 * m.W * m.W;
    m.NMT = (m.NCOMBO + 7) / 8;
    m.CH = form == 1 ? SG_CH_MASS : SG_CH_POIS;  // m-tiles per phase-3 item
    m.NCH = (m.NMT + m.CH - 1) / m.CH;
    m.TC = pad8_4(m.NCH * m.CH * 8);
    m.NCP = pad8_4(m.NCH * m.CH * 8);
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
    m.o_B2 = o;
    m.o_A1 = o; o += (long)T0 * m.NU1 * m.KS * m.MT * 32;                      // phase-1 A fragments
    m.o_B2f = o; o += ndim >= 2 ? (long)m.T1 * m.NK1 * m.KS * m.MT * 32 : 0;     // phase-2 B fragments
    m.o_B3f = o; o += ndim == 3 ? 2L * m.NK2 * m.KS3 * m.MT * 32 : 0;         // phase-3 B fragments (2 row planes)
    o = (o + 1) & ~1L;
    m.o_cmb = o; o += ndim == 3 ? (long)m.NCOMBO * 2 + 2 : 0;                  // per-combo {off, cnt01, row01, col01}
    {
        const int NW = 32;  // table sized for up to 32 warps (host and device layouts agree whatever the warp count)
        int nu2 = 0;
        for (int g = 0; g < (ndim >= 2 ? T.NG2 : 0); ++g) nu2 += T.g2n[g];
        m.NTAB = 3 * (NW + 1) + m.NG1 * T0 * m.NC1 + (ndim >= 2 ? T.NG2 * m.T1 * T0 : 0) + (ndim == 3 ? (P + 1) * m.NCH : 0) +
                 (m.NG1 + 1) + m.NU1 + (T.NG2 + 1) + nu2 + T.NF;
    }
    m.o_rb = o; o += ndim == 3 ? (long)T0 * m.T1 * kMmaT2 + 1 : 0;                // CSR start of every tile row (int64, -1: not owned)
    m.o_tab = o; o += (m.NTAB + 1) / 2;                                        // item schedule + unit tables (int)
    m.o_bar = o; o += 4;                                                       // 2 TMA mbarriers + 2 hand-over counters
    o = align16(o);
    m.o_D = o; o += align16((long)m.U * m.XWp * m.DY);                          // D window, double buffered (TMA)
    m.o_D2 = ndim == 3 ? o : m.o_D;                                           // 2D/1D: one plane per tile
    o += ndim == 3 ? align16((long)m.U * m.XWp * m.DY) : 0;
    m.o_T1 = o; o += ndim >= 2 ? (ndim == 3 ? 2L : 1L) * mma_t1_plane(m) : 0;  // 3D: 2 planes
    // T2 plane stride = 4 (mod 16) doubles: phase 3's A fragment takes its four k (z points, lane
    // bits 0-1) from consecutive planes and four consecutive combos per k (lane bits 2-3) in a
    // half-warp, so the four planes must start in distinct quarter-bank groups (was 4-way at 0 mod 16)
    m.T2PS = m.NG2 * m.TC;
    while (m.T2PS % 16 != 4) ++m.T2PS;
    m.o_T2 = o; o += ndim == 3 ? (long)mma_ns(ndim, P, form) * m.T2PS : 0;  // ring of T2 planes
    m.o_O = o;                                                                  // (no live partial sums: one z chain per entry)
    m.total = o;
    return m;
}

struct TileChoice { int T0, T1; };
__host__ __device__ constexpr TileChoice mma_tile(int ndim, int P, int form, bool rat) {
    const long cap = 224 * 1024 / 8;
    if (ndim == 1) return {32, 1};
    if (ndim == 2) {
#if defined(SG_FORCE2_FORM) && defined(SG_FORCE2_T0) && defined(SG_FORCE2_T1)
        if (form == SG_FORCE2_FORM && mma_geom(2, P, form, rat, SG_FORCE2_T0, SG_FORCE2_T1).total <= cap) return {SG_FORCE2_T0, SG_FORCE2_T1};
#endif
        // 2D bi-Laplacian, p = 3: a deeper y extent (2 x 5 instead of 3 x 3) halves the x-contraction
        // work per row (config 4: 7.04 -> 6.12 ms)
        if (form == 2 && P == 3 && mma_geom(2, P, form, rat, 2, 5).total <= cap) return {2, 5};
        // (3 x 3 tiles with an odd Gauss count start their TMA windows at odd y points: see tma_ysh)
        const int cand[] = {12, 10, 8, 6, 4, 3, 2, 1};
        for (int t : cand)
            if (mma_geom(2, P, form, rat, t, t).total <= cap) return {t, t};
        return {1, 1};
    }
#if defined(SG_FORCE_FORM) && defined(SG_FORCE_T0) && defined(SG_FORCE_T1)
    if (form == SG_FORCE_FORM && mma_geom(3, P, form, rat, SG_FORCE_T0, SG_FORCE_T1).total <= cap) return {SG_FORCE_T0, SG_FORCE_T1};
#endif
    // several CTAs per SM: 228 KB of shared memory per SM minus 1 KB reserved per CTA
    if (form == 1 && mma_minb(3, P, form, rat) > 1 &&
        mma_geom(3, P, form, rat, SG_MASS_T0, SG_MASS_T1).total <= (228L * 1024 / 8) / mma_minb(3, P, form, rat) - 128)
        return {SG_MASS_T0, SG_MASS_T1};
#if defined(SG_POIS_T0) && defined(SG_POIS_T1)
    if (form == 0 && mma_geom(3, P, form, rat, SG_POIS_T0, SG_POIS_T1).total <= cap) return {SG_POIS_T0, SG_POIS_T1};
#else
    // one row in x, as many as fit in y: phase 1 (the x contraction) runs once per y window of T1 + p
    // elements, so its work per row falls as 1/T1 (config 5 Poisson: 2x2 -> 1x5 tiles, 41.5 -> 33.8 ms)
    if (form == 0)  // Poisson / Stokes velocity (the 3D bi-Laplacian tables exceed the constexpr budget)
        for (int t1 = 8; t1 >= 3; --t1)
            if (mma_geom(3, P, form, rat, 1, t1).total <= cap) return {1, t1};
#endif
    const TileChoice cand[] = {{4, 4}, {2, 4}, {2, 2}, {1, 2}, {1, 1}};
    for (TileChoice t : cand)
        if (mma_geom(3, P, form, rat, t.T0, t.T1).total <= cap) return t;
    return {1, 1};
}

// ---- compile-time LPT schedule of the warp items of one barrier interval, emitted as a runtime table
// phase-1 items (group, i0l), phase-2 items (level-2 group, i1l, i0l), phase-3 items (r2, chunk);
// cost = DMMAs of the item's chains (+ a small epilogue constant).  3D: phases 1 and 2 share an
// interval (pipelined over planes) and phase 3 is placed on top of that load.  The item bodies are
// data driven (one copy of the code per phase: the unrolled-per-item form thrashed the I-cache).
// Table (ints): off1[NW+1] off2[NW+1] off3[NW+1] | items1 items2 items3 (grouped by warp) |
//   u1beg[NG1+1] u1ud[NU1] | u2beg[NG2+1] u2[NU2] | u3[NF]
// packed units: ga | gaT << 8 | kd << 16 | kdT << 20 | pair << 24, non-pair units first.
constexpr int kTabMax = 1024;
struct MmaTab {
    int v[kTabMax];
    int n;
    int o_off1, o_off2, o_off3, o_it1, o_it2, o_it3, o_u1b, o_u1ud, o_u2b, o_u2, o_u3;
};
__host__ __device__ constexpr int g2_blocks(const Tables& T, int g) { return T.g2n[g] + g2_npairs(T, g); }
__host__ __device__ constexpr int pack_unit(int ga, int gaT, int kd, int kdT, int pair) {
    return ga | (gaT << 8) | (kd << 16) | (kdT << 20) | (pair << 24);
}
__host__ __device__ constexpr MmaTab mma_tab(int ndim, int P, int form, bool rat) {
    const Tables T = make_tables(ndim, form, rat);
    const TileChoice tc = mma_tile(ndim, P, form, rat);
    const MmaGeom M = mma_geom(ndim, P, form, rat, tc.T0, tc.T1);
    const int NW = mma_warps(ndim, P, form, rat);
    MmaTab S{};
    const bool pr1 = false;  // p1_pair(T, ndim): paired phase-1 items measured no faster (config 5: 33.1 vs 32.7 ms)
    const int n1 = (pr1 ? (M.NG1 + 1) / 2 : M.NG1) * M.T0 * M.NC1;
    const int n2 = ndim >= 2 ? T.NG2 * M.T1 * M.T0 : 0;
    const int n3 = ndim == 3 ? M.NCH : 0;  // phase-3 items of a row plane: chunks of CH m-tiles
    int w1[512] = {}, w2[512] = {}, w3[512] = {};
    long load[64] = {};
    int cost[1024] = {};
    int kind[1024] = {}, idx[1024] = {};
    bool done[1024] = {};
    int n = 0;
    const int NBs = mma_spec_nb(ndim, form, P);
    int wlo = 0, whi = NW;  // warps the next lpt() pass may use
    auto lpt = [&]() {
        for (int it = 0; it < n; ++it) {
            int best = -1;
            for (int k = 0; k < n; ++k)
                if (!done[k] && (best < 0 || cost[k] > cost[best])) best = k;
            done[best] = true;
            int w = wlo;
            for (int v = wlo + 1; v < whi; ++v)
                if (load[v] < load[w]) w = v;
            load[w] += cost[best];
            if (kind[best] == 1) w1[idx[best]] = w;
            else if (kind[best] == 2) w2[idx[best]] = w;
            else w3[idx[best]] = w;
        }
        n = 0;
    };
    for (int k = 0; k < n1; ++k) {
        const int gk = k / (M.T0 * M.NC1);
        const int nun = pr1 ? (2 * gk + 1 < M.NG1 ? 2 : 1) : T.g1n[gk];
        cost[n] = nun * M.KS * M.MT * (M.NTY / M.NC1) + 2 + SG_P12_EPI * M.MT * (M.NTY / M.NC1);
        kind[n] = 1; idx[n] = k; done[n] = false; ++n;
    }
    if (ndim != 3) {  // 2D: phase 2 after its own barrier
        lpt();
        for (int v = 0; v < NW; ++v) load[v] = 0;
    }
    for (int k = 0; k < n2; ++k) {
        cost[n] = g2_blocks(T, k / (M.T1 * M.T0)) * M.KS * M.MT * M.MT + 2 + SG_P12_EPI * M.MT * M.MT;
        kind[n] = 2; idx[n] = k; done[n] = false; ++n;
    }
    if (NBs) whi = NW - NBs;
    lpt();
    if (NBs) {
        wlo = NW - NBs;
        whi = NW;
    }
    const int fb = T.NF + f_npairs(T);
    for (int k = 0; k < n3; ++k) {
        cost[n] = fb * M.KS3 * M.CH * M.MT + 2 + SG_P3_EPI * M.CH;  // + epilogue (live-sum update / CSR write)
        kind[n] = 3; idx[n] = k; done[n] = false; ++n;
    }
    lpt();
    // emit
    int o = 0;
    S.o_off1 = o; o += NW + 1;
    S.o_off2 = o; o += NW + 1;
    S.o_off3 = o; o += NW + 1;
    S.o_it1 = o; o += n1;
    S.o_it2 = o; o += n2;
    S.o_it3 = o; o += n3;
    int c1 = 0, c2 = 0, c3 = 0;
    for (int w = 0; w < NW; ++w) {
        S.v[S.o_off1 + w] = c1;
        S.v[S.o_off2 + w] = c2;
        S.v[S.o_off3 + w] = c3;
        for (int k = 0; k < n1; ++k) if (w1[k] == w) S.v[S.o_it1 + c1++] = k;
        for (int k = 0; k < n2; ++k) if (w2[k] == w) S.v[S.o_it2 + c2++] = k;
        for (int k = 0; k < n3; ++k) if (w3[k] == w) S.v[S.o_it3 + c3++] = k;
    }
    S.v[S.o_off1 + NW] = c1;
    S.v[S.o_off2 + NW] = c2;
    S.v[S.o_off3 + NW] = c3;
    S.o_u1b = o; o += M.NG1 + 1;
    S.o_u1ud = o; o += M.NU1;
    for (int g = 0; g <= M.NG1; ++g) S.v[S.o_u1b + g] = g1_unit_base(T, g);
    for (int g = 0; g < M.NG1; ++g)
        for (int u = 0; u < T.g1n[g]; ++u) S.v[S.o_u1ud + g1_unit_base(T, g) + u] = tri_index(T.g1mu[g][u], T.g1nu[g][u], T.MS);
    S.o_u2b = o; o += T.NG2 + 1;
    S.o_u2 = o;
    int c = 0;
    for (int g = 0; g < (ndim >= 2 ? T.NG2 : 0); ++g) {
        S.v[S.o_u2b + g] = c;
        for (int pass = 0; pass < 2; ++pass)
            for (int u = 0; u < T.g2n[g]; ++u) {
                if (T.g2pair[g][u] != pass) continue;
                const int ga = T.g2u[g][u], gaT = T.g1T[ga];
                S.v[S.o_u2 + c++] = pack_unit(ga, gaT, kslot1(T, kind1(T, ga)), kslot1(T, kind1(T, gaT)), pass);
            }
    }
    S.v[S.o_u2b + (ndim >= 2 ? T.NG2 : 0)] = c;
    o += c;
    S.o_u3 = o;
    c = 0;
    if (ndim == 3)
        for (int pass = 0; pass < 2; ++pass)
            for (int f = 0; f < T.NF; ++f) {
                if (T.fpair[f] != pass) continue;
                const int ga = T.fu[f], gaT = T.g2T[ga];
                S.v[S.o_u3 + c++] = pack_unit(ga, gaT, kslot2(T, kind2(T, ga)), kslot2(T, kind2(T, gaT)), pass);
            }
    o += c;
    S.n = o;
    return S;
}
template <int NDIM, int P, int FORM, bool RAT>
struct MmaTabS {
    static constexpr MmaTab S = mma_tab(NDIM, P, FORM, RAT);
};

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
    unsigned long long* dmma;    // executed DMMA instructions (per warp, summed per launch), or nullptr
    int z0;                      // z origin of the tile grid (rows)
    int run;                     // 2D: tiles per CTA (consecutive entries of the tile list)
    int dbg;                     // timing experiments only (SG_K4_DBG): skip 1 phase 3, 2 its epilogue, 4 phase 1, 8 phase 2
    int ntiles;                  // entries of the tile list (or tiles of the grid)
    int canon[3];                // B[d] holds bitwise equal values on all interior elements [p, S-1-p] (K2)
};

template <int NDIM, int P, int FORM, bool RAT>
__global__ void __launch_bounds__(32 * mma_warps(NDIM, P, FORM, RAT), mma_minb(NDIM, P, FORM, RAT)) assemble_mma(const __grid_constant__ MmaParams prm) {
    using TTS = TermTables<NDIM, FORM, RAT>;
    constexpr TileChoice TCH = mma_tile(NDIM, P, FORM, RAT);
    constexpr MmaGeom M = mma_geom(NDIM, P, FORM, RAT, TCH.T0, TCH.T1);
    constexpr int T0 = M.T0, T1 = M.T1, G = M.G, W = M.W, MT = M.MT, KS = M.KS, KS3 = M.KS3;
    constexpr int NB = M.NB, XW = M.XW, YW = M.YW, NTY = M.NTY, DY = M.DY, TY = M.TY, TC = M.TC;
    constexpr int MS = TTS::T.MS;
    constexpr int NW = mma_warps(NDIM, P, FORM, RAT);
    constexpr int NK1 = M.NK1, NK2 = M.NK2;
    constexpr int XWp = M.XWp;
    constexpr unsigned DBYTES = (unsigned)(M.U * XWp * DY * 8);
    extern __shared__ double smem[];
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    unsigned long long ndmma = 0;  // DMMA instructions this warp issues (reported per launch)
    unsigned nzero = 0;            // exact zeros this thread wrote to the CSR (3D; summed per launch)
    const int lr = lane >> 2, lk = lane & 3;

    // 2D: a CTA assembles a run of prm.run consecutive entries of the tile list (ordered column-major by
    // the host, so a run stays in one x column): the per-CTA set-up is paid once per run, the x-window
    // fragments once per column, and the next tile's D window streams in during phase 2
    const int run = (NDIM == 2 && prm.run > 1) ? prm.run : 1;
    const int t_first = (int)blockIdx.x * run;
    const int t_end = NDIM == 2 ? min(t_first + run, prm.ntiles) : t_first + 1;
    auto tile_at = [&](int t) { return prm.tiles ? prm.tiles[t] : t; };
    int tile = tile_at(t_first);
    int tc0 = tile % prm.tgrid[0], tc1 = (tile / prm.tgrid[0]) % prm.tgrid[1];
    const int tc2 = tile / (prm.tgrid[0] * prm.tgrid[1]);
    int b0 = tc0 * T0, b1 = tc1 * T1;
    const int b2 = prm.z0 + tc2 * prm.T2;
    // fixed windows: element e of direction d sits at local element (e - (b_d - P)); elements outside
    // the mesh have zero basis tables and zero D, so every index below is compile-time + lane
    int ew0 = b0 - P, ew1 = b1 - P;

    double* B0s = smem + M.o_B0;
    double* B1s = smem + M.o_B1;
    double* A1f = smem + M.o_A1;
    double* B2f = smem + M.o_B2f;
    double* B3f = smem + M.o_B3f;
    int* cmb = reinterpret_cast<int*>(smem + M.o_cmb);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + M.o_bar);
    // D window buffer of plane parity b (computed from smem so every access stays an LDS)
    auto Dbuf = [&](int b) -> double* { return smem + (b ? M.o_D2 : M.o_D); };
    double* T1s = smem + M.o_T1;
    double* T2s = smem + M.o_T2;

    // ---- item schedule + unit tables
    if (tid == 0) {
        int* tabw = reinterpret_cast<int*>(smem + M.o_tab);
        static_for<0, MmaTabS<NDIM, P, FORM, RAT>::S.n>([&](auto I) {
            constexpr int v = MmaTabS<NDIM, P, FORM, RAT>::S.v[decltype(I)::value];
            tabw[decltype(I)::value] = v;
        });
        if constexpr (NDIM == 3) {
            int* zr = reinterpret_cast<int*>(smem + M.o_rb + T0 * T1 * kMmaT2);
            zr[0] = INT_MAX;
            zr[1] = -1;
        }
    }
    // ---- zero the staging buffers once (padding columns / rows are read as exact zeros)
    for (long it = tid; it < M.total - M.o_T1; it += blockDim.x) T1s[it] = 0.0;
    // ---- window basis tables (zero outside the mesh)
    auto load_x = [&]() {
        for (int it = tid; it < XW * NB; it += blockDim.x) {
            const int e = ew0 + it / (G * NB);
            B0s[it] = (e >= 0 && e < prm.S[0]) ? prm.B[0][((long long)ew0 * G) * NB + it] : 0.0;
        }
    };
    auto load_y = [&]() {
        if constexpr (NDIM >= 2) {
            for (int it = tid; it < YW * NB; it += blockDim.x) {
                const int e = ew1 + it / (G * NB);
                B1s[it] = (e >= 0 && e < prm.S[1]) ? prm.B[1][((long long)ew1 * G) * NB + it] : 0.0;
            }
        }
    };
    load_x();
    load_y();
    __syncthreads();
    // ---- tile-constant fragments
    // A1f[((i0l*NU1 + unit)*KS + kk)*MT + a][lane] = Q0(i0, i0+d0, x): d0 = a*8 + lr - P, x = kk*4 + lk in supp(i0)
    auto frag_x = [&]() {
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
    };
    auto frag_y = [&]() {
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
    };
    frag_x();
    frag_y();
    if constexpr (NDIM == 3) {
        // per combo: {offset inside a row's j2 block (or -1), cnt0*cnt1, i0 + m0 i1, j0 + m0 j1}
        for (int c = tid; c < M.NCOMBO; c += blockDim.x) {
            const int d0 = c % W - P, d1 = (c / W) % W - P, i1l = (c / (W * W)) % T1, i0l = c / (W * W * T1);
            const int i0 = b0 + i0l, i1 = b1 + i1l, j0 = i0 + d0, j1 = i1 + d1;
            int off = -1, c01 = 0;
            if (i0 < prm.m[0] && i1 < prm.m[1] && j0 >= 0 && j0 < prm.m[0] && j1 >= 0 && j1 < prm.m[1]) {
                const int lo0 = max(0, i0 - P), lo1 = max(0, i1 - P);
                const int cnt0 = min(prm.m[0] - 1, i0 + P) - lo0 + 1, cnt1 = min(prm.m[1] - 1, i1 + P) - lo1 + 1;
                off = (j0 - lo0) + cnt0 * (j1 - lo1);
                c01 = cnt0 * cnt1;
            }
            cmb[4 * c + 0] = off;
            cmb[4 * c + 1] = c01 | ((c / (W * W)) << 16);  // cnt0*cnt1 | tile row of the combo << 16
            cmb[4 * c + 2] = i0 + prm.m[0] * i1;
            cmb[4 * c + 3] = j0 + prm.m[0] * j1;
        }
        int64_t* rb = reinterpret_cast<int64_t*>(smem + M.o_rb);
        int zlo = INT_MAX, zhi = -1;
        for (int t = tid; t < T0 * T1 * kMmaT2; t += blockDim.x) {
            const int i2 = b2 + t % kMmaT2, i1 = b1 + (t / kMmaT2) % T1, i0 = b0 + t / (kMmaT2 * T1);
            int64_t v = -1;
            if (i0 < prm.m[0] && i1 < prm.m[1] && i2 < prm.m[2] && t % kMmaT2 < prm.T2) {
                const int64_t row = (int64_t)i0 + (int64_t)prm.m[0] * i1 + (int64_t)prm.m[0] * prm.m[1] * i2;
                if (row >= prm.slab_lo && row < prm.slab_hi && (!prm.rowmask || prm.rowmask[row])) v = prm.rowstart[row];
            }
            rb[t] = v;
            if (v >= 0) {
                zlo = min(zlo, b2 + t % kMmaT2);
                zhi = max(zhi, b2 + t % kMmaT2);
            }
        }
        // z range of the rows this tile actually owns (restricted plans: only the needed layers)
        int* zr = reinterpret_cast<int*>(rb + T0 * T1 * kMmaT2);
        if (zlo <= zhi) {
            atomicMin(&zr[0], zlo);
            atomicMax(&zr[1], zhi);
        }
    }
    if constexpr (NDIM == 3) {
        __syncthreads();
        const int* zr = reinterpret_cast<const int*>(smem + M.o_rb + T0 * T1 * kMmaT2);
        if (zr[1] < zr[0]) return;  // no owned row in this tile
    }

    const long long G0 = prm.Gp[0];
    int elo2 = 0, ehi2 = 0;
    if constexpr (NDIM == 3) {
        const int* zrng = reinterpret_cast<const int*>(smem + M.o_rb + T0 * T1 * kMmaT2);
        elo2 = max(0, zrng[0] - P);
        ehi2 = min(prm.S[2] - 1, zrng[1]);
    }
    constexpr int GZ = NDIM == 3 ? G : 1;
    const int nplanes = (ehi2 - elo2 + 1) * GZ;
    const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&bars[0]);
    // A TMA box must start at a 16-byte aligned global address: with an odd Gauss count and an odd tile
    // extent in y the window's first y point (y fastest, 8 B each) can be odd (3 x 3 tiles at p = 2, 4:
    // the "illegal instruction" of profiles/r02_tma2d_matrix.txt).  Such a window is fetched from the
    // point before it and read one column further in (DY >= YW + 1 there: YW is odd).
    auto tma_ysh = [&](int e1) -> int {
        if constexpr (G % 2 == 0 || NDIM < 2) return 0;
        else return (prm.tma && NDIM >= 2) ? ((e1 * G) & 1) : 0;
    };
    static_assert(NDIM < 2 || G % 2 == 0 || T1 % 2 == 0 || DY >= YW + 1, "room for the shifted window");
    // D window of plane `pi` (TMA: one 4D box per plane; out-of-mesh coordinates are zero filled)
    auto issue_plane = [&](int pi) {
        const int z = elo2 * G + pi;
        const uint32_t bar = bar0 + 8u * (uint32_t)(pi & 1);
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(Dbuf(pi & 1));
        if (prm.dbg & 16) {  // timing experiment: no D traffic (the phase completes at once)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
            return;
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(DBYTES) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(dst),
            "l"(reinterpret_cast<uint64_t>(&prm.dmap)), "r"(ew1 * G - tma_ysh(ew1)), "r"(ew0 * G), "r"(0), "r"(z), "r"(bar)
            : "memory");
    };
    // TMA D windows: 3D (double-buffered pencil of planes), 2D (one window per tile, the next tile's
    // streamed during phase 2); SG_NO_TMA=1 selects plain loads (debug)
    constexpr bool kTma = NDIM >= 2;
    const bool use_tma = kTma && prm.tma;
    // warp-specialised 3D pipeline: plane j + 2 is issued into plane j's buffer as soon as the last
    // phase-1 warp has finished plane j (a shared counter), ~half an interval before the next barrier;
    // only the phase-1 warps wait for the D windows
    const bool early = use_tma && NDIM == 3 && mma_spec_nb(NDIM, FORM, P) > 0 && !(prm.dbg & 16);
    if (use_tma) {
        if (tid == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar0) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar0 + 8u) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
            reinterpret_cast<int*>(smem + M.o_bar + 3)[0] = 0;  // phase-1 warps done (early issue)
        }
        __syncthreads();
        if (tid == 0) issue_plane(0);
        if (tid == 0 && early && nplanes > 1) issue_plane(1);
    }
    // 2D: the D window of the run's k-th tile (TMA box at the tile's window origin; barrier k & 1)
    auto issue_tile = [&](int k, int t) {
        const int tt = tile_at(t);
        const int x0 = (tt % prm.tgrid[0]) * T0 - P, y0 = ((tt / prm.tgrid[0]) % prm.tgrid[1]) * T1 - P;
        const uint32_t bar = bar0 + 8u * (uint32_t)(k & 1);
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(Dbuf(0));
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(DBYTES) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(dst),
            "l"(reinterpret_cast<uint64_t>(&prm.dmap)), "r"(y0 * G - tma_ysh(y0)), "r"(x0 * G), "r"(0), "r"(0), "r"(bar)
            : "memory");
    };
    // make the D window of plane j resident in Dbuf[j & 1] (plain path: all threads load, then a barrier)
    auto get_plane = [&](int j) {
        double* Ds = Dbuf(j & 1);
        if (use_tma) {
            if (!early && tid == 0 && j + 1 < nplanes) issue_plane(j + 1);  // prefetch the next plane
            const uint32_t bar = bar0 + 8u * (uint32_t)(j & 1);
            const uint32_t par = (uint32_t)((j >> 1) & 1);
            uint32_t done = 0;
            while (!done) {
                asm volatile(
                    "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                    : "=r"(done)
                    : "r"(bar), "r"(par)
                    : "memory");
            }
            Ds += tma_ysh(ew1);
        } else {
            const long long gx0 = (long long)ew0 * G, gy0 = (long long)ew1 * G;
            const long long z = (long long)elo2 * G + j;
            const long long G1 = NDIM >= 2 ? prm.Gp[1] : 1;
            // (under warp specialisation only group A loads planes)
            const int nld = mma_spec_nb(NDIM, FORM, P) > 0 ? (NW - mma_spec_nb(NDIM, FORM, P)) * 32 : (int)blockDim.x;
            for (int it = tid; it < M.U * XWp * DY; it += nld) {
                const int y = it % DY, r = it / DY;
                const int u = r / XWp, x = r % XWp;
                const long long gx = gx0 + x, gy = gy0 + y;
                double v = 0.0;
                if (gx >= 0 && gx < G0 && gy >= 0 && gy < G1)
                    v = prm.D[((z * M.U + u) * G0 + gx) * (long long)prm.Dys + gy];
                Ds[r * DY + y] = v;
            }
            if constexpr (mma_spec_nb(NDIM, FORM, P) > 0) {
                asm volatile("bar.sync 1, %0;\n" ::"r"((NW - mma_spec_nb(NDIM, FORM, P)) * 32) : "memory");
            } else {
                __syncthreads();
            }
        }
        return Ds;
    };

    using TAB = MmaTabS<NDIM, P, FORM, RAT>;
    constexpr long T1SZ = mma_t1_plane(M);
    const int* tab = reinterpret_cast<const int*>(smem + M.o_tab);

    // ---------------- phase 1 (x): items (group, row i0l) -> T1[Gc][i0l][d0][y]
    auto phase1 = [&](const double* Ds, double* T1b) {
        if (prm.dbg & 4) return;
        const int qe = tab[TAB::S.o_off1 + warp + 1];
        for (int q = tab[TAB::S.o_off1 + warp]; q < qe; ++q) {
            const int k = tab[TAB::S.o_it1 + q];
            constexpr int NC1 = M.NC1, NTI = NTY / NC1;
            const int cc = k % NC1, Gc = k / (T0 * NC1), i0l = (k / NC1) % T0;
            double acc[MT][NTI][2];
#pragma unroll
            for (int a = 0; a < MT; ++a)
#pragma unroll
                for (int c = 0; c < NTI; ++c) acc[a][c][0] = acc[a][c][1] = 0.0;
            auto unit1 = [&](const int unit, const int ud) {
                const double* af = A1f + ((i0l * M.NU1 + unit) * KS) * MT * 32 + lane;
                const double* dpl = Ds + (ud * XWp) * DY + lr + cc * NTI * 8;
#pragma unroll
                for (int kk = 0; kk < KS; ++kk) {
                    const int s = kk * 4 + lk;
                    const int x = (s < (P + 1) * G) ? i0l * G + s : 0;
                    const double* drow = dpl + x * DY;
                    double afr[MT];
#pragma unroll
                    for (int a = 0; a < MT; ++a) afr[a] = af[(kk * MT + a) * 32];
#pragma unroll
                    for (int c = 0; c < NTI; ++c) {
                        const double bf = drow[c * 8];
#pragma unroll
                        for (int a = 0; a < MT; ++a) dmma(acc[a][c][0], acc[a][c][1], afr[a], bf);
                    }
                }
                        };
#if SG_STATIC_UNITS
            // the group's units and D components are compile-time constants (no table reads per unit)
            static_for<0, M.NG1>([&](auto GI) {
                constexpr int g = decltype(GI)::value;
                if (Gc != g) return;
                constexpr int ub = TAB::S.v[TAB::S.o_u1b + g], ue = TAB::S.v[TAB::S.o_u1b + g + 1];
                ndmma += (unsigned long long)(ue - ub) * KS * NTI * MT;
                static_for<ub, ue>([&](auto UI) {
                    constexpr int unit = decltype(UI)::value;
                    constexpr int ud = TAB::S.v[TAB::S.o_u1ud + unit];
                    unit1(unit, ud);
                });
            });
#else
            const int ue = tab[TAB::S.o_u1b + Gc + 1];
            ndmma += (unsigned long long)(ue - tab[TAB::S.o_u1b + Gc]) * KS * NTI * MT;
            for (int unit = tab[TAB::S.o_u1b + Gc]; unit < ue; ++unit) unit1(unit, tab[TAB::S.o_u1ud + unit]);
#endif
            if constexpr (NDIM == 1) {
                const int i0 = b0 + i0l;
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
                double* t1 = T1b + mma_t1_row(M, (Gc * T0 + i0l) * MT * 8 + lr);
#pragma unroll
                for (int a = 0; a < MT; ++a)
#pragma unroll
                    for (int c = 0; c < NTI; ++c) {
                        double* dst = t1 + a * (mma_t1_row(M, 8) - mma_t1_row(M, 0)) + (cc * NTI + c) * 8 + 2 * lk;
                        dst[0] = acc[a][c][0];
                        dst[1] = acc[a][c][1];
                    }
            }
        }
    };

    // ---------------- phase 2 (y): items (level-2 group, row i1l, row i0l)
    // 2D: final values into the CSR; 3D: T2 plane slot [g2][(i0l,i1l,d1,d0)]
    // Chains: non-pair units into accS in unit order, then each symmetric pair (A, B chains) folded
    // in as accS + (A + B) in order -- the mirror of the transposed entry's evaluation.
    auto phase2 = [&](const double* T1b, double* T2b) {
        if (prm.dbg & 8) return;
        constexpr int T1A = mma_t1_row(M, 8) - mma_t1_row(M, 0);  // T1 offset of 8 rows (one m-tile)
        if constexpr (NDIM >= 2) {
            const int qe = tab[TAB::S.o_off2 + warp + 1];
            for (int q = tab[TAB::S.o_off2 + warp]; q < qe; ++q) {
                const int k = tab[TAB::S.o_it2 + q];
                const int Gc = k / (T1 * T0), rem = k - Gc * (T1 * T0);
                const int i1l = rem / T0, r = rem - (rem / T0) * T0;
                const int i1 = b1 + i1l, i0 = b0 + r;
                if (i1 >= prm.m[1] || i0 >= prm.m[0]) continue;
                auto block = [&](int ga, int kd, double (&acc)[MT][MT][2]) {
                    const double* bfp = B2f + ((i1l * NK1 + kd) * KS) * MT * 32 + lane;
                    // y of support point s of row i1 is i1l*G + s (the support is contiguous)
                    const double* t1 = T1b + mma_t1_row(M, (ga * T0 + r) * MT * 8 + lr) + i1l * G + lk;
#pragma unroll
                    for (int kk = 0; kk < KS; ++kk) {
                        double bfs[MT];
#pragma unroll
                        for (int c = 0; c < MT; ++c) bfs[c] = bfp[(kk * MT + c) * 32];
#pragma unroll
                        for (int a = 0; a < MT; ++a) {
                            const double av = t1[a * T1A + kk * 4];
#pragma unroll
                            for (int c = 0; c < MT; ++c) dmma(acc[a][c][0], acc[a][c][1], av, bfs[c]);
                        }
                    }
                };
                // a symmetric pair's two chains, interleaved (independent accumulators)
                auto block2 = [&](int ga, int kd, int gb, int kb, double (&accA)[MT][MT][2], double (&accB)[MT][MT][2]) {
                    const double* bfa = B2f + ((i1l * NK1 + kd) * KS) * MT * 32 + lane;
                    const double* bfb = B2f + ((i1l * NK1 + kb) * KS) * MT * 32 + lane;
                    const double* ta = T1b + mma_t1_row(M, (ga * T0 + r) * MT * 8 + lr) + i1l * G + lk;
                    const double* tb = T1b + mma_t1_row(M, (gb * T0 + r) * MT * 8 + lr) + i1l * G + lk;
#pragma unroll
                    for (int kk = 0; kk < KS; ++kk) {
                        double fa[MT], fb[MT];
#pragma unroll
                        for (int c = 0; c < MT; ++c) {
                            fa[c] = bfa[(kk * MT + c) * 32];
                            fb[c] = bfb[(kk * MT + c) * 32];
                        }
#pragma unroll
                        for (int a = 0; a < MT; ++a) {
                            const double va = ta[a * T1A + kk * 4], vb = tb[a * T1A + kk * 4];
#pragma unroll
                            for (int c = 0; c < MT; ++c) {
                                dmma(accA[a][c][0], accA[a][c][1], va, fa[c]);
                                dmma(accB[a][c][0], accB[a][c][1], vb, fb[c]);
                            }
                        }
                    }
                };
                double accS[MT][MT][2];
#pragma unroll
                for (int a = 0; a < MT; ++a)
#pragma unroll
                    for (int c = 0; c < MT; ++c) accS[a][c][0] = accS[a][c][1] = 0.0;
                const int ue = tab[TAB::S.o_u2b + Gc + 1];
                ndmma += (unsigned long long)(ue - tab[TAB::S.o_u2b + Gc]) * KS * MT * MT;  // + one more per pair below
                [[maybe_unused]] int u = tab[TAB::S.o_u2b + Gc];
#if SG_P2_ILP
                {
                    // non-pair units (listed first) in two interleaved chains, even / odd units, added at
                    // the end: half the dependent DMMA depth.  Every unit is its own transpose, so the
                    // transposed entry evaluates the same sums in the same order (bitwise symmetry holds)
                    double accO[MT][MT][2];
                    bool odd = false;
#pragma unroll
                    for (int a = 0; a < MT; ++a)
#pragma unroll
                        for (int c = 0; c < MT; ++c) accO[a][c][0] = accO[a][c][1] = 0.0;
                    for (; u + 1 < ue; u += 2) {
                        const int d0 = tab[TAB::S.o_u2 + u], d1 = tab[TAB::S.o_u2 + u + 1];
                        if ((d0 >> 24) || (d1 >> 24)) break;
                        block2(d0 & 255, (d0 >> 16) & 15, d1 & 255, (d1 >> 16) & 15, accS, accO);
                        odd = true;
                    }
                    if (u < ue && !(tab[TAB::S.o_u2 + u] >> 24)) {
                        const int d = tab[TAB::S.o_u2 + u];
                        block(d & 255, (d >> 16) & 15, accS);
                        ++u;
                    }
                    if (odd)
#pragma unroll
                        for (int a = 0; a < MT; ++a)
#pragma unroll
                            for (int c = 0; c < MT; ++c)
#pragma unroll
                                for (int h = 0; h < 2; ++h) accS[a][c][h] = __dadd_rn(accS[a][c][h], accO[a][c][h]);
                }
#endif
                auto unit2 = [&](const int d) {
                    const int ga = d & 255, kd = (d >> 16) & 15;
                    if (!(d >> 24)) {
                        block(ga, kd, accS);
                    } else {
                        double tA[MT][MT][2], tB[MT][MT][2];
                        ndmma += KS * MT * MT;
#pragma unroll
                        for (int a = 0; a < MT; ++a)
#pragma unroll
                            for (int c = 0; c < MT; ++c) tA[a][c][0] = tA[a][c][1] = tB[a][c][0] = tB[a][c][1] = 0.0;
                        block2(ga, kd, (d >> 8) & 255, (d >> 20) & 15, tA, tB);
#pragma unroll
                        for (int a = 0; a < MT; ++a)
#pragma unroll
                            for (int c = 0; c < MT; ++c)
#pragma unroll
                                for (int h = 0; h < 2; ++h) accS[a][c][h] = __dadd_rn(accS[a][c][h], __dadd_rn(tA[a][c][h], tB[a][c][h]));
                    }
                };
#if SG_STATIC_UNITS && !SG_P2_ILP
                static_for<0, (NDIM >= 2 ? TTS::T.NG2 : 0)>([&](auto GI) {
                    constexpr int g = decltype(GI)::value;
                    if (Gc != g) return;
                    constexpr int ub = TAB::S.v[TAB::S.o_u2b + g], ue2 = TAB::S.v[TAB::S.o_u2b + g + 1];
                    static_for<ub, ue2>([&](auto UI) {
                        constexpr int d = TAB::S.v[TAB::S.o_u2 + decltype(UI)::value];
                        unit2(d);
                    });
                });
#else
                for (; u < ue; ++u) unit2(tab[TAB::S.o_u2 + u]);
#endif
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
                                double v = accS[a][c][h];
                                const int64_t col = (int64_t)j0 + (int64_t)prm.m[0] * j1;
                                if constexpr (RAT) v = v * (si * prm.sol_w[col]);
                                const int64_t pos = base + (j0 - lo0) + (int64_t)cnt0 * (j1 - lo1);
                                prm.data[pos] = v;
                                prm.indices[pos] = (int)col;
                                if (prm.zeros && v == 0.0) atomicAdd(prm.zeros, 1ull);
                            }
                    }
                } else {
                    double* t2 = T2b + Gc * TC + (r * T1 + i1l) * W * W;
#pragma unroll
                    for (int a = 0; a < MT; ++a) {
                        const int d0 = a * 8 + lr;
                        if (d0 >= W) continue;
#pragma unroll
                        for (int c = 0; c < MT; ++c)
#pragma unroll
                            for (int h = 0; h < 2; ++h) {
                                const int d1 = c * 8 + 2 * lk + h;
                                if (d1 < W) t2[d1 * W + d0] = accS[a][c][h];
                            }
                    }
                }
            }
        }
    };

    if constexpr (NDIM == 1) {
        const double* Ds = get_plane(0);
        phase1(Ds, T1s);
    } else if constexpr (NDIM == 2) {
        int colx = tc0;
        int ew0_prev = ew0, ew1_prev = ew1;  // windows whose fragments are in shared memory
        for (int t = t_first; t < t_end; ++t) {
            const int k = t - t_first;
            if (k > 0) {
                // next tile of the run: new y window; new x window only when the column changes
                tile = tile_at(t);
                tc0 = tile % prm.tgrid[0];
                tc1 = (tile / prm.tgrid[0]) % prm.tgrid[1];
                b0 = tc0 * T0;
                b1 = tc1 * T1;
                ew0 = b0 - P;
                ew1 = b1 - P;
                // windows made of interior elements carry identical tables (K2 canonicalises them),
                // so their fragments are reused as they are
                auto interior = [&](int ew, int nel, int S) { return ew >= P && ew + nel - 1 <= S - 1 - P; };
                const bool xin = prm.canon[0] && interior(ew0, T0 + P, prm.S[0]) && interior(ew0_prev, T0 + P, prm.S[0]);
                const bool yin = prm.canon[1] && interior(ew1, T1 + P, prm.S[1]) && interior(ew1_prev, T1 + P, prm.S[1]);
                const bool newx = tc0 != colx && !xin;
                const bool newy = !yin;
                colx = tc0;
                ew0_prev = ew0;
                ew1_prev = ew1;
                if (newx || newy) {
                    if (newx) load_x();
                    if (newy) load_y();
                    __syncthreads();
                    if (newx) frag_x();
                    if (newy) frag_y();
                    __syncthreads();
                }
            }
            const double* Ds;
            if (use_tma) {
                // the tile's box was issued by thread 0 (first tile: above; others: after the previous phase 1)
                const uint32_t bar = bar0 + 8u * (uint32_t)(k & 1);
                const uint32_t par = (uint32_t)((k >> 1) & 1);
                uint32_t done = 0;
                while (!done) {
                    asm volatile(
                        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                        : "=r"(done)
                        : "r"(bar), "r"(par)
                        : "memory");
                }
                Ds = Dbuf(0) + tma_ysh(ew1);
            } else {
                Ds = get_plane(0);
            }
            phase1(Ds, T1s);
            __syncthreads();
            // the D buffer is free: stream the next tile's window in while phase 2 runs
            if (use_tma && tid == 0 && t + 1 < t_end) issue_tile(k + 1, t + 1);
            phase2(T1s, nullptr);
            __syncthreads();
        }
    } else {
        // ---------------- 3D: one barrier interval per Gauss plane j (ascending z):
        //   phase 3(layer finished one interval ago; final entries straight to the CSR)
        //   | phase 1(plane j) | phase 2(plane j-1) | phase-3 fragments of the layer starting at j
        // T1 is double buffered by plane parity, T2 is a ring of G+1 plane slots, the phase-3
        // fragments are double buffered by layer parity.
        constexpr int NS = mma_ns(NDIM, P, FORM);
        constexpr int B3SZ = NK2 * KS3 * MT * 32;
        constexpr int CH = M.CH;
        constexpr int KZ = (P + 1) * G;  // z points of a row's support
        const int m01 = prm.m[0] * prm.m[1];
        const int* zrng = reinterpret_cast<const int*>(smem + M.o_rb + T0 * T1 * kMmaT2);
        const int zr0 = zrng[0], zr1 = zrng[1];
        const int nlayers = nplanes / G;
        // row planes elo2 .. elo2 + nsteps - 1; the rows above the last streamed layer (ehi2) have all
        // their layers streamed by then and follow it
        const int nsteps = nlayers + max(0, zr1 - ehi2);
        // phase-3 B fragments depend on the row plane only through the z tables of its layers i2-P .. i2:
        // on canonical tables (prm.canon[2]) every row plane with all of them interior (2P <= i2 <= S-1-P)
        // has the same fragments, so consecutive interior row planes share one buffer (no rebuild);
        // b3par(L) = buffer of row plane L (flips at every rebuilt row plane)
        const int b3La = prm.canon[2] ? 2 * P - elo2 : (1 << 29), b3Lb = prm.S[2] - 1 - P - elo2;
        auto b3reuse = [&](int L) { return L >= 1 && L - 1 >= b3La && L <= b3Lb; };
        auto b3par = [&](int L) {
            const int lo = max(b3La + 1, 1), hi = min(L, b3Lb);
            return (L - (hi >= lo ? hi - lo + 1 : 0)) & 1;
        };
        // ---- phase 3 (z) of row plane i2 = elo2 + L: every entry is one DMMA chain over the z points of
        // its row's support (layers i2-P .. i2 ascending; the column basis vanishes outside the shared
        // layers, so those terms add exact zeros), written straight to the CSR.  Items: chunks of CH m-tiles.
        auto phase3 = [&](const int L) {
            if (prm.dbg & 1) return;
            const int i2 = elo2 + L;
            if (i2 < zr0 || i2 > zr1) return;
            const double* B3b = B3f + b3par(L) * B3SZ;
            // T2 slot of this lane's z point s = kk*4 + lk: plane (i2 - P + s/G - elo2)*G + s%G of the stream
            int zslot[KS3];
#pragma unroll
            for (int kk = 0; kk < KS3; ++kk) {
                const int sz = kk * 4 + lk < KZ ? kk * 4 + lk : 0;
                const int rel = (i2 - P + sz / G - elo2) * G + sz % G;
                zslot[kk] = ((rel % NS) + NS) % NS;  // planes before the stream: zero fragments, any slot
            }
            const int64_t* rb = reinterpret_cast<const int64_t*>(smem + M.o_rb) + (i2 - b2);
            const int jlo2 = max(0, i2 - P);
            const int qe = tab[TAB::S.o_off3 + warp + 1];
            for (int q = tab[TAB::S.o_off3 + warp]; q < qe; ++q) {
                const int ch = tab[TAB::S.o_it3 + q];
                auto block = [&](int ga, int kd, double (&acc)[CH][MT][2]) {
                    const double* bfp = B3b + (kd * KS3) * MT * 32 + lane;
                    const double* t2b = T2s + ga * TC + ch * CH * 8 + lr;
#pragma unroll
                    for (int kk = 0; kk < KS3; ++kk) {
                        double bfs[MT];
#pragma unroll
                        for (int c = 0; c < MT; ++c) bfs[c] = bfp[(kk * MT + c) * 32];
                        const double* t2 = t2b + (long)zslot[kk] * M.T2PS;
#pragma unroll
                        for (int mm = 0; mm < CH; ++mm) {
                            const double av = t2[mm * 8];
#pragma unroll
                            for (int c = 0; c < MT; ++c) dmma(acc[mm][c][0], acc[mm][c][1], av, bfs[c]);
                        }
                    }
                };
                // two units' chains interleaved (independent accumulators)
                auto block2 = [&](int ga, int kd, int gb, int kb, double (&accA)[CH][MT][2], double (&accB)[CH][MT][2]) {
                    const double* bfa = B3b + (kd * KS3) * MT * 32 + lane;
                    const double* bfb = B3b + (kb * KS3) * MT * 32 + lane;
                    const double* t2a = T2s + ga * TC + ch * CH * 8 + lr;
                    const double* t2bb = T2s + gb * TC + ch * CH * 8 + lr;
#pragma unroll
                    for (int kk = 0; kk < KS3; ++kk) {
                        double fa[MT], fb[MT];
#pragma unroll
                        for (int c = 0; c < MT; ++c) {
                            fa[c] = bfa[(kk * MT + c) * 32];
                            fb[c] = bfb[(kk * MT + c) * 32];
                        }
                        const long zo = (long)zslot[kk] * M.T2PS;
#pragma unroll
                        for (int mm = 0; mm < CH; ++mm) {
                            const double va = t2a[zo + mm * 8], vb = t2bb[zo + mm * 8];
#pragma unroll
                            for (int c = 0; c < MT; ++c) {
                                dmma(accA[mm][c][0], accA[mm][c][1], va, fa[c]);
                                dmma(accB[mm][c][0], accB[mm][c][1], vb, fb[c]);
                            }
                        }
                    }
                };
                double accS[CH][MT][2];
#pragma unroll
                for (int mm = 0; mm < CH; ++mm)
#pragma unroll
                    for (int c = 0; c < MT; ++c) accS[mm][c][0] = accS[mm][c][1] = 0.0;
                ndmma += (unsigned long long)(TTS::T.NF + f_npairs(TTS::T)) * KS3 * CH * MT;  // compile-time per item
                [[maybe_unused]] int u = 0;
#if SG_P3_ILP
                {
                    // non-pair units in two interleaved chains (as phase 2)
                    double accO[CH][MT][2];
                    bool odd = false;
#pragma unroll
                    for (int mm = 0; mm < CH; ++mm)
#pragma unroll
                        for (int c = 0; c < MT; ++c) accO[mm][c][0] = accO[mm][c][1] = 0.0;
                    for (; u + 1 < TTS::T.NF; u += 2) {
                        const int d0 = tab[TAB::S.o_u3 + u], d1 = tab[TAB::S.o_u3 + u + 1];
                        if ((d0 >> 24) || (d1 >> 24)) break;
                        block2(d0 & 255, (d0 >> 16) & 15, d1 & 255, (d1 >> 16) & 15, accS, accO);
                        odd = true;
                    }
                    if (u < TTS::T.NF && !(tab[TAB::S.o_u3 + u] >> 24)) {
                        const int d = tab[TAB::S.o_u3 + u];
                        block(d & 255, (d >> 16) & 15, accS);
                        ++u;
                    }
                    if (odd)
#pragma unroll
                        for (int mm = 0; mm < CH; ++mm)
#pragma unroll
                            for (int c = 0; c < MT; ++c)
#pragma unroll
                                for (int h = 0; h < 2; ++h) accS[mm][c][h] = __dadd_rn(accS[mm][c][h], accO[mm][c][h]);
                }
#endif
                auto unit3 = [&](const int d) {
                    const int ga = d & 255, kd = (d >> 16) & 15;
                    if (!(d >> 24)) {
                        block(ga, kd, accS);
                    } else {
                        double tA[CH][MT][2], tB[CH][MT][2];
#pragma unroll
                        for (int mm = 0; mm < CH; ++mm)
#pragma unroll
                            for (int c = 0; c < MT; ++c) tA[mm][c][0] = tA[mm][c][1] = tB[mm][c][0] = tB[mm][c][1] = 0.0;
                        block2(ga, kd, (d >> 8) & 255, (d >> 20) & 15, tA, tB);
#pragma unroll
                        for (int mm = 0; mm < CH; ++mm)
#pragma unroll
                            for (int c = 0; c < MT; ++c)
#pragma unroll
                                for (int h = 0; h < 2; ++h) accS[mm][c][h] = __dadd_rn(accS[mm][c][h], __dadd_rn(tA[mm][c][h], tB[mm][c][h]));
                    }
                };
#if SG_STATIC_UNITS && !SG_P3_ILP
                static_for<0, TTS::T.NF>([&](auto UI) {
                    constexpr int d = TAB::S.v[TAB::S.o_u3 + decltype(UI)::value];
                    unit3(d);
                });
#else
                for (; u < TTS::T.NF; ++u) unit3(tab[TAB::S.o_u3 + u]);
#endif
                if (prm.dbg & 2) {
                    nzero += accS[0][0][0] == 0.0 ? 1u : 0u;
                    continue;
                }
                // final entries: row (combo's (i0, i1), i2), column (j0, j1, j2 = i2 + d2)
#pragma unroll
                for (int mm = 0; mm < CH; ++mm) {
                    const int combo = (ch * CH + mm) * 8 + lr;
                    if (combo >= M.NCOMBO) continue;
                    const int4 cb = reinterpret_cast<const int4*>(cmb)[combo];
                    const int64_t rowb = rb[(cb.y >> 16) * kMmaT2];
                    if (cb.x < 0 || rowb < 0) continue;
                    const int cnt01 = cb.y & 0xffff;
#pragma unroll
                    for (int c = 0; c < MT; ++c)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int d2 = c * 8 + 2 * lk + h - P;
                            const int j2 = i2 + d2;
                            if (d2 > P || j2 < 0 || j2 >= prm.m[2]) continue;
                            double v = accS[mm][c][h];
                            const int64_t pos = rowb + cb.x + (int64_t)cnt01 * (j2 - jlo2);
                            const int col = cb.w + m01 * j2;
                            if constexpr (RAT) v = v * (prm.sol_w[(int64_t)cb.z + (int64_t)m01 * i2] * prm.sol_w[col]);
                            nzero += v == 0.0 ? 1u : 0u;
                            prm.data[pos] = v;
                            prm.indices[pos] = col;
                        }
                }
            }
        };
        // ---- phase-3 B fragments of row plane i2 = elo2 + L (warps w0 .. w0+nw-1):
        // B3f[L&1][(slot*KS3 + kk)*MT + c][lane] = B^a2_{i2}(z_s) B^b2_{i2+d2}(z_s), s = kk*4 + lk, d2 = c*8 + lr - P
        auto build_b3 = [&](const int L, const int w0, const int nw) {
            const int i2 = elo2 + L;
            if (b3reuse(L)) return;
            double* B3b = B3f + b3par(L) * B3SZ;
            for (int slot = warp - w0; slot < NK2; slot += nw) {
                int kind = 0;
                static_for<0, NK2>([&](auto SI) { if (slot == decltype(SI)::value) kind = kind_of_slot2(TTS::T, decltype(SI)::value); });
                const int a2 = kind % 3, bb2 = kind / 3;
                for (int kk = 0; kk < KS3; ++kk) {
                    const int sz = kk * 4 + lk;
                    const int e = i2 - P + sz / G, r = P - sz / G;
                    for (int c = 0; c < MT; ++c) {
                        const int d2 = c * 8 + lr - P;
                        const int rj = r + d2;
                        double v = 0.0;
                        if (sz < KZ && d2 <= P && rj >= 0 && rj <= P && e >= 0 && e < prm.S[2]) {
                            const double* bz = prm.B[2] + ((long long)e * G + sz % G) * NB;
                            v = __dmul_rn(bz[a2 * (P + 1) + r], bz[bb2 * (P + 1) + rj]);
                        }
                        B3b[((slot * KS3 + kk) * MT + c) * 32 + lane] = v;
                    }
                }
            }
        };
        constexpr int NBW = mma_spec_nb(NDIM, FORM, P);
        if constexpr (NBW > 0) {
            // ---- warp-specialised pipeline: group A (phases 1-2, planes) / group B (phase 3, row planes),
            // handing over through two monotonic counters: ready = layers whose planes are in T2,
            // done = row planes finished (a T2 plane of layer l is free once row plane l + P is done)
            constexpr int NAW = NW - NBW;
            volatile int* cnt = reinterpret_cast<volatile int*>(smem + M.o_bar + 2);  // [0] ready, [1] done
            if (tid == 0) {
                cnt[0] = 0;
                cnt[1] = 0;
            }
            __syncthreads();
            auto wait_ge = [&](int which, int v) {
                for (long it = 0; cnt[which] < v; ++it) {
                    __nanosleep(64);
                    if (it > (1L << 26)) __trap();  // a lost hand-over aborts the launch instead of hanging the GPU
                }
                __threadfence_block();
            };
#ifdef SG_K4_PROF
            // clock64 breakdown per warp (experimental builds only): A: plane wait, phase 1, phase 2,
            // ring wait, barrier, loop; B: ready wait, barrier, phase 3, fragments, barrier, loop
            unsigned long long pf[6] = {0, 0, 0, 0, 0, 0};
#define SG_PF(k, stmt) { const long long t_ = clock64(); stmt; pf[k] += clock64() - t_; }
#else
#define SG_PF(k, stmt) { stmt; }
#endif
            if (warp < NAW) {
                // warps with phase-1 items (compile-time schedule) and their count
                constexpr int NP1W = [] {
                    int c = 0;
                    for (int w = 0; w < NW; ++w) c += TAB::S.v[TAB::S.o_off1 + w + 1] > TAB::S.v[TAB::S.o_off1 + w] ? 1 : 0;
                    return c;
                }();
                const bool has_p1 = tab[TAB::S.o_off1 + warp + 1] > tab[TAB::S.o_off1 + warp];
                int* p1cnt = reinterpret_cast<int*>(smem + M.o_bar + 3);
                SG_PF(5,
                for (int j = 0; j <= nplanes; ++j) {
                    const double* Ds = nullptr;
                    if (early) {
                        if (j < nplanes && has_p1) {
                            SG_PF(0, Ds = get_plane(j));
                            SG_PF(1, phase1(Ds, T1s + (j & 1) * T1SZ));
                            __syncwarp();
                            // the last phase-1 warp of plane j refills its buffer with plane j + 2
                            if (lane == 0 && atomicAdd(p1cnt, 1) == NP1W * (j + 1) - 1 && j + 2 < nplanes) issue_plane(j + 2);
                        }
                    } else {
                        SG_PF(0, Ds = j < nplanes ? get_plane(j) : nullptr);
                        SG_PF(1, if (j < nplanes) phase1(Ds, T1s + (j & 1) * T1SZ));
                    }
                    SG_PF(2, if (j >= 1) phase2(T1s + ((j - 1) & 1) * T1SZ, T2s + (long)((j - 1) % NS) * M.T2PS));
                    // before the next interval's phase 2 writes plane j over plane j - NS: the last row
                    // plane reading that plane's layer must be done
                    SG_PF(3, if (tid == 0 && j < nplanes && j >= NS) wait_ge(1, (j - NS) / G + P + 1));
                    SG_PF(4, asm volatile("bar.sync 1, %0;\n" ::"r"(NAW * 32) : "memory"));
                    if (tid == 0 && j >= 1 && j % G == 0) {
                        __threadfence_block();
                        cnt[0] = j / G;
                    }
                })
            } else {
                const int tb0 = NAW * 32;
                if (nsteps > 0) build_b3(0, NAW, NBW);
                SG_PF(5,
                for (int L = 0; L < nsteps; ++L) {
                    SG_PF(0, if (tid == tb0) wait_ge(0, min(L, nlayers - 1) + 1));
                    SG_PF(1, asm volatile("bar.sync 2, %0;\n" ::"r"(NBW * 32) : "memory"));
                    SG_PF(2, phase3(L));
                    SG_PF(3, if (L + 1 < nsteps) build_b3(L + 1, NAW, NBW));
                    SG_PF(4, asm volatile("bar.sync 2, %0;\n" ::"r"(NBW * 32) : "memory"));
                    if (tid == tb0) {
                        __threadfence_block();
                        cnt[1] = L + 1;
                    }
                })
            }
#ifdef SG_K4_PROF
            if (lane == 0 && prm.dmma)
                for (int k = 0; k < 6; ++k) atomicAdd(prm.dmma + 1 + warp * 8 + k, pf[k]);
            if (lane == 0 && prm.dmma && warp == 0) atomicAdd(prm.dmma + 1 + 32 * 8, 1ull);
#endif
#undef SG_PF
        } else {
            // one barrier interval per Gauss plane j: phase 3 (row plane whose last layer completed one
            // interval earlier) | phase 1 (plane j) | phase 2 (plane j-1) | fragments of the next row plane
            const int jend = max(nplanes, (nsteps + 1) * G) + 1;
            for (int j = 0; j <= jend; ++j) {
                const double* Ds = j < nplanes ? get_plane(j) : nullptr;
                if (j >= G + 1 && (j - 1) % G == 0 && (j - 1) / G - 1 < nsteps) phase3((j - 1) / G - 1);
                if (j < nplanes) phase1(Ds, T1s + (j & 1) * T1SZ);
                if (j >= 1 && j <= nplanes) phase2(T1s + ((j - 1) & 1) * T1SZ, T2s + (long)((j - 1) % NS) * M.T2PS);
                if (j % G == 0 && j / G < nsteps) build_b3(j / G, 0, NW);
                __syncthreads();
            }
        }
    }
    if (prm.dmma && lane == 0 && ndmma) atomicAdd(prm.dmma, ndmma);  // all lanes of a warp run the same items
    if constexpr (NDIM == 3) {
        for (int o = 16; o > 0; o >>= 1) nzero += __shfl_xor_sync(0xffffffffu, nzero, o);
        if (prm.zeros && lane == 0 && nzero) atomicAdd(prm.zeros, (unsigned long long)nzero);
    }
}

}  // namespace sg
