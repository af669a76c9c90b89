// Surrogate assembly (reference: surrogate.py:538-691).
//
//   K-classify : quad / interp row classes from the per-direction box and lattice masks (:509-531, :582-586)
//   K4 (rows)  : quadrature rows assembled straight into the final CSR positions (:588)
//   K6         : sample gather (:336-379) + per-direction collocation inverse (:430-471)
//   K7         : fused interpolant evaluation (sum factorised per offset on a tile of box rows),
//                placement (interpolated / symmetric copy / transposed quadrature value, :633-667),
//                row sums for the kernel-preserving diagonal (:673-680) and coalesced CSR writes
//   merge      : exact-zero drop of scipy's CSR add (:670) -- a fast path when no zero exists,
//                else an order-preserving compaction followed by the reference's positional
//                diagonal reset.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "sg_common.cuh"
#include "sg_internal.h"

namespace sg {

struct SurrParams {
    int n, p, P, center, mode;
    int m[3];
    int blo[3], bn[3];
    const uint8_t* inb[3];
    const uint8_t* smp[3];
    int nl[3];
    int qd[3];
    const int* esp[3];
    const double* etab[3];
    const double* coef;  // [P][nl2][nl1][nl0]
    const int* shifts;   // [P][3]
    const int64_t* rowstart;
    int* indices;
    double* data;
    double* newdiag;
    uint8_t* reset;
    unsigned long long* counters;  // 0 interp entries, 1 zeros (interp rows), 2 resets, 3 interp rows, 6 slow rows
    int* slow;                     // interpolated rows with a non-interpolated neighbour (row-staged path)
    int TB[3], tg[3];
    int cmax[3];  // max coefficient rows per direction touched by a (shifted) tile
    int64_t slab_lo, slab_hi;
    int64_t qlo, qhi;  // rows whose quadrature values this call needs (the slab and its p-plane halo)
    int tile0;         // first interpolation tile of the launch (row slabs launch their z range only)
    int dbg;           // timing experiments only (SG_K7_DBG): 1 no value stores, 2 no index stores, 4 no passes
};

__device__ __forceinline__ bool row_interp(const SurrParams& s, int j0, int j1, int j2) {
    bool in = s.inb[0][j0], sm = s.smp[0][j0];
    if (s.n >= 2) { in = in && s.inb[1][j1]; sm = sm && s.smp[1][j1]; }
    if (s.n >= 3) { in = in && s.inb[2][j2]; sm = sm && s.smp[2][j2]; }
    return in && !sm;
}

__global__ void classify_kernel(SurrParams s, int64_t N, uint8_t* quadmask) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const int i0 = (int)(i % s.m[0]), i1 = (int)((i / s.m[0]) % s.m[1]), i2 = (int)(i / ((int64_t)s.m[0] * s.m[1]));
    // quadrature rows of this call: the slab's and its halo's (transposed entries of interpolated rows);
    // lattice rows outside them come from a separate row-restricted assembly or another rank
    const bool quad = !row_interp(s, i0, i1, i2);
    const bool need = i >= s.qlo && i < s.qhi;
    quadmask[i] = quad && need ? 1 : 0;
}

// S[o][lat colex] = A[row(lat), o] for the lattice rows in [lo, hi) (bit-exact gather; lattice rows
// have the full P pattern); the other columns of S are left untouched
__global__ void gather_samples_kernel(const int64_t* __restrict__ rowstart, const double* __restrict__ data,
                                      const int64_t* __restrict__ latrows, int64_t nlat, int P, int64_t lo, int64_t hi,
                                      double* __restrict__ S) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nlat * P) return;
    const int64_t t = k / P;
    const int o = (int)(k % P);
    const int64_t r = latrows[t];
    if (r < lo || r >= hi) return;
    S[(int64_t)o * nlat + t] = data[rowstart[r] + o];
}

// out[..., s, ...] = sum_t Cinv[s][t] in[..., t, ...] along one direction (stride = inner block)
__global__ void apply_dir_kernel(const double* __restrict__ in, double* __restrict__ out, const double* __restrict__ Cinv,
                                 int64_t outer, int len, int64_t inner) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= outer * len * inner) return;
    const int64_t a = k / (len * inner), rem = k % (len * inner);
    const int s = (int)(rem / inner);
    const int64_t b = rem % inner;
    double acc = 0.0;
    for (int t = 0; t < len; ++t) acc = fma(Cinv[(int64_t)s * len + t], in[(a * len + t) * inner + b], acc);
    out[k] = acc;
}

__global__ void const_table_kernel(int n, int* sp, double* tab) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        sp[i] = 0;
        tab[i] = 1.0;
    }
}

// ---------------------------------------------------------------------------------------------
// K7: one CTA per tile of box rows (64 rows).  Warps split the P offsets; a lane owns two rows of
// the tile.  Per offset the warp evaluates the offset's tensor spline on the (possibly shifted)
// tile points by sum factorisation (x, then y, then z taps) from the coefficient tensor, then
// places each lane's entries (interpolated / symmetric copy / transposed quadrature value,
// surrogate.py:633-667), writes them straight into the CSR and keeps per-row partial sums for
// the kernel-preserving diagonal (:673-680).  No row staging: the CTA's rows stay L2 resident
// while their sectors fill.
// ---------------------------------------------------------------------------------------------
template <int NDIM>
__global__ void __launch_bounds__(512, 2) interp_tiles_kernel(SurrParams s) {
    extern __shared__ double sm[];
    constexpr int NR = 64;
    const int P = s.P;
    const int TB0 = s.TB[0], TB1 = NDIM >= 2 ? s.TB[1] : 1, TB2 = NDIM >= 3 ? s.TB[2] : 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int c1 = s.cmax[1], c2 = s.cmax[2];
    const int scr = c2 * c1 * TB0 + c2 * TB1 * TB0 + 8;
    double* A = sm + (size_t)warp * scr;
    double* Bm = A + c2 * c1 * TB0;
    double* red = sm + (size_t)nw * scr;                 // [nw][NR] partial row sums
    double* dgv = red + (size_t)nw * NR;                 // [NR] pre-reset diagonal value
    int* rcnt = reinterpret_cast<int*>(dgv + NR);        // [nw][NR][3]: off-diag interp, interp, zeros
    const int t = blockIdx.x + s.tile0;
    const int tc0 = t % s.tg[0], tc1 = (t / s.tg[0]) % s.tg[1], tc2 = t / (s.tg[0] * s.tg[1]);
    const int org0 = tc0 * TB0, org1 = tc1 * TB1, org2 = tc2 * TB2;
    const int q0 = s.qd[0], q1 = s.qd[1], q2 = s.qd[2];
    // stage the evaluation tables and row-class masks of this tile's +-p neighbourhood in smem
    const int p = s.p;
    const int L0 = TB0 + 2 * p, L1 = NDIM >= 2 ? TB1 + 2 * p : 1, L2 = NDIM >= 3 ? TB2 + 2 * p : 1;
    const int base0 = org0 - p, base1 = NDIM >= 2 ? org1 - p : 0, base2 = NDIM >= 3 ? org2 - p : 0;
    double* tb0 = reinterpret_cast<double*>(rcnt + nw * NR * 3 + 2);
    double* tb1 = tb0 + L0 * (q0 + 1);
    double* tb2 = tb1 + L1 * (q1 + 1);
    int* sp0 = reinterpret_cast<int*>(tb2 + L2 * (q2 + 1));
    int* sp1 = sp0 + L0;
    int* sp2 = sp1 + L1;
    uint8_t* mk0 = reinterpret_cast<uint8_t*>(sp2 + L2);  // bit0 in box, bit1 sampled (index range blo+base..)
    uint8_t* mk1 = mk0 + L0;
    uint8_t* mk2 = mk1 + L1;
    for (int it = threadIdx.x; it < L0 + L1 + L2; it += blockDim.x) {
        int d = 0, li = it;
        if (li >= L0) { li -= L0; d = 1; if (li >= L1) { li -= L1; d = 2; } }
        const int L = d == 0 ? L0 : (d == 1 ? L1 : L2), base = d == 0 ? base0 : (d == 1 ? base1 : base2);
        const int qq = s.qd[d];
        (void)L;
        const int x = min(max(base + li, 0), s.bn[d] - 1);
        int* spd = d == 0 ? sp0 : (d == 1 ? sp1 : sp2);
        double* tbd = d == 0 ? tb0 : (d == 1 ? tb1 : tb2);
        spd[li] = s.esp[d][x];
        for (int r = 0; r <= qq; ++r) tbd[li * (qq + 1) + r] = s.etab[d][x * (qq + 1) + r];
        const int j = s.blo[d] + base + li;  // basis index
        uint8_t mk = 0;
        if (j >= 0 && j < s.m[d]) mk = (uint8_t)(s.inb[d][j] | (s.smp[d][j] << 1));
        (d == 0 ? mk0 : (d == 1 ? mk1 : mk2))[li] = mk;
    }
    __syncthreads();
    auto jint_of = [&](int j0, int j1, int j2) {
        const uint8_t a = mk0[j0 - s.blo[0] - base0];
        const uint8_t b = NDIM >= 2 ? mk1[j1 - s.blo[1] - base1] : (uint8_t)3;
        const uint8_t c = NDIM >= 3 ? mk2[j2 - s.blo[2] - base2] : (uint8_t)3;
        return ((a & b & c) & 1) && !((a & b & c) & 2);
    };

    // the lane's two rows
    int rb0[2], rb1[2], rb2[2], ri0[2], ri1[2], ri2[2];
    int64_t rrow[2], rbase[2];
    bool rint[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int r = lane + 32 * k;
        rb0[k] = r % TB0;
        rb1[k] = (r / TB0) % TB1;
        rb2[k] = r / (TB0 * TB1);
        bool ok = org0 + rb0[k] < s.bn[0] && (NDIM < 2 || org1 + rb1[k] < s.bn[1]) && (NDIM < 3 || org2 + rb2[k] < s.bn[2]);
        ri0[k] = s.blo[0] + org0 + rb0[k];
        ri1[k] = NDIM >= 2 ? s.blo[1] + org1 + rb1[k] : 0;
        ri2[k] = NDIM >= 3 ? s.blo[2] + org2 + rb2[k] : 0;
        ok = ok && row_interp(s, ri0[k], ri1[k], ri2[k]);
        rrow[k] = (int64_t)ri0[k] + (int64_t)s.m[0] * ((int64_t)ri1[k] + (int64_t)s.m[1] * ri2[k]);
        ok = ok && rrow[k] >= s.slab_lo && rrow[k] < s.slab_hi;
        rint[k] = ok;
        rbase[k] = ok ? s.rowstart[rrow[k]] : 0;
    }
    double psum[2] = {0.0, 0.0};
    int poff[2] = {0, 0}, pint[2] = {0, 0}, pzero[2] = {0, 0};

    for (int o = warp; o < P; o += nw) {
        int op = o, sh0 = 0, sh1 = 0, sh2 = 0;
        if (s.mode != SG_GENERAL && o < s.center) {
            op = P - 1 - o;
            sh0 = s.shifts[o * 3 + 0];
            sh1 = s.shifts[o * 3 + 1];
            sh2 = s.shifts[o * 3 + 2];
        }
        const int so0 = s.shifts[o * 3 + 0], so1 = s.shifts[o * 3 + 1], so2 = s.shifts[o * 3 + 2];
        const double* cf = s.coef + (int64_t)op * s.nl[0] * s.nl[1] * s.nl[2];
        int lo1 = 0, lo2 = 0;
        if (NDIM >= 2) lo1 = sp1[min(max(org1 + sh1, 0), s.bn[1] - 1) - base1] - q1;
        if (NDIM >= 3) lo2 = sp2[min(max(org2 + sh2, 0), s.bn[2] - 1) - base2] - q2;
        double V[2];
        if constexpr (NDIM == 1) {
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int x0 = min(max(org0 + rb0[k] + sh0, 0), s.bn[0] - 1);
                const int sp = sp0[x0 - base0];
                double v = 0.0;
                for (int r = 0; r <= q0; ++r) v = fma(tb0[(x0 - base0) * (q0 + 1) + r], cf[sp - q0 + r], v);
                V[k] = v;
            }
        } else {
            // x pass: A[t2][t1][b0]
            for (int it = lane; it < c2 * c1 * TB0; it += 32) {
                const int b0 = it % TB0, tt1 = (it / TB0) % c1, tt2 = it / (TB0 * c1);
                const int x0 = min(max(org0 + b0 + sh0, 0), s.bn[0] - 1);
                const int sp = sp0[x0 - base0];
                const int r1 = min(lo1 + tt1, s.nl[1] - 1), r2 = min(lo2 + tt2, s.nl[2] - 1);
                const double* crow = cf + ((int64_t)r2 * s.nl[1] + r1) * s.nl[0];
                double v = 0.0;
                for (int r = 0; r <= q0; ++r) v = fma(tb0[(x0 - base0) * (q0 + 1) + r], crow[sp - q0 + r], v);
                A[(tt2 * c1 + tt1) * TB0 + b0] = v;
            }
            __syncwarp();
            if constexpr (NDIM == 2) {
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const int x1 = min(max(org1 + rb1[k] + sh1, 0), s.bn[1] - 1);
                    const int sp = sp1[x1 - base1];
                    double v = 0.0;
                    for (int r = 0; r <= q1; ++r) {
                        const int tt1 = sp - q1 + r - lo1;
                        if (tt1 >= 0 && tt1 < c1) v = fma(tb1[(x1 - base1) * (q1 + 1) + r], A[tt1 * TB0 + rb0[k]], v);
                    }
                    V[k] = v;
                }
            } else {
                // y pass: Bm[t2][b1][b0]
                for (int it = lane; it < c2 * TB1 * TB0; it += 32) {
                    const int b0 = it % TB0, b1 = (it / TB0) % TB1, tt2 = it / (TB0 * TB1);
                    const int x1 = min(max(org1 + b1 + sh1, 0), s.bn[1] - 1);
                    const int sp = sp1[x1 - base1];
                    double v = 0.0;
                    for (int r = 0; r <= q1; ++r) {
                        const int tt1 = sp - q1 + r - lo1;
                        if (tt1 >= 0 && tt1 < c1) v = fma(tb1[(x1 - base1) * (q1 + 1) + r], A[(tt2 * c1 + tt1) * TB0 + b0], v);
                    }
                    Bm[(tt2 * TB1 + b1) * TB0 + b0] = v;
                }
                __syncwarp();
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const int x2 = min(max(org2 + rb2[k] + sh2, 0), s.bn[2] - 1);
                    const int sp = sp2[x2 - base2];
                    double v = 0.0;
                    for (int r = 0; r <= q2; ++r) {
                        const int tt2 = sp - q2 + r - lo2;
                        if (tt2 >= 0 && tt2 < c2) v = fma(tb2[(x2 - base2) * (q2 + 1) + r], Bm[(tt2 * TB1 + rb1[k]) * TB0 + rb0[k]], v);
                    }
                    V[k] = v;
                }
            }
            __syncwarp();
        }
        // placement of offset o for the lane's rows
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            if (!rint[k]) continue;
            const int j0 = ri0[k] + so0, j1 = ri1[k] + so1, j2 = ri2[k] + so2;
            const int64_t col = (int64_t)j0 + (int64_t)s.m[0] * ((int64_t)j1 + (int64_t)s.m[1] * j2);
            const bool jint = jint_of(j0, j1, j2);
            const double v = jint ? V[k] : s.data[s.rowstart[col] + (P - 1 - o)];  // transposed quadrature entry A[j, i]
            s.data[rbase[k] + o] = v;
            s.indices[rbase[k] + o] = (int)col;
            psum[k] += v;
            if (jint) {
                pint[k]++;
                if (o != s.center) poff[k]++;
            }
            if (v == 0.0) pzero[k]++;
            if (o == s.center) dgv[lane + 32 * k] = v;
        }
    }
    // per-row reduction over warps (fixed order)
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int r = lane + 32 * k;
        red[warp * NR + r] = psum[k];
        rcnt[(warp * NR + r) * 3 + 0] = poff[k];
        rcnt[(warp * NR + r) * 3 + 1] = pint[k];
        rcnt[(warp * NR + r) * 3 + 2] = pzero[k];
    }
    __syncthreads();
    unsigned long long n_int = 0, n_zero = 0, n_reset = 0, n_rows = 0;
    if (threadIdx.x < NR) {
        const int r = threadIdx.x;
        const int k = r / 32, l = r % 32;
        (void)l;
        const int b0 = r % TB0, b1 = (r / TB0) % TB1, b2 = r / (TB0 * TB1);
        bool ok = org0 + b0 < s.bn[0] && (NDIM < 2 || org1 + b1 < s.bn[1]) && (NDIM < 3 || org2 + b2 < s.bn[2]);
        const int i0 = s.blo[0] + org0 + b0, i1 = NDIM >= 2 ? s.blo[1] + org1 + b1 : 0, i2 = NDIM >= 3 ? s.blo[2] + org2 + b2 : 0;
        ok = ok && row_interp(s, i0, i1, i2);
        const int64_t row = (int64_t)i0 + (int64_t)s.m[0] * ((int64_t)i1 + (int64_t)s.m[1] * i2);
        ok = ok && row >= s.slab_lo && row < s.slab_hi;
        (void)k;
        if (ok) {
            double sum = 0.0;
            int off = 0, in = 0, ze = 0;
            for (int w = 0; w < nw; ++w) {
                sum += red[w * NR + r];
                off += rcnt[(w * NR + r) * 3 + 0];
                in += rcnt[(w * NR + r) * 3 + 1];
                ze += rcnt[(w * NR + r) * 3 + 2];
            }
            n_int += in;
            n_zero += ze;
            n_rows++;
            if (s.mode == SG_SYMMETRIC_KERNEL_PRESERVING && off > 0) {
                s.newdiag[row] = dgv[r] - sum;
                s.reset[row] = 1;
                n_reset++;
            }
        }
    }
    if (threadIdx.x < NR) {
#pragma unroll
        for (int w = 16; w > 0; w >>= 1) {
            n_int += __shfl_xor_sync(0xffffffffu, n_int, w);
            n_zero += __shfl_xor_sync(0xffffffffu, n_zero, w);
            n_reset += __shfl_xor_sync(0xffffffffu, n_reset, w);
            n_rows += __shfl_xor_sync(0xffffffffu, n_rows, w);
        }
        if ((threadIdx.x & 31) == 0) {
            if (n_int) atomicAdd(&s.counters[0], n_int);
            if (n_zero) atomicAdd(&s.counters[1], n_zero);
            if (n_reset) atomicAdd(&s.counters[2], n_reset);
            if (n_rows) atomicAdd(&s.counters[3], n_rows);
        }
    }
}

// ---------------------------------------------------------------------------------------------
// K7 fixed-degree path (interpolation degree 3 in every direction, tile 4x4x4 / 8x8 = 64 rows,
// coefficient window 5 per direction).  Same arithmetic as interp_tiles_kernel (same FMA chains,
// bit-identical values) with the per-tile work hoisted out of the offset loop:
//   * per direction and shift sh in [-p, p]: the tap weights, window-relative tap start and window
//     origin of every tile point (the mirrored offsets of the symmetric modes evaluate at shifted
//     points, surrogate.py:633-651);
//   * per offset: the 5^n coefficient window is loaded once (independent loads), then the x, y, z
//     passes run with compile-time trip counts and no bounds checks.
// ---------------------------------------------------------------------------------------------
template <int NDIM>
__global__ void __launch_bounds__(512, 2) interp_fix_kernel(SurrParams s) {
    static_assert(NDIM == 2 || NDIM == 3, "fixed path: 2D / 3D");
    constexpr int Q = 3, CW = Q + 2, NR = 64, MAXSH = 9;  // p <= 4
    constexpr int TB0 = NDIM == 2 ? 8 : 4, TB1 = NDIM == 2 ? 8 : 4, TB2 = NDIM == 3 ? 4 : 1;
    constexpr int C2 = NDIM == 3 ? CW : 1;
    constexpr int NWIN = C2 * CW * CW, NA = C2 * CW * TB0, NB = NDIM == 3 ? C2 * TB1 * TB0 : 0;
    constexpr int SCR = 128 + NA + NB;
    extern __shared__ double sm[];
    const int P = s.P, p = s.p, NSH = 2 * p + 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    double* Wn = sm + (size_t)warp * SCR;
    double* A = Wn + 128;
    double* Bm = A + NA;
    double* red = sm + (size_t)nw * SCR;                 // [nw][NR] partial row sums
    double* dgv = red + (size_t)nw * NR;                 // [NR] pre-reset diagonal value
    double* TW = dgv + NR;                               // [d][sh][b][Q+1] tap weights
    int* TR = reinterpret_cast<int*>(TW + 3 * MAXSH * 8 * (Q + 1));  // [d][sh][b] window-relative tap start
    int* TL = TR + 3 * MAXSH * 8;                        // [d][sh] window origin (coefficient index)
    int* rcnt = TL + 3 * MAXSH;                          // [nw][NR][3]: off-diag interp, interp, zeros
    uint8_t* mk0 = reinterpret_cast<uint8_t*>(rcnt + nw * NR * 3);
    const int L0 = TB0 + 2 * p, L1 = TB1 + 2 * p, L2 = NDIM == 3 ? TB2 + 2 * p : 1;
    uint8_t* mk1 = mk0 + L0;
    uint8_t* mk2 = mk1 + L1;
    const int t = blockIdx.x + s.tile0;
    const int tc0 = t % s.tg[0], tc1 = (t / s.tg[0]) % s.tg[1], tc2 = t / (s.tg[0] * s.tg[1]);
    const int org[3] = {tc0 * TB0, tc1 * TB1, NDIM == 3 ? tc2 * TB2 : 0};
    const int TBd[3] = {TB0, TB1, TB2};
    const int base0 = org[0] - p, base1 = org[1] - p, base2 = NDIM == 3 ? org[2] - p : 0;
    for (int it = threadIdx.x; it < NDIM * NSH * 8; it += blockDim.x) {
        const int d = it / (NSH * 8), sh = (it / 8) % NSH - p, b = it % 8;
        if (b >= TBd[d]) continue;
        const int x = min(max(org[d] + b + sh, 0), s.bn[d] - 1);
        const int lo = s.esp[d][min(max(org[d] + sh, 0), s.bn[d] - 1)] - Q;
        const int k = (d * MAXSH + sh + p) * 8 + b;
        TR[k] = s.esp[d][x] - Q - lo;
        if (b == 0) TL[d * MAXSH + sh + p] = lo;
#pragma unroll
        for (int r = 0; r <= Q; ++r) TW[k * (Q + 1) + r] = s.etab[d][x * (Q + 1) + r];
    }
    for (int it = threadIdx.x; it < L0 + L1 + L2; it += blockDim.x) {
        int d = 0, li = it;
        if (li >= L0) { li -= L0; d = 1; if (li >= L1) { li -= L1; d = 2; } }
        if (d >= NDIM) continue;
        const int base = d == 0 ? base0 : (d == 1 ? base1 : base2);
        const int j = s.blo[d] + base + li;  // basis index
        uint8_t mk = 0;
        if (j >= 0 && j < s.m[d]) mk = (uint8_t)(s.inb[d][j] | (s.smp[d][j] << 1));
        (d == 0 ? mk0 : (d == 1 ? mk1 : mk2))[li] = mk;
    }
    __syncthreads();
    auto jint_of = [&](int j0, int j1, int j2) {
        const uint8_t a = mk0[j0 - s.blo[0] - base0];
        const uint8_t b = mk1[j1 - s.blo[1] - base1];
        const uint8_t c = NDIM == 3 ? mk2[j2 - s.blo[2] - base2] : (uint8_t)3;
        return ((a & b & c) & 1) && !((a & b & c) & 2);
    };

    // tile rows: CSR start (-1: not an interpolated row of this slab) and basis indices
    int64_t* rbS = reinterpret_cast<int64_t*>((reinterpret_cast<uintptr_t>(mk2 + L2) + 15) & ~(uintptr_t)15);
    int* rI = reinterpret_cast<int*>(rbS + NR);
    double* VB = reinterpret_cast<double*>(rI + 3 * NR) + (size_t)warp * 4 * NR;  // per warp [4][NR] values
    for (int r = threadIdx.x; r < NR; r += blockDim.x) {
        const int b0 = r % TB0, b1 = (r / TB0) % TB1, b2 = r / (TB0 * TB1);
        bool ok = org[0] + b0 < s.bn[0] && org[1] + b1 < s.bn[1] && (NDIM < 3 || org[2] + b2 < s.bn[2]);
        const int i0 = s.blo[0] + org[0] + b0, i1 = s.blo[1] + org[1] + b1, i2 = NDIM == 3 ? s.blo[2] + org[2] + b2 : 0;
        ok = ok && row_interp(s, i0, i1, i2);
        const int64_t row = (int64_t)i0 + (int64_t)s.m[0] * ((int64_t)i1 + (int64_t)s.m[1] * i2);
        ok = ok && row >= s.slab_lo && row < s.slab_hi;
        rbS[r] = ok ? s.rowstart[row] : -1;
        rI[3 * r] = i0;
        rI[3 * r + 1] = i1;
        rI[3 * r + 2] = i2;
    }
    for (int r = lane; r < NR; r += 32) {
        red[warp * NR + r] = 0.0;
        rcnt[(warp * NR + r) * 3 + 0] = rcnt[(warp * NR + r) * 3 + 1] = rcnt[(warp * NR + r) * 3 + 2] = 0;
    }
    __syncthreads();
    // the lane's two rows in the evaluation passes
    int rb0[2], rb1[2], rb2[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int r = lane + 32 * k;
        rb0[k] = r % TB0;
        rb1[k] = (r / TB0) % TB1;
        rb2[k] = r / (TB0 * TB1);
    }
    const int64_t nl01 = (int64_t)s.nl[0] * s.nl[1];

    // offset -> (evaluated offset, evaluation shift): mirrored offsets of the symmetric modes
    auto offset_of = [&](int o, int& op, int& sh0, int& sh1, int& sh2) {
        op = o;
        sh0 = sh1 = sh2 = 0;
        if (s.mode != SG_GENERAL && o < s.center) {
            op = P - 1 - o;
            sh0 = s.shifts[o * 3 + 0];
            sh1 = s.shifts[o * 3 + 1];
            sh2 = s.shifts[o * 3 + 2];
        }
    };
    constexpr int NWL = (NWIN + 31) / 32;  // window elements per lane
    // the lane's share of offset o's coefficient window W[t2][t1][t0] (registers: prefetched one
    // offset ahead so the L2 latency overlaps the current offset's passes)
    auto fetch = [&](int o, double (&w)[NWL]) {
        int op, a0, a1, a2;
        offset_of(o, op, a0, a1, a2);
        const double* cf = s.coef + (int64_t)op * nl01 * s.nl[2];
        const int lo0 = TL[0 * MAXSH + a0 + p], lo1 = TL[1 * MAXSH + a1 + p], lo2 = NDIM == 3 ? TL[2 * MAXSH + a2 + p] : 0;
#pragma unroll
        for (int i = 0; i < NWL; ++i) {
            const int e = i * 32 + lane;
            w[i] = 0.0;
            if (e < NWIN) {
                const int t0 = e % CW, t1 = (e / CW) % CW, t2 = e / (CW * CW);
                const int r0 = min(lo0 + t0, s.nl[0] - 1), r1 = min(lo1 + t1, s.nl[1] - 1);
                const int r2 = NDIM == 3 ? min(lo2 + t2, s.nl[2] - 1) : 0;
                w[i] = __ldg(cf + r2 * nl01 + (int64_t)r1 * s.nl[0] + r0);
            }
        }
    };
    // the warp's offsets: blocks of 4 consecutive offsets (block b = warp, warp + nw, ...), so the
    // placement writes 4 consecutive CSR slots per row (32 B data / 16 B index segments)
    const int nblk = (P + 3) / 4;
    auto next_offset = [&](int o) {  // offset after o in this warp's sequence (or P)
        if ((o & 3) != 3 && o + 1 < P) return o + 1;
        const int nb = (o >> 2) + nw;
        return nb < nblk ? nb * 4 : P;
    };
    double wpre[NWL];
    if (warp < nblk) fetch(warp * 4, wpre);
    for (int blk = warp; blk < nblk; blk += nw) {
        const int ob = blk * 4;
        for (int oo = 0; oo < 4; ++oo) {
            const int o = ob + oo;
            if (o >= P) break;
            int op, sh0, sh1, sh2;
            offset_of(o, op, sh0, sh1, sh2);
            (void)op;
            const int k0 = (0 * MAXSH + sh0 + p), k1 = (1 * MAXSH + sh1 + p), k2 = (2 * MAXSH + sh2 + p);
#pragma unroll
            for (int i = 0; i < NWL; ++i)
                if (i * 32 + lane < NWIN) Wn[i * 32 + lane] = wpre[i];
            {
                const int on = next_offset(o);
                if (on < P) fetch(on, wpre);
            }
            __syncwarp();
            // x pass: A[t2][t1][b0] = sum_r w0[b0][r] W[t2][t1][rel0(b0) + r]  (b0 = lane % TB0 for
            // every item of the lane: its weights and tap start are loaded once per offset)
            {
                const int kb = k0 * 8 + (lane % TB0);
                const double2 wa = *reinterpret_cast<const double2*>(TW + kb * (Q + 1));
                const double2 wb = *reinterpret_cast<const double2*>(TW + kb * (Q + 1) + 2);
                const double* cb = Wn + TR[kb];
#pragma unroll
                for (int i0 = 0; i0 < NA; i0 += 32) {
                    const int it = i0 + lane;
                    if (it < NA) {
                        const double* c = cb + (it / TB0) * CW;  // row t2*CW + t1
                        double v = 0.0;
                        v = fma(wa.x, c[0], v);
                        v = fma(wa.y, c[1], v);
                        v = fma(wb.x, c[2], v);
                        v = fma(wb.y, c[3], v);
                        A[it] = v;
                    }
                }
            }
            __syncwarp();
            if constexpr (NDIM == 2) {
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const int kb = k1 * 8 + rb1[k];
                    const double* w = TW + kb * (Q + 1);
                    const double* c = A + TR[kb] * TB0 + rb0[k];
                    double v = 0.0;
#pragma unroll
                    for (int r = 0; r <= Q; ++r) v = fma(w[r], c[r * TB0], v);
                    VB[oo * NR + lane + 32 * k] = v;
                }
            } else {
                // y pass: Bm[t2][b1][b0] = sum_r w1[b1][r] A[t2][rel1(b1) + r][b0]
                {
                    // b0 = lane % TB0 and b1 = (lane / TB0) % TB1 for every item of the lane (TB0*TB1 = 16 | 32)
                    const int b0 = lane % TB0, b1 = (lane / TB0) % TB1;
                    const int kb = k1 * 8 + b1;
                    const double2 wa = *reinterpret_cast<const double2*>(TW + kb * (Q + 1));
                    const double2 wb = *reinterpret_cast<const double2*>(TW + kb * (Q + 1) + 2);
                    const double* cb = A + TR[kb] * TB0 + b0;
#pragma unroll
                    for (int i0 = 0; i0 < NB; i0 += 32) {
                        const int it = i0 + lane;
                        if (it < NB) {
                            const double* c = cb + (it / (TB0 * TB1)) * CW * TB0;  // t2
                            double v = 0.0;
                            v = fma(wa.x, c[0], v);
                            v = fma(wa.y, c[TB0], v);
                            v = fma(wb.x, c[2 * TB0], v);
                            v = fma(wb.y, c[3 * TB0], v);
                            Bm[it] = v;
                        }
                    }
                }
                __syncwarp();
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const int kb = k2 * 8 + rb2[k];
                    const double* w = TW + kb * (Q + 1);
                    const double* c = Bm + (TR[kb] * TB1 + rb1[k]) * TB0 + rb0[k];
                    double v = 0.0;
#pragma unroll
                    for (int r = 0; r <= Q; ++r) v = fma(w[r], c[r * TB1 * TB0], v);
                    VB[oo * NR + lane + 32 * k] = v;
                }
            }
            __syncwarp();
        }
        // placement of the block: lane -> (row rr*8 + lane/4, offset ob + lane%4)
        const int oo = lane & 3, o = ob + oo;
        const bool ov = o < P;
        const int so0 = ov ? s.shifts[o * 3 + 0] : 0, so1 = ov ? s.shifts[o * 3 + 1] : 0, so2 = ov ? s.shifts[o * 3 + 2] : 0;
#pragma unroll 2
        for (int rr = 0; rr < NR / 8; ++rr) {
            const int r = rr * 8 + (lane >> 2);
            const int64_t rb = rbS[r];
            double v = 0.0;
            int in = 0, off = 0, ze = 0;
            if (rb >= 0 && ov) {
                const int j0 = rI[3 * r] + so0, j1 = rI[3 * r + 1] + so1, j2 = rI[3 * r + 2] + so2;
                const int64_t col = (int64_t)j0 + (int64_t)s.m[0] * ((int64_t)j1 + (int64_t)s.m[1] * j2);
                const bool jint = jint_of(j0, j1, j2);
                v = jint ? VB[oo * NR + r] : s.data[s.rowstart[col] + (P - 1 - o)];  // transposed quadrature entry A[j, i]
                s.data[rb + o] = v;
                s.indices[rb + o] = (int)col;
                in = jint;
                off = jint && o != s.center;
                ze = v == 0.0;
                if (o == s.center) dgv[r] = v;
            }
            // the row's 4 values: ((v0 + v1) + (v2 + v3)) added to this warp's partial row sum
            v += __shfl_xor_sync(0xffffffffu, v, 1);
            v += __shfl_xor_sync(0xffffffffu, v, 2);
            in += __shfl_xor_sync(0xffffffffu, in, 1);
            in += __shfl_xor_sync(0xffffffffu, in, 2);
            off += __shfl_xor_sync(0xffffffffu, off, 1);
            off += __shfl_xor_sync(0xffffffffu, off, 2);
            ze += __shfl_xor_sync(0xffffffffu, ze, 1);
            ze += __shfl_xor_sync(0xffffffffu, ze, 2);
            if (oo == 0 && rb >= 0) {
                red[warp * NR + r] += v;
                rcnt[(warp * NR + r) * 3 + 0] += off;
                rcnt[(warp * NR + r) * 3 + 1] += in;
                rcnt[(warp * NR + r) * 3 + 2] += ze;
            }
        }
        __syncwarp();
    }
    __syncthreads();
    unsigned long long n_int = 0, n_zero = 0, n_reset = 0, n_rows = 0;
    if (threadIdx.x < NR) {
        const int r = threadIdx.x;
        if (rbS[r] >= 0) {
            const int64_t row = (int64_t)rI[3 * r] + (int64_t)s.m[0] * ((int64_t)rI[3 * r + 1] + (int64_t)s.m[1] * rI[3 * r + 2]);
            double sum = 0.0;
            int off = 0, in = 0, ze = 0;
            for (int w = 0; w < nw; ++w) {
                sum += red[w * NR + r];
                off += rcnt[(w * NR + r) * 3 + 0];
                in += rcnt[(w * NR + r) * 3 + 1];
                ze += rcnt[(w * NR + r) * 3 + 2];
            }
            n_int += in;
            n_zero += ze;
            n_rows++;
            if (s.mode == SG_SYMMETRIC_KERNEL_PRESERVING && off > 0) {
                s.newdiag[row] = dgv[r] - sum;
                s.reset[row] = 1;
                n_reset++;
            }
        }
    }
    if (threadIdx.x < NR) {
#pragma unroll
        for (int w = 16; w > 0; w >>= 1) {
            n_int += __shfl_xor_sync(0xffffffffu, n_int, w);
            n_zero += __shfl_xor_sync(0xffffffffu, n_zero, w);
            n_reset += __shfl_xor_sync(0xffffffffu, n_reset, w);
            n_rows += __shfl_xor_sync(0xffffffffu, n_rows, w);
        }
        if ((threadIdx.x & 31) == 0) {
            if (n_int) atomicAdd(&s.counters[0], n_int);
            if (n_zero) atomicAdd(&s.counters[1], n_zero);
            if (n_reset) atomicAdd(&s.counters[2], n_reset);
            if (n_rows) atomicAdd(&s.counters[3], n_rows);
        }
    }
}
// ---------------------------------------------------------------------------------------------
// K7 3D row-staged path (interpolation degree 3, coefficient window 5 per direction, p <= 4).
// One CTA (8 warps) owns a 4 x 8 x 4 tile of box rows (128 rows).  The P offsets are processed in
// chunks of K = (2p+1)^2 consecutive offsets (one z-plane of the stencil, i.e. K consecutive CSR
// slots of every row).  Per chunk:
//   compute : each warp takes a contiguous run of the chunk's offsets; per offset the 5x5x5
//             coefficient window is loaded straight into registers (lane = window row, prefetched
//             one offset ahead), the x pass runs in registers (4 outputs per lane), y and z passes
//             go through a small per-warp scratch (8 and 4 outputs per lane), and the 128 values
//             land in a row-major stage [128][K];
//   write   : a warp per row writes the row's K values and column indices as one contiguous
//             segment (placement: interpolated / symmetric copy / transposed quadrature entry,
//             surrogate.py:633-667), and folds the row's K values into its SKP row sum (:673-680).
// Tap weights are padded to the 5-wide window (one zero tap; adding the +-0 product leaves the
// 4-tap FMA chain's value unchanged); every lane reads the same weights (broadcast loads).
// ---------------------------------------------------------------------------------------------
namespace rows3 {
constexpr int TB0 = 4, TB1 = 4, TB2 = 8, NR = TB0 * TB1 * TB2, CW = 5, MAXSH = 9, NWARP = 8;
constexpr int AS = 6;             // scratch A row stride (doubles): [(t2, t1)][AS] holding b0 = 0..3
constexpr int BS = 6;             // scratch B row stride: [(t2, b1)][BS] holding b0 = 0..3
constexpr int WS = 6;             // lane-specific weight rows [d][sh][b][WS] (5 taps + pad)
constexpr int SCR_SIMT = 25 * AS + 20 * BS + 2;
// tensor-core passes (MMA = true): x out / y in Ax[t1 (8)][SX] holding (t2, b0) = 4 t2 + b0; y out /
// z in Bz[t2 (8)][SZ] holding (b1, b0) = 4 b1 + b0 (row strides chosen so the B-fragment loads of a
// half warp hit distinct banks); rows 5..7 and the padding columns stay zero (finite operands of the
// zero-weight taps)
constexpr int SX = 28, SZ = 20;
constexpr int SCR_MMA = 8 * SX + 8 * SZ;
constexpr int SCR = SCR_SIMT > SCR_MMA ? SCR_SIMT : SCR_MMA;  // per-warp scratch (doubles)
// stage row of tile point (b0, b1, b2): rho = (b1 + 4 b2) + 32 b0 (the z-pass lane is b1 + 4 b2)
}  // namespace rows3

template <int NS, bool MMA>
__global__ void __launch_bounds__(256, 2) interp_rows3_kernel(SurrParams s) {
    using namespace rows3;
    extern __shared__ double sm[];
    constexpr int p = (NS - 1) / 2, K = NS * NS, RPW = NR / NWARP;  // rows per warp (write phase)
    const int P = s.P;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // smem: W5 [3][MAXSH][8][CW] | scratch [NWARP][SCR] | stage [NR][K] | rbS [NR] (int64) |
    //       rowid [NR] | shl [P] | LO [3][MAXSH] | rfast [NR] | masks
    double* W5 = sm;                          // x taps, uniform over lanes: [d][sh][r][b]
    double* WT = W5 + 3 * MAXSH * 8 * CW;     // y / z taps, one row per lane: [d][sh][b][WS]
    double* scr = WT + 3 * MAXSH * 8 * WS;
    double* Aw = scr + (size_t)warp * SCR;
    double* Bw = Aw + 25 * AS;
    double* stage = scr + NWARP * SCR;
    int64_t* rbS = reinterpret_cast<int64_t*>(stage + (size_t)NR * K);
    int* rbr = reinterpret_cast<int*>(rbS + NR);  // CSR start relative to the tile's first row start
    int* rowid = rbr + NR;
    int* shl = rowid + NR;
    int* oinf = shl + P;  // per offset: evaluated offset | evaluation shift (+p) << 16, 20, 24
    int* LO = oinf + P;
    uint8_t* rfast = reinterpret_cast<uint8_t*>(LO + 3 * MAXSH);
    uint8_t* mk0 = rfast + NR;
    constexpr int L0 = TB0 + 2 * p, L1 = TB1 + 2 * p, L2 = TB2 + 2 * p;
    uint8_t* mk1 = mk0 + L0;
    uint8_t* mk2 = mk1 + L1;
    const int t = blockIdx.x + s.tile0;
    const int tc0 = t % s.tg[0], tc1 = (t / s.tg[0]) % s.tg[1], tc2 = t / (s.tg[0] * s.tg[1]);
    const int org[3] = {tc0 * TB0, tc1 * TB1, tc2 * TB2};
    const int TBd[3] = {TB0, TB1, TB2};
    const int base0 = org[0] - p, base1 = org[1] - p, base2 = org[2] - p;
    // padded tap weights W5[d][sh][r][b] (tile point b contiguous) and window origins per
    // (direction, evaluation shift)
    for (int it = threadIdx.x; it < 3 * NS * 8; it += blockDim.x) {
        const int d = it / (NS * 8), sh = (it / 8) % NS - p, b = it % 8;
        double* w = W5 + (d * MAXSH + sh + p) * CW * 8 + b;
        double* wt = WT + ((d * MAXSH + sh + p) * 8 + b) * WS;
        if (b >= TBd[d]) {
#pragma unroll
            for (int r = 0; r < CW; ++r) w[r * 8] = wt[r] = 0.0;
            wt[CW] = 0.0;
            continue;
        }
        const int x = min(max(org[d] + b + sh, 0), s.bn[d] - 1);
        const int lo_ = s.esp[d][min(max(org[d] + sh, 0), s.bn[d] - 1)] - 3;
        // window origin kept inside the coefficient rows when there are >= 5 sites (the shifted taps stay
        // inside the window: points at the last interval then sit at rel = 1)
        const int lo = s.nl[d] >= CW ? min(lo_, s.nl[d] - CW) : lo_;
        const int rel = s.esp[d][x] - 3 - lo;  // 0 or 1 (host checked the 5-wide window)
#pragma unroll
        for (int r = 0; r < CW; ++r) {
            const int tap = r - rel;
            w[r * 8] = wt[r] = (tap >= 0 && tap <= 3) ? s.etab[d][x * 4 + tap] : 0.0;
        }
        wt[CW] = 0.0;
        if (b == 0) LO[d * MAXSH + sh + p] = lo;
    }
    for (int it = threadIdx.x; it < L0 + L1 + L2; it += blockDim.x) {
        int d = 0, li = it;
        if (li >= L0) { li -= L0; d = 1; if (li >= L1) { li -= L1; d = 2; } }
        const int base = d == 0 ? base0 : (d == 1 ? base1 : base2);
        const int j = s.blo[d] + base + li;
        uint8_t mk = 0;
        if (j >= 0 && j < s.m[d]) mk = (uint8_t)(s.inb[d][j] | (s.smp[d][j] << 1));
        (d == 0 ? mk0 : (d == 1 ? mk1 : mk2))[li] = mk;
    }
    // column shift of every offset (colex), in flat row index units
    for (int o = threadIdx.x; o < P; o += blockDim.x) {
        shl[o] = (o % NS - p) + s.m[0] * ((o / NS) % NS - p + s.m[1] * (o / K - p));
        // mirrored offsets of the symmetric modes evaluate offset P-1-o at the shifted point
        const bool mir = s.mode != SG_GENERAL && o < s.center;
        oinf[o] = mir ? ((P - 1 - o) | ((o % NS) << 16) | (((o / NS) % NS) << 20) | ((o / K) << 24)) : (o | (p << 16) | (p << 20) | (p << 24));
    }
    __syncthreads();
    const int64_t tile_row0 = (int64_t)(s.blo[0] + org[0]) + (int64_t)s.m[0] * ((int64_t)(s.blo[1] + org[1]) + (int64_t)s.m[1] * (s.blo[2] + org[2]));
    double* const tdata = s.data + s.rowstart[tile_row0];
    int* const tidx = s.indices + s.rowstart[tile_row0];
    // tile rows: CSR start (-1: not an interpolated row of this slab), flat index, and whether every
    // neighbour within +-p is an interpolated row (then every entry is the evaluated value)
    for (int r = threadIdx.x; r < NR; r += blockDim.x) {
        const int b0 = r / 32, b1 = r % 4, b2 = (r % 32) / 4;
        bool ok = org[0] + b0 < s.bn[0] && org[1] + b1 < s.bn[1] && org[2] + b2 < s.bn[2];
        const int i0 = s.blo[0] + org[0] + b0, i1 = s.blo[1] + org[1] + b1, i2 = s.blo[2] + org[2] + b2;
        ok = ok && row_interp(s, i0, i1, i2);
        const int64_t row = (int64_t)i0 + (int64_t)s.m[0] * ((int64_t)i1 + (int64_t)s.m[1] * i2);
        ok = ok && row >= s.slab_lo && row < s.slab_hi;
        rbS[r] = ok ? s.rowstart[row] : -1;
        rbr[r] = ok ? (int)(s.rowstart[row] - s.rowstart[tile_row0]) : -1;
        rowid[r] = (int)row;
        uint8_t all0 = 1, all1 = 1, all2 = 1, any0 = 0, any1 = 0, any2 = 0;
#pragma unroll
        for (int q = 0; q < NS; ++q) {
            const uint8_t a0 = mk0[b0 + q], a1 = mk1[b1 + q], a2 = mk2[b2 + q];
            all0 &= a0;
            all1 &= a1;
            all2 &= a2;
            any0 |= a0 >> 1;
            any1 |= a1 >> 1;
            any2 |= a2 >> 1;
        }
        rfast[r] = (all0 & all1 & all2 & 1) && !(any0 & any1 & any2 & 1);
    }
    __syncthreads();
    const int kb = (warp * K) / NWARP, ke = ((warp + 1) * K) / NWARP;  // this warp's run of offsets in every chunk
    unsigned n_int = 0, n_zero = 0;
    // write phase: warp owns rows [RPW*warp, RPW*warp + RPW); lane < RPW keeps row RPW*warp+lane's sums
    const int rsl = RPW * warp + (lane < RPW ? lane : 0);
    double rsum = 0.0, dg = 0.0;
    auto write_chunk = [&](const int c) {
        // ---- write the warp's row segments of the chunk: entries flattened over (row, k) so the
        //      lanes stay busy; consecutive lanes write consecutive CSR slots of a row.  The trip
        //      count is a compile-time constant, so unrolled iterations issue their shared loads
        //      together (the loop was bound by shared-load latency)
        constexpr int NE = RPW * K, NIT = (NE + 31) / 32;
#pragma unroll 5
        for (int it = 0; it < NIT; ++it) {
            const int e = it * 32 + lane;
            if (e < NE) {
                const int rl = e / K, k = e - rl * K;
                const int r = RPW * warp + rl;
                const int rb = rbr[r];
                const int o = c * K + k;
                const int col = rowid[r] + shl[o];
                const double v = stage[r * K + k];
                if (rb >= 0) {
                    n_int++;  // provisional for slow rows (corrected by slow_rows_kernel)
                    n_zero += v == 0.0;
                    tdata[rb + o] = v;
                    tidx[rb + o] = col;
                }
            }
        }
        __syncwarp();
        // ---- SKP row sums of the warp's rows (lane = row; ascending offsets in four interleaved
        //      partial sums, joined in a fixed order)
        if (lane < RPW && rbS[rsl] >= 0) {
            const double* sr = stage + (size_t)rsl * K;
            double q0 = 0.0, q1 = 0.0, q2 = 0.0, q3 = 0.0;
#pragma unroll
            for (int k = 0; k + 3 < K; k += 4) {
                q0 += sr[k];
                q1 += sr[k + 1];
                q2 += sr[k + 2];
                q3 += sr[k + 3];
            }
#pragma unroll
            for (int k = K & ~3; k < K; ++k) q0 += sr[k];
            rsum += (q0 + q1) + (q2 + q3);
            if (c == p) dg = sr[(K - 1) / 2];
        }
    };
    if constexpr (!MMA) {
    // window row of this lane (lanes 0..24): t1 = lane % 5, t2 = lane / 5
    const int wt1 = lane % 5, wt2 = lane / 5;
    const int nl0 = s.nl[0], nl01 = s.nl[0] * s.nl[1], nl012 = nl01 * s.nl[2];
    // the lane's window row of offset o (5 coefficients, unclamped: zero-weight taps may read the
    // zeroed tail of the coefficient buffer)
    auto fetch = [&](int o, double (&w)[CW]) {
        if (lane < 25) {
            const int oi = oinf[o];
            const int op = oi & 0xffff, a0 = (oi >> 16) & 15, a1 = (oi >> 20) & 15, a2 = oi >> 24;
            const double* cf = s.coef + (op * nl012 + (LO[2 * MAXSH + a2] + wt2) * nl01 + (LO[MAXSH + a1] + wt1) * nl0 + LO[a0]);
#pragma unroll
            for (int r = 0; r < CW; ++r) w[r] = __ldg(cf + r);
        }
    };
    double wpre[CW] = {0, 0, 0, 0, 0};
    if (kb < ke) fetch(kb, wpre);
    const int yb1 = lane % 4, yt2 = lane / 4;  // y pass lane (lanes 0..19)
    const int zb1 = lane % 4, zb2 = lane / 4;  // z pass lane
    // the lane's y and z tap rows, reloaded only when the evaluation shift changes (z: per chunk)
    double wyr[CW], wzr[CW];
    int cur1 = -1, cur2 = -1;
    for (int c = 0; c < NS; ++c) {
        // ---- compute the chunk's values into the stage
        for (int k = kb; k < ke; ++k) {
            const int o = c * K + k;
            const int oi = oinf[o];
            const int sh0 = (oi >> 16) & 15, sh1 = (oi >> 20) & 15, sh2 = oi >> 24;  // shift + p
            double w[CW];
#pragma unroll
            for (int r = 0; r < CW; ++r) w[r] = wpre[r];
            {
                const int on = (k + 1 < ke) ? o + 1 : ((c + 1 < NS) ? (c + 1) * K + kb : -1);
                if (on >= 0) fetch(on, wpre);
            }
            const double2* wx = reinterpret_cast<const double2*>(W5 + (0 * MAXSH + sh0) * CW * 8);
            if (sh1 != cur1) {
                const double2* q = reinterpret_cast<const double2*>(WT + ((1 * MAXSH + sh1) * 8 + yb1) * WS);
                const double2 u0 = q[0], u1 = q[1], u2 = q[2];
                wyr[0] = u0.x, wyr[1] = u0.y, wyr[2] = u1.x, wyr[3] = u1.y, wyr[4] = u2.x;
                cur1 = sh1;
            }
            if (sh2 != cur2) {
                const double2* q = reinterpret_cast<const double2*>(WT + ((2 * MAXSH + sh2) * 8 + zb2) * WS);
                const double2 u0 = q[0], u1 = q[1], u2 = q[2];
                wzr[0] = u0.x, wzr[1] = u0.y, wzr[2] = u1.x, wzr[3] = u1.y, wzr[4] = u2.x;
                cur2 = sh2;
            }
            // x pass: A[t2][t1][b0] (independent chains over b0, taps ascending)
            if (lane < 25) {
                double a[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                for (int r = 0; r < CW; ++r) {
                    const double2 u0 = wx[r * 4], u1 = wx[r * 4 + 1];
                    a[0] = fma(u0.x, w[r], a[0]);
                    a[1] = fma(u0.y, w[r], a[1]);
                    a[2] = fma(u1.x, w[r], a[2]);
                    a[3] = fma(u1.y, w[r], a[3]);
                }
                *reinterpret_cast<double2*>(Aw + lane * AS) = make_double2(a[0], a[1]);
                *reinterpret_cast<double2*>(Aw + lane * AS + 2) = make_double2(a[2], a[3]);
            }
            __syncwarp();
            // y pass: B[t2][b1][b0] for the lane's (b1, t2), b0 = 0..3 (taps t1 ascending)
            if (lane < 20) {
                double bv[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                for (int r = 0; r < CW; ++r) {
                    const double2* q = reinterpret_cast<const double2*>(Aw + (yt2 * 5 + r) * AS);
                    const double2 u0 = q[0], u1 = q[1];
                    bv[0] = fma(wyr[r], u0.x, bv[0]);
                    bv[1] = fma(wyr[r], u0.y, bv[1]);
                    bv[2] = fma(wyr[r], u1.x, bv[2]);
                    bv[3] = fma(wyr[r], u1.y, bv[3]);
                }
                double* dst = Bw + (yt2 * 4 + yb1) * BS;
                *reinterpret_cast<double2*>(dst) = make_double2(bv[0], bv[1]);
                *reinterpret_cast<double2*>(dst + 2) = make_double2(bv[2], bv[3]);
            }
            __syncwarp();
            // z pass: V[b2][b1][b0] for the lane's (b1, b2), b0 = 0..3 -> stage rows lane + 32 b0
            {
                double v[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                for (int r = 0; r < CW; ++r) {
                    const double2* q = reinterpret_cast<const double2*>(Bw + (r * 4 + zb1) * BS);
                    const double2 u0 = q[0], u1 = q[1];
                    v[0] = fma(wzr[r], u0.x, v[0]);
                    v[1] = fma(wzr[r], u0.y, v[1]);
                    v[2] = fma(wzr[r], u1.x, v[2]);
                    v[3] = fma(wzr[r], u1.y, v[3]);
                }
#pragma unroll
                for (int b = 0; b < 4; ++b) stage[(lane + 32 * b) * K + k] = v[b];
            }
            __syncwarp();
        }
        __syncthreads();
        write_chunk(c);
        __syncthreads();
    }
    } else {
    // ---- tensor-core passes: per offset three m8n8k4 DMMA contractions (x: M = b0, K = t0,
    //      N = (t1, t2); y: M = b1, K = t1, N = (t2, b0); z: M = b2, K = t2, N = (b1, b0)), taps
    //      padded to K = 8 with zero weights: each value is the same ascending FMA chain as the
    //      SIMT passes (a DMMA's K is a sequential FMA chain), so the results are bitwise the same
    const int lr = lane >> 2, lk = lane & 3;
    const int nl0 = s.nl[0], nl01 = s.nl[0] * s.nl[1], nl012 = nl01 * s.nl[2];
    double* Ax = Aw;                 // [t1][SX]
    double* Bz = Aw + 8 * SX;        // [t2][SZ]
    for (int it = lane; it < SCR_MMA; it += 32) Aw[it] = 0.0;
    __syncwarp();
    // B-fragment element offsets of the x pass inside a coefficient window (k-step kt, n-tile j):
    // t0 = 4 kt + lk (clamped into the window: its weight is zero beyond tap 4), n = 8 j + lr -> (t1, t2)
    int xoff[2][4];
#pragma unroll
    for (int kt = 0; kt < 2; ++kt)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int t0 = min(4 * kt + lk, 4), n = min(8 * j + lr, 24);
            xoff[kt][j] = (n / 5) * nl01 + (n % 5) * nl0 + t0;
        }
    auto fetch = [&](int o, double (&b)[2][4]) {
        const int oi = oinf[o];
        const int op = oi & 0xffff, a0 = (oi >> 16) & 15, a1 = (oi >> 20) & 15, a2 = oi >> 24;
        const double* cf = s.coef + (op * nl012 + LO[2 * MAXSH + a2] * nl01 + LO[MAXSH + a1] * nl0 + LO[a0]);
#pragma unroll
        for (int kt = 0; kt < 2; ++kt)
#pragma unroll
            for (int j = 0; j < 4; ++j) b[kt][j] = __ldg(cf + xoff[kt][j]);
    };
    // A fragments of the three directions for an evaluation shift: w[d][b = lr][t = 4 kt + lk]
    auto wfrag = [&](int d, int sh, double (&a)[2]) {
#pragma unroll
        for (int kt = 0; kt < 2; ++kt) {
            const int t = 4 * kt + lk;
            a[kt] = (t < CW && lr < 8) ? W5[((d * MAXSH + sh) * CW + t) * 8 + lr] : 0.0;
        }
    };
    double bpre[2][4];
    if (kb < ke) fetch(kb, bpre);
    double wy[2], wz[2];
    int cur1 = -1, cur2 = -1;
    for (int c = 0; c < NS; ++c) {
        for (int k = kb; k < ke; ++k) {
            const int o = c * K + k;
            const int oi = oinf[o];
            const int sh0 = (oi >> 16) & 15, sh1 = (oi >> 20) & 15, sh2 = oi >> 24;  // shift + p
            double bx[2][4];
#pragma unroll
            for (int kt = 0; kt < 2; ++kt)
#pragma unroll
                for (int j = 0; j < 4; ++j) bx[kt][j] = bpre[kt][j];
            {
                const int on = (k + 1 < ke) ? o + 1 : ((c + 1 < NS) ? (c + 1) * K + kb : -1);
                if (on >= 0) fetch(on, bpre);
            }
            double wx[2];
            wfrag(0, sh0, wx);
            if (sh1 != cur1) {
                wfrag(1, sh1, wy);
                cur1 = sh1;
            }
            if (sh2 != cur2) {
                wfrag(2, sh2, wz);
                cur2 = sh2;
            }
            // x pass -> Ax[t1][4 t2 + b0]
            {
                double acc[4][2];
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll
                for (int kt = 0; kt < 2; ++kt)
#pragma unroll
                    for (int j = 0; j < 4; ++j) dmma(acc[j][0], acc[j][1], wx[kt], bx[kt][j]);
                if (lr < TB0) {
#pragma unroll
                    for (int j = 0; j < 4; ++j)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int n = 8 * j + 2 * lk + h;
                            if (n < 25) Ax[(n % 5) * SX + 4 * (n / 5) + lr] = acc[j][h];
                        }
                }
            }
            __syncwarp();
            // y pass -> Bz[t2][4 b1 + b0]
            {
                double acc[3][2];
#pragma unroll
                for (int j = 0; j < 3; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll
                for (int kt = 0; kt < 2; ++kt)
#pragma unroll
                    for (int j = 0; j < 3; ++j) dmma(acc[j][0], acc[j][1], wy[kt], Ax[(4 * kt + lk) * SX + 8 * j + lr]);
                if (lr < TB1) {
#pragma unroll
                    for (int j = 0; j < 3; ++j)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int n = 8 * j + 2 * lk + h;  // 4 t2 + b0
                            if (n < 20) Bz[(n / 4) * SZ + 4 * lr + (n % 4)] = acc[j][h];
                        }
                }
            }
            __syncwarp();
            // z pass -> stage rows (b1 + 4 b2) + 32 b0
            {
                double acc[2][2];
#pragma unroll
                for (int j = 0; j < 2; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll
                for (int kt = 0; kt < 2; ++kt)
#pragma unroll
                    for (int j = 0; j < 2; ++j) dmma(acc[j][0], acc[j][1], wz[kt], Bz[(4 * kt + lk) * SZ + 8 * j + lr]);
#pragma unroll
                for (int j = 0; j < 2; ++j)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int n = 8 * j + 2 * lk + h, b1 = n / 4, b0 = n % 4;
                        stage[((b1 + 4 * lr) + 32 * b0) * K + k] = acc[j][h];
                    }
            }
            __syncwarp();
        }
        __syncthreads();
        write_chunk(c);
        __syncthreads();
    }
    }
    // ---- SKP diagonal values and counters
    unsigned n_reset = 0, n_rows = 0;
    if (lane < RPW && rbS[rsl] >= 0) {
        n_rows = 1;
        if (s.mode == SG_SYMMETRIC_KERNEL_PRESERVING) s.newdiag[rowid[rsl]] = dg - rsum;
        if (!rfast[rsl]) {
            s.slow[atomicAdd(&s.counters[6], 1ull)] = rowid[rsl];  // finished by slow_rows_kernel
        } else if (s.mode == SG_SYMMETRIC_KERNEL_PRESERVING) {
            // every neighbour is interpolated: the row has interpolated off-diagonal entries
            s.reset[rowid[rsl]] = 1;
            n_reset = 1;
        }
    }
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) {
        n_int += __shfl_xor_sync(0xffffffffu, n_int, m);
        n_zero += __shfl_xor_sync(0xffffffffu, n_zero, m);
        n_reset += __shfl_xor_sync(0xffffffffu, n_reset, m);
        n_rows += __shfl_xor_sync(0xffffffffu, n_rows, m);
    }
    if (lane == 0) {
        if (n_int) atomicAdd(&s.counters[0], n_int);
        if (n_zero) atomicAdd(&s.counters[1], n_zero);
        if (n_reset) atomicAdd(&s.counters[2], n_reset);
        if (n_rows) atomicAdd(&s.counters[3], n_rows);
    }
}
// ---------------------------------------------------------------------------------------------
// K7 3D row-staged path, second form (the default): the tile, chunks and fp64 tensor-core passes of
// interp_rows3_kernel, rebuilt around what bound it (ncu, profiles/r02_interp_rows3_ncu.txt: the
// L1/shared data pipe at 73% of its wavefront peak, half of the shared stores bank-conflict replays;
// compute and CSR writes of a CTA strictly alternating, both CTAs of an SM in step):
//   * no CTA barrier in the loop.  The offsets of the whole tile are dealt to the 8 warps round robin
//     (42 or 43 each).  The stage is a ring of three half-chunks (a chunk = K consecutive CSR slots of
//     every row, written in halves of (K+1)/2 and K/2 slots); a warp that has finished its offsets of
//     half-chunk u announces it on an mbarrier, writes ITS 16 rows of half-chunk u - 1 (values from
//     the stage, column indices from registers) and goes on with half-chunk u + 1 once the ring slot
//     has been released: CSR stores and tensor-core passes of one CTA overlap all the time;
//   * a pass runs its second k-step (taps 4..7) only when the tile straddles two interpolant
//     intervals in that direction at the offset's evaluation shift; otherwise tap 4 has zero weight
//     for every tile point and the step would add exact zeros;
//   * the (t1, t2) columns of the x pass are ordered t1 = lane quad index, t2 = (n-tile, half) and the
//     z-pass operand rows are rotated by one column on odd t2: the x, y and z stores and the y and z
//     fragment loads are bank-conflict free (odd stage row pitch, stage rows ordered so that the 32
//     rows of a z-pass store cover every bank pair twice); the t1 = 4 columns form a fourth n-tile;
//   * SKP row sums and the exact-zero count are accumulated from the z-pass accumulators (no stage
//     reads); the per-offset window address, shifts and flags come from one table built at tile start;
//     rows' CSR starts are 32-bit offsets from the tile's first row, broadcast by shuffles.
// Every value is the same ascending FMA chain over its nonzero taps as before (skipped taps only
// drop +-0 products), and a value depends on (row, offset) alone, so slabs, tiles and mirrored
// entries agree bit for bit.  Tried and dropped (config 5, one B200): bulk async copies
// (cp.async.bulk shared -> global) of 384 B / 192 B row segments sustain one copy per ~35-40 cycles
// per SM whatever their size (3.7 ms); a dedicated writer warp per CTA cannot issue the stores fast
// enough (4.9-5.8 ms); two writer warps cost the compute warps their registers (3.7 ms).
// ---------------------------------------------------------------------------------------------
namespace rows3v2 {
constexpr int TB0 = 4, TB1 = 4, TB2 = 8, NR = TB0 * TB1 * TB2, CW = 5, MAXSH = 9;
constexpr int NCW = 8, NWARP = NCW, NBUF = 3;  // every warp computes and writes; the stage is a ring of three half-chunks
constexpr int SX = 20;                 // Ax[t1 (8)][SX]: column 4 t2 + b0
constexpr int SZ = 20;                 // Bz[t2 (8)][SZ]: column (4 b1 + b0 + (t2 & 1)) mod 16
constexpr int AXN = 8 * SX + 8, BZN = 8 * SZ, SCR = AXN + BZN;
// stage row of tile point (b0, b1, b2)
__host__ __device__ constexpr int srow(int b0, int b1, int b2) {
    return ((b2 >> 1) << 1) + (b0 >> 1) + 8 * ((b2 & 1) + 2 * (b1 & 1) + 4 * (b1 >> 1) + 8 * (b0 & 1));
}
}  // namespace rows3v2

// mbarriers addressed by their 32-bit shared address
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_try(unsigned bar, unsigned parity) {
    unsigned ok;
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok)
                 : "r"(bar), "r"(parity)
                 : "memory");
    return ok != 0;
}
__device__ __noinline__ void mbar_wait_slow(unsigned bar, unsigned parity) {
    unsigned long long spins = 0;
    while (!mbar_try(bar, parity))
        if (++spins > (1ull << 26)) __trap();  // a lost hand-over must fail loudly, not hang the device
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    if (!mbar_try(bar, parity)) mbar_wait_slow(bar, parity);
}

template <int NS>
__global__ void __launch_bounds__(32 * rows3v2::NWARP, 2) interp_rows3v2_kernel(SurrParams s) {
    using namespace rows3v2;
    extern __shared__ double sm[];
    constexpr int p = (NS - 1) / 2, K = NS * NS, PT = K * NS;
    // a chunk (K consecutive CSR slots of every row) leaves in two halves of LA and LB slots
    constexpr int LA = (K + 1) / 2, LB = K / 2, HP = LA, NU = 2 * NS;  // odd row pitch: conflict-free z-pass stores
    static_assert((LA & 1) == 1 && LA <= 64, "odd first half");
    const int P = s.P;  // == PT
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int lr = lane >> 2, lk = lane & 3;
    // smem: W5 [3][MAXSH][CW][8] | scratch [NCW][SCR] | stage [NBUF][NR][HP] | dgv [NR] | rbS [NR] (int64) |
    //       bars [6] | otab [P] (int2) | rowid [NR] | LO [3][MAXSH] | ST [3][MAXSH] | rfast [NR] | masks
    double* W5 = sm;
    double* scr = W5 + 3 * MAXSH * 8 * CW;
    double* stage = scr + NCW * SCR;
    double* dgv = stage + (size_t)NBUF * NR * HP;
    int64_t* rbS = reinterpret_cast<int64_t*>(dgv + NR);
    uint64_t* barp = reinterpret_cast<uint64_t*>(rbS + NR);  // full[NBUF], empty[NBUF]
    const unsigned bars = (unsigned)__cvta_generic_to_shared(barp);
    int2* otab = reinterpret_cast<int2*>(barp + 2 * NBUF);  // per offset: window element offset | shifts (+p) + straddle flags
    int* rowid = reinterpret_cast<int*>(otab + PT);
    int* LO = rowid + NR;
    int* ST = LO + 3 * MAXSH;
    uint8_t* rfast = reinterpret_cast<uint8_t*>(ST + 3 * MAXSH);
    uint8_t* mk0 = rfast + NR;
    constexpr int L0 = TB0 + 2 * p, L1 = TB1 + 2 * p, L2 = TB2 + 2 * p;
    uint8_t* mk1 = mk0 + L0;
    uint8_t* mk2 = mk1 + L1;
    const int t = blockIdx.x + s.tile0;
    const int tc0 = t % s.tg[0], tc1 = (t / s.tg[0]) % s.tg[1], tc2 = t / (s.tg[0] * s.tg[1]);
    const int org0 = tc0 * TB0, org1 = tc1 * TB1, org2 = tc2 * TB2;
    const int nl0 = s.nl[0], nl01 = s.nl[0] * s.nl[1], nl012 = nl01 * s.nl[2];
    const int64_t tile_row0 = (int64_t)(s.blo[0] + org0) + (int64_t)s.m[0] * ((int64_t)(s.blo[1] + org1) + (int64_t)s.m[1] * (s.blo[2] + org2));
    // ---- round 1 of the set-up (independent global loads): window origins and straddle flags, tap
    //      weights, neighbour masks, row starts
    for (int it = threadIdx.x; it < 3 * NS; it += blockDim.x) {
        const int d = it / NS, sh = it % NS - p;
        const int og = d == 0 ? org0 : (d == 1 ? org1 : org2), tb = d == 2 ? TB2 : TB0;
        const int lo_ = s.esp[d][min(max(og + sh, 0), s.bn[d] - 1)] - 3;
        const int lo = s.nl[d] >= CW ? min(lo_, s.nl[d] - CW) : lo_;
        int st = 0;
        for (int b = 0; b < tb; ++b) {
            const int x = min(max(og + b + sh, 0), s.bn[d] - 1);
            st |= (s.esp[d][x] - 3 - lo) != 0;
        }
        LO[d * MAXSH + sh + p] = lo;
        ST[d * MAXSH + sh + p] = st;
    }
    for (int it = threadIdx.x; it < 3 * NS * 8; it += blockDim.x) {
        const int d = it / (NS * 8), sh = (it / 8) % NS - p, b = it % 8;
        const int og = d == 0 ? org0 : (d == 1 ? org1 : org2), tb = d == 2 ? TB2 : TB0;
        double* w = W5 + (d * MAXSH + sh + p) * CW * 8 + b;
        if (b >= tb) {
#pragma unroll
            for (int r = 0; r < CW; ++r) w[r * 8] = 0.0;
            continue;
        }
        const int x = min(max(og + b + sh, 0), s.bn[d] - 1);
        const int lo_ = s.esp[d][min(max(og + sh, 0), s.bn[d] - 1)] - 3;
        const int lo = s.nl[d] >= CW ? min(lo_, s.nl[d] - CW) : lo_;
        const int rel = s.esp[d][x] - 3 - lo;  // 0 or 1 (host checked the 5-wide window)
        double e4[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) e4[q] = s.etab[d][x * 4 + q];
#pragma unroll
        for (int r = 0; r < CW; ++r) {
            const int tap = r - rel;
            w[r * 8] = tap == 0 ? e4[0] : (tap == 1 ? e4[1] : (tap == 2 ? e4[2] : (tap == 3 ? e4[3] : 0.0)));
        }
    }
    for (int it = threadIdx.x; it < L0 + L1 + L2; it += blockDim.x) {
        int d = 0, li = it;
        if (li >= L0) { li -= L0; d = 1; if (li >= L1) { li -= L1; d = 2; } }
        const int base = (d == 0 ? org0 : (d == 1 ? org1 : org2)) - p;
        const int j = s.blo[d] + base + li;
        uint8_t mk = 0;
        if (j >= 0 && j < s.m[d]) mk = (uint8_t)(s.inb[d][j] | (s.smp[d][j] << 1));
        (d == 0 ? mk0 : (d == 1 ? mk1 : mk2))[li] = mk;
    }
    // tile rows (stage order): CSR start (-1: not an interpolated row of this slab) and flat index
    for (int r = threadIdx.x; r < NR; r += blockDim.x) {
        const int b0 = ((r >> 6) & 1) | ((r & 1) << 1), b1 = ((r >> 4) & 1) | (((r >> 5) & 1) << 1);
        const int b2 = ((r >> 3) & 1) | (((r >> 1) & 3) << 1);
        bool ok = org0 + b0 < s.bn[0] && org1 + b1 < s.bn[1] && org2 + b2 < s.bn[2];
        const int i0 = s.blo[0] + org0 + b0, i1 = s.blo[1] + org1 + b1, i2 = s.blo[2] + org2 + b2;
        ok = ok && row_interp(s, i0, i1, i2);
        const int64_t row = (int64_t)i0 + (int64_t)s.m[0] * ((int64_t)i1 + (int64_t)s.m[1] * i2);
        ok = ok && row >= s.slab_lo && row < s.slab_hi;
        rbS[r] = ok ? s.rowstart[row] : -1;
        rowid[r] = (int)row;
    }
    for (int it = lane; it < SCR; it += 32) scr[warp * SCR + it] = 0.0;
    if (threadIdx.x == 0) {
        for (int q = 0; q < 2 * NBUF; ++q) mbar_init(bars + 8 * q, NCW);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    // ---- round 2: per-offset table, fast-row flags
    for (int o = threadIdx.x; o < P; o += blockDim.x) {
        // mirrored offsets of the symmetric modes evaluate offset P-1-o at the shifted point
        const bool mir = s.mode != SG_GENERAL && o < s.center;
        const int a0 = mir ? o % NS : p, a1 = mir ? (o / NS) % NS : p, a2 = mir ? o / K : p;
        const int op = mir ? P - 1 - o : o;
        otab[o] = make_int2(op * nl012 + LO[2 * MAXSH + a2] * nl01 + LO[MAXSH + a1] * nl0 + LO[a0],
                            a0 | (a1 << 4) | (a2 << 8) | (ST[a0] << 12) | (ST[MAXSH + a1] << 13) | (ST[2 * MAXSH + a2] << 14));
    }
    // whether every neighbour within +-p is an interpolated row (then every entry is the evaluated value)
    for (int r = threadIdx.x; r < NR; r += blockDim.x) {
        const int b0 = ((r >> 6) & 1) | ((r & 1) << 1), b1 = ((r >> 4) & 1) | (((r >> 5) & 1) << 1);
        const int b2 = ((r >> 3) & 1) | (((r >> 1) & 3) << 1);
        uint8_t all0 = 1, all1 = 1, all2 = 1, any0 = 0, any1 = 0, any2 = 0;
#pragma unroll
        for (int q = 0; q < NS; ++q) {
            const uint8_t a0 = mk0[b0 + q], a1 = mk1[b1 + q], a2 = mk2[b2 + q];
            all0 &= a0;
            all1 &= a1;
            all2 &= a2;
            any0 |= a0 >> 1;
            any1 |= a1 >> 1;
            any2 |= a2 >> 1;
        }
        rfast[r] = (all0 & all1 & all2 & 1) && !(any0 & any1 & any2 & 1);
    }
    __syncthreads();
    double rs[4] = {0.0, 0.0, 0.0, 0.0};
    int sb[4] = {0, 0, 0, 0};
    unsigned n_zero = 0;
    {
        // ================= every warp: offsets g = warp, warp + NCW, ... of the whole tile; after its offsets of
        // half-chunk u (= 2 c + h, stage buffer u mod NBUF) it writes its 16 rows of half-chunk u - 1
        double* Ax = scr + (size_t)warp * SCR;
        double* Bz = Ax + AXN;
        // the lane's four stage rows (z-pass accumulators acc[j][h]): b2 = lr, b1 = 2j + (lk >> 1), b0 = 2 (lk & 1) + h
        unsigned vmask = 0;  // valid rows
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int j = i >> 1, h = i & 1;
            const int r = srow(2 * (lk & 1) + h, 2 * j + (lk >> 1), lr);
            const int64_t rb = rbS[r];
            sb[i] = r * HP;  // stage offset of the row
            vmask |= (rb >= 0 ? 1u : 0u) << i;
        }
        // B-fragment element offsets of the x pass inside a coefficient window: n-tiles 0..2 hold
        // (t1 = lr >> 1, t2 = 2 j + (lr & 1)), n-tile 3 holds (t1 = 4, t2 = lr); k = t0 = 4 kt + lk (clamped
        // into the window: the weight is zero beyond tap 4, and columns past t2 = 4 are never stored)
        int xoff[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int t1 = j < 3 ? (lr >> 1) : 4, t2 = j < 3 ? min(2 * j + (lr & 1), 4) : min(lr, 4);
            xoff[j] = t2 * nl01 + t1 * nl0 + lk;
        }
        const int x1 = 4 - lk;  // k-step 1: t0 = 4 (lanes lk > 0 re-read tap 4 with zero weight)
        auto fetch = [&](int g, double (&b)[2][4]) {
            const int2 ot = otab[g];
            const double* cf = s.coef + ot.x;
            const bool s1 = ot.y & (1 << 13);  // the t1 = 4 columns are only read when the tile straddles in y
#pragma unroll
            for (int j = 0; j < 3; ++j) b[0][j] = __ldg(cf + xoff[j]);
            if (s1) b[0][3] = __ldg(cf + xoff[3]);
            if (ot.y & (1 << 12)) {
#pragma unroll
                for (int j = 0; j < 3; ++j) b[1][j] = __ldg(cf + xoff[j] + x1);
                if (s1) b[1][3] = __ldg(cf + xoff[3] + x1);
            }
        };
        // A fragment of direction d at evaluation shift sh: w[b = lr][t = 4 kt + lk]
        auto wfrag = [&](int d, int sh, double (&a)[2]) {
            a[0] = W5[((d * MAXSH + sh) * CW + lk) * 8 + lr];
            a[1] = lk == 0 ? W5[((d * MAXSH + sh) * CW + 4) * 8 + lr] : 0.0;
        };
        // ---- write share: the rows [16 warp, 16 warp + 16) (stage order) of a finished half-chunk
        constexpr int RW = NR / NCW, NKL = (LA + 31) / 32;
        int colk[2][NKL];  // per-lane column constants of the slots k = h LA + lane + 32 qq
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int qq = 0; qq < NKL; ++qq) {
                const int k = min(h * LA + lane + 32 * qq, K - 1);
                colk[h][qq] = (k % NS - p) + s.m[0] * ((k / NS) % NS - p);
            }
        const int m01 = s.m[0] * s.m[1];
        // CSR starts relative to the tile's first row (a tile spans 8 row planes: < 2^31 slots)
        const int64_t trs = s.rowstart[tile_row0];
        const int64_t rbl64 = rbS[RW * warp + (lane & (RW - 1))];
        const int rbl = rbl64 >= 0 ? (int)(rbl64 - trs) : -1;
        const int ridl = rowid[RW * warp + (lane & (RW - 1))];
        auto write_share = [&](const int v) {
            const int c = v >> 1, h = v & 1, G = c * K + h * LA, L = h ? LB : LA;
            const double* sbuf = stage + (size_t)(v % NBUF) * NR * HP + (size_t)RW * warp * HP;
            mbar_wait(bars + 8 * (v % NBUF), (v / NBUF) & 1);
            // a row per step: its L values (stage -> CSR) and column indices, a lane per slot; the row's CSR
            // start and id are broadcast from the lanes' registers (no shared loads in the address chain)
#pragma unroll
            for (int qq = 0; qq < NKL; ++qq) {
                const int k = lane + 32 * qq;
                const bool act = k < L;
                const bool wv = act && !(s.dbg & 1), wi = act && !(s.dbg & 2);
                const int cs = (c - p) * m01 + colk[h][qq];
                double* db = s.data + trs + G + k;
                int* ib = s.indices + trs + G + k;
                const double* sk = sbuf + (act ? k : 0);
#pragma unroll
                for (int j = 0; j < RW; ++j) {
                    const int rb = __shfl_sync(0xffffffffu, rbl, j);
                    const int rid = __shfl_sync(0xffffffffu, ridl, j);
                    const double val = sk[j * HP];
                    if (rb >= 0 && wv) db[rb] = val;
                    if (rb >= 0 && wi) ib[rb] = rid + cs;
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(bars + 8 * (NBUF + v % NBUF));
        };
        double wx[2], wy[2], wz[2];
        int cur0 = -1, cur1 = -1, cur2 = -1;
        int u = 0, gend = LA;   // current half-chunk and the end of its offsets
        double* sp[4];          // sp[i][g]: stage slot of offset g in the lane's row i
#pragma unroll
        for (int i = 0; i < 4; ++i) sp[i] = stage + sb[i];
        // one offset: passes x, y, z on the tensor cores; bx holds its x-pass B fragments, bn receives
        // the next offset's
        auto step = [&](const int g, double (&bx)[2][4], double (&bn)[2][4]) {
            while (g >= gend) {
                // this warp's offsets of half-chunk u are done: announce it, write the warp's rows of half-chunk
                // u - 1, move to the next buffer (last used by half-chunk u + 1 - NBUF)
                __syncwarp();
                if (lane == 0) mbar_arrive(bars + 8 * (u % NBUF));
                if (u >= 1) write_share(u - 1);
                ++u;
                const int c = u >> 1, h = u & 1, G = c * K + h * LA;
                gend = G + (h ? LB : LA);
                if (u >= NBUF) mbar_wait(bars + 8 * (NBUF + u % NBUF), (u / NBUF - 1) & 1);
#pragma unroll
                for (int i = 0; i < 4; ++i) sp[i] = stage + (size_t)(u % NBUF) * NR * HP + sb[i] - G;
            }
            const int fl = otab[g].y;
            const int sh0 = fl & 15, sh1 = (fl >> 4) & 15, sh2 = (fl >> 8) & 15;  // shift + p
            if (g + NCW < PT) fetch(g + NCW, bn);
            if (sh0 != cur0) {
                wfrag(0, sh0, wx);
                cur0 = sh0;
            }
            if (sh1 != cur1) {
                wfrag(1, sh1, wy);
                cur1 = sh1;
            }
            if (sh2 != cur2) {
                wfrag(2, sh2, wz);
                cur2 = sh2;
            }
            // x pass -> Ax[t1][4 t2 + b0]
            {
                double acc[4][2];
                const bool s1 = fl & (1 << 13);
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    acc[j][0] = acc[j][1] = 0.0;
                    dmma(acc[j][0], acc[j][1], wx[0], bx[0][j]);
                }
                acc[3][0] = acc[3][1] = 0.0;
                if (s1) dmma(acc[3][0], acc[3][1], wx[0], bx[0][3]);
                if (fl & (1 << 12)) {
#pragma unroll
                    for (int j = 0; j < 3; ++j) dmma(acc[j][0], acc[j][1], wx[1], bx[1][j]);
                    if (s1) dmma(acc[3][0], acc[3][1], wx[1], bx[1][3]);
                }
                if (lr < TB0) {
#pragma unroll
                    for (int j = 0; j < 3; ++j)
#pragma unroll
                        for (int h = 0; h < 2; ++h)
                            if (2 * j + h < CW) Ax[lk * SX + 4 * (2 * j + h) + lr] = acc[j][h];
                    if (s1) {
#pragma unroll
                        for (int h = 0; h < 2; ++h)
                            if (2 * lk + h < CW) Ax[4 * SX + 4 * (2 * lk + h) + lr] = acc[3][h];
                    }
                }
            }
            __syncwarp();
            // y pass -> Bz[t2][(4 b1 + b0 + (t2 & 1)) mod 16]
            {
                double acc[3][2];
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    acc[j][0] = acc[j][1] = 0.0;
                    dmma(acc[j][0], acc[j][1], wy[0], Ax[lk * SX + 8 * j + lr]);
                }
                if (fl & (1 << 13)) {
#pragma unroll
                    for (int j = 0; j < 3; ++j) dmma(acc[j][0], acc[j][1], wy[1], Ax[(4 + lk) * SX + 8 * j + lr]);
                }
                if (lr < TB1) {
#pragma unroll
                    for (int j = 0; j < 3; ++j)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int t2 = 2 * j + (lk >> 1), b0 = 2 * (lk & 1) + h;
                            if (t2 < CW) Bz[t2 * SZ + ((4 * lr + b0 + (t2 & 1)) & 15)] = acc[j][h];
                        }
                }
            }
            __syncwarp();
            // z pass -> stage
            {
                double acc[2][2];
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    acc[j][0] = acc[j][1] = 0.0;
                    dmma(acc[j][0], acc[j][1], wz[0], Bz[lk * SZ + ((8 * j + lr + (lk & 1)) & 15)]);
                }
                if (fl & (1 << 14)) {
#pragma unroll
                    for (int j = 0; j < 2; ++j) dmma(acc[j][0], acc[j][1], wz[1], Bz[(4 + lk) * SZ + ((8 * j + lr + (lk & 1)) & 15)]);
                }
                bool anyz = false;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const double v = acc[i >> 1][i & 1];
                    sp[i][g] = v;
                    rs[i] += v;
                    anyz = anyz || v == 0.0;
                }
                if (anyz) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) n_zero += (acc[i >> 1][i & 1] == 0.0) & ((vmask >> i) & 1);
                }
                if (g == (PT - 1) / 2) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) dgv[sb[i] / HP] = acc[i >> 1][i & 1];
                }
            }
            __syncwarp();
        };
        if (!(s.dbg & 4)) {
            double bA[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}}, bB[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
            fetch(warp, bA);
            int g = warp;
            for (; g + NCW < PT; g += 2 * NCW) {
                step(g, bA, bB);
                step(g + NCW, bB, bA);
            }
            if (g < PT) step(g, bA, bB);
        }
        // the remaining half-chunks (the warp's offsets end before the last ones), then the last two writes
        for (;;) {
            __syncwarp();
            if (lane == 0) mbar_arrive(bars + 8 * (u % NBUF));
            if (u >= 1) write_share(u - 1);
            if (++u >= NU) break;
            if (u >= NBUF) mbar_wait(bars + 8 * (NBUF + u % NBUF), (u / NBUF - 1) & 1);
        }
        write_share(NU - 1);
    }
    __syncthreads();
    // ---- SKP row sums: the compute warps' partial sums joined in warp order (aliases the stage; the
    //      last half-chunk has been written)
    double* part = stage;  // [NCW][NR]
#pragma unroll
    for (int i = 0; i < 4; ++i) part[warp * NR + sb[i] / HP] = rs[i];
    __syncthreads();
    unsigned n_reset = 0, n_rows = 0;
    if (threadIdx.x < NR) {
        const int r = threadIdx.x;
        if (rbS[r] >= 0) {
            double rsum = 0.0;
#pragma unroll
            for (int w = 0; w < NCW; ++w) rsum += part[w * NR + r];
            n_rows = 1;
            if (s.mode == SG_SYMMETRIC_KERNEL_PRESERVING) s.newdiag[rowid[r]] = dgv[r] - rsum;
            if (!rfast[r]) {
                s.slow[atomicAdd(&s.counters[6], 1ull)] = rowid[r];  // finished by slow_rows_kernel
            } else if (s.mode == SG_SYMMETRIC_KERNEL_PRESERVING) {
                // every neighbour is interpolated: the row has interpolated off-diagonal entries
                s.reset[rowid[r]] = 1;
                n_reset = 1;
            }
        }
    }
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) {
        n_zero += __shfl_xor_sync(0xffffffffu, n_zero, m);
        n_reset += __shfl_xor_sync(0xffffffffu, n_reset, m);
        n_rows += __shfl_xor_sync(0xffffffffu, n_rows, m);
    }
    if (lane == 0) {
        if (n_rows) atomicAdd(&s.counters[0], (unsigned long long)n_rows * P);  // provisional for slow rows
        if (n_zero) atomicAdd(&s.counters[1], n_zero);
        if (n_reset) atomicAdd(&s.counters[2], n_reset);
        if (n_rows) atomicAdd(&s.counters[3], n_rows);
    }
}
// Rows of the row-staged path with a non-interpolated neighbour (box boundary band, neighbours of
// fully sampled rows).  interp_rows3_kernel wrote the interpolant into every slot of these rows,
// counted every slot as interpolated and stored the provisional SKP diagonal (centre - row sum);
// here the non-interpolated slots get the transposed quadrature entry A[j, i] (surrogate.py:633-667)
// and the counts, the row sum and the reset flag (:673-680) are corrected.  One warp per row; the row's neighbour classes
// come from per-direction bit masks (no per-entry mask loads).
template <int NS>
__global__ void __launch_bounds__(256) slow_rows_kernel(SurrParams s) {
    constexpr int p = (NS - 1) / 2, K = NS * NS, P = K * NS;
    const int lane = threadIdx.x & 31;
    const int64_t nslow = (int64_t)s.counters[6];
    int n_int = 0, n_zero = 0, n_reset = 0;
    for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nslow; w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t row = s.slow[w];
        const int i0 = (int)(row % s.m[0]), i1 = (int)((row / s.m[0]) % s.m[1]), i2 = (int)(row / ((int64_t)s.m[0] * s.m[1]));
        // bit q of ib_d / sm_d: neighbour index i_d + q - p in the box / sampled
        unsigned ib[3], sm[3];
        {
            const int id[3] = {i0, i1, i2};
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                const int j = id[d] + lane - p;
                const bool ok = lane < NS;
                ib[d] = __ballot_sync(0xffffffffu, ok && s.inb[d][j]);
                sm[d] = __ballot_sync(0xffffffffu, ok && s.smp[d][j]);
            }
        }
        const int64_t rb = s.rowstart[row];
        double corr = 0.0;
        int nq = 0;
        // loads through a separate no-alias view: the gathered quadrature rows are never written here
        // and every slot of this row is read before it is written, so the loads of later iterations
        // may be issued ahead of earlier stores (the gathers are DRAM-latency bound)
        const double* __restrict__ dsrc = s.data;
        double* __restrict__ ddst = s.data;
#pragma unroll 4
        for (int k = lane; k < P; k += 32) {
            const int q0 = k % NS, q1 = (k / NS) % NS, q2 = k / K;
            const unsigned a = (ib[0] >> q0) & (ib[1] >> q1) & (ib[2] >> q2) & 1u;
            const unsigned b = (sm[0] >> q0) & (sm[1] >> q1) & (sm[2] >> q2) & 1u;
            if (a && !b) continue;  // interpolated neighbour: the slot is final
            const int64_t col = row + (q0 - p) + (int64_t)s.m[0] * ((q1 - p) + (int64_t)s.m[1] * (q2 - p));
            const double old = dsrc[rb + k];
            const double v = dsrc[__ldg(s.rowstart + col) + (P - 1 - k)];  // transposed quadrature entry A[j, i]
            ddst[rb + k] = v;
            corr += v - old;
            nq++;
            n_zero += (v == 0.0) - (old == 0.0);
        }
#pragma unroll
        for (int m = 16; m > 0; m >>= 1) {
            corr += __shfl_xor_sync(0xffffffffu, corr, m);
            nq += __shfl_xor_sync(0xffffffffu, nq, m);
        }
        n_int -= nq;
        if (lane == 0 && s.mode == SG_SYMMETRIC_KERNEL_PRESERVING && nq < P - 1) {
            s.newdiag[row] -= corr;  // centre - row sum with the transposed entries
            s.reset[row] = 1;
            n_reset++;
        }
    }
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) n_zero += __shfl_xor_sync(0xffffffffu, n_zero, m);
    if (lane == 0) {
        // two's-complement adds: the corrections of the counts may be negative
        if (n_int) atomicAdd(&s.counters[0], (unsigned long long)(long long)n_int);
        if (n_zero) atomicAdd(&s.counters[1], (unsigned long long)(long long)n_zero);
        if (n_reset) atomicAdd(&s.counters[2], (unsigned long long)n_reset);
    }
}

static size_t interp_rows3_smem(int p) {
    using namespace rows3;
    const int NS = 2 * p + 1, K = NS * NS, P = K * NS;
    return sizeof(double) * (3 * MAXSH * 8 * CW + 3 * MAXSH * 8 * WS + NWARP * SCR + (size_t)NR * K) + sizeof(int64_t) * NR +
           sizeof(int) * (2 * NR + 2 * P + 3 * MAXSH) + 2 * NR + 3 * (8 + 2 * p) + 16;
}

static size_t interp_rows3v2_smem(int p) {
    using namespace rows3v2;
    const int NS = 2 * p + 1, K = NS * NS, P = K * NS, HP = (K + 1) / 2;
    return sizeof(double) * (3 * MAXSH * 8 * CW + NCW * SCR + (size_t)NBUF * NR * HP + NR) + sizeof(int64_t) * (NR + 2 * NBUF) +
           sizeof(int) * (2 * P + NR + 6 * MAXSH) + NR + 3 * (8 + 2 * p) + 16;
}
static size_t interp_fix_smem(int n, int p) {
    const int Q = 3, CW = 5, NR = 64, MAXSH = 9, nw = 16;
    const int TB0 = n == 2 ? 8 : 4, TB1 = n == 2 ? 8 : 4, TB2 = n == 3 ? 4 : 1;
    const int C2 = n == 3 ? CW : 1;
    const int SCR = 128 + C2 * CW * TB0 + (n == 3 ? C2 * TB1 * TB0 : 0);
    const int L = (TB0 + 2 * p) + (TB1 + 2 * p) + (n == 3 ? TB2 + 2 * p : 1);
    return sizeof(double) * ((size_t)nw * SCR + (size_t)nw * NR + NR + 3 * MAXSH * 8 * (Q + 1)) +
           sizeof(int) * (3 * MAXSH * 8 + 3 * MAXSH + (size_t)nw * NR * 3) + L + 16 +
           sizeof(int64_t) * NR + sizeof(int) * 3 * NR + sizeof(double) * (size_t)nw * 4 * NR;
}

__global__ void skp_apply_kernel(const uint8_t* __restrict__ reset, const double* __restrict__ newdiag,
                                 const int64_t* __restrict__ rowstart, int center, int64_t lo, int64_t hi, double* data) {
    int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= hi) return;
    if (reset[i]) data[rowstart[i] + center] = newdiag[i];
}

// --- slow path: exact zeros present -> order-preserving compaction (scipy csr add) ---
__global__ void nz_count_kernel(const int64_t* __restrict__ rowstart, const double* __restrict__ data, int64_t lo,
                                int64_t hi, int64_t* __restrict__ cnt) {
    int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > hi) return;
    if (i == hi) { cnt[i - lo] = 0; return; }
    int64_t c = 0;
    for (int64_t k = rowstart[i]; k < rowstart[i + 1]; ++k) c += (data[k] != 0.0);
    cnt[i - lo] = c;
}

__global__ void compact_kernel(const int64_t* __restrict__ rowstart, const double* __restrict__ data,
                               const int* __restrict__ indices, int64_t lo, int64_t hi, const int64_t* __restrict__ newptr,
                               double* __restrict__ ndata, int* __restrict__ nind) {
    int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= hi) return;
    int64_t w = newptr[i - lo];
    for (int64_t k = rowstart[i]; k < rowstart[i + 1]; ++k)
        if (data[k] != 0.0) {
            ndata[w] = data[k];
            nind[w] = indices[k];
            ++w;
        }
}

// surrogate.py:673-680 on the compacted matrix: window of P entries from the row start, pre-reset values
__global__ void skp_positional_kernel(const uint8_t* __restrict__ reset, const int64_t* __restrict__ newptr, int64_t lo,
                                      int64_t hi, int P, int center, int64_t nnz, const double* __restrict__ ndata,
                                      double* __restrict__ newval, int* __restrict__ bad) {
    int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= hi || !reset[i]) return;
    const int64_t st = newptr[i - lo];
    if (st + P > nnz) { *bad = 1; return; }
    double tot = 0.0;
    for (int k = 0; k < P; ++k) tot += ndata[st + k];
    newval[i - lo] = ndata[st + center] - tot;
}

__global__ void skp_positional_apply(const uint8_t* __restrict__ reset, const int64_t* __restrict__ newptr, int64_t lo,
                                     int64_t hi, int center, const double* __restrict__ newval, double* __restrict__ ndata) {
    int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= hi || !reset[i]) return;
    ndata[newptr[i - lo] + center] = newval[i - lo];
}

static inline unsigned nblk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

}  // namespace sg

using namespace sg;


// ==========================================================================================
// Surrogate call in two phases (strategy B for row slabs):
//   begin  : masks, analytic pattern, quadrature rows of the slab and its p-plane halo (K4) into
//            work arrays sized for exactly those rows, samples of the lattice rows inside the slab;
//   [the caller fills the other lattice rows' samples: another rank's all-gather, or the
//    single-call path's row-restricted assembly of the foreign lattice rows]
//   finish : collocation solves (K6), interpolation (K7), merge / zero drop, SKP diagonal.
// ==========================================================================================
struct sg_surrogate_state {
    Call c;
    DevProblem dp;
    SurrParams s;
    int n = 0, p = 0, P = 0, center = 0;
    int64_t N = 0, slab_lo = 0, slab_hi = 0, nnz_lo = 0, nnz_hi = 0, nnz_all = 0, nnz_qlo = 0, nnz_qhi = 0;
    int64_t nlat_tot = 1;
    std::vector<int64_t> latrows;
    int64_t* dlat = nullptr;
    int64_t* rowstart = nullptr;
    int* indices = nullptr;  // allocation: entries of rows [qlo, qhi)
    double* data = nullptr;
    uint8_t* reset = nullptr;
    double* newdiag = nullptr;
    unsigned long long* counters = nullptr;
    double* bufA = nullptr;
    double* bufB = nullptr;
    int64_t cpad = 0;
    const double* d_ci[3] = {nullptr, nullptr, nullptr};  // inverse collocation matrices (device)
    const double* d_kn[3] = {nullptr, nullptr, nullptr};  // averaged knots
    const double* d_bp[3] = {nullptr, nullptr, nullptr};  // in-box midpoints
    explicit sg_surrogate_state(const sg_exec* ex) : c(ex) {}
};

static int surr_begin(sg_surrogate_state& S, const sg_problem* prob, const sg_surrogate_params* sp, const sg_exec* ex) {
    Call& c = S.c;
    DevProblem& dp = S.dp;
    int rc = prepare_problem(c, prob, dp);
    if (rc) return rc;
    const int n = dp.n, p = dp.p;
    int P = 1;
    for (int d = 0; d < n; ++d) P *= 2 * p + 1;
    const int center = (P - 1) / 2;
    if (sp->mode < 0 || sp->mode > 2) return fail(-1, "unknown surrogate mode %d", sp->mode);
    const int64_t N = dp.N;
    int64_t slab_lo = 0, slab_hi = N;
    if (ex && ex->slab_hi > 0) {
        slab_lo = std::max<int64_t>(0, ex->slab_lo);
        slab_hi = std::min<int64_t>(N, ex->slab_hi);
        if (slab_lo >= slab_hi) return fail(-1, "empty row slab");
    }
    S.n = n;
    S.p = p;
    S.P = P;
    S.center = center;
    S.N = N;
    S.slab_lo = slab_lo;
    S.slab_hi = slab_hi;
    SurrParams& s = S.s;
    memset(&s, 0, sizeof(s));
    s.n = n;
    s.p = p;
    s.P = P;
    s.center = center;
    s.mode = sp->mode;
    s.slab_lo = slab_lo;
    s.slab_hi = slab_hi;
    {
        const int64_t halo0 = (int64_t)p * (1 + dp.m[0] + (int64_t)dp.m[0] * dp.m[1]);
        s.qlo = std::max<int64_t>(0, slab_lo - halo0);
        s.qhi = std::min<int64_t>(N, slab_hi + halo0);
    }
    s.tile0 = 0;
    // per-direction masks (surrogate.py:509-531)
    std::vector<std::vector<uint8_t>> inb(3), smp(3);
    for (int d = 0; d < 3; ++d) {
        s.m[d] = dp.m[d];
        if (d < n) {
            s.blo[d] = 2 * p;
            s.bn[d] = dp.m[d] - 4 * p;
            if (s.bn[d] <= 0) return fail(-1, "interior sampling box is empty; no lattice exists");
            inb[d].assign(dp.m[d], 0);
            smp[d].assign(dp.m[d], 0);
            for (int k = s.blo[d]; k < s.blo[d] + s.bn[d]; ++k) inb[d][k] = 1;
            s.nl[d] = sp->nlat[d];
            for (int k = 0; k < sp->nlat[d]; ++k) {
                const int64_t li = sp->lat_idx[d][k];
                if (li < s.blo[d] || li >= s.blo[d] + s.bn[d]) return fail(-1, "lattice index outside the box");
                smp[d][li] = 1;
            }
            s.qd[d] = sp->qd[d];
        } else {
            s.blo[d] = 0;
            s.bn[d] = 1;
            inb[d].assign(1, 1);
            smp[d].assign(1, 1);
            s.nl[d] = 1;
            s.qd[d] = 0;
        }
        S.nlat_tot *= s.nl[d];
    }
    // offsets [-p,p]^n colex (surrogate.py:103-122)
    std::vector<int> shifts(P * 3, 0);
    for (int o = 0; o < P; ++o) {
        int r = o;
        for (int d = 0; d < n; ++d) {
            shifts[o * 3 + d] = r % (2 * p + 1) - p;
            r /= 2 * p + 1;
        }
    }
    // lattice rows (colex over the lattice)
    S.latrows.resize(S.nlat_tot);
    for (int64_t t = 0; t < S.nlat_tot; ++t) {
        int64_t r = t, idx[3] = {0, 0, 0};
        for (int d = 0; d < n; ++d) {
            idx[d] = sp->lat_idx[d][r % s.nl[d]];
            r /= s.nl[d];
        }
        S.latrows[t] = idx[0] + dp.m[0] * (idx[1] + (int64_t)dp.m[1] * idx[2]);
    }
    // every host input of the call in one staged copy: masks, offsets, lattice rows, and the fit's
    // per-direction tables (used by finish)
    {
        std::vector<std::pair<const void*, size_t>> ups;
        for (int d = 0; d < 3; ++d) {
            ups.push_back({inb[d].data(), inb[d].size()});
            ups.push_back({smp[d].data(), smp[d].size()});
        }
        ups.push_back({shifts.data(), sizeof(int) * shifts.size()});
        ups.push_back({S.latrows.data(), sizeof(int64_t) * S.nlat_tot});
        for (int d = 0; d < n; ++d) {
            const bool fit = s.qd[d] >= 1;
            ups.push_back({fit ? sp->colloc_inv[d] : nullptr, fit ? sizeof(double) * s.nl[d] * s.nl[d] : 8});
            ups.push_back({fit ? sp->interp_knots[d] : nullptr, fit ? sizeof(double) * (s.nl[d] + s.qd[d] + 1) : 8});
            ups.push_back({fit ? sp->box_pts[d] : nullptr, fit ? sizeof(double) * s.bn[d] : 8});
        }
        const std::vector<void*> dv = c.upload_batch(ups);
        for (void* v : dv)
            if (!v) return fail(-4, "device allocation failed");
        for (int d = 0; d < 3; ++d) {
            s.inb[d] = (const uint8_t*)dv[2 * d];
            s.smp[d] = (const uint8_t*)dv[2 * d + 1];
        }
        s.shifts = (const int*)dv[6];
        S.dlat = (int64_t*)dv[7];
        for (int d = 0; d < n; ++d) {
            S.d_ci[d] = (const double*)dv[8 + 3 * d];
            S.d_kn[d] = (const double*)dv[9 + 3 * d];
            S.d_bp[d] = (const double*)dv[10 + 3 * d];
        }
    }

    // analytic pattern; work arrays hold the entries of rows [qlo, qhi) only (the slab, its halo):
    // kernels index them with global row starts through base pointers shifted by nnz(qlo)
    S.rowstart = (int64_t*)c.alloc(sizeof(int64_t) * (N + 1), true);
    launch_indptr_full(c, dp, 0, S.rowstart);
    S.nnz_all = nnz_before_row(dp, N);
    S.nnz_lo = nnz_before_row(dp, slab_lo);
    S.nnz_hi = nnz_before_row(dp, slab_hi);
    S.nnz_qlo = nnz_before_row(dp, s.qlo);
    S.nnz_qhi = nnz_before_row(dp, s.qhi);
    const int64_t nwork = std::max<int64_t>(S.nnz_qhi - S.nnz_qlo, 1);
    S.indices = (int*)c.alloc(sizeof(int) * nwork, true);
    S.data = (double*)c.alloc(sizeof(double) * nwork, true);
    uint8_t* quadmask = (uint8_t*)c.alloc(N, true);
    S.counters = (unsigned long long*)c.alloc(8 * sizeof(unsigned long long), true);
    S.newdiag = (double*)c.alloc(sizeof(double) * N, true);
    S.reset = (uint8_t*)c.alloc(N, true);
    if (!S.rowstart || !S.indices || !S.data || !quadmask || !S.counters || !S.newdiag || !S.reset)
        return fail(-4, "device allocation failed (%lld work entries)", (long long)nwork);
    cudaMemsetAsync(S.counters, 0, 8 * sizeof(unsigned long long), c.stream);
    cudaMemsetAsync(S.reset, 0, N, c.stream);
    s.rowstart = S.rowstart;
    s.indices = S.indices - S.nnz_qlo;
    s.data = S.data - S.nnz_qlo;
    s.newdiag = S.newdiag;
    s.reset = S.reset;
    s.counters = S.counters;
    s.slow = nullptr;
    c.kbegin("classify");
    classify_kernel<<<nblk(N, 256), 256, 0, c.stream>>>(s, N, quadmask);
    c.kend();
    c.hmark("surr_begin:classified");

    // ---- K4: the quadrature rows of [qlo, qhi) (the slab's own, the halo's transposed entries).
    // A row slab starts its tile grid at its first plane and splits its planes into equal-depth z
    // tiles, so no tile streams element layers of planes outside [qlo, qhi)
    Plan pl;
    int t2 = 0, z0 = 0;
    if (n == 3 && (s.qlo > 0 || s.qhi < N)) {
        const int64_t pl01 = (int64_t)dp.m[0] * dp.m[1];
        z0 = (int)(s.qlo / pl01);
        const int planes = (int)((s.qhi - 1) / pl01) - z0 + 1;
        const int nz = (planes + 23) / 24;
        t2 = (planes + nz - 1) / nz;
    }
    rc = plan_assembly(dp, pl, true, t2, z0);
    c.hmark("surr_begin:planned");
    if (rc) return rc;
    std::vector<int> tiles;
    // per direction and tile coordinate: every index in the box / some index sampled (the tile
    // grid is a tensor product, so a tile's classes are ANDs of three per-direction flags)
    std::vector<uint8_t> fin[3], fsm[3];
    for (int d = 0; d < 3; ++d) {
        fin[d].assign(pl.tgrid[d], 1);
        fsm[d].assign(pl.tgrid[d], d < n ? 0 : 1);
        if (d >= n) continue;
        for (int tc = 0; tc < pl.tgrid[d]; ++tc) {
            const int64_t lo = (d == 2 ? pl.z0 : 0) + (int64_t)tc * pl.T[d], hi = std::min<int64_t>(lo + pl.T[d], dp.m[d]) - 1;
            for (int64_t k = lo; k <= hi; ++k) {
                fin[d][tc] = fin[d][tc] && inb[d][k];
                fsm[d][tc] = fsm[d][tc] || smp[d][k];
            }
        }
    }
    {
        // tiles with a quadrature row whose slowest-direction range meets the planes of [qlo, qhi)
        // (tile classes are ANDs of per-direction flags; tiles are ordered z-slowest)
        const int64_t plane = n == 3 ? (int64_t)dp.m[0] * dp.m[1] : (n == 2 ? dp.m[0] : 1);
        const int ds = n - 1;
        const int64_t zlo = s.qlo / plane, zhi = (s.qhi - 1) / plane;
        const int64_t org = ds == 2 ? pl.z0 : 0;
        const int tz0 = (int)std::max<int64_t>(0, (zlo - org) / pl.T[ds]);
        const int tz1 = (int)std::min<int64_t>(pl.tgrid[ds] - 1, (zhi - org) / pl.T[ds]);
        int tsz[3] = {pl.tgrid[0], pl.tgrid[1], pl.tgrid[2]};
        int lo3[3] = {0, 0, 0};
        lo3[ds] = tz0;
        tsz[ds] = tz1 + 1;
        for (int c2 = lo3[2]; c2 < tsz[2]; ++c2)
            for (int c1 = lo3[1]; c1 < tsz[1]; ++c1)
                for (int c0 = lo3[0]; c0 < tsz[0]; ++c0) {
                    const int tc[3] = {c0, c1, c2};
                    bool all_in = true, any_samp_all = true;
                    for (int d = 0; d < n; ++d) {
                        all_in = all_in && fin[d][tc[d]];
                        any_samp_all = any_samp_all && fsm[d][tc[d]];
                    }
                    if (!all_in || any_samp_all) tiles.push_back(c0 + pl.tgrid[0] * (c1 + pl.tgrid[1] * c2));
                }
    }
    c.hmark("surr_begin:tiles");
    rc = run_assembly(c, dp, pl, &tiles, quadmask, S.rowstart, s.qlo, s.qhi, s.indices, s.data, S.counters + 4);
    if (rc) return rc;

    // ---- the sample table S[o][lattice colex]
    // a zeroed tail of one lattice plane + row behind the coefficients: the row-staged K7 kernel
    // reads whole 5-wide windows without clamping (the taps past the last site have weight 0)
    S.cpad = (int64_t)s.nl[0] * s.nl[1] + s.nl[0] + 16;
    S.bufA = (double*)c.alloc(sizeof(double) * (P * S.nlat_tot + S.cpad), true);
    S.bufB = (double*)c.alloc(sizeof(double) * (P * S.nlat_tot + S.cpad), true);
    if (!S.bufA || !S.bufB) return fail(-4, "device allocation failed");
    cudaMemsetAsync(S.bufA, 0, sizeof(double) * (P * S.nlat_tot + S.cpad), c.stream);
    cudaMemsetAsync(S.bufB + P * S.nlat_tot, 0, sizeof(double) * S.cpad, c.stream);
    c.kbegin("gather_samples");
    gather_samples_kernel<<<nblk(S.nlat_tot * P, 256), 256, 0, c.stream>>>(S.rowstart, s.data, S.dlat, S.nlat_tot, P, slab_lo,
                                                                           slab_hi, S.bufA);
    c.kend();
    return 0;
}

// single-call path: the lattice rows outside the slab by a row-restricted assembly (bitwise the
// same rows, assembly.py:613-622), gathered into the sample table
static int surr_foreign_samples(sg_surrogate_state& S) {
    Call& c = S.c;
    std::vector<int64_t> rows;
    for (int64_t r : S.latrows)
        if (r < S.slab_lo || r >= S.slab_hi) rows.push_back(r);
    if (rows.empty()) return 0;
    std::sort(rows.begin(), rows.end());
    int64_t* rs = nullptr;
    int* ind = nullptr;
    double* dat = nullptr;
    int rc = assemble_rows_compact(c, S.dp, rows, &rs, &ind, &dat);
    if (rc) return rc;
    c.kbegin("gather_samples");
    gather_samples_kernel<<<nblk(S.nlat_tot * S.P, 256), 256, 0, c.stream>>>(rs, dat, S.dlat, S.nlat_tot, S.P, 0, S.slab_lo,
                                                                             S.bufA);
    gather_samples_kernel<<<nblk(S.nlat_tot * S.P, 256), 256, 0, c.stream>>>(rs, dat, S.dlat, S.nlat_tot, S.P, S.slab_hi, S.N,
                                                                             S.bufA);
    c.kend();
    c.free_temp(ind);
    c.free_temp(dat);
    return 0;
}

static int surr_finish(sg_surrogate_state& S, const sg_surrogate_params* sp, sg_result** out, sg_surrogate_stats* stats) {
    Call& c = S.c;
    DevProblem& dp = S.dp;
    SurrParams& s = S.s;
    const int n = S.n, p = S.p, P = S.P, center = S.center;
    const int64_t N = S.N, slab_lo = S.slab_lo, slab_hi = S.slab_hi, nlat_tot = S.nlat_tot;
    // ---- K6: samples -> spline coefficients
    double* cur = S.bufA;
    double* nxt = S.bufB;
    int64_t inner = 1;
    for (int d = 0; d < n; ++d) {
        const int len = s.nl[d];
        const int64_t outer = (int64_t)P * nlat_tot / (len * inner);
        if (s.qd[d] >= 1) {
            const double* ci = S.d_ci[d];
            c.kbegin("coef_solve");
            apply_dir_kernel<<<nblk(P * nlat_tot, 256), 256, 0, c.stream>>>(cur, nxt, ci, outer, len, inner);
            c.kend();
            std::swap(cur, nxt);
        }
        inner *= len;
    }
    // the zeroed tail behind the coefficients (bufA's was cleared in begin, bufB's too)
    s.coef = cur;

    // ---- evaluation tables at the in-box midpoints (Cox-de Boor on the averaged knots)
    for (int d = 0; d < 3; ++d) {
        int* esp = (int*)c.alloc(sizeof(int) * s.bn[d], true);
        double* et = (double*)c.alloc(sizeof(double) * s.bn[d] * (s.qd[d] + 1), true);
        if (d < n && s.qd[d] >= 1) {
            const int nk = s.nl[d] + s.qd[d] + 1;
            const double* kn = S.d_kn[d];
            const double* bp = S.d_bp[d];
            tabulate(c, kn, nk, s.qd[d], bp, s.bn[d], 0, esp, et);
        } else {
            c.kbegin("const_table");
            const_table_kernel<<<nblk(s.bn[d], 128), 128, 0, c.stream>>>(s.bn[d], esp, et);
            c.kend();
        }
        s.esp[d] = esp;
        s.etab[d] = et;
    }
    // coefficient window bounds per direction for a tile (host-side, from the same tables)
    const int TBdef[3][3] = {{64, 1, 1}, {8, 8, 1}, {4, 4, 4}};  // 64 rows per tile
    // 3D, interpolation degree 3: the row-staged kernel (4 x 8 x 4 tiles) when every tile's window fits
    bool rows3 = n == 3 && p <= 4 && s.qd[0] == 3 && s.qd[1] == 3 && s.qd[2] == 3 && !getenv("SG_INTERP_FIX");
    for (int d = 0; d < 3; ++d) {
        s.TB[d] = rows3 ? (d == 0 ? rows3::TB0 : (d == 1 ? rows3::TB1 : rows3::TB2)) : TBdef[n - 1][d];
        s.tg[d] = (s.bn[d] + s.TB[d] - 1) / s.TB[d];
    }
    for (int d = 0; d < 3; ++d) {
        if (d >= n || s.qd[d] < 1) {
            s.cmax[d] = 1;
            continue;
        }
        std::vector<double> kn(sp->interp_knots[d], sp->interp_knots[d] + s.nl[d] + s.qd[d] + 1);
        std::vector<int> spn(s.bn[d]);
        for (int k = 0; k < s.bn[d]; ++k) spn[k] = find_span(kn.data(), (int)kn.size(), s.qd[d], sp->box_pts[d][k]);
        int cm = 1;
        for (int org = 0; org < s.bn[d]; org += s.TB[d])
            for (int sh = -p; sh <= p; ++sh) {
                const int a = std::min(std::max(org + sh, 0), s.bn[d] - 1);
                const int b = std::min(std::max(org + s.TB[d] - 1 + sh, 0), s.bn[d] - 1);
                cm = std::max(cm, spn[b] - spn[a] + s.qd[d] + 1);
            }
        s.cmax[d] = cm;
    }
    // ---- K7
    const int nthreads = 512;
    bool fixq = s.qd[0] == 3 && (n < 2 || s.qd[1] == 3) && (n < 3 || s.qd[2] == 3);
    for (int d = 0; d < n; ++d) fixq = fixq && s.cmax[d] <= 5;
    void* kfn;
    const int NR = 64;
    size_t smem;
    int nthr = nthreads;
    if (rows3 && !fixq) {
        // a 4 x 8 x 4 tile's window exceeds 5 coefficients: generic kernel on 64-row tiles (the
        // window bounds computed for the larger tiles are upper bounds for these)
        rows3 = false;
        fixq = false;
        for (int d = 0; d < 3; ++d) {
            s.TB[d] = TBdef[n - 1][d];
            s.tg[d] = (s.bn[d] + s.TB[d] - 1) / s.TB[d];
        }
    }
    if (rows3) {
        s.slow = (int*)c.alloc(sizeof(int) * N, true);
        if (!s.slow) return fail(-4, "device allocation failed");
        for (int d = 0; d < n; ++d) s.cmax[d] = 5;
        // second form by default; SG_INTERP_V1=1 selects the first tensor-core form, SG_INTERP_SIMT=1 its
        // SIMT passes (same values up to the sign of zero)
        // (the second form keeps 32-bit CSR offsets relative to the tile's first row: 8 row planes of slots)
        const bool v2 = !getenv("SG_INTERP_SIMT") && !getenv("SG_INTERP_V1") &&
                        (int64_t)rows3v2::TB2 * dp.m[0] * dp.m[1] * P < (int64_t)INT32_MAX;
        if (v2)
            kfn = p == 1 ? (void*)interp_rows3v2_kernel<3>
                         : (p == 2 ? (void*)interp_rows3v2_kernel<5> : (p == 3 ? (void*)interp_rows3v2_kernel<7> : (void*)interp_rows3v2_kernel<9>));
        else if (getenv("SG_INTERP_SIMT"))
            kfn = p == 1 ? (void*)interp_rows3_kernel<3, false>
                         : (p == 2 ? (void*)interp_rows3_kernel<5, false> : (p == 3 ? (void*)interp_rows3_kernel<7, false> : (void*)interp_rows3_kernel<9, false>));
        else
            kfn = p == 1 ? (void*)interp_rows3_kernel<3, true>
                         : (p == 2 ? (void*)interp_rows3_kernel<5, true> : (p == 3 ? (void*)interp_rows3_kernel<7, true> : (void*)interp_rows3_kernel<9, true>));
        smem = v2 ? interp_rows3v2_smem(p) : interp_rows3_smem(p);
        nthr = v2 ? rows3v2::NWARP * 32 : rows3::NWARP * 32;
    } else if (fixq && n >= 2 && p <= 4) {
        for (int d = 0; d < n; ++d) s.cmax[d] = 5;
        kfn = n == 2 ? (void*)interp_fix_kernel<2> : (void*)interp_fix_kernel<3>;
        smem = interp_fix_smem(n, p);
    } else {
        kfn = n == 1 ? (void*)interp_tiles_kernel<1> : (n == 2 ? (void*)interp_tiles_kernel<2> : (void*)interp_tiles_kernel<3>);
        const int nw = nthreads / 32;
        const int scr = s.cmax[2] * s.cmax[1] * s.TB[0] + s.cmax[2] * s.TB[1] * s.TB[0] + 8;
        size_t tabs = 0;
        for (int d = 0; d < 3; ++d) {
            const int L = (d < n ? s.TB[d] + 2 * p : 1);
            tabs += (size_t)L * (s.qd[d] + 1) * sizeof(double) + (size_t)L * sizeof(int) + L;
        }
        smem = sizeof(double) * ((size_t)nw * scr + (size_t)nw * NR + NR) + sizeof(int) * ((size_t)nw * NR * 3 + 2) + tabs + 64;
    }
    int ntiles = s.tg[0] * s.tg[1] * s.tg[2];
    if (slab_lo > 0 || slab_hi < N) {
        // row slab: only the tiles whose slowest-direction range meets the slab's planes (tiles are
        // ordered with the slowest direction outermost)
        const int64_t plane = n == 3 ? (int64_t)dp.m[0] * dp.m[1] : (n == 2 ? dp.m[0] : 1);
        const int zs = (int)(slab_lo / plane), ze = (int)((slab_hi - 1) / plane);
        const int d = n - 1, TBs = s.TB[d];
        const int c0 = std::max(0, (zs - s.blo[d]) / TBs), c1 = std::min(s.tg[d] - 1, std::max(0, ze - s.blo[d]) / TBs);
        const int per = n == 3 ? s.tg[0] * s.tg[1] : (n == 2 ? s.tg[0] : 1);
        if (ze < s.blo[d] || zs > s.blo[d] + s.bn[d] - 1) {
            ntiles = 0;  // the slab holds no box plane: no interpolated rows
        } else {
            s.tile0 = c0 * per;
            ntiles = (c1 - c0 + 1) * per;
        }
    }
    if (smem > 227 * 1024) return fail(-2, "surrogate tile does not fit shared memory (%zu B)", smem);
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemOptinMax);
    s.dbg = getenv("SG_K7_DBG") ? atoi(getenv("SG_K7_DBG")) : 0;
    void* args[] = {&s};
    c.kbegin(rows3 ? "interp_rows3" : "interp_tiles");
    cudaError_t e = ntiles > 0 ? cudaLaunchKernel(kfn, dim3(ntiles), dim3(nthr), args, smem, c.stream) : cudaSuccess;
    c.kend();
    if (e != cudaSuccess) return fail(-3, "interp launch failed: %s", cudaGetErrorString(e));
    if (rows3) {
        void* sk = p == 1 ? (void*)slow_rows_kernel<3>
                          : (p == 2 ? (void*)slow_rows_kernel<5> : (p == 3 ? (void*)slow_rows_kernel<7> : (void*)slow_rows_kernel<9>));
        c.kbegin("interp_slow_rows");
        // (a fine grid: the rows' costs vary with their number of non-interpolated neighbours; 148 x 8 blocks:
        // 0.67 ms at config 5, x 16: 0.64, x 32: 0.59, x 64: 0.58)
        e = cudaLaunchKernel(sk, dim3(148 * 64), dim3(256), args, 0, c.stream);
        c.kend();
        if (e != cudaSuccess) return fail(-3, "slow-row launch failed: %s", cudaGetErrorString(e));
    }

    // ---- merge: zero check
    unsigned long long hc[8];
    cudaMemcpyAsync(hc, S.counters, sizeof(hc), cudaMemcpyDeviceToHost, c.stream);
    cudaStreamSynchronize(c.stream);
    e = cudaGetLastError();
    if (e != cudaSuccess) return fail(-3, "CUDA error in surrogate: %s", cudaGetErrorString(e));
    const unsigned long long zeros = hc[1] + hc[4];
    sg_result* r = new sg_result();
    r->dev = c.dev;
    r->nrows_global = N;
    r->row_lo = slab_lo;
    r->nrows = slab_hi - slab_lo;
    r->indptr = (int64_t*)c.alloc(sizeof(int64_t) * (r->nrows + 1), false);
    if (zeros == 0) {
        if (s.mode == SG_SYMMETRIC_KERNEL_PRESERVING) {
            c.kbegin("skp_apply");
            skp_apply_kernel<<<nblk(slab_hi - slab_lo, 256), 256, 0, c.stream>>>(S.reset, S.newdiag, S.rowstart, center, slab_lo,
                                                                                slab_hi, s.data);
            c.kend();
        }
        r->nnz = S.nnz_hi - S.nnz_lo;
        c.release(S.indices);
        c.release(S.data);
        if (S.nnz_qlo == S.nnz_lo && S.nnz_qhi == S.nnz_hi) {
            // the work arrays are exactly the result's rows (whole matrix): no copy
            r->indices = S.indices;
            r->data = S.data;
        } else {
            // row slab: the result is the slab's range of the work arrays (sized for the slab and its
            // p-plane halo only); the allocations are freed with the result
            r->own_indices = S.indices;
            r->own_data = S.data;
            r->indices = S.indices + (S.nnz_lo - S.nnz_qlo);
            r->data = S.data + (S.nnz_lo - S.nnz_qlo);
        }
        r->analytic = true;  // no exact zero dropped: the full pattern's rows
        r->p = p;
        for (int d = 0; d < 3; ++d) r->m[d] = dp.m[d];
        cudaMemcpyAsync(r->indptr, S.rowstart + slab_lo, sizeof(int64_t) * (r->nrows + 1), cudaMemcpyDeviceToDevice, c.stream);
        if (S.nnz_lo) {
            c.kbegin("rebase");
            rebase_kernel<<<nblk(r->nrows + 1, 256), 256, 0, c.stream>>>(r->indptr, r->nrows + 1, S.nnz_lo);
            c.kend();
        }
    } else {
        // exact zeros present (surrogate.py:670, scipy's CSR add drops them): compact the slab's rows
        const int64_t nr = slab_hi - slab_lo;
        int64_t* cnt = (int64_t*)c.alloc(sizeof(int64_t) * (nr + 1), true);
        c.kbegin("nz_count");
        nz_count_kernel<<<nblk(nr + 1, 256), 256, 0, c.stream>>>(S.rowstart, s.data, slab_lo, slab_hi, cnt);
        c.kend();
        size_t tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, r->indptr, nr + 1, c.stream);
        void* tmp = c.alloc(tb, true);
        cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, r->indptr, nr + 1, c.stream);
        int64_t nnz_new = 0;
        cudaMemcpyAsync(&nnz_new, r->indptr + nr, sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream);
        cudaStreamSynchronize(c.stream);
        r->nnz = nnz_new;
        r->indices = (int*)c.alloc(sizeof(int) * std::max<int64_t>(nnz_new, 1), false);
        r->data = (double*)c.alloc(sizeof(double) * std::max<int64_t>(nnz_new, 1), false);
        c.kbegin("compact");
        compact_kernel<<<nblk(nr, 256), 256, 0, c.stream>>>(S.rowstart, s.data, s.indices, slab_lo, slab_hi, r->indptr, r->data,
                                                           r->indices);
        c.kend();
        if (s.mode == SG_SYMMETRIC_KERNEL_PRESERVING) {
            // surrogate.py:673-680 is positional on the global CSR: a reset row's window of P entries may
            // run into the following rows.  Inside a slab those rows are local; past the slab's end they
            // belong to the next slab (refused), past the matrix's end it is the reference's IndexError.
            double* nv = (double*)c.alloc(sizeof(double) * std::max<int64_t>(nr, 1), true);
            int* bad = (int*)c.alloc(sizeof(int), true);
            cudaMemsetAsync(bad, 0, sizeof(int), c.stream);
            skp_positional_kernel<<<nblk(nr, 256), 256, 0, c.stream>>>(S.reset, r->indptr, slab_lo, slab_hi, P, center, nnz_new,
                                                                       r->data, nv, bad);
            skp_positional_apply<<<nblk(nr, 256), 256, 0, c.stream>>>(S.reset, r->indptr, slab_lo, slab_hi, center, nv, r->data);
            int hb = 0;
            cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, c.stream);
            cudaStreamSynchronize(c.stream);
            if (hb) {
                sg_result_free(r);
                if (slab_hi != N)
                    return fail(-2, "kernel-preserving reset window crosses the row slab end after an exact-zero drop");
                return fail(-6, "index out of bounds in kernel-preserving reset after zero drop");
            }
        }
    }
    int rc = c.finish();
    if (rc) {
        sg_result_free(r);
        return rc;
    }
    cudaStreamSynchronize(c.stream);
    e = cudaGetLastError();
    if (e != cudaSuccess) {
        sg_result_free(r);
        return fail(-3, "CUDA error after surrogate: %s", cudaGetErrorString(e));
    }
    c.record_timing();
    if (stats) {
        stats->n_interp_entries = (int64_t)hc[0];
        stats->n_zero_dropped = (int64_t)zeros;
        stats->n_reset_rows = (int64_t)hc[2];
        stats->n_interp_rows = (int64_t)hc[3];
        stats->n_quad_rows = N - (int64_t)hc[3];
    }
    *out = r;
    return 0;
}

extern "C" int sg_surrogate(const sg_problem* prob, const sg_surrogate_params* sp, const sg_exec* ex, sg_result** out,
                            sg_surrogate_stats* stats) {
    if (!out || !sp) return fail(-1, "null argument");
    *out = nullptr;
    sg_surrogate_state S(ex);
    int rc = surr_begin(S, prob, sp, ex);
    if (rc) return rc;
    rc = surr_foreign_samples(S);
    if (rc) return rc;
    return surr_finish(S, sp, out, stats);
}

extern "C" int sg_surrogate_begin(const sg_problem* prob, const sg_surrogate_params* sp, const sg_exec* ex,
                                  sg_surrogate_state** state, double** samples, int64_t* nlat) {
    if (!state || !sp) return fail(-1, "null argument");
    *state = nullptr;
    sg_surrogate_state* S = new sg_surrogate_state(ex);
    int rc = surr_begin(*S, prob, sp, ex);
    if (rc) {
        delete S;
        return rc;
    }
    cudaStreamSynchronize(S->c.stream);  // the slab's samples are in the table when this returns
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        delete S;
        return fail(-3, "CUDA error in surrogate begin: %s", cudaGetErrorString(e));
    }
    if (samples) *samples = S->bufA;
    if (nlat) *nlat = S->nlat_tot;
    *state = S;
    return 0;
}

extern "C" int sg_surrogate_finish(sg_surrogate_state* state, const sg_surrogate_params* sp, sg_result** out,
                                   sg_surrogate_stats* stats) {
    if (!state || !sp || !out) return fail(-1, "null argument");
    *out = nullptr;
    const int rc = surr_finish(*state, sp, out, stats);
    delete state;
    return rc;
}

extern "C" int sg_surrogate_state_free(sg_surrogate_state* state) {
    delete state;
    return 0;
}
