// Shared device helpers: Cox-de Boor, constexpr form/term tables, kernel parameter blocks.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <type_traits>
#include <utility>

#ifndef SG_MAX_P
#define SG_MAX_P 5
#endif
#define SG_MAX_PG 8

namespace sg {

// one fp64 tensor-core MMA (m8n8k4, row.col): {c0, c1} += A(lane) x B(lane); bitwise a sequential FMA
// chain over its K (profiles/fp64_peak.txt)
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    // not volatile: the MMA's only effects are its outputs, so the compiler may schedule the shared
    // loads of later operands ahead of it (hides the LDS latency of the operand chains)
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}


enum { POISSON = 0, MASS = 1, BIHARMONIC = 2 };

// ---------------------------------------------------------------------------------------------
// Cox-de Boor (NURBS book A2.2/A2.3), the algorithm of bspline.py:45-109.  Written with explicit
// round-to-nearest intrinsics (no FMA contraction) so the tables are bit-identical to the
// reference's Python-scalar evaluation.
// ---------------------------------------------------------------------------------------------
__host__ __device__ inline int find_span(const double* knots, int nknots, int p, double x) {
    // largest span with knots[span] <= x (searchsorted side=right minus one), clamped to [p, nb-1]
    int lo = 0, hi = nknots;  // first index with knots[idx] > x
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (knots[mid] <= x) lo = mid + 1; else hi = mid;
    }
    int span = lo - 1;
    int nb = nknots - p - 1;
    if (span < p) span = p;
    if (span > nb - 1) span = nb - 1;
    return span;
}

#ifdef __CUDA_ARCH__
#define SG_MUL(a, b) __dmul_rn((a), (b))
#define SG_ADD(a, b) __dadd_rn((a), (b))
#define SG_SUB(a, b) __dsub_rn((a), (b))
#else
#define SG_MUL(a, b) ((a) * (b))
#define SG_ADD(a, b) ((a) + (b))
#define SG_SUB(a, b) ((a) - (b))
#endif

// ders[(k)*(p+1)+r], k = 0..nu ; returns span
__host__ __device__ inline int basis_ders(const double* knots, int nknots, int p, double x, int nu, double* ders) {
    const int span = find_span(knots, nknots, p, x);
    double left[SG_MAX_PG + 1], right[SG_MAX_PG + 1];
    double ndu[SG_MAX_PG + 1][SG_MAX_PG + 1];
    ndu[0][0] = 1.0;
    for (int j = 1; j <= p; ++j) {
        left[j] = SG_SUB(x, knots[span + 1 - j]);
        right[j] = SG_SUB(knots[span + j], x);
        double saved = 0.0;
        for (int r = 0; r < j; ++r) {
            ndu[j][r] = SG_ADD(right[r + 1], left[j - r]);
            double temp = ndu[r][j - 1] / ndu[j][r];
            ndu[r][j] = SG_ADD(saved, SG_MUL(right[r + 1], temp));
            saved = SG_MUL(left[j - r], temp);
        }
        ndu[j][j] = saved;
    }
    for (int k = 0; k <= nu; ++k)
        for (int r = 0; r <= p; ++r) ders[k * (p + 1) + r] = 0.0;
    for (int r = 0; r <= p; ++r) ders[r] = ndu[r][p];
    const int nd = nu < p ? nu : p;
    double a[2][SG_MAX_PG + 1];
    for (int r = 0; r <= p; ++r) {
        int s1 = 0, s2 = 1;
        a[0][0] = 1.0;
        for (int k = 1; k <= nd; ++k) {
            double d = 0.0;
            const int rk = r - k, pk = p - k;
            if (r >= k) {
                a[s2][0] = a[s1][0] / ndu[pk + 1][rk];
                d = SG_MUL(a[s2][0], ndu[rk][pk]);
            }
            const int j1 = (rk >= -1) ? 1 : -rk;
            const int j2 = (r - 1 <= pk) ? k - 1 : p - r;
            for (int j = j1; j <= j2; ++j) {
                a[s2][j] = SG_SUB(a[s1][j], a[s1][j - 1]) / ndu[pk + 1][rk + j];
                d = SG_ADD(d, SG_MUL(a[s2][j], ndu[rk + j][pk]));
            }
            if (r <= pk) {
                a[s2][k] = -a[s1][k - 1] / ndu[pk + 1][r];
                d = SG_ADD(d, SG_MUL(a[s2][k], ndu[r][pk]));
            }
            ders[k * (p + 1) + r] = d;
            int t = s1; s1 = s2; s2 = t;
        }
    }
    double fac = (double)p;
    for (int k = 1; k <= nd; ++k) {
        for (int r = 0; r <= p; ++r) ders[k * (p + 1) + r] = SG_MUL(ders[k * (p + 1) + r], fac);
        fac = SG_MUL(fac, (double)(p - k));
    }
    return span;
}

// CSR pattern counts: row k of a 1D factor couples columns [max(0,k-p), min(m-1,k+p)];
// pre1d(k) = sum_{k'<k} cnt1d(k') in closed form.  (The colex prefix factorises per direction.)
__host__ __device__ inline int64_t cnt1d(int64_t k, int64_t m, int p) {
    const int64_t hi = (m - 1 < k + p) ? m - 1 : k + p;
    const int64_t lo = (k - p > 0) ? k - p : 0;
    return hi - lo + 1;
}
__host__ __device__ inline int64_t pre1d(int64_t k, int64_t m, int p) {
    // sum_{k'<k} [min(m-1, k'+p) - max(0, k'-p) + 1], valid for any m >= 1 (also degenerate m=1 axes)
    int64_t c = m - 1 - p;
    c = c < 0 ? 0 : (c > k ? k : c);
    int64_t s = c * (c - 1) / 2 + c * p + (k - c) * (m - 1) + k;
    const int64_t t = k - 1 - p;
    if (t >= 1) s -= t * (t + 1) / 2;
    return s;
}

// ---------------------------------------------------------------------------------------------
// Form algebra.  Every square form is written as
//     A_ij = s_i s_j  sum_q  sum_{mu,nu in Mset} D_{mu nu}(q) d^mu B_i(q) d^nu B_j(q)
// with B the tensor B-spline basis, Mset a set of parametric derivative multi-indices and D a
// symmetric per-point matrix built from the geometry (and the NURBS weight function W for a
// rational space, s_i = w_i).  This is the reference's integrand (assembly.py:531-548 plus the
// quotient rule of assembly.py:496-517) with the weight quotient folded into D.
// A multi-index is encoded as code = a0 + 3 a1 + 9 a2.
// ---------------------------------------------------------------------------------------------
__host__ __device__ constexpr int acode(int code, int d) { return d == 0 ? code % 3 : (d == 1 ? (code / 3) % 3 : code / 9); }
__host__ __device__ constexpr int aorder(int code) { return acode(code, 0) + acode(code, 1) + acode(code, 2); }

__host__ __device__ constexpr int form_deriv(int form) { return form == POISSON ? 1 : (form == MASS ? 0 : 2); }
__host__ __device__ constexpr int form_lo(int form, bool rat) { return rat ? 0 : (form == MASS ? 0 : 1); }
__host__ __device__ constexpr int geo_deriv(int form) { return form == BIHARMONIC ? 2 : 1; }

__host__ __device__ constexpr bool code_ok(int code, int ndim, int lo, int hi) {
    return (ndim >= 3 || acode(code, 2) == 0) && (ndim >= 2 || acode(code, 1) == 0) && aorder(code) >= lo &&
           aorder(code) <= hi;
}

struct Tables {
    // Mset
    int MS;
    int mcode[10];
    // level-1 groups (after contracting direction 0): key (a1mu, a1nu, a2mu, a2nu) = 0..80
    int NG1;
    int g1key[81];
    int g1n[81];              // units per group
    int g1mu[81][36];         // unit: Mset index of mu  (for pairs: the (mu,nu) with mu<nu)
    int g1nu[81][36];
    int g1pair[81][36];       // 1 = symmetric pair {(mu,nu),(nu,mu)}
    int g1T[81];              // index of the transposed group
    // level-2 groups (after contracting direction 1): key (a2mu, a2nu) = 0..8
    int NG2;
    int g2key[9];
    int g2n[9];
    int g2u[9][81];           // unit: level-1 group index
    int g2pair[9][81];        // pair with its transpose
    int g2T[9];
    // final units over level-2 groups (3D) / level-1 groups (2D) / terms (1D use g1 of the single group)
    int NF;
    int fu[81];
    int fpair[81];
};

__host__ __device__ constexpr int tri_index(int a, int b, int MS) {
    // index of (min,max) in the packed upper triangle, row-major over a<=b
    int lo = a < b ? a : b, hi = a < b ? b : a;
    return lo * MS - (lo * (lo - 1)) / 2 + (hi - lo);
}

__host__ __device__ constexpr Tables make_tables(int ndim, int form, bool rat) {
    Tables T{};
    const int lo = form_lo(form, rat), hi = form_deriv(form);
    T.MS = 0;
    for (int c = 0; c < 27; ++c)
        if (code_ok(c, ndim, lo, hi)) T.mcode[T.MS++] = c;
    // keys of terms
    auto key1 = [&](int mu, int nu) {
        return acode(T.mcode[mu], 1) + 3 * acode(T.mcode[nu], 1) + 9 * acode(T.mcode[mu], 2) + 27 * acode(T.mcode[nu], 2);
    };
    auto key1T = [](int k) {
        int a = k % 3, b = (k / 3) % 3, c = (k / 9) % 3, d = k / 27;
        return b + 3 * a + 9 * d + 27 * c;
    };
    T.NG1 = 0;
    for (int k = 0; k < 81; ++k) {
        bool present = false;
        for (int mu = 0; mu < T.MS; ++mu)
            for (int nu = 0; nu < T.MS; ++nu)
                if (key1(mu, nu) == k) present = true;
        if (present) T.g1key[T.NG1++] = k;
    }
    for (int g = 0; g < T.NG1; ++g) {
        const int k = T.g1key[g], kT = key1T(k);
        T.g1n[g] = 0;
        for (int h = 0; h < T.NG1; ++h)
            if (T.g1key[h] == kT) T.g1T[g] = h;
        if (k == kT) {
            for (int mu = 0; mu < T.MS; ++mu)
                for (int nu = mu; nu < T.MS; ++nu)
                    if (key1(mu, nu) == k) {
                        T.g1mu[g][T.g1n[g]] = mu;
                        T.g1nu[g][T.g1n[g]] = nu;
                        T.g1pair[g][T.g1n[g]] = (mu != nu) ? 1 : 0;
                        T.g1n[g]++;
                    }
        } else {
            const int prim = k < kT ? k : kT;
            for (int mu = 0; mu < T.MS; ++mu)
                for (int nu = 0; nu < T.MS; ++nu)
                    if (key1(mu, nu) == prim) {
                        if (k == prim) { T.g1mu[g][T.g1n[g]] = mu; T.g1nu[g][T.g1n[g]] = nu; }
                        else { T.g1mu[g][T.g1n[g]] = nu; T.g1nu[g][T.g1n[g]] = mu; }
                        T.g1pair[g][T.g1n[g]] = 0;
                        T.g1n[g]++;
                    }
        }
    }
    // level 2
    auto key2of1 = [](int k1) { return (k1 / 9) % 3 + 3 * (k1 / 27); };
    auto key2T = [](int k) { return (k / 3) + 3 * (k % 3); };
    T.NG2 = 0;
    for (int k = 0; k < 9; ++k) {
        bool present = false;
        for (int g = 0; g < T.NG1; ++g)
            if (key2of1(T.g1key[g]) == k) present = true;
        if (present) T.g2key[T.NG2++] = k;
    }
    for (int g = 0; g < T.NG2; ++g) {
        const int k = T.g2key[g], kT = key2T(k);
        T.g2n[g] = 0;
        for (int h = 0; h < T.NG2; ++h)
            if (T.g2key[h] == kT) T.g2T[g] = h;
        if (k == kT) {
            for (int a = 0; a < T.NG1; ++a) {
                if (key2of1(T.g1key[a]) != k) continue;
                const int aT = T.g1T[a];
                if (aT < a) continue;  // already listed as a pair
                T.g2u[g][T.g2n[g]] = a;
                T.g2pair[g][T.g2n[g]] = (aT != a) ? 1 : 0;
                T.g2n[g]++;
            }
        } else {
            const int prim = k < kT ? k : kT;
            for (int a = 0; a < T.NG1; ++a) {
                if (key2of1(T.g1key[a]) != prim) continue;
                T.g2u[g][T.g2n[g]] = (k == prim) ? a : T.g1T[a];
                T.g2pair[g][T.g2n[g]] = 0;
                T.g2n[g]++;
            }
        }
    }
    // final units
    T.NF = 0;
    if (ndim == 3) {
        for (int g = 0; g < T.NG2; ++g) {
            const int gT = T.g2T[g];
            if (gT < g) continue;
            T.fu[T.NF] = g;
            T.fpair[T.NF] = (gT != g) ? 1 : 0;
            T.NF++;
        }
    } else if (ndim == 2) {
        for (int a = 0; a < T.NG1; ++a) {
            const int aT = T.g1T[a];
            if (aT < a) continue;
            T.fu[T.NF] = a;
            T.fpair[T.NF] = (aT != a) ? 1 : 0;
            T.NF++;
        }
    }
    return T;
}

template <int NDIM, int FORM, bool RAT>
struct TermTables {
    static constexpr Tables T = make_tables(NDIM, FORM, RAT);
};

// compile-time loop helper
template <int I, class F, int... K>
__device__ __forceinline__ void static_for_impl(F& f, std::integer_sequence<int, K...>) {
    (f(std::integral_constant<int, I + K>{}), ...);
}
template <int I, int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
    if constexpr (I < N) static_for_impl<I>(f, std::make_integer_sequence<int, N - I>{});
}

// ---------------------------------------------------------------------------------------------
// Kernel parameter block of the tiled assembly kernel.
// ---------------------------------------------------------------------------------------------
struct AsmParams {
    int n, p, g;
    int m[3], S[3];              // basis counts, spans (1 for unused directions)
    const double* B[3];          // solution tables  [S*g][nu+1][p+1]
    const double* sol_w;         // N (rational) or nullptr
    const double* D;             // per-point form tensor from K3, [Gp2][U][Gp0][Dys]
    int Gp[3];                   // Gauss points per direction
    int Dys;                     // y stride of D
    // tiling
    int T[3];                    // rows per tile per direction
    int tgrid[3];                // tiles per direction
    const int* tiles;            // tile ids to process (colex over tgrid), or nullptr = all
    int ypad;                    // padded window size along direction 1
    int off_B0, off_B1, off_D, off_T1, off_T2, off_misc;   // smem layout (doubles)
    // rows & outputs
    const uint8_t* rowmask;      // per-row selection (nullptr = all rows)
    const int64_t* rowstart;     // output position of each row's first entry
    int64_t slab_lo, slab_hi;    // owned row range (colex flat); rows outside are skipped
    int* indices;
    double* data;
    unsigned long long* zeros;   // optional: count of exact zeros written (surrogate merge check)
};

}  // namespace sg
