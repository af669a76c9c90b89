// Device-resident consumer of the assembled CSR: sparse matrix-vector product
// and the conjugate-gradient solve of surriga/solvers.py:74-155 (`solve_spd` with
// method="conjugate-gradient", preconditioner "none" or "diagonal"), run on the matrix where the
// assembly left it (no 8.9 GB D2H of the CSR at config 5).
//
//   spmv_dot      y = A d (sub-warp per row, lanes strided over the row's nonzeros, fixed shuffle
//                 tree) fused with the per-block partial sums of d.y
//   cg_update     x += a d, r -= a Ad, z = r (/ diag), partial sums of r.r and r.z; a = rz / curv is
//                 read from device scalars (no host round trip between the kernels)
//   cg_direction  d = z + (rz_new / rz) d
//   reduce_*      block partials summed in a fixed order by one block -> every result is
//                 deterministic (bitwise reproducible run to run)
// One CG iteration = 5 kernels captured once in a CUDA graph and replayed; the host reads the two
// scalars it needs for the reference's checks (curvature <= 0, |r| <= target) once per iteration.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "../../include/surriga_b200.h"
#include "sg_internal.h"

namespace sg {
namespace solve {

constexpr int kThreads = 256;
constexpr int kMaxBlocks = 148 * 8;  // partial-sum slots (grid-stride kernels)

// y[i] = sum_k a_ik x_k for rows handled by a group of VS lanes; returns the group's partial
// sum of x_i * y_i through `dot` (only meaningful on the group's first lane)
template <int VS>
__global__ void __launch_bounds__(kThreads) spmv_dot_kernel(int64_t nrows, const int64_t* __restrict__ ip,
                                                           const int* __restrict__ ix, const double* __restrict__ a,
                                                           const double* __restrict__ x, double* __restrict__ y,
                                                           double* __restrict__ partial) {
    __shared__ double red[kThreads / 32];
    // every lane of a warp runs the same number of row iterations (the group shuffles below use the
    // full mask): warp w takes rows [w*RPW, w*RPW + RPW) of each sweep, RPW = 32 / VS groups per warp
    constexpr int RPW = 32 / VS;
    const int lane = threadIdx.x & (VS - 1);
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int sub = (threadIdx.x & 31) / VS;
    double dot = 0.0;
    for (int64_t base = warp * RPW; base < nrows; base += nwarps * RPW) {
        const int64_t row = base + sub;
        const bool ok = row < nrows;
        const int64_t b = ok ? ip[row] : 0, e = ok ? ip[row + 1] : 0;
        double s = 0.0;
        for (int64_t k = b + lane; k < e; k += VS) s = fma(__ldcs(a + k), x[__ldcs(ix + k)], s);
#pragma unroll
        for (int m = VS / 2; m > 0; m >>= 1) s += __shfl_xor_sync(0xffffffffu, s, m, VS);
        if (lane == 0 && ok) {
            y[row] = s;
            if (partial) dot = fma(x[row], s, dot);
        }
    }
    if (!partial) return;
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, m);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = dot;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kThreads / 32; ++w) t += red[w];
        partial[blockIdx.x] = t;
    }
}

// sum of nb partials (columns of `partial`, stride kMaxBlocks) -> out[c], fixed order
__global__ void reduce_kernel(const double* __restrict__ partial, int nb, int ncols, double* __restrict__ out) {
    __shared__ double red[kThreads];
    for (int c = 0; c < ncols; ++c) {
        double t = 0.0;
        for (int i = threadIdx.x; i < nb; i += blockDim.x) t += partial[c * kMaxBlocks + i];
        red[threadIdx.x] = t;
        __syncthreads();
        for (int s = blockDim.x / 2; s > 0; s >>= 1) {
            if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
            __syncthreads();
        }
        if (threadIdx.x == 0) out[c] = red[0];
        __syncthreads();
    }
}

// scalars: [0] rz, [1] curv (d.Ad), [2] r.r, [3] rz_new
__global__ void __launch_bounds__(kThreads) cg_update_kernel(int64_t n, const double* __restrict__ sc, double* __restrict__ x,
                                                            double* __restrict__ r, double* __restrict__ z,
                                                            const double* __restrict__ d, const double* __restrict__ Ad,
                                                            const double* __restrict__ diag, double* __restrict__ partial) {
    __shared__ double red[2][kThreads / 32];
    const double alpha = sc[0] / sc[1];
    double rr = 0.0, rz = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        x[i] = fma(alpha, d[i], x[i]);
        const double ri = fma(-alpha, Ad[i], r[i]);
        r[i] = ri;
        const double zi = diag ? ri / diag[i] : ri;
        z[i] = zi;
        rr = fma(ri, ri, rr);
        rz = fma(ri, zi, rz);
    }
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) {
        rr += __shfl_xor_sync(0xffffffffu, rr, m);
        rz += __shfl_xor_sync(0xffffffffu, rz, m);
    }
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = rr;
        red[1][threadIdx.x >> 5] = rz;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int w = 0; w < kThreads / 32; ++w) {
            a += red[0][w];
            b += red[1][w];
        }
        partial[blockIdx.x] = a;
        partial[kMaxBlocks + blockIdx.x] = b;
    }
}

__global__ void cg_direction_kernel(int64_t n, double* __restrict__ sc, const double* __restrict__ z, double* __restrict__ d) {
    const double beta = sc[3] / sc[0];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        d[i] = fma(beta, d[i], z[i]);
}

__global__ void cg_roll_kernel(double* sc) {
    if (threadIdx.x == 0) sc[0] = sc[3];
}

// x = 0, r = b, z = r (/ diag), d = z; partials of r.z and b.b
__global__ void __launch_bounds__(kThreads) cg_init_kernel(int64_t n, const double* __restrict__ b, const double* __restrict__ diag,
                                                          double* __restrict__ x, double* __restrict__ r, double* __restrict__ z,
                                                          double* __restrict__ d, double* __restrict__ partial) {
    __shared__ double red[2][kThreads / 32];
    double rz = 0.0, bb = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double bi = b[i];
        const double zi = diag ? bi / diag[i] : bi;
        x[i] = 0.0;
        r[i] = bi;
        z[i] = zi;
        d[i] = zi;
        rz = fma(bi, zi, rz);
        bb = fma(bi, bi, bb);
    }
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) {
        rz += __shfl_xor_sync(0xffffffffu, rz, m);
        bb += __shfl_xor_sync(0xffffffffu, bb, m);
    }
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = rz;
        red[1][threadIdx.x >> 5] = bb;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, c = 0.0;
        for (int w = 0; w < kThreads / 32; ++w) {
            a += red[0][w];
            c += red[1][w];
        }
        partial[blockIdx.x] = a;
        partial[kMaxBlocks + blockIdx.x] = c;
    }
}

// diagonal entry of every row (0 when the row stores none), binary search in the sorted columns
__global__ void diag_kernel(int64_t nrows, int64_t row_lo, const int64_t* __restrict__ ip, const int* __restrict__ ix,
                            const double* __restrict__ a, double* __restrict__ diag, int* __restrict__ nonpos) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nrows; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = ip[i], hi = ip[i + 1];
        const int col = (int)(i + row_lo);
        double v = 0.0;
        while (lo < hi) {
            const int64_t mid = (lo + hi) / 2;
            if (ix[mid] < col) lo = mid + 1;
            else hi = mid;
        }
        if (lo < ip[i + 1] && ix[lo] == col) v = a[lo];
        diag[i] = v;
        if (!(v > 0.0)) atomicOr(nonpos, 1);
    }
}

// res = A x - b (for the reference's final residual check)
__global__ void sub_kernel(int64_t n, const double* __restrict__ b, double* __restrict__ y, double* __restrict__ partial) {
    __shared__ double red[kThreads / 32];
    double s = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double v = y[i] - b[i];
        y[i] = v;
        s = fma(v, v, s);
    }
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) s += __shfl_xor_sync(0xffffffffu, s, m);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kThreads / 32; ++w) t += red[w];
        partial[blockIdx.x] = t;
    }
}

static int grid_for(int64_t n, int per_thread_groups = 1) {
    const int64_t need = (n * per_thread_groups + kThreads - 1) / kThreads;
    return (int)std::max<int64_t>(1, std::min<int64_t>(need, kMaxBlocks));
}

struct Spmv {
    int vs = 32;
    int grid = 1;
    void* fn = nullptr;
};

static Spmv plan_spmv(const sg_result* A) {
    Spmv s;
    const double avg = A->nrows ? (double)A->nnz / (double)A->nrows : 0.0;
    s.vs = avg >= 96 ? 32 : (avg >= 24 ? 16 : (avg >= 8 ? 8 : 4));
    s.fn = s.vs == 32 ? (void*)spmv_dot_kernel<32>
                      : (s.vs == 16 ? (void*)spmv_dot_kernel<16> : (s.vs == 8 ? (void*)spmv_dot_kernel<8> : (void*)spmv_dot_kernel<4>));
    s.grid = grid_for(A->nrows, s.vs);
    return s;
}

static void launch_spmv(const Spmv& s, cudaStream_t st, const sg_result* A, const double* x, double* y, double* partial) {
    int64_t n = A->nrows;
    const int64_t* ip = A->indptr;
    const int* ix = A->indices;
    const double* a = A->data;
    void* args[] = {&n, &ip, &ix, &a, &x, &y, &partial};
    cudaLaunchKernel(s.fn, dim3(s.grid), dim3(kThreads), args, 0, st);
}

}  // namespace solve
}  // namespace sg

using namespace sg;
using namespace sg::solve;

extern "C" {

int sg_result_from_host(int32_t device, int64_t nrows, int64_t nnz, const int64_t* indptr, const int32_t* indices,
                        const double* data, sg_result** out) {
    if (!out || !indptr || (nnz > 0 && (!indices || !data))) return fail(-1, "null argument");
    if (nrows < 0 || nnz < 0) return fail(-1, "negative size");
    *out = nullptr;
    sg_exec ex{device, nullptr, 0, 0};
    Call c(&ex);
    sg_result* r = new sg_result();
    r->dev = device;
    r->nrows = r->nrows_global = nrows;
    r->nnz = nnz;
    r->indptr = (int64_t*)c.alloc(sizeof(int64_t) * (nrows + 1), false);
    r->indices = (int*)c.alloc(sizeof(int) * std::max<int64_t>(nnz, 1), false);
    r->data = (double*)c.alloc(sizeof(double) * std::max<int64_t>(nnz, 1), false);
    if (!r->indptr || !r->indices || !r->data) {
        sg_result_free(r);
        return fail(-4, "device allocation failed");
    }
    cudaMemcpyAsync(r->indptr, indptr, sizeof(int64_t) * (nrows + 1), cudaMemcpyHostToDevice, c.stream);
    if (nnz) {
        cudaMemcpyAsync(r->indices, indices, sizeof(int) * nnz, cudaMemcpyHostToDevice, c.stream);
        cudaMemcpyAsync(r->data, data, sizeof(double) * nnz, cudaMemcpyHostToDevice, c.stream);
    }
    cudaStreamSynchronize(c.stream);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        sg_result_free(r);
        return fail(-3, "CUDA error in upload: %s", cudaGetErrorString(e));
    }
    *out = r;
    return 0;
}

int sg_spmv(const sg_result* A, const double* x, double* y, const sg_exec* ex) {
    if (!A || !x || !y) return fail(-1, "null argument");
    if (A->nrows != A->nrows_global || A->row_lo != 0) return fail(-1, "sg_spmv needs a whole square matrix");
    sg_exec e0{A->dev, ex ? ex->stream : nullptr, 0, 0};
    Call c(&e0);
    const int64_t n = A->nrows;
    double* dx = (double*)c.upload(x, sizeof(double) * std::max<int64_t>(n, 1));
    double* dy = (double*)c.alloc(sizeof(double) * std::max<int64_t>(n, 1), true);
    Spmv s = plan_spmv(A);
    c.kbegin("spmv");
    launch_spmv(s, c.stream, A, dx, dy, nullptr);
    c.kend();
    int rc = c.finish();
    if (rc) return rc;
    cudaMemcpyAsync(y, dy, sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream);
    cudaStreamSynchronize(c.stream);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(-3, "CUDA error in spmv: %s", cudaGetErrorString(e));
    c.record_timing();
    return 0;
}

int sg_cg_solve(const sg_result* A, const double* b, double* x, double tol, int64_t maxit, int32_t precond,
                const sg_exec* ex, sg_cg_stats* stats) {
    if (!A || !b || !x || !stats) return fail(-1, "null argument");
    if (A->nrows != A->nrows_global || A->row_lo != 0) return fail(-1, "sg_cg_solve needs a whole square matrix");
    if (maxit < 1) return fail(-1, "max_iterations must be at least 1");
    *stats = sg_cg_stats{};
    sg_exec e0{A->dev, ex ? ex->stream : nullptr, 0, 0};
    Call c(&e0);
    const int64_t n = A->nrows;
    const size_t vb = sizeof(double) * std::max<int64_t>(n, 1);
    double* db = (double*)c.upload(b, vb);
    double* dx = (double*)c.alloc(vb, true);
    double* dr = (double*)c.alloc(vb, true);
    double* dz = (double*)c.alloc(vb, true);
    double* dd = (double*)c.alloc(vb, true);
    double* dAd = (double*)c.alloc(vb, true);
    double* diag = nullptr;
    double* part = (double*)c.alloc(sizeof(double) * 2 * kMaxBlocks, true);
    double* sc = (double*)c.alloc(sizeof(double) * 8, true);
    int* nonpos = (int*)c.alloc(sizeof(int), true);
    double* hsc = nullptr;
    if (!db || !dx || !dr || !dz || !dd || !dAd || !part || !sc || !nonpos) return fail(-4, "device allocation failed");
    if (cudaMallocHost(&hsc, sizeof(double) * 8) != cudaSuccess) return fail(-4, "pinned allocation failed");
    struct HostFree {
        double* p;
        ~HostFree() { cudaFreeHost(p); }
    } hf{hsc};
    cudaMemsetAsync(sc, 0, sizeof(double) * 8, c.stream);
    const int gv = grid_for(n);
    if (precond == 1) {
        diag = (double*)c.alloc(vb, true);
        cudaMemsetAsync(nonpos, 0, sizeof(int), c.stream);
        c.kbegin("diag");
        diag_kernel<<<gv, kThreads, 0, c.stream>>>(n, 0, A->indptr, A->indices, A->data, diag, nonpos);
        c.kend();
        int hnp = 0;
        cudaMemcpyAsync(&hnp, nonpos, sizeof(int), cudaMemcpyDeviceToHost, c.stream);
        cudaStreamSynchronize(c.stream);
        if (hnp) {
            stats->status = SG_CG_NONPOSITIVE_DIAGONAL;
            return 0;
        }
    }
    c.kbegin("cg_init");
    cg_init_kernel<<<gv, kThreads, 0, c.stream>>>(n, db, diag, dx, dr, dz, dd, part);
    reduce_kernel<<<1, kThreads, 0, c.stream>>>(part, gv, 2, sc + 4);  // sc[4] = r.z, sc[5] = b.b
    cudaMemcpyAsync(sc, sc + 4, sizeof(double), cudaMemcpyDeviceToDevice, c.stream);
    c.kend();
    cudaMemcpyAsync(hsc, sc, sizeof(double) * 8, cudaMemcpyDeviceToHost, c.stream);
    cudaStreamSynchronize(c.stream);
    const double normb = std::sqrt(hsc[5]);
    const double target = tol * normb;
    Spmv sp = plan_spmv(A);

    // one iteration as a CUDA graph: Ad = A d, curv = d.Ad, update, |r|^2 and r.z, new direction
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t gexec = nullptr;
    cudaStream_t cap;
    cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking);
    cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal);
    launch_spmv(sp, cap, A, dd, dAd, part);
    reduce_kernel<<<1, kThreads, 0, cap>>>(part, sp.grid, 1, sc + 1);
    cg_update_kernel<<<gv, kThreads, 0, cap>>>(n, sc, dx, dr, dz, dd, dAd, diag, part);
    reduce_kernel<<<1, kThreads, 0, cap>>>(part, gv, 2, sc + 2);
    cg_direction_kernel<<<gv, kThreads, 0, cap>>>(n, sc, dz, dd);
    cg_roll_kernel<<<1, 32, 0, cap>>>(sc);  // rz <- rz_new (after the direction used both)
    cudaMemcpyAsync(hsc, sc, sizeof(double) * 4, cudaMemcpyDeviceToHost, cap);
    cudaError_t e = cudaStreamEndCapture(cap, &graph);
    if (e == cudaSuccess) e = cudaGraphInstantiate(&gexec, graph, 0);
    cudaStreamDestroy(cap);
    if (e != cudaSuccess) {
        if (graph) cudaGraphDestroy(graph);
        return fail(-3, "CG graph capture failed: %s", cudaGetErrorString(e));
    }
    stats->status = SG_CG_MAX_ITERATIONS;
    c.kbegin("cg_iterations");
    int64_t it = 1;
    for (; it <= maxit; ++it) {
        cudaGraphLaunch(gexec, c.stream);
        cudaStreamSynchronize(c.stream);
        // hsc: [0] rz (already rolled), [1] curv, [2] r.r, [3] rz_new
        if (!(hsc[1] > 0.0)) {  // solvers.py:138-141 (curv <= 0; NaN counts as a failure too)
            stats->status = SG_CG_NEGATIVE_CURVATURE;
            break;
        }
        if (std::sqrt(hsc[2]) <= target) {  // solvers.py:144-145
            stats->status = SG_CG_CONVERGED;
            break;
        }
    }
    c.kend();
    stats->iterations = std::min(it, maxit);
    cudaGraphExecDestroy(gexec);
    cudaGraphDestroy(graph);
    // relative residual |A x - b| / |b| of the returned iterate (solvers.py:108-110, 151)
    launch_spmv(sp, c.stream, A, dx, dAd, nullptr);
    sub_kernel<<<gv, kThreads, 0, c.stream>>>(n, db, dAd, part);
    reduce_kernel<<<1, kThreads, 0, c.stream>>>(part, gv, 1, sc + 6);
    cudaMemcpyAsync(hsc + 6, sc + 6, sizeof(double), cudaMemcpyDeviceToHost, c.stream);
    cudaMemcpyAsync(x, dx, sizeof(double) * n, cudaMemcpyDeviceToHost, c.stream);
    int rc = c.finish();
    if (rc) return rc;
    cudaStreamSynchronize(c.stream);
    e = cudaGetLastError();
    if (e != cudaSuccess) return fail(-3, "CUDA error in CG: %s", cudaGetErrorString(e));
    stats->norm_b = normb;
    stats->rel_residual = normb > 0.0 ? std::sqrt(hsc[6]) / normb : 0.0;
    c.record_timing();
    return 0;
}

}  // extern "C"
