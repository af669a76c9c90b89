// Internal host-side structures shared by the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <chrono>
#include <string>
#include <utility>
#include <atomic>
#include <vector>

#include "../../include/surriga_b200.h"

struct sg_result {
    int dev = 0;
    int64_t nrows = 0;         // rows held (slab)
    int64_t nrows_global = 0;  // N of the matrix
    int64_t row_lo = 0;        // first global row held
    int64_t nnz = 0;
    int64_t* indptr = nullptr;  // device, nrows+1 (relative to this result)
    int* indices = nullptr;     // device
    double* data = nullptr;     // device
    int64_t tiles = 0;
    void* stream_hint = nullptr;
    void* own_indices = nullptr;  // allocations to free when indices / data point inside a larger buffer
    void* own_data = nullptr;
    bool exported = false;  // device pointers handed out (sg_result_device_ptrs): free waits for the device
    // the result holds full rows of the square basis-overlap pattern (no row restriction, no exact-zero
    // drop): its column indices are a closed-form function of (m, p, row) and the host copy generates
    // them on host threads while the values stream over PCIe instead of copying them
    bool analytic = false;
    int p = 0;
    int64_t m[3] = {1, 1, 1};
};

namespace sg {

// opt-in ceiling for dynamic shared memory set once per kernel function: the attribute is shared by
// every caller of the function, so per-launch sizes would race between concurrent library calls
constexpr int kSmemOptinMax = 227 * 1024;

int fail(int code, const char* fmt, ...);

// One API call: stream, stream-ordered temporaries, per-kernel event timing.
struct Call {
    int dev = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    std::vector<void*> temps;
    struct KEv {
        std::string name;
        cudaEvent_t a, b;
        double host_ms = 0.0;  // host time of the launch since the call started (SG_TRACE)
    };
    std::chrono::steady_clock::time_point t_host0;
    std::vector<std::pair<const char*, double>> hmarks;  // host-only timeline marks (SG_TRACE)
    void hmark(const char* what);
    std::vector<KEv> kev;
    int launches = 0;
    unsigned long long* dmma = nullptr;  // device counter of executed DMMA instructions (K4)
    explicit Call(const sg_exec* ex);
    ~Call();
    void* alloc(size_t bytes, bool temp);
    void release(void* p);  // hand a temporary over to a result (no free at call end)
    void free_temp(void* p);  // free a temporary early (stream ordered)
    void* upload(const void* host, size_t bytes);
    // several host inputs in one device allocation and one staged copy (device pointers in order)
    // defer: items >= 256 KB are packed by the copy pool while the host goes on; their copies are
    // issued by flush_uploads(), which kbegin() calls before any kernel except tabulate / indptr_full
    std::vector<void*> upload_batch(const std::vector<std::pair<const void*, size_t>>& items, bool defer = false);
    struct Pending { void* d; const void* h; size_t bytes; };
    std::vector<Pending> pending;
    std::atomic<int>* pending_left = nullptr;
    void flush_uploads();
    void kbegin(const char* name, bool kernel = true);  // kernel=false: a copy (timed, not counted)
    void kend();
    int finish();
    void record_timing();
};

struct DevProblem {
    sg_problem pr;
    int n = 0, p = 0, g = 0, nu = 0, nug = 0;
    int m[3], S[3], mg[3];
    int64_t N = 0, Ng = 0;
    bool rational = false;
    bool geo_poly = false;     // geometry weights all exactly 1: K3 skips the quotient rule
    int canon[3] = {0, 0, 0};  // solution tables of direction d canonicalised on interior elements (K2)
    double* B[3];
    int* bspan[3];
    double* qw[3];
    double* G[3];
    int* gspan[3];
    std::vector<int> hgspan[3];
    double* hom = nullptr;
    double* sol_w = nullptr;
    double* D = nullptr;
    int Dys = 1;
    int64_t last_tiles = 0;
    int last_T[3];
    size_t last_smem = 0;
};

struct Plan {
    bool mma = false;            // fp64 tensor-core tile kernel (sg_tile_mma.cuh) vs SIMT fallback
    void* kfn = nullptr;
    int kmax = 1, nthreads = 512;
    int T[3], tgrid[3], ypad, off[6];
    int z0 = 0;                  // z origin of the tile grid (row slabs start their tiles at their first plane)
    size_t smem = 0;
    int64_t ntiles = 0;
};

int prepare_problem(Call& c, const sg_problem* pr, DevProblem& dp);
int plan_assembly(DevProblem& dp, Plan& pl, bool restricted = false, int t2 = 0, int z0 = 0);
void tile_box(const Plan& pl, const DevProblem& dp, int64_t t, int64_t lo[3], int64_t hi[3]);
int64_t tile_of_row(const Plan& pl, const DevProblem& dp, int64_t r);
int run_assembly(Call& c, DevProblem& dp, const Plan& pl, const std::vector<int>* tiles, const uint8_t* d_rowmask,
                 const int64_t* d_rowstart, int64_t slab_lo, int64_t slab_hi, int* d_indices, double* d_data,
                 unsigned long long* d_zeros);
void launch_indptr_full(Call& c, const DevProblem& dp, int64_t base, int64_t* rowstart);
// entries before row r of the full basis-overlap pattern (closed form, host)
int64_t nnz_before_row(const DevProblem& dp, int64_t r);
// rows= assembly of sorted unique `rows` into call temporaries (rowstart over all N rows)
int assemble_rows_compact(Call& c, DevProblem& dp, const std::vector<int64_t>& rows, int64_t** d_rowstart, int** d_ind,
                          double** d_dat);
int launch_assembly(Call& c, DevProblem& dp, const uint8_t* d_rowmask, const int64_t* d_rowstart, const int64_t* h_rows,
                    int64_t nrows, int64_t slab_lo, int64_t slab_hi, int* d_indices, double* d_data);
int tabulate(Call& c, const double* d_knots, int nk, int p, const double* d_pts, int npts, int nu, int* d_span,
             double* d_tab);

__global__ void rebase_kernel(int64_t* a, int64_t n, int64_t sub);

// host: closed-form columns of full-pattern rows [r0, r1) of a result starting at global row row_lo
// (sg_hostcols.cpp; AVX2 + non-temporal stores when the CPU has them)
void stream_copy(void* dst, const void* src, size_t n);  // non-temporal stores (staging for DMA)
void gen_columns_avx2(int64_t r0, int64_t r1, int64_t row_lo, const int64_t* m, int p, int32_t* out);
void gen_columns_base(int64_t r0, int64_t r1, int64_t row_lo, const int64_t* m, int p, int32_t* out);
inline void gen_columns(int64_t r0, int64_t r1, int64_t row_lo, const int64_t* m, int p, int32_t* out) {
    static const bool avx2 = __builtin_cpu_supports("avx2");
    if (avx2) gen_columns_avx2(r0, r1, row_lo, m, p, out);
    else gen_columns_base(r0, r1, row_lo, m, p, out);
}

}  // namespace sg
