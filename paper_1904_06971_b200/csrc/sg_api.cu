// C-ABI entry points (include/surriga_b200.h): workspace management, basis tabulation (K2),
// analytic CSR row pointers (K1), tile planning and launch of the assembly kernel (K4),
// result handles, transfers and checksums.
#include <cub/cub.cuh>

#include <sys/mman.h>
#include <sched.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <deque>
#include <functional>
#include <mutex>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <cmath>
#include <string>
#include <thread>
#include <vector>

#include "../../include/surriga_b200.h"
#include "sg_common.cuh"
#include "sg_geom.cuh"
#include "sg_tile_mma.cuh"
#include "sg_internal.h"

namespace sg {

// ------------------------------------------------------------------------------------------
// errors / timing (thread local: the library is re-entrant, ctypes releases the GIL)
// ------------------------------------------------------------------------------------------
static thread_local std::string g_err;
static thread_local double g_last_ms = 0.0;
static thread_local int g_last_launches = 0;
static thread_local std::vector<std::pair<std::string, double>> g_ktimes;
static thread_local unsigned long long g_last_dmma = 0;
#ifdef SG_K4_PROF
constexpr int kProfN = 2 + 32 * 8;  // DMMA count, per-warp clock sums, CTA count
#else
constexpr int kProfN = 1;
#endif

int fail(int code, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

// Small host inputs (knots, Gauss points, masks, tables) are staged through a per-thread pinned arena,
// so their copies are truly asynchronous: a pageable cudaMemcpyAsync blocks the host until the stream
// reaches it, which serialised host planning behind every kernel already queued (~0.5 ms of device
// idle per call at config 5).  The arena is rewound when the last live Call of the thread has been
// destroyed (every Call synchronises its stream before it dies, so no staged copy is pending).
static void pool_memcpy(void* dst, const void* src, size_t n);  // parallel host memcpy (copy pool)
static void copy_pool_run(std::vector<std::function<void()>>& fns, std::atomic<int>* left);
static void copy_pool_wait(std::atomic<int>* left);

struct PinnedArena {
    char* base = nullptr;
    size_t cap = 0, off = 0;
    int users = 0;
    bool tried = false;
};
static thread_local PinnedArena g_arena;
constexpr size_t kArenaBytes = 64u << 20;

Call::Call(const sg_exec* ex) {
    g_arena.users++;
    dev = ex ? ex->device : 0;
    cudaSetDevice(dev);
    if (ex && ex->stream) {
        stream = (cudaStream_t)ex->stream;
        own_stream = false;
    } else {
        cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking);
        own_stream = true;
    }
    static thread_local bool pool_set[64] = {false};
    if (dev >= 0 && dev < 64 && !pool_set[dev]) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        pool_set[dev] = true;
    }
    cudaEventCreate(&ev0);
    cudaEventCreate(&ev1);
    cudaEventRecord(ev0, stream);
    t_host0 = std::chrono::steady_clock::now();
    launches = 0;
}

Call::~Call() {
    flush_uploads();  // the pool must be done with the staging arena before it is reused
    for (void* p : temps)
        if (p) cudaFreeAsync(p, stream);
    for (auto& k : kev) {
        cudaEventDestroy(k.a);
        cudaEventDestroy(k.b);
    }
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    cudaStreamSynchronize(stream);  // staged uploads are complete (no-op when the call already synchronised)
    if (own_stream) cudaStreamDestroy(stream);
    if (--g_arena.users == 0) g_arena.off = 0;
}

void* Call::alloc(size_t bytes, bool temp) {
    void* p = nullptr;
    if (bytes == 0) bytes = 8;
    if (cudaMallocAsync(&p, bytes, stream) != cudaSuccess) return nullptr;
    if (temp) temps.push_back(p);
    return p;
}

void Call::release(void* p) {
    for (auto& t : temps)
        if (t == p) t = nullptr;
}

void Call::free_temp(void* p) {
    if (!p) return;
    for (auto& t : temps)
        if (t == p) {
            t = nullptr;
            cudaFreeAsync(p, stream);
        }
}

void* Call::upload(const void* host, size_t bytes) {
    void* d = alloc(bytes, true);
    if (!d || !host || !bytes) return d;
    if (!g_arena.tried) {
        g_arena.tried = true;
        if (cudaMallocHost((void**)&g_arena.base, kArenaBytes) == cudaSuccess) g_arena.cap = kArenaBytes;
        else g_arena.base = nullptr;
    }
    const size_t need = (bytes + 255) & ~size_t(255);
    if (g_arena.base && g_arena.off + need <= g_arena.cap) {
        char* h = g_arena.base + g_arena.off;
        stream_copy(h, host, bytes);
        g_arena.off += need;
        cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, stream);
    } else {
        cudaMemcpyAsync(d, host, bytes, cudaMemcpyHostToDevice, stream);
    }
    return d;
}

std::vector<void*> Call::upload_batch(const std::vector<std::pair<const void*, size_t>>& items, bool defer) {
    // one device allocation, one pinned staging block, one copy: per-upload API overhead (allocation,
    // memcpy call, copy launch) was ~5-10 us each; large items are packed by the host copy pool
    hmark("upload_batch:start");
    std::vector<void*> out(items.size(), nullptr);
    size_t total = 0;
    std::vector<size_t> off(items.size());
    for (size_t k = 0; k < items.size(); ++k) {
        off[k] = total;
        total += (std::max<size_t>(items[k].second, 8) + 255) & ~size_t(255);
    }
    if (!g_arena.tried) {
        g_arena.tried = true;
        if (cudaMallocHost((void**)&g_arena.base, kArenaBytes) == cudaSuccess) g_arena.cap = kArenaBytes;
        else g_arena.base = nullptr;
    }
    if (!g_arena.base || g_arena.off + total > g_arena.cap) {
        for (size_t k = 0; k < items.size(); ++k) out[k] = upload(items[k].first, items[k].second);
        return out;
    }
    char* d = (char*)alloc(total, true);
    if (!d) return out;
    char* h = g_arena.base + g_arena.off;
    g_arena.off += total;
    std::vector<size_t> big;
    for (size_t k = 0; k < items.size(); ++k) {
        out[k] = d + off[k];
        if (!items[k].first || !items[k].second) continue;
        if (items[k].second >= (256u << 10)) big.push_back(k);
        else stream_copy(h + off[k], items[k].first, items[k].second);
    }
    if (defer && !big.empty()) {
        // small items now (the runs between large ones), large ones packed in the background
        flush_uploads();
        std::vector<std::function<void()>> fns;
        for (size_t k : big) {
            const size_t n = items[k].second, piece = std::max<size_t>(512u << 10, (n + 3) / 4);
            for (size_t lo = 0; lo < n; lo += piece) {
                const size_t len = std::min(piece, n - lo);
                char* dst = h + off[k] + lo;
                const char* src = (const char*)items[k].first + lo;
                fns.push_back([=] { stream_copy(dst, src, len); });
            }
            pending.push_back({d + off[k], h + off[k], n});
        }
        pending_left = new std::atomic<int>(0);
        copy_pool_run(fns, pending_left);
        kbegin("h2d_inputs", false);
        size_t lo = 0;
        for (size_t k : big) {
            if (off[k] > lo) cudaMemcpyAsync(d + lo, h + lo, off[k] - lo, cudaMemcpyHostToDevice, stream);
            lo = off[k] + ((items[k].second + 255) & ~size_t(255));
        }
        if (total > lo) cudaMemcpyAsync(d + lo, h + lo, total - lo, cudaMemcpyHostToDevice, stream);
        kend();
        hmark("upload_batch:small issued");
        return out;
    }
    for (size_t k : big) pool_memcpy(h + off[k], items[k].first, items[k].second);
    hmark("upload_batch:packed");
    kbegin("h2d_inputs", false);
    cudaMemcpyAsync(d, h, total, cudaMemcpyHostToDevice, stream);
    kend();
    return out;
}

void Call::flush_uploads() {
    if (!pending_left) return;
    hmark("flush_uploads:enter");
    copy_pool_wait(pending_left);
    hmark("flush_uploads:packed");
    delete pending_left;
    pending_left = nullptr;
    KEv k;
    k.name = "h2d_deferred";
    k.host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_host0).count();
    cudaEventCreate(&k.a);
    cudaEventCreate(&k.b);
    cudaEventRecord(k.a, stream);
    for (auto& p : pending) cudaMemcpyAsync(p.d, p.h, p.bytes, cudaMemcpyHostToDevice, stream);
    cudaEventRecord(k.b, stream);
    kev.push_back(k);
    pending.clear();
}

void Call::kbegin(const char* name, bool kernel) {
    if (pending_left && kernel && strcmp(name, "tabulate") != 0 && strcmp(name, "indptr_full") != 0) flush_uploads();
    KEv k;
    k.name = name;
    k.host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_host0).count();
    cudaEventCreate(&k.a);
    cudaEventCreate(&k.b);
    cudaEventRecord(k.a, stream);
    kev.push_back(k);
    if (kernel) launches++;
}
void Call::hmark(const char* what) {
    static const bool on = getenv("SG_TRACE") != nullptr;
    if (on) hmarks.push_back({what, std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_host0).count()});
}
void Call::kend() { cudaEventRecord(kev.back().b, stream); }

int Call::finish() {
    flush_uploads();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(-3, "CUDA launch error: %s", cudaGetErrorString(e));
    cudaEventRecord(ev1, stream);
    return 0;
}

void Call::record_timing() {
    // called after the caller synchronised; collects device times
    float ms = 0.f;
    if (cudaEventSynchronize(ev1) == cudaSuccess && cudaEventElapsedTime(&ms, ev0, ev1) == cudaSuccess) g_last_ms = ms;
    g_last_launches = launches;
    g_last_dmma = 0;
    if (dmma) cudaMemcpy(&g_last_dmma, dmma, sizeof(g_last_dmma), cudaMemcpyDeviceToHost);
#ifdef SG_K4_PROF
    if (dmma) {
        // per-warp clock64 sums of the warp-specialised K4 loop (experimental build), cycles per CTA
        std::vector<unsigned long long> pf(kProfN);
        cudaMemcpy(pf.data(), dmma, sizeof(unsigned long long) * kProfN, cudaMemcpyDeviceToHost);
        const double nct = std::max(1ull, pf[1 + 32 * 8]);
        fprintf(stderr, "[k4 prof] CTAs %.0f; per warp, kcycles per CTA: A = plane-wait p1 p2 ring-wait bar loop | B = ready-wait bar p3 b3frag bar loop\n", nct);
        for (int w = 0; w < 32; ++w) {
            const unsigned long long* q = pf.data() + 1 + w * 8;
            if (!q[5]) continue;
            fprintf(stderr, "[k4 prof] warp %2d:", w);
            for (int k = 0; k < 6; ++k) fprintf(stderr, " %8.1f", q[k] / nct / 1e3);
            fprintf(stderr, "\n");
        }
    }
#endif
    g_ktimes.clear();
    for (auto& k : kev) {
        float t = 0.f;
        cudaEventElapsedTime(&t, k.a, k.b);
        g_ktimes.push_back({k.name, (double)t});
    }
    if (getenv("SG_TRACE")) {
        // device timeline of the call (start offset / duration) next to the host time of each launch
        fprintf(stderr, "[sg trace] call total %.3f ms\n", ms);
        for (auto& k : kev) {
            float t0 = 0.f, t1 = 0.f;
            cudaEventElapsedTime(&t0, ev0, k.a);
            cudaEventElapsedTime(&t1, k.a, k.b);
            fprintf(stderr, "[sg trace]   %-18s dev start %8.3f dur %7.3f  host launch %8.3f\n", k.name.c_str(), t0, t1, k.host_ms);
        }
        for (auto& h : hmarks) fprintf(stderr, "[sg trace]   host mark %-24s %8.3f\n", h.first, h.second);
    }
}

// ------------------------------------------------------------------------------------------
// K2: Cox-de Boor tables at many points (bspline.py:112-124), one thread per point
// ------------------------------------------------------------------------------------------
__global__ void tabulate_kernel(const double* __restrict__ knots, int nk, int p, const double* __restrict__ pts, int npts,
                                int nu, int* __restrict__ span_out, double* __restrict__ tab_out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= npts) return;
    double ders[(SG_MAX_PG + 1) * 3];
    const int span = basis_ders(knots, nk, p, pts[i], nu, ders);
    if (span_out) span_out[i] = span;
    const int w = (nu + 1) * (p + 1);
    for (int k = 0; k < w; ++k) tab_out[(long long)i * w + k] = ders[k];
}

// Are the knots uniform and every element's Gauss points the same affine image of one reference set
// (to 1e-13 of the span width)?  Only then do interior elements share their basis values.
static bool uniform_points(const double* kn, int p, int S, const double* x, int g) {
    const double h = (kn[p + S] - kn[p]) / S;
    if (!(h > 0.0)) return false;
    const double tol = 1e-13 * h;
    for (int e = 0; e <= S; ++e)
        if (std::fabs(kn[p + e] - (kn[p] + e * h)) > tol) return false;
    for (int e = 0; e < S; ++e)
        for (int q = 0; q < g; ++q)
            if (std::fabs((x[e * g + q] - kn[p + e]) - (x[q] - kn[p])) > tol) return false;
    return true;
}

// several tabulations in one launch (blockIdx.y = job): the per-direction solution and geometry
// tables of a call are tiny, so their launch overhead dominated the call's prologue
struct TabJob {
    const double* knots;
    const double* pts;
    int* span;
    double* tab;
    int nk, p, npts, nu;
    int g, canon;  // canon: points of interior elements take the first interior element's values
};
struct TabJobs {
    TabJob j[6];
    int n;
};

__global__ void tabulate_multi_kernel(TabJobs jobs) {
    const TabJob& J = jobs.j[blockIdx.y];
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= J.npts) return;
    double ders[(SG_MAX_PG + 1) * 3];
    // uniform open knots: on an interior element (every nonzero function interior, e in [p, S-1-p])
    // the basis values at the q-th Gauss point are the same numbers on every such element; they are
    // taken from element p, so all interior elements carry bitwise identical tables (and tiles whose
    // windows are interior share their fragments, sg_tile_mma.cuh 2D runs)
    const int S = J.npts / J.g, e = i / J.g;
    const bool canon = J.canon && e > J.p && e <= S - 1 - J.p;
    int span = basis_ders(J.knots, J.nk, J.p, J.pts[canon ? J.p * J.g + i % J.g : i], J.nu, ders);
    if (canon) span += e - J.p;
    if (J.span) J.span[i] = span;
    const int w = (J.nu + 1) * (J.p + 1);
    for (int k = 0; k < w; ++k) J.tab[(long long)i * w + k] = ders[k];
}

int tabulate(Call& c, const double* d_knots, int nk, int p, const double* d_pts, int npts, int nu, int* d_span,
             double* d_tab) {
    if (npts <= 0) return 0;
    c.kbegin("tabulate");
    tabulate_kernel<<<(npts + 127) / 128, 128, 0, c.stream>>>(d_knots, nk, p, d_pts, npts, nu, d_span, d_tab);
    c.kend();
    return 0;
}

// ------------------------------------------------------------------------------------------
// K1: analytic row pointers of the basis-overlap pattern.  Row i has prod_d cnt_d(i_d) columns,
// cnt(k) = min(m-1,k+p) - max(0,k-p) + 1; the colex prefix factorises per direction.
// ------------------------------------------------------------------------------------------
struct Dims {
    int64_t m[3];
    int p;
};

__global__ void indptr_full_kernel(Dims D, int64_t N, int64_t base, int64_t* __restrict__ rowstart) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > N) return;
    if (i == N) {
        int64_t tot = 1;
        for (int d = 0; d < 3; ++d) tot *= pre1d(D.m[d], D.m[d], D.p);
        rowstart[N] = tot - base;
        return;
    }
    const int64_t i0 = i % D.m[0], i1 = (i / D.m[0]) % D.m[1], i2 = i / (D.m[0] * D.m[1]);
    const int p = D.p;
    const int64_t t0 = pre1d(D.m[0], D.m[0], p), t1 = pre1d(D.m[1], D.m[1], p);
    rowstart[i] = pre1d(i2, D.m[2], p) * t1 * t0 +
                  cnt1d(i2, D.m[2], p) * (pre1d(i1, D.m[1], p) * t0 + cnt1d(i1, D.m[1], p) * pre1d(i0, D.m[0], p)) - base;
}

__global__ void row_counts_kernel(Dims D, int64_t N, const uint8_t* __restrict__ mask, int64_t* __restrict__ counts) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > N) return;
    if (i == N) { counts[N] = 0; return; }
    const int64_t i0 = i % D.m[0], i1 = (i / D.m[0]) % D.m[1], i2 = i / (D.m[0] * D.m[1]);
    const int p = D.p;
    counts[i] = mask[i] ? cnt1d(i0, D.m[0], p) * cnt1d(i1, D.m[1], p) * cnt1d(i2, D.m[2], p) : 0;
}

__global__ void rebase_kernel(int64_t* a, int64_t n, int64_t sub) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] -= sub;
}

__global__ void scatter_mask_kernel(const int64_t* __restrict__ rows, int64_t n, uint8_t* __restrict__ mask) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) mask[rows[i]] = 1;
}


int64_t nnz_before_row(const DevProblem& dp, int64_t r) {
    if (r >= dp.N) {
        int64_t tot = 1;
        for (int d = 0; d < 3; ++d) tot *= pre1d(dp.m[d], dp.m[d], dp.p);
        return tot;
    }
    const int64_t i0 = r % dp.m[0], i1 = (r / dp.m[0]) % dp.m[1], i2 = r / ((int64_t)dp.m[0] * dp.m[1]);
    const int64_t t0 = pre1d(dp.m[0], dp.m[0], dp.p), t1 = pre1d(dp.m[1], dp.m[1], dp.p);
    return pre1d(i2, dp.m[2], dp.p) * t1 * t0 +
           cnt1d(i2, dp.m[2], dp.p) * (pre1d(i1, dp.m[1], dp.p) * t0 + cnt1d(i1, dp.m[1], dp.p) * pre1d(i0, dp.m[0], dp.p));
}

int assemble_rows_compact(Call& c, DevProblem& dp, const std::vector<int64_t>& rows, int64_t** d_rowstart, int** d_ind,
                          double** d_dat) {
    // the rows= path of sg_assemble into call temporaries: rowstart over all N rows (zero-length
    // rows outside `rows`), entries of the listed rows only
    const int64_t N = dp.N;
    Dims D;
    for (int d = 0; d < 3; ++d) D.m[d] = dp.m[d];
    D.p = dp.p;
    int64_t* rowstart = (int64_t*)c.alloc(sizeof(int64_t) * (N + 1), true);
    uint8_t* mask = (uint8_t*)c.alloc(N + 1, true);
    int64_t* counts = (int64_t*)c.alloc(sizeof(int64_t) * (N + 1), true);
    if (!rowstart || !mask || !counts) return fail(-4, "device allocation failed");
    cudaMemsetAsync(mask, 0, N + 1, c.stream);
    int64_t nnz = 0;
    for (int64_t r : rows) {
        const int64_t i0 = r % dp.m[0], i1 = (r / dp.m[0]) % dp.m[1], i2 = r / ((int64_t)dp.m[0] * dp.m[1]);
        nnz += cnt1d(i0, dp.m[0], dp.p) * cnt1d(i1, dp.m[1], dp.p) * cnt1d(i2, dp.m[2], dp.p);
    }
    if (!rows.empty()) {
        int64_t* drows = (int64_t*)c.upload(rows.data(), sizeof(int64_t) * rows.size());
        scatter_mask_kernel<<<(unsigned)((rows.size() + 255) / 256), 256, 0, c.stream>>>(drows, (int64_t)rows.size(), mask);
    }
    row_counts_kernel<<<(unsigned)((N + 1 + 255) / 256), 256, 0, c.stream>>>(D, N, mask, counts);
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, counts, rowstart, N + 1, c.stream);
    void* tmp = c.alloc(tmp_bytes, true);
    cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, counts, rowstart, N + 1, c.stream);
    int* ind = (int*)c.alloc(sizeof(int) * std::max<int64_t>(nnz, 1), true);
    double* dat = (double*)c.alloc(sizeof(double) * std::max<int64_t>(nnz, 1), true);
    if (!ind || !dat) return fail(-4, "device allocation failed");
    *d_rowstart = rowstart;
    *d_ind = ind;
    *d_dat = dat;
    if (rows.empty()) return 0;
    return launch_assembly(c, dp, mask, rowstart, rows.data(), (int64_t)rows.size(), 0, N, ind, dat);
}

void launch_indptr_full(Call& c, const DevProblem& dp, int64_t base, int64_t* rowstart) {
    Dims D;
    for (int d = 0; d < 3; ++d) D.m[d] = dp.m[d];
    D.p = dp.p;
    c.kbegin("indptr_full");
    indptr_full_kernel<<<(unsigned)((dp.N + 1 + 255) / 256), 256, 0, c.stream>>>(D, dp.N, base, rowstart);
    c.kend();
}

// ------------------------------------------------------------------------------------------
// problem upload + tables
// ------------------------------------------------------------------------------------------
int prepare_problem(Call& c, const sg_problem* pr, DevProblem& dp) {
    if (!pr) return fail(-1, "null problem");
    if (pr->n < 1 || pr->n > 3) return fail(-1, "supported dimensions: 1, 2, 3");
    if (pr->p < 1) return fail(-1, "degree p=%d must be at least 1", pr->p);
    if (pr->g < 1) return fail(-1, "gauss=%d must be at least 1", pr->g);
    // valid for the reference (any p >= 1, any Gauss count) but outside what this build instantiates:
    // "unsupported configuration", not an invalid argument
    if (pr->p > SG_MAX_P) return fail(-2, "degree p=%d is not supported by this build (p <= %d)", pr->p, SG_MAX_P);
    if (pr->g > 8) return fail(-2, "gauss=%d is not supported by this build (gauss <= 8)", pr->g);
    if (pr->geo_p < 1 || pr->geo_p > SG_MAX_PG) return fail(-1, "geometry degree %d unsupported", pr->geo_p);
    if (pr->form < 0 || pr->form > 2) return fail(-1, "unknown form %d", pr->form);
    if (pr->form == BIHARMONIC && pr->p < 2) return fail(-1, "the fourth-order form needs degree >= 2 for C^1 continuity");
    dp.pr = *pr;
    dp.n = pr->n;
    dp.p = pr->p;
    dp.g = pr->g;
    dp.nu = form_deriv(pr->form);
    dp.nug = geo_deriv(pr->form);
    dp.N = 1;
    dp.Ng = 1;
    for (int d = 0; d < 3; ++d) {
        if (d < pr->n) {
            dp.m[d] = pr->m[d];
            dp.S[d] = pr->m[d] - pr->p;
            dp.mg[d] = pr->geo_m[d];
            if (dp.S[d] < 1 || pr->m[d] < 2 * pr->p + 1) return fail(-1, "basis count m=%d below 2p+1=%d", pr->m[d], 2 * pr->p + 1);
        } else {
            dp.m[d] = 1;
            dp.S[d] = 1;
            dp.mg[d] = 1;
        }
        dp.N *= dp.m[d];
        dp.Ng *= dp.mg[d];
    }
    dp.rational = pr->sol_w != nullptr;
    // uploads; the 2n tables (solution and geometry bases per direction) in one launch
    TabJobs jobs;
    jobs.n = 0;
    int maxpts = 0;
    // every host input of the problem in one staged copy
    std::vector<std::pair<const void*, size_t>> ups;
    for (int d = 0; d < pr->n; ++d) {
        const int npts = dp.S[d] * dp.g;
        ups.push_back({pr->knots[d], sizeof(double) * (dp.m[d] + dp.p + 1)});
        ups.push_back({pr->qpts[d], sizeof(double) * npts});
        ups.push_back({pr->qwts[d], sizeof(double) * dp.g});
        ups.push_back({pr->geo_knots[d], sizeof(double) * (dp.mg[d] + pr->geo_p + 1)});
    }
    ups.push_back({pr->geo_hom, sizeof(double) * dp.Ng * (pr->n + 1)});
    if (dp.rational) ups.push_back({pr->sol_w, sizeof(double) * dp.N});
    const std::vector<void*> dv = c.upload_batch(ups, true);
    for (void* v : dv)
        if (!v) return fail(-4, "device allocation failed");
    dp.hom = (double*)dv[4 * pr->n];
    // unit weights: a polynomial map (the reference's GeometryMap.is_polynomial, geometry.py:167)
    dp.geo_poly = true;
    for (int64_t i = 0; i < dp.Ng && dp.geo_poly; ++i) dp.geo_poly = pr->geo_hom[i * (pr->n + 1) + pr->n] == 1.0;
    dp.sol_w = dp.rational ? (double*)dv[4 * pr->n + 1] : nullptr;
    // the 4n tables in one allocation (cudaMallocAsync is ~5 us per call on the host)
    size_t tab_bytes = 0;
    auto carve = [&](size_t b) { const size_t o = tab_bytes; tab_bytes += (b + 255) & ~size_t(255); return o; };
    size_t o_tab[3][4];
    for (int d = 0; d < pr->n; ++d) {
        const size_t npts = (size_t)dp.S[d] * dp.g;
        o_tab[d][0] = carve(sizeof(double) * npts * (dp.nu + 1) * (dp.p + 1));
        o_tab[d][1] = carve(sizeof(int) * npts);
        o_tab[d][2] = carve(sizeof(double) * npts * (dp.nug + 1) * (pr->geo_p + 1));
        o_tab[d][3] = carve(sizeof(int) * npts);
    }
    char* tabs = (char*)c.alloc(tab_bytes, true);
    if (!tabs) return fail(-4, "device allocation failed");
    for (int d = 0; d < pr->n; ++d) {
        const int npts = dp.S[d] * dp.g;
        maxpts = std::max(maxpts, npts);
        double* kn = (double*)dv[4 * d];
        double* qp = (double*)dv[4 * d + 1];
        dp.qw[d] = (double*)dv[4 * d + 2];
        dp.B[d] = (double*)(tabs + o_tab[d][0]);
        dp.bspan[d] = (int*)(tabs + o_tab[d][1]);
        dp.canon[d] = uniform_points(pr->knots[d], dp.p, dp.S[d], pr->qpts[d], dp.g) ? 1 : 0;
        jobs.j[jobs.n++] = TabJob{kn, qp, dp.bspan[d], dp.B[d], dp.m[d] + dp.p + 1, dp.p, npts, dp.nu, dp.g, dp.canon[d]};
        double* gk = (double*)dv[4 * d + 3];
        dp.G[d] = (double*)(tabs + o_tab[d][2]);
        dp.gspan[d] = (int*)(tabs + o_tab[d][3]);
        jobs.j[jobs.n++] = TabJob{gk, qp, dp.gspan[d], dp.G[d], dp.mg[d] + pr->geo_p + 1, pr->geo_p, npts, dp.nug, dp.g, 0};
        // host copies of geometry spans for the smem bound
        std::vector<double> hk(pr->geo_knots[d], pr->geo_knots[d] + dp.mg[d] + pr->geo_p + 1);
        dp.hgspan[d].resize(npts);
        for (int i = 0; i < npts; ++i)
            dp.hgspan[d][i] = find_span(hk.data(), (int)hk.size(), pr->geo_p, pr->qpts[d][i]);
    }
    c.hmark("prepare:tables allocated");
    c.kbegin("tabulate");
    tabulate_multi_kernel<<<dim3((maxpts + 127) / 128, jobs.n), 128, 0, c.stream>>>(jobs);
    c.kend();
    for (int d = pr->n; d < 3; ++d) {
        dp.qw[d] = nullptr;
        dp.B[d] = nullptr;
        dp.G[d] = nullptr;
        dp.gspan[d] = nullptr;
        dp.hgspan[d].assign(1, 0);
    }
    return 0;
}

// ------------------------------------------------------------------------------------------
// tile planning + kernel launch
// ------------------------------------------------------------------------------------------
#define SG_DECL(nd, f) extern void* assemble_kernel_##nd##_##f(int p, bool rat, int* kmax);
SG_DECL(1, 0) SG_DECL(1, 1) SG_DECL(1, 2) SG_DECL(2, 0) SG_DECL(2, 1) SG_DECL(2, 2) SG_DECL(3, 0) SG_DECL(3, 1) SG_DECL(3, 2)
#undef SG_DECL

#define SG_DECLK(nd, f, r) extern void* kernel_ptr_##nd##_##f##_##r(int which, int p, int* kmax);
SG_DECLK(1, 0, 0) SG_DECLK(1, 0, 1) SG_DECLK(1, 1, 0) SG_DECLK(1, 1, 1) SG_DECLK(1, 2, 0) SG_DECLK(1, 2, 1)
SG_DECLK(2, 0, 0) SG_DECLK(2, 0, 1) SG_DECLK(2, 1, 0) SG_DECLK(2, 1, 1) SG_DECLK(2, 2, 0) SG_DECLK(2, 2, 1)
SG_DECLK(3, 0, 0) SG_DECLK(3, 0, 1) SG_DECLK(3, 1, 0) SG_DECLK(3, 1, 1) SG_DECLK(3, 2, 0) SG_DECLK(3, 2, 1)
#undef SG_DECLK

static void* kernel_ptr(int n, int form, bool rat, int which, int p, int* kmax) {
    typedef void* (*Fn)(int, int, int*);
    static const Fn tab[3][3][2] = {
        {{kernel_ptr_1_0_0, kernel_ptr_1_0_1}, {kernel_ptr_1_1_0, kernel_ptr_1_1_1}, {kernel_ptr_1_2_0, kernel_ptr_1_2_1}},
        {{kernel_ptr_2_0_0, kernel_ptr_2_0_1}, {kernel_ptr_2_1_0, kernel_ptr_2_1_1}, {kernel_ptr_2_2_0, kernel_ptr_2_2_1}},
        {{kernel_ptr_3_0_0, kernel_ptr_3_0_1}, {kernel_ptr_3_1_0, kernel_ptr_3_1_1}, {kernel_ptr_3_2_0, kernel_ptr_3_2_1}}};
    if (n < 1 || n > 3 || form < 0 || form > 2) return nullptr;
    int km = 1;
    void* f = tab[n - 1][form][rat ? 1 : 0](which, p, &km);
    if (kmax) *kmax = km;
    return f;
}

static void* get_mma_kernel(int n, int form, int p, bool rat, int* nthreads) { return kernel_ptr(n, form, rat, 1, p, nthreads); }

static void* get_kernel(int n, int form, int p, bool rat, int* kmax) { return kernel_ptr(n, form, rat, 0, p, kmax); }

struct Layout {
    int T[3];
    int ypad;
    size_t off[6];  // B0, B1, D, T1, T2, misc
    size_t total;   // doubles
};

static Layout make_layout(const DevProblem& dp, int T0, int T1, int T2) {
    const int n = dp.n, P = dp.p, g = dp.g;
    const Tables TT = make_tables(n, dp.pr.form, dp.rational);
    const int MS = TT.MS, U = MS * (MS + 1) / 2;
    const int NB = (dp.nu + 1) * (P + 1);
    const int W2P = 2 * P + 1;
    Layout L;
    L.T[0] = T0;
    L.T[1] = n >= 2 ? T1 : 1;
    L.T[2] = n >= 3 ? T2 : 1;
    const int X0 = (std::min(T0 + P, dp.S[0])) * g;
    const int X1 = n >= 2 ? (std::min(L.T[1] + P, dp.S[1])) * g : 1;
    L.ypad = n >= 2 ? (X1 | 1) : 1;
    size_t sz[6];
    sz[0] = (size_t)X0 * NB;
    sz[1] = n >= 2 ? (size_t)X1 * NB : 0;
    sz[2] = (size_t)U * X0 * L.ypad;
    sz[3] = n >= 2 ? (size_t)TT.NG1 * T0 * W2P * L.ypad : 0;
    sz[4] = n == 3 ? (size_t)TT.NG2 * T0 * W2P * L.T[1] * W2P : 0;
    sz[5] = NB + 8;
    size_t o = 0;
    for (int k = 0; k < 6; ++k) {
        L.off[k] = o;
        o += sz[k];
        o = (o + 1) & ~size_t(1);
    }
    L.total = o;
    return L;
}

static const size_t kSmemCap = 227 * 1024;

static int choose_layout(const DevProblem& dp, int kmax, int nthreads, Layout& out) {
    const int n = dp.n, P = dp.p;
    const int W2P = 2 * P + 1;
    for (int T = (n == 1 ? 256 : 16); T >= 1; --T) {
        const int T2 = n == 3 ? 16 : 1;
        Layout L = make_layout(dp, T, T, T2);
        if (L.total * sizeof(double) > kSmemCap) continue;
        if (n == 3 && (size_t)T * W2P * T * W2P * (P + 1) > (size_t)kmax * nthreads) continue;
        out = L;
        return 0;
    }
    return fail(-2, "no tile configuration fits shared memory for this problem (p=%d, n=%d)", P, n);
}

// ------------------------------------------------------------------------------------------
// K3 launch: per-point form tensor D on the blocks of points the selected tiles read
// ------------------------------------------------------------------------------------------
static void* get_geom_kernel(int n, int form, bool rat, bool poly) { return kernel_ptr(n, form, rat, poly ? 3 : 2, 1, nullptr); }

struct GeomMark {
    int n, P, g, T[3], tg[3], S[3], BX, BY, nbx, nby, z0;
    int m[3];
    const uint8_t* rowmask;  // restricted plans: rows the tiles own (nullptr: every row of the slab)
    int64_t slab_lo, slab_hi;
};
// geometry blocks needed by a tile list: the element window [lo - P, lo + T - 1] of every tile
__global__ void geom_mark_kernel(GeomMark m, const int* __restrict__ tiles, int64_t ntiles, uint8_t* __restrict__ mask) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ntiles) return;
    const int t = tiles[i];
    const int tc[3] = {t % m.tg[0], (t / m.tg[0]) % m.tg[1], t / (m.tg[0] * m.tg[1])};
    int64_t plo[3] = {0, 0, 0}, phi[3] = {0, 0, 0};
    int64_t rlo[3], rhi[3];  // the tile's row box
    for (int d = 0; d < 3; ++d) {
        rlo[d] = (d == 2 ? m.z0 : 0) + (int64_t)tc[d] * m.T[d];
        rhi[d] = min((int64_t)m.m[d] - 1, rlo[d] + m.T[d] - 1);
    }
    if (m.n == 3) {
        // slowest direction: only the rows the tile owns (the kernel streams just their layers; a
        // tile kept for a few sampled rows needs a few planes of D, not its whole depth)
        int64_t zlo = INT64_MAX, zhi = -1;
        for (int64_t i2 = rlo[2]; i2 <= rhi[2]; ++i2)
            for (int64_t i1 = rlo[1]; i1 <= rhi[1]; ++i1)
                for (int64_t i0 = rlo[0]; i0 <= rhi[0]; ++i0) {
                    const int64_t row = i0 + (int64_t)m.m[0] * (i1 + (int64_t)m.m[1] * i2);
                    if (row >= m.slab_lo && row < m.slab_hi && (!m.rowmask || m.rowmask[row])) {
                        zlo = min(zlo, i2);
                        zhi = max(zhi, i2);
                    }
                }
        if (zhi < 0) return;
        rlo[2] = zlo;
        rhi[2] = zhi;
    }
    for (int d = 0; d < m.n; ++d) {
        const int64_t e0 = max((int64_t)0, rlo[d] - m.P), e1 = min((int64_t)m.S[d] - 1, rhi[d]);
        plo[d] = e0 * m.g;
        phi[d] = (e1 + 1) * m.g - 1;
    }
    for (int64_t z = plo[2]; z <= phi[2]; ++z)
        for (int64_t by = plo[1] / m.BY; by <= phi[1] / m.BY; ++by)
            for (int64_t bx = plo[0] / m.BX; bx <= phi[0] / m.BX; ++bx) mask[bx + m.nbx * (by + m.nby * z)] = 1;
}

static int env_int(const char* name, int dflt) {
    const char* v = getenv(name);
    return (v && *v) ? atoi(v) : dflt;
}

int compute_D(Call& c, DevProblem& dp, const Plan& pl, const std::vector<int>* tiles, const uint8_t* d_rowmask,
              int64_t slab_lo, int64_t slab_hi) {
    const int n = dp.n, g = dp.g, P = dp.p, pg = dp.pr.geo_p;
    const Tables TT = make_tables(n, dp.pr.form, dp.rational);
    const int U = TT.MS * (TT.MS + 1) / 2;
    const int NU = dp.nu, NUG = dp.nug;
    const int NB = (NU + 1) * (P + 1), NBG = (NUG + 1) * (pg + 1);
    GeomParams gp;
    memset(&gp, 0, sizeof(gp));
    gp.p = P;
    gp.g = g;
    gp.pg = pg;
    for (int d = 0; d < 3; ++d) {
        gp.m[d] = dp.m[d];
        gp.mg[d] = dp.mg[d];
        gp.B[d] = dp.B[d];
        gp.qw[d] = dp.qw[d];
        gp.gspan[d] = dp.gspan[d];
        gp.G[d] = dp.G[d];
        gp.Gp[d] = d < n ? dp.S[d] * g : 1;
    }
    gp.sol_w = dp.sol_w;
    gp.hom = dp.hom;
    gp.coef = dp.pr.coefficient;
    gp.U = U;
    gp.Dys = n >= 2 ? ((gp.Gp[1] + 1) & ~1) : 1;
    dp.Dys = gp.Dys;
    // Points per block: 32 x 32 for restricted plans (16 x 16 measured slower: the per-block table set-up
    // dominates; larger blocks compute more unneeded points); whole-mesh plans take 32 x 256 where it fits
    // (a warp shares x and walks y: the per-plane Hz / Hx preparation and its barriers are amortised over
    // 8x the points; config 5: Poisson 2.10 -> 1.67 ms, mass 1.69 -> 1.18 ms; 32 x 128: 1.72 / 1.25,
    // 32 x 512: 1.78 / 1.22, 64 x 256: 1.79 / 1.23, 16 x 256: 1.69 / 1.20)
    const int C = n + 1;
    const int NCg = n == 3 ? (NUG + 1) * (NUG + 2) / 2 : NUG + 1;
    const int NCw = n == 3 ? (NU + 1) * (NU + 2) / 2 : NU + 1;
    auto gbound = [&](int d, int B) {
        int mx = 1;
        if (d >= n) return 1;
        for (int s0 = 0; s0 < gp.Gp[d]; s0 += B) {
            const int s1 = std::min(gp.Gp[d], s0 + B) - 1;
            mx = std::max(mx, dp.hgspan[d][s1] - dp.hgspan[d][s0] + pg + 1);
        }
        return mx;
    };
    auto set_layout = [&](int BX, int BY) -> size_t {
        gp.BX = BX;
        gp.BY = BY;
        gp.nbx = (gp.Gp[0] + gp.BX - 1) / gp.BX;
        gp.nby = (gp.Gp[1] + gp.BY - 1) / gp.BY;
        // 3D: several z-planes per block (the x/y tables and spans are loaded once), enough blocks for
        // every SM several times over
        gp.ZB = 1;
        if (n == 3)
            while (gp.ZB < env_int("SG_GEOM_ZB", 8) && (int64_t)gp.nbx * gp.nby * ((gp.Gp[2] + 2 * gp.ZB - 1) / (2 * gp.ZB)) >= 8 * 148) gp.ZB *= 2;
        // function-range bounds per block
        gp.GN0 = gbound(0, gp.BX);
        gp.GN1 = gbound(1, gp.BY);
        gp.WN0 = (gp.BX + g - 1) / g + 1 + P;
        gp.WN1 = n >= 2 ? (gp.BY + g - 1) / g + 1 + P : 1;
        size_t sz[13];
        sz[0] = (size_t)gp.BX * NBG;
        sz[1] = n >= 2 ? (size_t)gp.BY * (NBG | 1) : 0;
        sz[2] = gp.BX / 2 + 1;
        sz[3] = gp.BY / 2 + 1;
        sz[4] = dp.rational ? (size_t)gp.BX * NB : 0;
        sz[5] = (dp.rational && n >= 2) ? (size_t)gp.BY * (NB | 1) : 0;
        sz[6] = gp.BX / 2 + 1;
        sz[7] = gp.BY / 2 + 1;
        sz[8] = n == 3 ? (size_t)gp.GN0 * gp.GN1 * C * (NUG + 1) : 0;
        sz[9] = n >= 2 ? (size_t)gp.BX * gp.GN1 * C * NCg : 0;
        sz[10] = (n == 3 && dp.rational) ? (size_t)gp.WN0 * gp.WN1 * (NU + 1) : 0;
        sz[11] = (n >= 2 && dp.rational) ? (size_t)gp.BX * gp.WN1 * NCw : 0;
        sz[12] = 64 + gp.BX + gp.BY + 8;
        int* offs[13] = {&gp.off_G0, &gp.off_G1, &gp.off_gs0, &gp.off_gs1, &gp.off_B0, &gp.off_B1, &gp.off_ws0,
                         &gp.off_ws1, &gp.off_Hz, &gp.off_Hy, &gp.off_Wz, &gp.off_Wy, &gp.off_misc};
        size_t o = 0;
        for (int k = 0; k < 13; ++k) {
            *offs[k] = (int)o;
            o += sz[k];
            o = (o + 1) & ~size_t(1);
        }
        return o * sizeof(double);
    };
    size_t smem = 0;
    if (n >= 2 && !tiles && !getenv("SG_GEOM_BY") && !getenv("SG_GEOM_BX")) {
        for (int by : {256, 128, 64}) {
            if (by >= 2 * gp.Gp[1]) continue;  // a block taller than the mesh buys nothing
            smem = set_layout(32, by);
            if (smem <= 72 * 1024) break;  // three blocks per SM
            smem = 0;
        }
    }
    if (!smem) {
        const int bxy = (n == 3 && tiles) ? env_int("SG_GEOM_BXY_RESTR", 32) : 32;
        smem = set_layout(n == 1 ? 256 : env_int("SG_GEOM_BX", bxy), n >= 2 ? env_int("SG_GEOM_BY", bxy) : 1);
    }
    const int64_t nblk_all = (int64_t)gp.nbx * gp.nby * gp.Gp[2];
    if (smem > kSmemCap) return fail(-2, "geometry block does not fit shared memory (%zu B)", smem);
    const size_t npts = (size_t)gp.Gp[0] * gp.Dys * gp.Gp[2];
    c.hmark("compute_D:layout");
    gp.D = (double*)c.alloc(sizeof(double) * npts * U, true);
    c.hmark("compute_D:alloc");
    if (!gp.D) return fail(-4, "device allocation of the D tensor failed (%zu MB)", sizeof(double) * npts * U >> 20);
    dp.D = gp.D;
    if (tiles) {
        // blocks touched by the tiles' element windows, marked on the device (no host loop)
        if (tiles->empty()) return 0;
        const int* dt = (const int*)c.upload(tiles->data(), sizeof(int) * tiles->size());
        uint8_t* mask = (uint8_t*)c.alloc(nblk_all, true);
        cudaMemsetAsync(mask, 0, nblk_all, c.stream);
        GeomMark gm;
        gm.n = n;
        gm.P = P;
        gm.g = g;
        for (int d = 0; d < 3; ++d) {
            gm.T[d] = pl.T[d];
            gm.tg[d] = pl.tgrid[d];
            gm.S[d] = dp.S[d];
        }
        gm.z0 = pl.z0;
        for (int d = 0; d < 3; ++d) gm.m[d] = dp.m[d];
        gm.rowmask = d_rowmask;
        gm.slab_lo = slab_lo;
        gm.slab_hi = slab_hi;
        gm.BX = gp.BX;
        gm.BY = gp.BY;
        gm.nbx = gp.nbx;
        gm.nby = gp.nby;
        c.kbegin("geom_mark");
        geom_mark_kernel<<<(unsigned)((tiles->size() + 127) / 128), 128, 0, c.stream>>>(gm, dt, (int64_t)tiles->size(), mask);
        c.kend();
        gp.blockmask = mask;
    }
    void* kfn = get_geom_kernel(n, dp.pr.form, dp.rational, dp.geo_poly && !getenv("SG_GEO_QUOTIENT"));
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemOptinMax);
    void* args[] = {&gp};
    const int64_t nb = (int64_t)gp.nbx * gp.nby * ((gp.Gp[2] + gp.ZB - 1) / gp.ZB);
    c.kbegin("geom_D");
    cudaError_t e = cudaLaunchKernel(kfn, dim3((unsigned)nb), dim3(256), args, smem, c.stream);
    c.kend();
    if (e != cudaSuccess) return fail(-3, "geometry launch failed: %s", cudaGetErrorString(e));
    return 0;
}

// TMA descriptor of the D tensor [Gp2][U][Gp0][Dys] (fetched through the runtime's driver entry point)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static int encode_dmap(CUtensorMap* map, const double* D, int Dys, const int Gp[3], int U, int DY, int XW) {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
            return fail(-3, "cuTensorMapEncodeTiled unavailable");
        fn = (EncodeTiledFn)p;
    }
    cuuint64_t dims[4] = {(cuuint64_t)Gp[1], (cuuint64_t)Gp[0], (cuuint64_t)U, (cuuint64_t)Gp[2]};
    cuuint64_t strides[3] = {(cuuint64_t)Dys * 8, (cuuint64_t)Gp[0] * Dys * 8, (cuuint64_t)U * Gp[0] * Dys * 8};
    cuuint32_t box[4] = {(cuuint32_t)DY, (cuuint32_t)XW, (cuuint32_t)U, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void*)D, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(-3, "cuTensorMapEncodeTiled failed (%d): box {%d,%d,%d,1}", (int)r, DY, XW, U);
    return 0;
}

// tile depth in z (rows) for restricted plans (quadrature rows, rows=); whole-matrix plans choose theirs
constexpr int kT2Restricted = 24;

static bool plan_mma(DevProblem& dp, Plan& pl, int t2, int z0) {
    const int n = dp.n, P = dp.p, g = dp.g;
    if (P > 4 || g != P + 1 || getenv("SG_NO_MMA")) return false;
    int nthreads = 0;
    void* kfn = get_mma_kernel(n, dp.pr.form, P, dp.rational, &nthreads);
    if (!kfn) return false;
    const TileChoice tc = mma_tile(n, P, dp.pr.form, dp.rational);
    const MmaGeom M = mma_geom(n, P, dp.pr.form, dp.rational, tc.T0, tc.T1);
    if (M.total * 8 > (long)kSmemCap) return false;
    pl.mma = true;
    pl.kfn = kfn;
    pl.nthreads = nthreads;
    pl.T[0] = M.T0;
    pl.T[1] = M.T1;
    // z depth of a tile: deeper tiles recompute fewer halo planes per owned plane (the p element
    // layers below a tile are streamed again by the tile below); restricted plans (surrogate
    // quadrature rows, rows=) touch few planes per tile and prefer shallower tiles
    if (n == 3) {
        if (t2 <= 0) t2 = env_int("SG_T2_FULL", 0);
        if (t2 <= 0) {
            // whole-matrix plans: the fewest, deepest z tiles (<= kMmaT2 rows, equal depths) that still
            // give every SM several tiles (config 5: two tiles of 66 rows, 48.4 -> 41.5 ms for Poisson)
            int sms = 148, dev = 0;
            cudaGetDevice(&dev);  // the calling Call has selected its device
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            const int64_t xy = (int64_t)((dp.m[0] + M.T0 - 1) / M.T0) * ((dp.m[1] + M.T1 - 1) / M.T1);
            const int nzr = dp.m[2] - z0;  // planes from the grid origin
            int nz = (nzr + kMmaT2 - 1) / kMmaT2;
            while (xy * nz < 8LL * sms && nz < nzr) ++nz;
            t2 = (nzr + nz - 1) / nz;
        }
        pl.T[2] = std::min(kMmaT2, std::max(1, t2));
        pl.z0 = z0;
    } else {
        pl.T[2] = 1;
        pl.z0 = 0;
    }
    for (int d = 0; d < 3; ++d) pl.tgrid[d] = (dp.m[d] - (d == 2 ? pl.z0 : 0) + pl.T[d] - 1) / pl.T[d];
    pl.smem = M.total * sizeof(double);
    pl.ntiles = (int64_t)pl.tgrid[0] * pl.tgrid[1] * pl.tgrid[2];
    return true;
}

int plan_assembly(DevProblem& dp, Plan& pl, bool restricted, int t2, int z0) {
    // restricted plans: 24 row planes per tile; 3D p = 3 Poisson-type forms on deep meshes take 48 (config 5
    // surrogate call 13.09 -> 12.68 ms, 66: 12.74, 96: 12.85; mass and p = 2 are faster at 24: 6.65 vs 6.83, 1.85 vs 1.91)
    if (t2 <= 0 && restricted)
        t2 = env_int("SG_T2_RESTR", (dp.n == 3 && dp.pr.form == 0 && dp.p == 3 && dp.m[2] >= 96) ? 48 : kT2Restricted);
    pl.mma = false;
    pl.z0 = 0;
    if (plan_mma(dp, pl, t2, z0)) return 0;
    pl.kfn = get_kernel(dp.n, dp.pr.form, dp.p, dp.rational, &pl.kmax);
    if (!pl.kfn) return fail(-2, "no kernel instantiated for n=%d p=%d form=%d", dp.n, dp.p, dp.pr.form);
    pl.nthreads = 512;
    Layout L;
    int rc = choose_layout(dp, pl.kmax, pl.nthreads, L);
    if (rc) return rc;
    for (int d = 0; d < 3; ++d) {
        pl.T[d] = L.T[d];
        pl.tgrid[d] = (dp.m[d] + L.T[d] - 1) / L.T[d];
    }
    pl.ypad = L.ypad;
    for (int k = 0; k < 6; ++k) pl.off[k] = (int)L.off[k];
    pl.smem = L.total * sizeof(double);
    pl.ntiles = (int64_t)pl.tgrid[0] * pl.tgrid[1] * pl.tgrid[2];
    return 0;
}

void tile_box(const Plan& pl, const DevProblem& dp, int64_t t, int64_t lo[3], int64_t hi[3]) {
    int64_t tc[3] = {t % pl.tgrid[0], (t / pl.tgrid[0]) % pl.tgrid[1], t / ((int64_t)pl.tgrid[0] * pl.tgrid[1])};
    for (int d = 0; d < 3; ++d) {
        lo[d] = (d == 2 ? pl.z0 : 0) + tc[d] * pl.T[d];
        hi[d] = std::min<int64_t>(lo[d] + pl.T[d], dp.m[d]) - 1;
    }
}

int64_t tile_of_row(const Plan& pl, const DevProblem& dp, int64_t r) {
    const int64_t i0 = r % dp.m[0], i1 = (r / dp.m[0]) % dp.m[1], i2 = r / ((int64_t)dp.m[0] * dp.m[1]);
    return (i0 / pl.T[0]) + pl.tgrid[0] * ((i1 / pl.T[1]) + (int64_t)pl.tgrid[1] * ((i2 - pl.z0) / pl.T[2]));
}

int run_assembly(Call& c, DevProblem& dp, const Plan& pl, const std::vector<int>* tiles, const uint8_t* d_rowmask,
                 const int64_t* d_rowstart, int64_t slab_lo, int64_t slab_hi, int* d_indices, double* d_data,
                 unsigned long long* d_zeros) {
    if (tiles && tiles->empty()) return 0;
    c.hmark("run_assembly:start");
    int rc = compute_D(c, dp, pl, tiles, d_rowmask, slab_lo, slab_hi);
    c.hmark("run_assembly:D launched");
    if (rc) return rc;
    if (pl.mma) {
        MmaParams mp;
        memset(&mp, 0, sizeof(mp));
        for (int d = 0; d < 3; ++d) {
            mp.m[d] = dp.m[d];
            mp.S[d] = dp.S[d];
            mp.B[d] = dp.B[d];
            mp.canon[d] = d < dp.n ? dp.canon[d] : 0;
            mp.tgrid[d] = pl.tgrid[d];
            mp.Gp[d] = d < dp.n ? dp.S[d] * dp.g : 1;
        }
        mp.T2 = pl.T[2];
        mp.sol_w = dp.sol_w;
        mp.D = dp.D;
        mp.Dys = dp.Dys;
        mp.tma = getenv("SG_NO_TMA") ? 0 : 1;
        if (dp.n >= 2) {
            const TileChoice tc = mma_tile(dp.n, dp.p, dp.pr.form, dp.rational);
            const MmaGeom M = mma_geom(dp.n, dp.p, dp.pr.form, dp.rational, tc.T0, tc.T1);
            int rc2 = encode_dmap(&mp.dmap, dp.D, dp.Dys, mp.Gp, M.U, M.DY, M.XWp);
            if (rc2) return rc2;
        }
        mp.rowmask = d_rowmask;
        mp.rowstart = d_rowstart;
        mp.slab_lo = slab_lo;
        mp.slab_hi = slab_hi;
        mp.indices = d_indices;
        mp.data = d_data;
        mp.zeros = d_zeros;
        mp.z0 = pl.z0;
        mp.dbg = env_int("SG_K4_DBG", 0);
        if (!c.dmma) {
            c.dmma = (unsigned long long*)c.alloc(sizeof(unsigned long long) * kProfN, true);
            if (c.dmma) cudaMemsetAsync(c.dmma, 0, sizeof(unsigned long long) * kProfN, c.stream);
        }
        mp.dmma = c.dmma;
        int64_t nb = pl.ntiles;
        mp.run = 1;
        if (dp.n == 2) {
            // runs of tiles along y (column-major list): one CTA per run, ~8 waves of runs over the SMs
            std::vector<int> col;
            if (tiles) col = *tiles;
            else {
                col.resize(pl.ntiles);
                for (int64_t t = 0; t < pl.ntiles; ++t) col[t] = (int)t;
            }
            const int tg0 = pl.tgrid[0];
            if (tiles) {
                // bucket by x column, ascending tile order inside a column (counting sort)
                std::vector<int> start(tg0 + 1, 0);
                for (int t : col) start[t % tg0 + 1]++;
                for (int c2 = 0; c2 < tg0; ++c2) start[c2 + 1] += start[c2];
                std::vector<int> out(col.size());
                for (int t : col) out[start[t % tg0]++] = t;
                col.swap(out);
            } else {
                const int tg1 = (int)(pl.ntiles / tg0);
                for (int c0 = 0, k = 0; c0 < tg0; ++c0)
                    for (int c1 = 0; c1 < tg1; ++c1) col[k++] = c0 + tg0 * c1;
            }
            int sms = 148;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.dev);
            const int64_t want = 8LL * sms;
            mp.run = (int)std::max<int64_t>(1, ((int64_t)col.size() + want - 1) / want);
            if (const char* e = getenv("SG_RUN2D")) mp.run = std::max(1, atoi(e));
            mp.ntiles = (int)col.size();
            mp.tiles = (const int*)c.upload(col.data(), sizeof(int) * col.size());
            nb = ((int64_t)col.size() + mp.run - 1) / mp.run;
        } else if (dp.n == 3 && !getenv("SG_NO_RASTER")) {
            // 3D launch order: the CTAs resident together (one wave) cover a compact patch of tiles in (x, y)
            // and sweep z in step, so a D plane fetched for one tile's window is still in L2 for the
            // neighbours whose windows overlap it.  (Plain x-fastest order made a wave a 131 x 1 strip: the
            // y halo was re-read from HBM by the next wave, 25 GB of DRAM reads for the 6.4 GB D of config 5.)
            const TileChoice tc = mma_tile(3, dp.p, dp.pr.form, dp.rational);
            int sms = 148;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.dev);
            const int resident = sms * mma_minb(3, dp.p, dp.pr.form, dp.rational);
            // patch of PX x PY tiles, PX PY ~ resident, as square as possible in rows (PX T0 ~ PY T1)
            int PY = std::max(1, (int)std::lround(std::sqrt((double)resident * tc.T0 / tc.T1)));
            int PX = std::max(1, resident / PY);
            if (const char* e = getenv("SG_RASTER_PX")) PX = std::max(1, atoi(e));
            if (const char* e = getenv("SG_RASTER_PY")) PY = std::max(1, atoi(e));
            const int tg0 = pl.tgrid[0], tg1 = pl.tgrid[1];
            std::vector<int> ord;
            if (tiles) ord = *tiles;
            else {
                ord.resize(pl.ntiles);
                for (int64_t q = 0; q < pl.ntiles; ++q) ord[q] = (int)q;
            }
            const int npx = (tg0 + PX - 1) / PX;
            auto key = [&](int q) -> int64_t {
                const int c0 = q % tg0, c1 = (q / tg0) % tg1, c2 = q / (tg0 * tg1);
                const int64_t patch = (int64_t)(c1 / PY) * npx + c0 / PX;
                return (((int64_t)c2 * ((int64_t)npx * ((tg1 + PY - 1) / PY)) + patch) * PY + c1 % PY) * PX + c0 % PX;
            };
            std::vector<std::pair<int64_t, int>> ks(ord.size());
            for (size_t q = 0; q < ord.size(); ++q) ks[q] = {key(ord[q]), ord[q]};
            std::sort(ks.begin(), ks.end());
            for (size_t q = 0; q < ord.size(); ++q) ord[q] = ks[q].second;
            mp.tiles = (const int*)c.upload(ord.data(), sizeof(int) * ord.size());
            nb = (int64_t)ord.size();
            mp.ntiles = (int)nb;
        } else if (tiles) {
            mp.tiles = (const int*)c.upload(tiles->data(), sizeof(int) * tiles->size());
            nb = (int64_t)tiles->size();
            mp.ntiles = (int)nb;
        } else {
            mp.ntiles = (int)nb;
        }
        cudaFuncSetAttribute(pl.kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemOptinMax);
        void* args[] = {&mp};
        c.hmark("run_assembly:pre-launch");
        c.kbegin("assemble_mma");
        cudaError_t e = cudaLaunchKernel(pl.kfn, dim3((unsigned)nb), dim3(pl.nthreads), args, pl.smem, c.stream);
        c.kend();
        if (e != cudaSuccess)
            return fail(-3, "assembly (mma) launch failed: %s (smem %zu B, %lld tiles)", cudaGetErrorString(e), pl.smem, (long long)nb);
        dp.last_tiles = nb;
        c.free_temp(dp.D);  // stream ordered: released once the kernel is done with it
        dp.D = nullptr;
        return 0;
    }
    AsmParams prm;
    memset(&prm, 0, sizeof(prm));
    prm.n = dp.n;
    prm.p = dp.p;
    prm.g = dp.g;
    for (int d = 0; d < 3; ++d) {
        prm.m[d] = dp.m[d];
        prm.S[d] = dp.S[d];
        prm.B[d] = dp.B[d];
        prm.T[d] = pl.T[d];
        prm.tgrid[d] = pl.tgrid[d];
        prm.Gp[d] = d < dp.n ? dp.S[d] * dp.g : 1;
    }
    prm.sol_w = dp.sol_w;
    prm.D = dp.D;
    prm.Dys = dp.Dys;
    prm.ypad = pl.ypad;
    int* offs[6] = {&prm.off_B0, &prm.off_B1, &prm.off_D, &prm.off_T1, &prm.off_T2, &prm.off_misc};
    for (int k = 0; k < 6; ++k) *offs[k] = pl.off[k];
    prm.rowmask = d_rowmask;
    prm.rowstart = d_rowstart;
    prm.slab_lo = slab_lo;
    prm.slab_hi = slab_hi;
    prm.indices = d_indices;
    prm.data = d_data;
    prm.zeros = d_zeros;
    int64_t nblocks = pl.ntiles;
    if (tiles) {
        prm.tiles = (const int*)c.upload(tiles->data(), sizeof(int) * tiles->size());
        nblocks = (int64_t)tiles->size();
    }
    cudaFuncSetAttribute(pl.kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemOptinMax);
    void* args[] = {&prm};
    c.kbegin("assemble_tiles");
    cudaError_t e = cudaLaunchKernel(pl.kfn, dim3((unsigned)nblocks), dim3(pl.nthreads), args, pl.smem, c.stream);
    c.kend();
    if (e != cudaSuccess)
        return fail(-3, "assembly launch failed: %s (smem %zu B, %lld tiles)", cudaGetErrorString(e), pl.smem, (long long)nblocks);
    dp.last_tiles = nblocks;
    c.free_temp(dp.D);
    dp.D = nullptr;
    return 0;
}

int launch_assembly(Call& c, DevProblem& dp, const uint8_t* d_rowmask, const int64_t* d_rowstart, const int64_t* h_rows,
                    int64_t nrows, int64_t slab_lo, int64_t slab_hi, int* d_indices, double* d_data) {
    Plan pl;
    const bool full_slab = (slab_lo <= 0 && slab_hi >= dp.N);
    int t2 = 0, z0 = 0;
    if (!h_rows && !full_slab && dp.n == 3) {
        // row slab (multi-GPU): the tile grid starts at the slab's first plane and its z tiles split
        // the slab's planes evenly, so no tile straddles a slab edge (one halo per slab)
        const int64_t pl01 = (int64_t)dp.m[0] * dp.m[1];
        z0 = (int)(std::max<int64_t>(0, slab_lo) / pl01);
        const int planes = (int)((std::min<int64_t>(dp.N, slab_hi) - 1) / pl01) - z0 + 1;
        const int nz = (planes + kMmaT2 - 1) / kMmaT2;
        t2 = (planes + nz - 1) / nz;
    }
    c.hmark("launch_assembly:start");
    int rc = plan_assembly(dp, pl, h_rows != nullptr, t2, z0);
    c.hmark("launch_assembly:planned");
    if (rc) return rc;
    if (!h_rows && full_slab) return run_assembly(c, dp, pl, nullptr, d_rowmask, d_rowstart, slab_lo, slab_hi, d_indices, d_data, nullptr);
    const int64_t pl01 = (int64_t)dp.m[0] * dp.m[1];
    if (!h_rows && dp.n == 3 && slab_lo % pl01 == 0 && (slab_hi % pl01 == 0 || slab_hi >= dp.N)) {
        // plane-aligned slab on a grid starting at its first plane: the tiles of the z-tile rows
        // covering the slab's planes, a contiguous index range (no per-tile test)
        const int64_t ze = (std::min<int64_t>(dp.N, slab_hi) - 1) / pl01;
        const int64_t nzt = std::min<int64_t>(pl.tgrid[2], (ze - pl.z0) / pl.T[2] + 1);
        std::vector<int> tiles((size_t)(nzt * pl.tgrid[0] * pl.tgrid[1]));
        for (size_t t = 0; t < tiles.size(); ++t) tiles[t] = (int)t;
        c.hmark("launch_assembly:tiles");
        return run_assembly(c, dp, pl, &tiles, d_rowmask, d_rowstart, slab_lo, slab_hi, d_indices, d_data, nullptr);
    }
    std::vector<uint8_t> mark(pl.ntiles, 0);
    if (h_rows) {
        for (int64_t k = 0; k < nrows; ++k)
            if (h_rows[k] >= slab_lo && h_rows[k] < slab_hi) mark[tile_of_row(pl, dp, h_rows[k])] = 1;
    } else {
        for (int64_t t = 0; t < pl.ntiles; ++t) {
            int64_t lo[3], hi[3];
            tile_box(pl, dp, t, lo, hi);
            const int64_t flo = lo[0] + dp.m[0] * (lo[1] + (int64_t)dp.m[1] * lo[2]);
            const int64_t fhi = hi[0] + dp.m[0] * (hi[1] + (int64_t)dp.m[1] * hi[2]);
            if (fhi >= slab_lo && flo < slab_hi) mark[t] = 1;
        }
    }
    std::vector<int> tiles;
    for (int64_t t = 0; t < pl.ntiles; ++t)
        if (mark[t]) tiles.push_back((int)t);
    c.hmark("launch_assembly:tiles");
    return run_assembly(c, dp, pl, &tiles, d_rowmask, d_rowstart, slab_lo, slab_hi, d_indices, d_data, nullptr);
}

// ------------------------------------------------------------------------------------------
// checksum (fixed-order reduction: deterministic)
// ------------------------------------------------------------------------------------------
__global__ void checksum_partial(const int64_t* __restrict__ indptr, const double* __restrict__ data, int64_t nrows,
                                 double* __restrict__ part) {
    // part[block*5 + k]
    __shared__ double sh[5][256];
    double s[5] = {0, 0, 0, 0, 0};
    const int64_t per = (nrows + gridDim.x - 1) / gridDim.x;
    const int64_t r0 = blockIdx.x * per, r1 = min(nrows, r0 + per);
    for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
        double rs = 0.0;
        for (int64_t k = indptr[r]; k < indptr[r + 1]; ++k) {
            const double a = data[k];
            s[1] += a;
            s[2] += a * a;
            s[3] += fabs(a);
            rs += a;
        }
        s[0] += (double)(indptr[r + 1] - indptr[r]);
        s[4] += fabs(rs);
    }
    for (int k = 0; k < 5; ++k) sh[k][threadIdx.x] = s[k];
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w)
            for (int k = 0; k < 5; ++k) sh[k][threadIdx.x] += sh[k][threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0)
        for (int k = 0; k < 5; ++k) part[blockIdx.x * 5 + k] = sh[k][0];
}

}  // namespace sg

using namespace sg;

// ==========================================================================================
// C ABI
// ==========================================================================================
extern "C" {

const char* sg_last_error(void) { return g_err.c_str(); }
const char* sg_version(void) { return "surriga_b200 0.1.0 (sm_100a)"; }
int sg_max_degree(void) { return SG_MAX_P; }

int sg_last_dmma_count(int64_t* count) {
    if (!count) return fail(-1, "null argument");
    *count = (int64_t)g_last_dmma;
    return 0;
}

int sg_last_timing(double* ms_total, int32_t* launches) {
    if (ms_total) *ms_total = g_last_ms;
    if (launches) *launches = g_last_launches;
    return 0;
}

int sg_last_kernel_times(char* names, int32_t names_cap, double* ms, int32_t cap, int32_t* count) {
    std::string s;
    int k = 0;
    for (auto& kt : g_ktimes) {
        if (k < cap && ms) ms[k] = kt.second;
        if (!s.empty()) s += ",";
        s += kt.first;
        k++;
    }
    if (names && names_cap > 0) {
        strncpy(names, s.c_str(), names_cap - 1);
        names[names_cap - 1] = 0;
    }
    if (count) *count = k;
    return 0;
}

int sg_assemble(const sg_problem* prob, const int64_t* rows, int64_t nrows, const sg_exec* ex, sg_result** out) {
    if (!out) return fail(-1, "null output handle");
    *out = nullptr;
    Call c(ex);
    DevProblem dp;
    int rc = prepare_problem(c, prob, dp);
    if (rc) return rc;
    int64_t slab_lo = 0, slab_hi = dp.N;
    if (ex && ex->slab_hi > 0) {
        slab_lo = std::max<int64_t>(0, ex->slab_lo);
        slab_hi = std::min<int64_t>(dp.N, ex->slab_hi);
        if (slab_lo >= slab_hi) return fail(-1, "empty row slab");
    }
    for (int64_t k = 0; rows && k < nrows; ++k) {
        if (rows[k] < 0 || rows[k] >= dp.N) return fail(-1, "row index out of range");
        if (k && rows[k] <= rows[k - 1]) return fail(-1, "rows must be sorted and unique");
    }
    Dims D;
    for (int d = 0; d < 3; ++d) D.m[d] = dp.m[d];
    D.p = dp.p;
    sg_result* r = new sg_result();
    r->dev = c.dev;
    r->nrows_global = dp.N;
    r->row_lo = slab_lo;
    r->nrows = slab_hi - slab_lo;
    const int64_t N = dp.N;
    int64_t* rowstart = (int64_t*)c.alloc(sizeof(int64_t) * (N + 1), true);
    uint8_t* mask = nullptr;
    if (!rows) {
        // full pattern; slab rows rebased so the slab's first entry sits at 0
        int64_t base = 0;
        if (slab_lo > 0) {
            const int64_t i0 = slab_lo % dp.m[0], i1 = (slab_lo / dp.m[0]) % dp.m[1], i2 = slab_lo / ((int64_t)dp.m[0] * dp.m[1]);
            const int64_t t0 = pre1d(dp.m[0], dp.m[0], dp.p), t1 = pre1d(dp.m[1], dp.m[1], dp.p);
            base = pre1d(i2, dp.m[2], dp.p) * t1 * t0 +
                   cnt1d(i2, dp.m[2], dp.p) * (pre1d(i1, dp.m[1], dp.p) * t0 + cnt1d(i1, dp.m[1], dp.p) * pre1d(i0, dp.m[0], dp.p));
        }
        c.kbegin("indptr_full");
        indptr_full_kernel<<<(unsigned)((N + 1 + 255) / 256), 256, 0, c.stream>>>(D, N, base, rowstart);
        c.kend();
    } else {
        mask = (uint8_t*)c.alloc(N + 1, true);
        cudaMemsetAsync(mask, 0, N + 1, c.stream);
        std::vector<int64_t> sel;
        for (int64_t k = 0; k < nrows; ++k)
            if (rows[k] >= slab_lo && rows[k] < slab_hi) sel.push_back(rows[k]);
        if (!sel.empty()) {
            int64_t* drows = (int64_t*)c.upload(sel.data(), sizeof(int64_t) * sel.size());
            c.kbegin("rows_mask");
            scatter_mask_kernel<<<(unsigned)((sel.size() + 255) / 256), 256, 0, c.stream>>>(drows, (int64_t)sel.size(), mask);
            c.kend();
        }
        int64_t* counts = (int64_t*)c.alloc(sizeof(int64_t) * (N + 1), true);
        c.kbegin("row_counts");
        row_counts_kernel<<<(unsigned)((N + 1 + 255) / 256), 256, 0, c.stream>>>(D, N, mask, counts);
        c.kend();
        size_t tmp_bytes = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, counts, rowstart, N + 1, c.stream);
        void* tmp = c.alloc(tmp_bytes, true);
        c.kbegin("row_scan");
        cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, counts, rowstart, N + 1, c.stream);
        c.kend();
    }
    // nnz of this result: closed form (whole pattern) or the listed rows' counts -- no round trip
    int64_t nnz_lo = 0, nnz_hi = 0;
    if (!rows) {
        nnz_hi = nnz_before_row(dp, slab_hi) - nnz_before_row(dp, slab_lo);  // rowstart is already rebased
    } else {
        for (int64_t k = 0; k < nrows; ++k) {
            const int64_t rr = rows[k];
            if (rr < slab_lo || rr >= slab_hi) continue;
            const int64_t i0 = rr % dp.m[0], i1 = (rr / dp.m[0]) % dp.m[1], i2 = rr / ((int64_t)dp.m[0] * dp.m[1]);
            nnz_hi += cnt1d(i0, dp.m[0], dp.p) * cnt1d(i1, dp.m[1], dp.p) * cnt1d(i2, dp.m[2], dp.p);
        }
    }
    r->nnz = nnz_hi - nnz_lo;
    // result arrays (owned by the handle)
    r->indptr = (int64_t*)c.alloc(sizeof(int64_t) * (r->nrows + 1), false);
    r->indices = (int*)c.alloc(sizeof(int) * std::max<int64_t>(r->nnz, 1), false);
    r->data = (double*)c.alloc(sizeof(double) * std::max<int64_t>(r->nnz, 1), false);
    if (!r->indptr || !r->indices || !r->data) {
        delete r;
        return fail(-4, "device allocation failed (nnz=%lld)", (long long)(nnz_hi - nnz_lo));
    }
    // rowstart relative to the slab start -> write positions directly into the result arrays
    if (nnz_lo != 0) {
        // shift: rowstart -= nnz_lo (only for rows of this slab; others are skipped by the kernel)
        c.kbegin("rebase");
        rebase_kernel<<<(unsigned)((N + 1 + 255) / 256), 256, 0, c.stream>>>(rowstart, N + 1, nnz_lo);
        c.kend();
    }
    cudaMemcpyAsync(r->indptr, rowstart + slab_lo, sizeof(int64_t) * (r->nrows + 1), cudaMemcpyDeviceToDevice, c.stream);
    if (r->nnz > 0) {
        rc = launch_assembly(c, dp, mask, rowstart, rows, nrows, slab_lo, slab_hi, r->indices, r->data);
        if (rc) {
            sg_result_free(r);
            return rc;
        }
    }
    r->stream_hint = nullptr;
    rc = c.finish();
    if (rc) {
        sg_result_free(r);
        return rc;
    }
    cudaStreamSynchronize(c.stream);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        sg_result_free(r);
        return fail(-3, "CUDA error after assembly: %s", cudaGetErrorString(e));
    }
    c.record_timing();
    r->tiles = dp.last_tiles;
    if (!rows) {
        r->analytic = true;
        r->p = dp.p;
        for (int d = 0; d < 3; ++d) r->m[d] = dp.m[d];
    }
    *out = r;
    return 0;
}

int sg_result_sizes(const sg_result* r, int64_t* nrows, int64_t* nnz) {
    if (!r) return fail(-1, "null result");
    if (nrows) *nrows = r->nrows;
    if (nnz) *nnz = r->nnz;
    return 0;
}

}  // extern "C"

namespace sg {
// Device -> host copy of large result arrays.  PCIe D2H runs at ~57 GB/s into pinned memory, but
// pinning the caller's buffer costs more than it saves (2-8 GB/s), so the copy goes through a
// pinned staging ring (R x 64 MB): the DMA engine fills slot k+1.. while a persistent pool of host
// threads copies slot k into the caller's pageable buffer (first-touch page faults spread over the
// pool, transparent huge pages requested on the destination).
struct CopyPool {
    std::vector<std::thread> th;
    std::mutex mu;
    std::condition_variable cv, done_cv;
    struct Task { char* dst; const char* src; size_t len; std::atomic<int>* left; std::function<void()> fn; };
    std::deque<Task> q;
    bool stop = false;
    explicit CopyPool(int n) {
        for (int t = 0; t < n; ++t)
            th.emplace_back([this] {
                for (;;) {
                    Task tk;
                    {
                        std::unique_lock<std::mutex> lk(mu);
                        cv.wait(lk, [this] { return stop || !q.empty(); });
                        if (stop && q.empty()) return;
                        tk = q.front();
                        q.pop_front();
                    }
                    if (tk.fn) tk.fn();
                    else memcpy(tk.dst, tk.src, tk.len);
                    if (tk.left->fetch_sub(1) == 1) {
                        std::lock_guard<std::mutex> lk(mu);
                        done_cv.notify_all();
                    }
                }
            });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> lk(mu);
            stop = true;
        }
        cv.notify_all();
        for (auto& t : th) t.join();
    }
    void submit(char* dst, const char* src, size_t n, std::atomic<int>* left, size_t piece) {
        const int np = (int)((n + piece - 1) / piece);
        left->store(np);
        {
            std::lock_guard<std::mutex> lk(mu);
            for (int p = 0; p < np; ++p) {
                const size_t lo = (size_t)p * piece, len = std::min(piece, n - lo);
                q.push_back({dst + lo, src + lo, len, left});
            }
        }
        wake(np);
    }
    void wake(int tasks) {
        // as many workers as tasks: waking all 16 for a 4-piece copy cost more than the copy (VM hosts)
        if (tasks >= (int)th.size()) cv.notify_all();
        else
            for (int t = 0; t < tasks; ++t) cv.notify_one();
    }
    void run(std::vector<std::function<void()>>& fns, std::atomic<int>* left) {
        left->store((int)fns.size());
        {
            std::lock_guard<std::mutex> lk(mu);
            for (auto& f : fns) q.push_back({nullptr, nullptr, 0, left, f});
        }
        wake((int)fns.size());
    }
    void wait(std::atomic<int>* left, bool help = false) {
        // help: the waiting thread runs queued tasks itself (workers parked on an idle VM vCPU can take
        // ~100 us to wake); not in the D2H ring, whose thread must stay free to issue the next chunk
        std::unique_lock<std::mutex> lk(mu);
        while (left->load() != 0) {
            if (help && !q.empty()) {
                Task tk = q.front();
                q.pop_front();
                lk.unlock();
                if (tk.fn) tk.fn();
                else memcpy(tk.dst, tk.src, tk.len);
                lk.lock();
                if (tk.left->fetch_sub(1) == 1) done_cv.notify_all();
                continue;
            }
            done_cv.wait(lk);
        }
    }
};
static CopyPool& copy_pool() {
    static CopyPool pool((int)std::max(2u, std::min(16u, std::thread::hardware_concurrency())));
    return pool;
}
static void copy_pool_run(std::vector<std::function<void()>>& fns, std::atomic<int>* left) { copy_pool().run(fns, left); }
static void copy_pool_wait(std::atomic<int>* left) { copy_pool().wait(left, true); }

static void pool_memcpy(void* dst, const void* src, size_t n) {
    // packs pinned staging for an upload: streaming stores (stream_copy, sg_hostcols.cpp)
    const size_t piece = std::max<size_t>(512u << 10, (n + 3) / 4);
    std::vector<std::function<void()>> fns;
    for (size_t lo = 0; lo < n; lo += piece) {
        const size_t len = std::min(piece, n - lo);
        fns.push_back([=] { stream_copy((char*)dst + lo, (const char*)src + lo, len); });
    }
    std::atomic<int> left(0);
    copy_pool().run(fns, &left);
    copy_pool().wait(&left, true);
}

constexpr int kRingMax = 16;
struct Stager {
    int dev = -1;
    cudaStream_t st = nullptr;
    char* buf[kRingMax] = {};
    cudaEvent_t ev[kRingMax];
    std::atomic<int> left[kRingMax];
    int ring = 0;
    size_t chunk = 0, piece = 0;
};
static thread_local Stager g_stage;

static void want_huge_pages(void* p, size_t n) {
    const uintptr_t a = ((uintptr_t)p + (2u << 20) - 1) & ~(uintptr_t)((2u << 20) - 1);
    const uintptr_t e = ((uintptr_t)p + n) & ~(uintptr_t)((2u << 20) - 1);
    if (e > a) madvise((void*)a, e - a, MADV_HUGEPAGE);
}

static size_t env_size(const char* name, size_t dflt) {
    const char* v = getenv(name);
    return v ? (size_t)atof(v) : dflt;
}
static int stager_init(int dev) {
    Stager& S = g_stage;
    if (S.dev != dev || !S.buf[0]) {
        for (int k = 0; k < kRingMax; ++k)
            if (S.buf[k]) cudaFreeHost(S.buf[k]), S.buf[k] = nullptr;
        // ring geometry (tunable for experiments; defaults measured on the B200 host)
        S.chunk = env_size("SG_D2H_CHUNK_KB", 64 * 1024) << 10;
        S.ring = (int)std::min<size_t>(kRingMax, std::max<size_t>(2, env_size("SG_D2H_RING", 4)));
        S.piece = std::max<size_t>(64 << 10, env_size("SG_D2H_PIECE_KB", 4096) << 10);
        for (int k = 0; k < S.ring; ++k)
            if (cudaHostAlloc((void**)&S.buf[k], S.chunk, cudaHostAllocDefault) != cudaSuccess) {
                S.buf[0] = nullptr;
                return fail(-4, "pinned staging allocation failed");
            }
        if (!S.st) {
            cudaStreamCreateWithFlags(&S.st, cudaStreamNonBlocking);
            for (int k = 0; k < kRingMax; ++k) cudaEventCreateWithFlags(&S.ev[k], cudaEventDisableTiming);
        }
        S.dev = dev;
    }
    copy_pool();
    return 0;
}

static int d2h(void* dst, const void* src, size_t bytes, int dev) {
    if (bytes == 0) return 0;
    if (bytes < (8u << 20)) {
        if (cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost) != cudaSuccess) return fail(-3, "D2H copy failed");
        return 0;
    }
    // destinations registered with the driver (reused host result buffers, _lib._HostPool): DMA
    // straight into them, no staging copy
    cudaPointerAttributes pa;
    if (cudaPointerGetAttributes(&pa, dst) == cudaSuccess && pa.type == cudaMemoryTypeHost) {
        cudaStream_t st = nullptr;
        cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
        const cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st);
        const cudaError_t e2 = cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
        if (e != cudaSuccess || e2 != cudaSuccess) return fail(-3, "D2H copy failed");
        return 0;
    }
    cudaGetLastError();  // clear a possible "invalid value" from the attribute query
    if (int rc = stager_init(dev)) return rc;
    Stager& S = g_stage;
    const size_t chunk = S.chunk, piece = S.piece;
    const int kRing = S.ring;
    want_huge_pages(dst, bytes);
    CopyPool& pool = copy_pool();
    const size_t nch = (bytes + chunk - 1) / chunk;
    auto issue = [&](size_t k) {
        const size_t off = k * chunk, len = std::min(chunk, bytes - off);
        cudaMemcpyAsync(S.buf[k % kRing], (const char*)src + off, len, cudaMemcpyDeviceToHost, S.st);
        cudaEventRecord(S.ev[k % kRing], S.st);
    };
    for (size_t k = 0; k < std::min<size_t>(nch, kRing); ++k) issue(k);
    for (size_t k = 0; k < nch; ++k) {
        const int s = (int)(k % kRing);
        if (cudaEventSynchronize(S.ev[s]) != cudaSuccess) return fail(-3, "D2H copy failed");
        const size_t off = k * chunk, len = std::min(chunk, bytes - off);
        pool.submit((char*)dst + off, S.buf[s], len, &S.left[s], piece);
        if (k >= 1) {  // slot of chunk k-1 is free once its host copy finished: refill it
            const int ps = (int)((k - 1) % kRing);
            pool.wait(&S.left[ps]);
            if (k - 1 + kRing < nch) issue(k - 1 + kRing);
        }
    }
    pool.wait(&S.left[(nch - 1) % kRing]);
    return 0;
}
}  // namespace sg

extern "C" {

int sg_host_register(void* ptr, size_t bytes) {
    if (!ptr || !bytes) return 0;
    const cudaError_t e = cudaHostRegister(ptr, bytes, cudaHostRegisterDefault);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(-3, "cudaHostRegister failed: %s", cudaGetErrorString(e));
    }
    return 0;
}

int sg_host_unregister(void* ptr) {
    if (!ptr) return 0;
    const cudaError_t e = cudaHostUnregister(ptr);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(-3, "cudaHostUnregister failed: %s", cudaGetErrorString(e));
    }
    return 0;
}

int sg_host_staging_init(int device) {
    cudaSetDevice(device);
    return sg::stager_init(device);
}

int sg_result_copy_i64(const sg_result* r, int64_t* indptr, int32_t* indices, double* data) {
    if (!r) return fail(-1, "null result");
    cudaSetDevice(r->dev);
    // every call that creates a result synchronises its stream before returning the handle, so no
    // device-wide synchronisation here: a copy can overlap the next assembly on the same device
    int rc = 0;
    std::vector<int64_t> ipv;
    int64_t* ip = indptr;
    if (!ip && indices && r->analytic) {
        ipv.resize(r->nrows + 1);
        ip = ipv.data();
    }
    if (ip && (rc = d2h(ip, r->indptr, sizeof(int64_t) * (r->nrows + 1), r->dev))) return rc;
    if (r->nnz > 0) {
        if (indices && r->analytic && !getenv("SG_COPY_INDICES")) {
            // closed-form columns on the host pool, concurrent with the values' D2H
            std::atomic<int> left(0);
            std::vector<std::function<void()>> fns;
            const int nt = 64;  // small tasks: staging copies of a concurrent pageable D2H interleave in the queue
            int64_t r0 = 0;
            for (int t = 0; t < nt && r0 < r->nrows; ++t) {
                int64_t r1 = r->nrows;
                if (t + 1 < nt) {  // balance by entries
                    const int64_t target = ip[0] + (ip[r->nrows] - ip[0]) * (t + 1) / nt;
                    r1 = std::max<int64_t>(r0, (int64_t)(std::upper_bound(ip, ip + r->nrows + 1, target) - ip) - 1);
                }
                fns.push_back([r, ip, indices, r0, r1] { gen_columns(r0, r1, r->row_lo, r->m, r->p, indices + (ip[r0] - ip[0])); });
                r0 = r1;
            }
            copy_pool().run(fns, &left);
            if (data) rc = d2h(data, r->data, sizeof(double) * r->nnz, r->dev);
            copy_pool().wait(&left);
            if (rc) return rc;
        } else {
            if (indices && (rc = d2h(indices, r->indices, sizeof(int32_t) * r->nnz, r->dev))) return rc;
            if (data && (rc = d2h(data, r->data, sizeof(double) * r->nnz, r->dev))) return rc;
        }
    }
    return 0;
}

int sg_result_copy(const sg_result* r, int32_t* indptr, int32_t* indices, double* data) {
    if (!r) return fail(-1, "null result");
    if (r->nnz >= INT32_MAX) return fail(-1, "nnz exceeds int32; use sg_result_copy_i64");
    std::vector<int64_t> ip(r->nrows + 1);
    int rc = sg_result_copy_i64(r, ip.data(), indices, data);
    if (rc) return rc;
    if (indptr)
        for (int64_t k = 0; k <= r->nrows; ++k) indptr[k] = (int32_t)ip[k];
    return 0;
}

int sg_result_device_ptrs(const sg_result* r, void** indptr_i64, void** indices_i32, void** data_f64) {
    if (!r) return fail(-1, "null result");
    const_cast<sg_result*>(r)->exported = true;
    if (indptr_i64) *indptr_i64 = r->indptr;
    if (indices_i32) *indices_i32 = r->indices;
    if (data_f64) *data_f64 = r->data;
    return 0;
}

int sg_result_checksum(const sg_result* r, double out[5]) {
    if (!r) return fail(-1, "null result");
    cudaSetDevice(r->dev);
    const int nb = 256;
    double* part = nullptr;
    cudaMalloc(&part, sizeof(double) * nb * 5);
    if (r->nrows > 0) checksum_partial<<<nb, 256>>>(r->indptr, r->data, r->nrows, part);
    else cudaMemset(part, 0, sizeof(double) * nb * 5);
    std::vector<double> h(nb * 5);
    cudaMemcpy(h.data(), part, sizeof(double) * nb * 5, cudaMemcpyDeviceToHost);
    cudaFree(part);
    for (int k = 0; k < 5; ++k) {
        double s = 0.0;
        for (int b = 0; b < nb; ++b) s += h[b * 5 + k];
        out[k] = s;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(-3, "checksum failed: %s", cudaGetErrorString(e));
    return 0;
}

int sg_result_free(sg_result* r) {
    if (!r) return 0;
    cudaSetDevice(r->dev);
    // the library's own calls on a result synchronise their streams before returning, so a result
    // whose device pointers were never handed out is freed without waiting for other threads' work;
    // once sg_result_device_ptrs exported them, a consumer may still read them on any stream: wait
    // for the whole device before the memory can be reused
    if (r->exported) cudaDeviceSynchronize();
    if (r->indptr) cudaFreeAsync(r->indptr, 0);
    if (r->own_indices) cudaFreeAsync(r->own_indices, 0);
    else if (r->indices) cudaFreeAsync(r->indices, 0);
    if (r->own_data) cudaFreeAsync(r->own_data, 0);
    else if (r->data) cudaFreeAsync(r->data, 0);
    cudaStreamSynchronize(0);
    delete r;
    return 0;
}

}  // extern "C"
