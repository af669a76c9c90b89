// MatrixMarket writer (reference: surriga/assembly.py:304-312
// `save_matrix_market(path, A)` -> scipy mmwrite(field="real", precision=16, symmetry=...)).
//
// The only on-disk output of the assembly path.  The reference prints 16 significant digits,
// which does not round-trip every double (its own test_assembly.py:182-190 asks for a bitwise
// round trip); this writer prints the shortest representation that reads back to the same double
// (std::to_chars), so load_matrix_market(save_matrix_market(A)) is bitwise A.
//
// Layout as mmwrite's coordinate format: header, "%", "N M nnz", then 1-based "i j value" lines;
// symmetric matrices store the lower triangle (j <= i).  Rows are formatted in parallel by a pool
// of host threads into per-thread buffers (balanced by entry count) and written in order, block by
// block, so the memory held stays bounded for the 22 GB text of a config-5 matrix.
#include <charconv>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/surriga_b200.h"
#include "sg_internal.h"

namespace sg {

static void format_rows(const int64_t* ip, const int32_t* ix, const double* a, int64_t r0, int64_t r1, int64_t row_base,
                        bool lower, std::string& out) {
    char buf[96];
    for (int64_t i = r0; i < r1; ++i) {
        const int64_t gi = i + row_base;
        for (int64_t k = ip[i]; k < ip[i + 1]; ++k) {
            const int64_t j = ix[k];
            if (lower && j > gi) continue;
            char* p = buf;
            p = std::to_chars(p, buf + sizeof(buf), gi + 1).ptr;
            *p++ = ' ';
            p = std::to_chars(p, buf + sizeof(buf), j + 1).ptr;
            *p++ = ' ';
            p = std::to_chars(p, buf + sizeof(buf), a[k]).ptr;  // shortest round-trip form
            *p++ = '\n';
            out.append(buf, p - buf);
        }
    }
}

static int write_mm(const char* path, int64_t nrows, int64_t ncols, const int64_t* ip, const int32_t* ix, const double* a,
                    int symmetric, int nthreads) {
    if (!path) return fail(-1, "null path");
    if (symmetric && nrows != ncols) return fail(-1, "a symmetric MatrixMarket file needs a square matrix");
    if (nthreads <= 0) nthreads = (int)std::max(1u, std::thread::hardware_concurrency());
    FILE* f = fopen(path, "wb");
    if (!f) return fail(-5, "cannot open %s for writing", path);
    int64_t count = 0;
    if (symmetric) {
        for (int64_t i = 0; i < nrows; ++i)
            for (int64_t k = ip[i]; k < ip[i + 1]; ++k) count += ix[k] <= i;
    } else {
        count = ip[nrows];
    }
    fprintf(f, "%%%%MatrixMarket matrix coordinate real %s\n%%\n%lld %lld %lld\n", symmetric ? "symmetric" : "general",
            (long long)nrows, (long long)ncols, (long long)count);
    // blocks of about 8M entries, each split over the threads by entry count
    const int64_t block = 8 << 20;
    std::vector<std::string> bufs(nthreads);
    int64_t r = 0;
    bool ok = true;
    while (r < nrows && ok) {
        int64_t rend = r;
        while (rend < nrows && ip[rend] - ip[r] < block) ++rend;
        if (rend == r) rend = r + 1;
        const int64_t e0 = ip[r], e1 = ip[rend];
        std::vector<int64_t> cut(nthreads + 1, r);
        cut[nthreads] = rend;
        for (int t = 1; t < nthreads; ++t) {
            const int64_t target = e0 + (e1 - e0) * t / nthreads;
            int64_t lo = cut[t - 1], hi = rend;
            while (lo < hi) {  // first row whose start >= target
                const int64_t mid = (lo + hi) / 2;
                if (ip[mid] < target) lo = mid + 1;
                else hi = mid;
            }
            cut[t] = lo;
        }
        std::vector<std::thread> th;
        for (int t = 0; t < nthreads; ++t) {
            bufs[t].clear();
            th.emplace_back([&, t] { format_rows(ip, ix, a, cut[t], cut[t + 1], 0, symmetric != 0, bufs[t]); });
        }
        for (auto& x : th) x.join();
        for (int t = 0; t < nthreads && ok; ++t) ok = fwrite(bufs[t].data(), 1, bufs[t].size(), f) == bufs[t].size();
        r = rend;
    }
    ok = (fclose(f) == 0) && ok;
    return ok ? 0 : fail(-5, "write error on %s", path);
}

}  // namespace sg

using namespace sg;

extern "C" {

int sg_write_matrix_market_host(const char* path, int64_t nrows, int64_t ncols, const int64_t* indptr, const int32_t* indices,
                                const double* data, int32_t symmetric, int32_t nthreads) {
    if (!indptr || (indptr[nrows] > 0 && (!indices || !data))) return fail(-1, "null argument");
    return write_mm(path, nrows, ncols, indptr, indices, data, symmetric, nthreads);
}

int sg_write_matrix_market(const sg_result* A, int64_t ncols, const char* path, int32_t symmetric, int32_t nthreads) {
    if (!A) return fail(-1, "null result");
    if (A->row_lo != 0 || A->nrows != A->nrows_global) return fail(-1, "MatrixMarket output needs a whole matrix");
    std::vector<int64_t> ip(A->nrows + 1);
    std::vector<int32_t> ix(std::max<int64_t>(A->nnz, 1));
    std::vector<double> d(std::max<int64_t>(A->nnz, 1));
    int rc = sg_result_copy_i64(A, ip.data(), ix.data(), d.data());
    if (rc) return rc;
    return write_mm(path, A->nrows, ncols > 0 ? ncols : A->nrows, ip.data(), ix.data(), d.data(), symmetric, nthreads);
}

}  // extern "C"
