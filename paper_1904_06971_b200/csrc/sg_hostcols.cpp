// Host-side closed-form column indices of full-pattern CSR rows (sg_result_copy*): the int32 columns
// of rows [r0, r1) written to out (the slice of the caller's indices array starting at row r0).
// Interior rows (all 2p+1 neighbours per direction present) are the row index plus one fixed shift
// table; the stream is staged in a small buffer and written with non-temporal stores (no
// read-for-ownership of the destination lines: the copy runs next to a 57 GB/s DMA into host memory).
// Compiled twice (Makefile): -mavx2 -DSG_GEN_NAME=gen_columns_avx2 and -DSG_GEN_NAME=gen_columns_base;
// sg_api.cu dispatches on the CPU at run time.  The base build also holds stream_copy (SSE2).
#ifdef __AVX2__
#include <immintrin.h>
#else
#include <emmintrin.h>
#endif
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <vector>

namespace sg {

namespace {

struct Sink {
    int32_t* dst;
    int32_t buf[8192 + 512];
    int n = 0;
    void flush() {
        int32_t* d = dst;
        int i = 0;
#ifdef __AVX2__
        {
            // head up to 32-byte alignment, streamed body, tail
            while (i < n && (reinterpret_cast<uintptr_t>(d + i) & 31)) {
                d[i] = buf[i];
                ++i;
            }
            for (; i + 8 <= n; i += 8) _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i), _mm256_loadu_si256(reinterpret_cast<const __m256i*>(buf + i)));
        }
#endif
        for (; i < n; ++i) d[i] = buf[i];
        dst += n;
        n = 0;
    }
};

void gen(int64_t r0, int64_t r1, int64_t row_lo, const int64_t* m, int p, int32_t* out) {
    const int64_t m0 = m[0], m1 = m[1], m2 = m[2], m01 = m0 * m1;
    const int W = 2 * p + 1;
    std::vector<int32_t> shift((size_t)W * W * W);
    int k = 0;
    for (int d2 = -p; d2 <= p; ++d2)
        for (int d1 = -p; d1 <= p; ++d1)
            for (int d0 = -p; d0 <= p; ++d0) shift[k++] = (int32_t)(d0 + m0 * d1 + m01 * d2);
    const int P = k;
    Sink* s = new Sink();
    s->dst = out;
    for (int64_t rr = r0; rr < r1; ++rr) {
        const int64_t row = row_lo + rr;
        const int64_t i0 = row % m0, i1 = (row / m0) % m1, i2 = row / m01;
        if (s->n + P > 8192) s->flush();
        int32_t* o = s->buf + s->n;
        if (i0 >= p && i0 + p < m0 && i1 >= p && i1 + p < m1 && i2 >= p && i2 + p < m2) {
            const int32_t rv = (int32_t)row;
            for (int j = 0; j < P; ++j) o[j] = rv + shift[j];
            s->n += P;
        } else {
            const int64_t a0 = std::max<int64_t>(0, i0 - p), b0 = std::min<int64_t>(m0 - 1, i0 + p);
            const int64_t a1 = std::max<int64_t>(0, i1 - p), b1 = std::min<int64_t>(m1 - 1, i1 + p);
            const int64_t a2 = std::max<int64_t>(0, i2 - p), b2 = std::min<int64_t>(m2 - 1, i2 + p);
            int c = 0;
            for (int64_t j2 = a2; j2 <= b2; ++j2)
                for (int64_t j1 = a1; j1 <= b1; ++j1) {
                    const int32_t base = (int32_t)(m01 * j2 + m0 * j1);
                    for (int64_t j0 = a0; j0 <= b0; ++j0) o[c++] = base + (int32_t)j0;
                }
            s->n += c;
        }
    }
    s->flush();
#ifdef __AVX2__
    _mm_sfence();
#endif
    delete s;
}

}  // namespace

void SG_GEN_NAME(int64_t r0, int64_t r1, int64_t row_lo, const int64_t* m, int p, int32_t* out) {
    gen(r0, r1, row_lo, m, p, out);
}

#ifndef __AVX2__
// Copy into pinned staging memory that a DMA engine reads next: streaming (non-temporal) stores leave
// no dirty lines in the writing core's cache, so the device's reads are not served by snoops.  A 2 MB
// upload packed by the copy pool ran at ~7 GB/s over PCIe with plain stores, ~45 GB/s like this.
void stream_copy(void* dst, const void* src, size_t n) {
    char* d = (char*)dst;
    const char* s = (const char*)src;
    const size_t head = std::min(n, (size_t)((16 - ((uintptr_t)d & 15)) & 15));
    memcpy(d, s, head);
    d += head;
    s += head;
    n -= head;
    const size_t nv = n / 16;
    for (size_t i = 0; i < nv; ++i)
        _mm_stream_si128((__m128i*)d + i, _mm_loadu_si128((const __m128i*)s + i));
    memcpy(d + nv * 16, s + nv * 16, n - nv * 16);
    _mm_sfence();
}
#endif

}  // namespace sg
