// host copy rates into pinned staging (why does packing a 2 MB upload take ~0.25 ms?)
// nvcc -O2 -o hostcopy hostcopy.cu && ./hostcopy
#include <cuda_runtime.h>
#include <emmintrin.h>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
static double now() { return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
static void nt(char* d, const char* s, size_t n) {
    for (size_t i = 0; i < n / 16; ++i) _mm_stream_si128((__m128i*)d + i, _mm_loadu_si128((const __m128i*)s + i));
    _mm_sfence();
}
int main() {
    const size_t n = 2165248;
    char* pin; cudaMallocHost((void**)&pin, 64 << 20);
    std::vector<char> src(n, 1), dst(n);
    memset(pin, 0, 64 << 20);
    printf("hardware_concurrency %u\n", std::thread::hardware_concurrency());
    for (int rep = 0; rep < 3; ++rep) {
        double t0 = now(); memcpy(pin, src.data(), n); double t1 = now();
        nt(pin, src.data(), n); double t2 = now();
        memcpy(dst.data(), src.data(), n); double t3 = now();
        printf("memcpy->pinned %.1f us  nt->pinned %.1f us  memcpy->heap %.1f us\n", t1 - t0, t2 - t1, t3 - t2);
    }
    for (int T : {1, 2, 4, 8, 16}) {
        double best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
            double t0 = now();
            std::vector<std::thread> th;
            size_t piece = (n + T - 1) / T;
            for (int t = 0; t < T; ++t) th.emplace_back([&, t] { size_t lo = t * piece, len = std::min(piece, n - lo); nt(pin + lo, src.data() + lo, len & ~15ul); });
            for (auto& x : th) x.join();
            best = std::min(best, now() - t0);
        }
        printf("threads %2d nt (incl. spawn) %.1f us\n", T, best);
    }
    char* d; cudaMalloc(&d, n);
    cudaStream_t st; cudaStreamCreate(&st);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 3; ++rep) {
            if (mode == 0) memcpy(pin, src.data(), n);
            if (mode == 1) nt(pin, src.data(), n);
            if (mode == 2) { std::thread t([&] { memcpy(pin, src.data(), n); }); t.join(); }
            cudaEventRecord(a, st); cudaMemcpyAsync(d, pin, n, cudaMemcpyHostToDevice, st); cudaEventRecord(b, st);
            cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b);
            printf("mode %d (0 memcpy,1 nt,2 other-thread memcpy) h2d %.1f us\n", mode, ms * 1e3);
        }
    }
    return 0;
}
