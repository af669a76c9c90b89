// DMMA (mma.sync m8n8k4 f64) latency / ILP sweep: one CTA per SM, W warps, C independent chains per warp.
#include <cstdio>
#include <cuda_runtime.h>
template <int C>
__global__ void k(double* out, int iters, long long* cyc) {
    double acc[C][2];
    const double a = threadIdx.x * 1e-9, b = 1.0 + 1e-12;
#pragma unroll
    for (int c = 0; c < C; ++c) acc[c][0] = acc[c][1] = c;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < C; ++c)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a), "d"(b));
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int c = 0; c < C; ++c) s += acc[c][0] + acc[c][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int C>
void run(int warps, double* d, long long* cyc) {
    const int iters = 4096;
    k<C><<<148, warps * 32>>>(d, 64, cyc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<C><<<148, warps * 32>>>(d, iters, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    double tf = 148.0 * warps * 32 * 2.0 * 256 / 32 * C * iters * 1.0 / (ms * 1e-3) / 1e12 * 1.0;
    // per warp-instruction: 8x8x4 = 256 FMA = 512 flop
    tf = 148.0 * warps * C * (double)iters * 512.0 / (ms * 1e-3) / 1e12;
    printf("warps/SM %2d chains/warp %d : %.2f TFLOP/s  cycles per chain step %.1f\n", warps, C, tf, (double)c / iters);
}
int main() {
    double* d; long long* cyc;
    cudaMalloc(&d, 148 * 1024 * 8); cudaMalloc(&cyc, 8);
    for (int w : {1, 4, 8, 16}) { run<1>(w, d, cyc); run<2>(w, d, cyc); run<4>(w, d, cyc); run<8>(w, d, cyc); }
    return 0;
}
