// DMMA (mma.sync m8n8k4 f64) latency / throughput per SM: W warps, C independent accumulator chains
// per warp, N dependent steps per chain.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_lat dmma_lat.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int C>
__global__ void k(double* out, int N, long long* cyc) {
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    double acc[C][2];
    for (int c = 0; c < C; ++c) acc[c][0] = acc[c][1] = c;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int c = 0; c < C; ++c)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a), "d"(b));
    }
    __syncthreads();
    long long t1 = clock64();
    double s = 0;
    for (int c = 0; c < C; ++c) s += acc[c][0] + acc[c][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int C>
void run(int W, int N) {
    double* o; long long* c; cudaMalloc(&o, 148 * 1024 * 8); cudaMalloc(&c, 8);
    k<C><<<148, 32 * W>>>(o, N, c);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<C><<<148, 32 * W>>>(o, N, c);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long cy; cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
    const double dmma_per_sm = (double)W * C * N;
    printf("warps %2d chains %d: %.1f cycles per dependent step, %.2f cycles per DMMA per SM, %.1f TF/s\n", W, C,
           (double)cy / N, (double)cy / dmma_per_sm, 148.0 * dmma_per_sm * 512 / (ms * 1e-3) / 1e12);
    cudaFree(o); cudaFree(c);
}
int main() {
    const int N = 4096;
    for (int W : {1, 4, 8, 16, 20, 24, 32}) { run<1>(W, N); run<2>(W, N); run<4>(W, N); }
    return 0;
}
