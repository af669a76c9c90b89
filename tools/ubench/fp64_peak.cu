// fp64 throughput microbenchmark: DFMA (SIMT) vs DMMA (mma.sync m8n8k4 f64).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters) {
    double a[8], b = 1.0000001, c = 0.9999999;
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
    }
    double s = 0;
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 1234.5) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
    double acc[4][2];
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
    for (int k = 0; k < 4; ++k) acc[k][0] = acc[k][1] = 0.0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(acc[k][0]), "+d"(acc[k][1]) : "d"(a), "d"(b));
    }
    double s = 0;
    for (int k = 0; k < 4; ++k) s += acc[k][0] + acc[k][1];
    if (s == 1234.5) out[0] = s;
}

int main() {
    double* d;
    cudaMalloc(&d, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
        int iters = 20000;
        for (int tpb : {256, 512, 1024}) {
            dim3 grid(sms * 2), blk(tpb);
            dfma_kernel<<<grid, blk>>>(d, 100);
            cudaEventRecord(a);
            dfma_kernel<<<grid, blk>>>(d, iters);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            double flops = 2.0 * 8 * iters * (double)grid.x * tpb;
            printf("DFMA tpb=%d: %.2f TFLOP/s\n", tpb, flops / ms / 1e9);
            dmma_kernel<<<grid, blk>>>(d, 100);
            cudaEventRecord(a);
            dmma_kernel<<<grid, blk>>>(d, iters);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            flops = 2.0 * 256 * 4 * iters * (double)grid.x * (tpb / 32);
            printf("DMMA tpb=%d: %.2f TFLOP/s\n", tpb, flops / ms / 1e9);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
