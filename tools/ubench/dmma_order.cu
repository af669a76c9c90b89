// Does mma.sync m8n8k4 f64 compute c + a0 b0 + a1 b1 + a2 b2 + a3 b3 as a sequential FMA chain
// (k = 0..3), or with a different association / single rounding?
#include <cstdio>
#include <cstdlib>
#include <cmath>
__global__ void k(const double* A, const double* B, const double* Cin, double* D) {
    int l = threadIdx.x;
    double a = A[(l / 4) * 4 + (l % 4)];          // row=l/4, col(k)=l%4
    double b = B[(l % 4) * 8 + (l / 4)];          // row(k)=l%4, col=l/4
    double c0 = Cin[(l / 4) * 8 + 2 * (l % 4)], c1 = Cin[(l / 4) * 8 + 2 * (l % 4) + 1];
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
    D[(l / 4) * 8 + 2 * (l % 4)] = c0;
    D[(l / 4) * 8 + 2 * (l % 4) + 1] = c1;
}
int main() {
    double hA[32], hB[32], hC[64], hD[64];
    double *dA, *dB, *dC, *dD;
    cudaMalloc(&dA, 256); cudaMalloc(&dB, 256); cudaMalloc(&dC, 512); cudaMalloc(&dD, 512);
    srand(1);
    long seq = 0, rev = 0, pair = 0, exact1 = 0, total = 0;
    for (int trial = 0; trial < 2000; ++trial) {
        for (int i = 0; i < 32; ++i) { hA[i] = (rand() / (double)RAND_MAX - 0.5) * pow(10.0, rand() % 17 - 8); hB[i] = (rand() / (double)RAND_MAX - 0.5) * pow(10.0, rand() % 17 - 8); }
        for (int i = 0; i < 64; ++i) hC[i] = (rand() / (double)RAND_MAX - 0.5) * pow(10.0, rand() % 17 - 8);
        cudaMemcpy(dA, hA, 256, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice); cudaMemcpy(dC, hC, 512, cudaMemcpyHostToDevice);
        k<<<1, 32>>>(dA, dB, dC, dD);
        cudaMemcpy(hD, dD, 512, cudaMemcpyDeviceToHost);
        for (int r = 0; r < 8; ++r) for (int c = 0; c < 8; ++c) {
            double s = hC[r * 8 + c];
            for (int q = 0; q < 4; ++q) s = fma(hA[r * 4 + q], hB[q * 8 + c], s);
            double t = hC[r * 8 + c];
            for (int q = 3; q >= 0; --q) t = fma(hA[r * 4 + q], hB[q * 8 + c], t);
            // pairwise: (c + (a0b0 + a1b1)) + (a2b2 + a3b3) as fma chains
            long double e = hC[r * 8 + c];
            for (int q = 0; q < 4; ++q) e += (long double)hA[r * 4 + q] * hB[q * 8 + c];
            double g = hD[r * 8 + c];
            seq += (g == s); rev += (g == t); exact1 += (g == (double)e); total++;
        }
    }
    printf("DMMA == sequential fma k0..3: %ld/%ld, reverse: %ld, ~exact(long double): %ld\n", seq, total, rev, exact1);
    return 0;
}
