// Microbenchmark: fp64 DADD/DFMA dependent-chain latency and per-SM throughput on the B200.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat_kernel(double* out, long long* cyc, double a, double b, int n) {
    double x = a;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < n; ++i) x = x + b;          // dependent DADD chain
    long long t1 = clock64();
    double y = a;
    long long t2 = clock64();
#pragma unroll 16
    for (int i = 0; i < n; ++i) y = fma(y, b, a);   // dependent DFMA chain
    long long t3 = clock64();
    out[threadIdx.x] = x + y;
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t3 - t2; }
}

template <int ILP>
__global__ void tput_kernel(double* out, double a, double b, int n) {
    double x[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) x[k] = a + k;
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < ILP; ++k) x[k] = fma(x[k], b, a);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < ILP; ++k) s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    double* out; long long* cyc;
    cudaMalloc(&out, 1 << 26); cudaMalloc(&cyc, 16);
    const int n = 4096;
    lat_kernel<<<1, 32>>>(out, cyc, 1.0, 1e-9, n);
    long long h[2]; cudaMemcpy(h, cyc, 16, cudaMemcpyDeviceToHost);
    printf("dependent DADD latency: %.2f cycles, DFMA: %.2f cycles\n", (double)h[0] / n, (double)h[1] / n);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int warps : {4, 8, 12, 16, 32}) {
        const int iters = 20000;
        tput_kernel<8><<<sms, warps * 32>>>(out, 1.0, 0.999999, 100);
        cudaEventRecord(e0);
        tput_kernel<8><<<sms, warps * 32>>>(out, 1.0, 0.999999, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double ops = (double)sms * warps * 32 * iters * 8;
        printf("warps/SM=%2d ILP=8: %.3f T DFMA/s = %.1f per SM per clk at %d MHz\n", warps, ops / ms / 1e9,
               ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    }
    return 0;
}
