// Microbenchmark of the transport row arithmetic in isolation (registers only):
//   A: incremental form  y += dy (4 DADD) ; C = L-|yn|-|yt|-|yb| (3 DADD) ; Q += C v (DFMA) ; S += C (DADD)
//   B: FMA form          y = fma(r, dy, y0) (4 DFMA) ; C = (L-|yn|)-(|yt|+|yb|) (3 DADD) ; Q, S as A
// Reports fp64 instructions per SM per clock (peak 32 warp-lanes... = 64 lane-ops/clk/SM).
#include <cstdio>
#include <cuda_runtime.h>

template <int R, bool FMA>
__global__ void __launch_bounds__(256, 1) rowmix(double* out, const double* in, int iters) {
    double Q[R], S[R], v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) { Q[r] = 0; S[r] = 0; v[r] = in[(threadIdx.x + r) & 255]; }
    double y0 = in[1] * threadIdx.x, y1 = in[2], y2 = in[3], L = in[4];
    double d0 = in[5], d1 = in[6], d2 = in[7], dL = in[8];
    for (int it = 0; it < iters; ++it) {
        double a = y0, b = y1, c = y2, l = L;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            double C;
            if (FMA) {
                const double rr = (double)r;
                const double yn = fma(rr, d0, y0), yt = fma(rr, d1, y1), yb = fma(rr, d2, y2), Lr = fma(rr, dL, L);
                C = (Lr - fabs(yn)) - (fabs(yt) + fabs(yb));
            } else {
                C = l - fabs(a) - fabs(b) - fabs(c);
                a += d0; b += d1; c += d2; l += dL;
            }
            Q[r] = fma(C, v[r], Q[r]);
            S[r] += C;
        }
        y0 += 1e-3; L += 2e-3;   // new "neighbour"
    }
    double s = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) s += Q[r] + S[r];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int R, bool FMA>
void run(int sms, int clk, double* out, double* in, int warps) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 4000;
    rowmix<R, FMA><<<sms, warps * 32>>>(out, in, 10);
    cudaEventRecord(e0);
    rowmix<R, FMA><<<sms, warps * 32>>>(out, in, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double instr = (double)sms * warps * 32 * iters * R * 9;   // 9 fp64 per row
    printf("R=%d %s warps/SM=%d: %.1f fp64 lane-ops per SM per clk (%.0f%% of 64)\n", R, FMA ? "FMA " : "INCR", warps,
           instr / (ms * 1e-3) / sms / (clk * 1e3), instr / (ms * 1e-3) / sms / (clk * 1e3) / 64 * 100);
}

int main() {
    double *out, *in;
    cudaMalloc(&out, 1 << 24); cudaMalloc(&in, 1 << 16);
    cudaMemset(in, 0, 1 << 16);
    int sms, clk;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    for (int w : {4, 8}) {
        run<25, false>(sms, clk, out, in, w);
        run<25, true>(sms, clk, out, in, w);
    }
    return 0;
}
