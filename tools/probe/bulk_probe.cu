// Bulk-copy (cp.async.bulk) streaming probe: one producer warp per block streams NC copies of S bytes
// from a large DRAM-resident buffer into an NS-deep shared-memory ring; consumer warps wait on the
// full barrier and release the stage.  Reports GB/s for (S, NS, copies per stage, row stride).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../../paper_2408_02350_b200/csrc/async.cuh"
using namespace bgk;

__global__ void __launch_bounds__(416, 1) k_probe(const char* __restrict__ src, size_t nbytes, int S, int NS, int nrow,
                                                  int ncopy, long stride, int nconsumer, int mode, int P) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + 200 * 1024);
    uint64_t* empty = full + 64;
    const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
    const int SB = (S * ncopy + 127) / 128 * 128;
    if (tid == 0) {
        for (int q = 0; q < NS; ++q) { mbar_init(full + q, 1); mbar_init(empty + q, nconsumer); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // block b reads rows b*nrow .. : row r at offset (r * stride) % nbytes, ncopy pieces of S bytes
    if (wp == nconsumer && mode == 0) {
        for (int u = 0; u < nrow; ++u) {
            const int q = u % NS;
            if (u >= NS) mbar_wait(empty + q, (uint32_t)(u / NS - 1) & 1u);
            if (lane == 0) mbar_expect_tx(full + q, (uint32_t)(S * ncopy));
            __syncwarp();
            const size_t off = ((size_t)(blockIdx.x * (size_t)nrow + u) * stride) % (nbytes - S * ncopy - 4096);
            const size_t off128 = off / 128 * 128;
            if (lane < ncopy) bulk_load(sm + (size_t)q * SB + lane * S, src + off128 + (size_t)lane * S, S, full + q);
        }
    } else if (wp == nconsumer && mode == 1) {      // lane l issues row u0 + l (ncopy == 1), P rows per step
        for (int u0 = 0; u0 < nrow; u0 += P) {
            const int u = u0 + lane;
            if (lane < P && u < nrow) {
                const int q = u % NS;
                if (u >= NS) mbar_wait(empty + q, (uint32_t)(u / NS - 1) & 1u);
                mbar_expect_tx(full + q, (uint32_t)S);
                const size_t off = ((size_t)(blockIdx.x * (size_t)nrow + u) * stride) % (nbytes - S - 4096);
                bulk_load(sm + (size_t)q * SB, src + off / 128 * 128, S, full + q);
            }
            __syncwarp();
        }
    } else if (wp == nconsumer && mode == 3) {      // row u issued by lane u % 32, one row at a time
        for (int u = 0; u < nrow; ++u) {
            const int q = u % NS;
            if (lane == (u & 31)) {
                if (u >= NS) mbar_wait(empty + q, (uint32_t)(u / NS - 1) & 1u);
                mbar_expect_tx(full + q, (uint32_t)S);
                const size_t off = ((size_t)(blockIdx.x * (size_t)nrow + u) * stride) % (nbytes - S - 4096);
                bulk_load(sm + (size_t)q * SB, src + off / 128 * 128, S, full + q);
            }
            __syncwarp();
        }
    } else if (wp == nconsumer && mode == 8) {      // lanes 0,1 issue rows u, u+1 in one instruction, then 2x25x4 DFMA
        double x0 = lane, x1 = lane + 1, x2 = lane + 2, x3 = lane + 3;
        for (int u0 = 0; u0 < nrow; u0 += 2) {
            const int u = u0 + lane;
            const int q = u % NS;
            if (lane < 2 && u < nrow) {
                if (u >= NS) mbar_wait(empty + q, (uint32_t)(u / NS - 1) & 1u);
                mbar_expect_tx(full + q, (uint32_t)S);
                const size_t off = ((size_t)(blockIdx.x * (size_t)nrow + u) * stride) % (nbytes - S - 4096);
                bulk_load(sm + (size_t)q * SB, src + off / 128 * 128, S, full + q);
            }
            __syncwarp();
            for (int k = 0; k < 2 * P; ++k) {
                x0 = fma(x0, 1.0000001, 0.5); x1 = fma(x1, 1.0000001, 0.5);
                x2 = fma(x2, 1.0000001, 0.5); x3 = fma(x3, 1.0000001, 0.5);
            }
        }
        if (x0 + x1 + x2 + x3 == 12345.0) full[0] = 1;
    } else if (wp == nconsumer && mode == 9) {      // expect_tx for row u issued one row EARLY (separate), copy now
        double x0 = lane, x1 = lane + 1, x2 = lane + 2, x3 = lane + 3;
        if (lane == 0) mbar_expect_tx(full + 0, (uint32_t)S);
        for (int u = 0; u < nrow; ++u) {
            const int q = u % NS;
            if (u >= NS) mbar_wait(empty + q, (uint32_t)(u / NS - 1) & 1u);
            if (lane == 0) {
                const size_t off = ((size_t)(blockIdx.x * (size_t)nrow + u) * stride) % (nbytes - S - 4096);
                bulk_load(sm + (size_t)q * SB, src + off / 128 * 128, S, full + q);
                const int q1 = (u + 1) % NS;
                if (u + 1 < nrow) {
                    if (u + 1 >= NS) mbar_wait(empty + q1, (uint32_t)((u + 1) / NS - 1) & 1u);
                    mbar_expect_tx(full + q1, (uint32_t)S);
                }
            }
            for (int k = 0; k < P; ++k) {
                x0 = fma(x0, 1.0000001, 0.5); x1 = fma(x1, 1.0000001, 0.5);
                x2 = fma(x2, 1.0000001, 0.5); x3 = fma(x3, 1.0000001, 0.5);
            }
        }
        if (x0 + x1 + x2 + x3 == 12345.0) full[0] = 1;
    } else if (wp == nconsumer && mode >= 5) {      // lane 0 issues a row, then ~P*4 dependent-free DFMAs per lane
        double x0 = lane, x1 = lane + 1, x2 = lane + 2, x3 = lane + 3;
        for (int u = 0; u < nrow; ++u) {
            const int q = u % NS;
            if (u >= NS) mbar_wait(empty + q, (uint32_t)(u / NS - 1) & 1u);
            if (lane == 0 && mode != 6) {
                mbar_expect_tx(full + q, (uint32_t)S);
                const size_t off = ((size_t)(blockIdx.x * (size_t)nrow + u) * stride) % (nbytes - S - 4096);
                bulk_load(sm + (size_t)q * SB, src + off / 128 * 128, S, full + q);
            }
            if (mode == 6 && lane == 0) mbar_arrive(full + q);
            for (int k = 0; k < P; ++k) {
                x0 = fma(x0, 1.0000001, 0.5); x1 = fma(x1, 1.0000001, 0.5);
                x2 = fma(x2, 1.0000001, 0.5); x3 = fma(x3, 1.0000001, 0.5);
            }
        }
        if (x0 + x1 + x2 + x3 == 12345.0) full[0] = 1;
    } else if (wp == nconsumer && mode == 2) {      // no wait on empty at all (NS >= nrow impossible) -> issue only
        for (int u = 0; u < nrow; ++u) {
            const int q = u % NS;
            if (u >= NS) mbar_wait(empty + q, (uint32_t)(u / NS - 1) & 1u);
            if (lane == 0) {
                mbar_expect_tx(full + q, (uint32_t)S);
                const size_t off = ((size_t)(blockIdx.x * (size_t)nrow + u) * stride) % (nbytes - S - 4096);
                bulk_load(sm + (size_t)q * SB, src + off / 128 * 128, S, full + q);
            }
        }
    } else if (wp < nconsumer) {
        for (int u = 0; u < nrow; ++u) {
            const int q = u % NS;
            mbar_wait(full + q, (uint32_t)(u / NS) & 1u);
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + q);
        }
    }
    __syncthreads();
}

int main() {
    const size_t nbytes = (size_t)8 << 30;
    char* buf;
    cudaMalloc(&buf, nbytes);
    cudaMemset(buf, 1, nbytes);
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024 + 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    struct Cfg { int S, ncopy, NS; long stride; int mode, P; };
    Cfg cfgs[] = {{8192, 1, 12, 128000, 5, 25}, {8192, 1, 12, 128000, 6, 25}, {8192, 1, 12, 128000, 8, 25},
                  {8192, 1, 12, 128000, 9, 25}, {8192, 1, 12, 128000, 5, 100}, {8192, 1, 12, 128000, 8, 100},
                  {8192, 1, 12, 128000, 9, 100},
                  {8192, 1, 20, 128000, 1, 4}, {8192, 1, 20, 128000, 1, 8}, {8192, 1, 24, 128000, 1, 12},
                  {4096, 1, 40, 128000, 1, 8}, {4096, 1, 40, 128000, 1, 16},
                  {16384, 1, 12, 128000, 1, 4}};
    for (auto& c : cfgs) {
        const int nrow = 400, blocks = 148 * 4;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            k_probe<<<blocks, 416, 200 * 1024 + 1024>>>(buf, nbytes, c.S, c.NS, nrow, c.ncopy, c.stride, 12, c.mode, c.P);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
        }
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = (double)blocks * nrow * c.S * c.ncopy;
        printf("S=%6d x%d NS=%2d stride=%7ld mode=%d P=%2d : %.3f ms  %.2f TB/s  (%s)\n", c.S, c.ncopy, c.NS, c.stride, c.mode, c.P, ms,
               bytes / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
