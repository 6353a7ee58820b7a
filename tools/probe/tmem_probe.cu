// Probe: TMEM alloc / st / ld pattern of k_transport_pair_tm in isolation (hang check).
#include <cstdint>
#include <cstdio>
// TMEM swap of the active particle's accumulators (Q[25], Sc[25] = 100 32-bit words per lane):
// store them to slot `to`, load slot `from` into the same registers.  32x32b shape: lane l of the
// warp's quadrant, columns [slot, slot + 100).
__device__ __forceinline__ void tm_store100(uint32_t taddr, const uint32_t (&w)[100]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x64.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32, %33, %34, %35, %36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, %48, %49, %50, %51, %52, %53, %54, %55, %56, %57, %58, %59, %60, %61, %62, %63, %64};" :: "r"(taddr + 0u), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15]), "r"(w[16]), "r"(w[17]), "r"(w[18]), "r"(w[19]), "r"(w[20]), "r"(w[21]), "r"(w[22]), "r"(w[23]), "r"(w[24]), "r"(w[25]), "r"(w[26]), "r"(w[27]), "r"(w[28]), "r"(w[29]), "r"(w[30]), "r"(w[31]), "r"(w[32]), "r"(w[33]), "r"(w[34]), "r"(w[35]), "r"(w[36]), "r"(w[37]), "r"(w[38]), "r"(w[39]), "r"(w[40]), "r"(w[41]), "r"(w[42]), "r"(w[43]), "r"(w[44]), "r"(w[45]), "r"(w[46]), "r"(w[47]), "r"(w[48]), "r"(w[49]), "r"(w[50]), "r"(w[51]), "r"(w[52]), "r"(w[53]), "r"(w[54]), "r"(w[55]), "r"(w[56]), "r"(w[57]), "r"(w[58]), "r"(w[59]), "r"(w[60]), "r"(w[61]), "r"(w[62]), "r"(w[63]) : "memory");
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" :: "r"(taddr + 64u), "r"(w[64]), "r"(w[65]), "r"(w[66]), "r"(w[67]), "r"(w[68]), "r"(w[69]), "r"(w[70]), "r"(w[71]), "r"(w[72]), "r"(w[73]), "r"(w[74]), "r"(w[75]), "r"(w[76]), "r"(w[77]), "r"(w[78]), "r"(w[79]), "r"(w[80]), "r"(w[81]), "r"(w[82]), "r"(w[83]), "r"(w[84]), "r"(w[85]), "r"(w[86]), "r"(w[87]), "r"(w[88]), "r"(w[89]), "r"(w[90]), "r"(w[91]), "r"(w[92]), "r"(w[93]), "r"(w[94]), "r"(w[95]) : "memory");
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" :: "r"(taddr + 96u), "r"(w[96]), "r"(w[97]), "r"(w[98]), "r"(w[99]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tm_load100(uint32_t taddr, uint32_t (&w)[100]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32, %33, %34, %35, %36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, %48, %49, %50, %51, %52, %53, %54, %55, %56, %57, %58, %59, %60, %61, %62, %63}, [%64];" : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]), "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15]), "=r"(w[16]), "=r"(w[17]), "=r"(w[18]), "=r"(w[19]), "=r"(w[20]), "=r"(w[21]), "=r"(w[22]), "=r"(w[23]), "=r"(w[24]), "=r"(w[25]), "=r"(w[26]), "=r"(w[27]), "=r"(w[28]), "=r"(w[29]), "=r"(w[30]), "=r"(w[31]), "=r"(w[32]), "=r"(w[33]), "=r"(w[34]), "=r"(w[35]), "=r"(w[36]), "=r"(w[37]), "=r"(w[38]), "=r"(w[39]), "=r"(w[40]), "=r"(w[41]), "=r"(w[42]), "=r"(w[43]), "=r"(w[44]), "=r"(w[45]), "=r"(w[46]), "=r"(w[47]), "=r"(w[48]), "=r"(w[49]), "=r"(w[50]), "=r"(w[51]), "=r"(w[52]), "=r"(w[53]), "=r"(w[54]), "=r"(w[55]), "=r"(w[56]), "=r"(w[57]), "=r"(w[58]), "=r"(w[59]), "=r"(w[60]), "=r"(w[61]), "=r"(w[62]), "=r"(w[63]) : "r"(taddr + 0u) : "memory");
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];" : "=r"(w[64]), "=r"(w[65]), "=r"(w[66]), "=r"(w[67]), "=r"(w[68]), "=r"(w[69]), "=r"(w[70]), "=r"(w[71]), "=r"(w[72]), "=r"(w[73]), "=r"(w[74]), "=r"(w[75]), "=r"(w[76]), "=r"(w[77]), "=r"(w[78]), "=r"(w[79]), "=r"(w[80]), "=r"(w[81]), "=r"(w[82]), "=r"(w[83]), "=r"(w[84]), "=r"(w[85]), "=r"(w[86]), "=r"(w[87]), "=r"(w[88]), "=r"(w[89]), "=r"(w[90]), "=r"(w[91]), "=r"(w[92]), "=r"(w[93]), "=r"(w[94]), "=r"(w[95]) : "r"(taddr + 64u) : "memory");
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(w[96]), "=r"(w[97]), "=r"(w[98]), "=r"(w[99]) : "r"(taddr + 96u) : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(128, 2) k(double* out, int iters) {
    __shared__ uint32_t tm_base;
    extern __shared__ unsigned char dyn[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    if (wib == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"((uint32_t)__cvta_generic_to_shared(&tm_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tlane = tm_base + ((uint32_t)((wib & 3) * 32) << 16);
    uint32_t w[100];
    for (int i = 0; i < 100; ++i) w[i] = threadIdx.x * 1000 + i + blockIdx.x;
    double acc = 0;
    for (int it = 0; it < iters; ++it) {
        tm_store100(tlane + (it & 1) * 100u, w);
        tm_load100(tlane + ((it + 1) & 1) * 100u, w);
        acc += w[lane];
    }
    out[blockIdx.x * 128 + threadIdx.x] = acc + dyn[0];
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (wib == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm_base));
}
int main() {
    double* out;
    cudaMalloc(&out, 148 * 8 * 128 * 8);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 106 * 1024);
    k<<<148 * 8, 128, 106 * 1024>>>(out, 100);
    cudaError_t e = cudaDeviceSynchronize();
    printf("probe: %s\n", cudaGetErrorString(e));
    return 0;
}
