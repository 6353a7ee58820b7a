// cells.cuh -- Morton (Z-order) codes of the neighbour-search cells, shared by the neighbour
// search (neighbors.cu) and particle management (manage.cu).
#pragma once

#include <stdint.h>

namespace bgk {

// Cells are numbered along a Morton (Z-order) curve, so consecutive cells -- and the
// cell-ordered interior list the transport kernel walks -- form compact 3D blobs: the
// neighbour rows a block of consecutive particles needs stay within a small, L2-resident
// window.  Up to 10 bits per axis in 3D (1024 cells per axis) and 16 in 2D.
__host__ __device__ __forceinline__ uint32_t spread3(uint32_t v) {
    v &= 0x3ffu;
    v = (v | (v << 16)) & 0x030000ffu;
    v = (v | (v << 8)) & 0x0300f00fu;
    v = (v | (v << 4)) & 0x030c30c3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}
__host__ __device__ __forceinline__ uint32_t compact3(uint32_t v) {
    v &= 0x09249249u;
    v = (v | (v >> 2)) & 0x030c30c3u;
    v = (v | (v >> 4)) & 0x0300f00fu;
    v = (v | (v >> 8)) & 0x030000ffu;
    v = (v | (v >> 16)) & 0x3ffu;
    return v;
}
__host__ __device__ __forceinline__ uint32_t spread2(uint32_t v) {
    v &= 0xffffu;
    v = (v | (v << 8)) & 0x00ff00ffu;
    v = (v | (v << 4)) & 0x0f0f0f0fu;
    v = (v | (v << 2)) & 0x33333333u;
    v = (v | (v << 1)) & 0x55555555u;
    return v;
}
__host__ __device__ __forceinline__ uint32_t compact2(uint32_t v) {
    v &= 0x55555555u;
    v = (v | (v >> 1)) & 0x33333333u;
    v = (v | (v >> 2)) & 0x0f0f0f0fu;
    v = (v | (v >> 4)) & 0x00ff00ffu;
    v = (v | (v >> 8)) & 0x0000ffffu;
    return v;
}
template <int D>
__device__ __forceinline__ int cell_code(int cx, int cy, int cz) {
    if constexpr (D == 3) return (int)(spread3(cx) | (spread3(cy) << 1) | (spread3(cz) << 2));
    else return (int)(spread2(cx) | (spread2(cy) << 1));
}
template <int D>
__device__ __forceinline__ void cell_decode(int code, int& cx, int& cy, int& cz) {
    if constexpr (D == 3) {
        cx = (int)compact3((uint32_t)code);
        cy = (int)compact3((uint32_t)code >> 1);
        cz = (int)compact3((uint32_t)code >> 2);
    } else {
        cx = (int)compact2((uint32_t)code);
        cy = (int)compact2((uint32_t)code >> 1);
        cz = 0;
    }
}

}  // namespace bgk
