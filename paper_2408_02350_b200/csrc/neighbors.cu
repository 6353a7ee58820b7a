// neighbors.cu -- cell-linked-list neighbour search.
//
// N(i) = { j != i : ((x_j-x_i)^2 + (y_j-y_i)^2) + (z_j-z_i)^2 <= h2 } with every
// operation rounded (__dsub_rn/__dmul_rn/__dadd_rn, no FMA), ascending j, so the
// lists are bit-identical to a brute-force O(N^2) scan with the same arithmetic.
//
// Pipeline (all on the caller's stream, no host sync):
//   k_cell_assign  particle -> cell (edge >= h, 3^d sweep suffices), counts
//   k_scan         exclusive scan of cell counts (single block)
//   k_cell_fill    scatter particle ids into cells, k_cell_sort: ascending per cell
//   k_compact_*    interior particles in cell order -> transport processing order (multi-block)
//   k_nb_count     warp per particle: lanes test the 3^d cells' candidates, ballot+popc
//   k_scan         exclusive scan of counts -> CSR offsets (int64)
//   k_nb_fill      warp per particle: ballot compaction into shared memory, rank sort, store
#include <algorithm>
#include <climits>

#include "bgk_internal.cuh"
#include "cells.cuh"

namespace bgk {

namespace {

constexpr int kScanThreads = 1024;

// exclusive scan of n int32 counts into out[0..n] (out[n] = total); one block of 1024.
template <typename Tout>
__global__ void __launch_bounds__(kScanThreads) k_scan(const int32_t* __restrict__ in, Tout* __restrict__ out,
                                                        int64_t n) {
    __shared__ int64_t wsum[32];
    const int t = threadIdx.x;
    const int64_t chunk = (n + kScanThreads - 1) / kScanThreads;
    const int64_t b = t * chunk, e = min(n, b + chunk);
    int64_t local = 0;
    for (int64_t i = b; i < e; ++i) local += in[i];
    __syncwarp();                    // reconverge after the data-dependent loop before the shuffles
    // block exclusive scan of `local`
    const int lane = t & 31, wid = t >> 5;
    int64_t v = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int64_t u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
    }
    if (lane == 31) wsum[wid] = v;
    __syncthreads();
    if (wid == 0) {
        int64_t w = wsum[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int64_t u = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += u;
        }
        wsum[lane] = w;
    }
    __syncthreads();
    int64_t run = v - local + (wid > 0 ? wsum[wid - 1] : 0);
    for (int64_t i = b; i < e; ++i) {
        out[i] = (Tout)run;
        run += in[i];
    }
    if (t == kScanThreads - 1) out[n] = (Tout)(run);
    if (n == 0 && t == 0) out[0] = 0;
}

template <int D>
__global__ void k_cell_assign(const double* __restrict__ x, int64_t N, double L, double inv_e0, double inv_e1,
                              double inv_e2, int nc0, int nc1, int nc2, int32_t* __restrict__ cell_of,
                              int32_t* __restrict__ cell_cnt, int64_t* err) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    const double inv[3] = {inv_e0, inv_e1, inv_e2};
    const int nc[3] = {nc0, nc1, nc2};
    int cidx[3] = {0, 0, 0};
    bool ok = true;
#pragma unroll
    for (int a = 0; a < D; ++a) {
        double v = x[i * D + a];
        if (!(v >= 0.0 && v <= L)) ok = false;
        int c = (int)floor(v * inv[a]);
        cidx[a] = min(max(c, 0), nc[a] - 1);
    }
    if (!ok) latch_error(err, BGK_E_OUT_OF_DOMAIN, i);
    const int cell = cell_code<D>(cidx[0], cidx[1], cidx[2]);
    cell_of[i] = cell;
    atomicAdd(cell_cnt + cell, 1);
}

__global__ void k_cell_fill(int64_t N, const int32_t* __restrict__ cell_of, const int32_t* __restrict__ cell_start,
                            int32_t* __restrict__ cell_fill, int32_t* __restrict__ cell_pts) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    int c = cell_of[i];
    int pos = cell_start[c] + atomicAdd(cell_fill + c, 1);
    cell_pts[pos] = (int32_t)i;
}

// ascending particle ids inside each cell: one warp per cell, rank sort of up to 64 ids held two
// per lane (ids are distinct, so rank = number of smaller ids); larger cells fall back to an
// insertion sort by one lane
__global__ void k_cell_sort(int ncell, const int32_t* __restrict__ cell_start, int32_t* __restrict__ cell_pts) {
    const int lane = threadIdx.x & 31;
    const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (c >= ncell) return;
    const int b = cell_start[c], e = cell_start[c + 1], n = e - b;
    if (n <= 64) {
        const int v0 = lane < n ? cell_pts[b + lane] : INT_MAX;
        const int v1 = lane + 32 < n ? cell_pts[b + lane + 32] : INT_MAX;
        int r0 = 0, r1 = 0;
        for (int k = 0; k < 32; ++k) {
            const int u0 = __shfl_sync(0xffffffffu, v0, k), u1 = __shfl_sync(0xffffffffu, v1, k);
            r0 += (u0 < v0) + (u1 < v0);
            r1 += (u0 < v1) + (u1 < v1);
        }
        __syncwarp();
        if (lane < n) cell_pts[b + r0] = v0;
        if (lane + 32 < n) cell_pts[b + r1] = v1;
        return;
    }
    if (lane != 0) return;
    for (int q = b + 1; q < e; ++q) {
        int v = cell_pts[q], r = q - 1;
        while (r >= b && cell_pts[r] > v) {
            cell_pts[r + 1] = cell_pts[r];
            --r;
        }
        cell_pts[r + 1] = v;
    }
}

// exclusive scan of n int32 counts into out[0..n] (int64) with many blocks: per-block sums, a
// single-block scan of the sums, then each block scans its chunk from its offset
__global__ void __launch_bounds__(256) k_bsum(const int32_t* __restrict__ in, int64_t n, int64_t chunk,
                                              int32_t* __restrict__ bsum) {
    __shared__ int wsum[8];
    const int64_t b = blockIdx.x * chunk, e = min(n, b + chunk);
    int acc = 0;
    for (int64_t i = b + threadIdx.x; i < e; i += 256) acc += in[i];
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < 8; ++w) t += wsum[w];
        bsum[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(256) k_bscan(const int32_t* __restrict__ in, int64_t n, int64_t chunk,
                                               const int64_t* __restrict__ boff, int64_t nblk,
                                               int64_t* __restrict__ out) {
    __shared__ int64_t wsum[8];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int64_t base = boff[blockIdx.x];
    const int64_t b = blockIdx.x * chunk, e = min(n, b + chunk);
    for (int64_t i0 = b; i0 < e; i0 += 256) {
        const int64_t i = i0 + threadIdx.x;
        const int64_t v = i < e ? in[i] : 0;
        int64_t x = v;                                       // inclusive warp scan
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t u = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += u;
        }
        if (lane == 31) wsum[wid] = x;
        __syncthreads();
        int64_t before = 0, total = 0;
        for (int w = 0; w < 8; ++w) {
            before += w < wid ? wsum[w] : 0;
            total += wsum[w];
        }
        if (i < e) out[i] = base + before + x - v;
        base += total;
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[n] = boff[nblk];
}

void scan_counts(bgk_ctx* c, const int32_t* in, int64_t* out, int64_t n, cudaStream_t s) {
    if (n <= 32768) {                    // small clouds (2D workloads): one block, one launch
        k_scan<int64_t><<<1, kScanThreads, 0, s>>>(in, out, n);
        return;
    }
    const int64_t nblk = std::max<int64_t>(1, std::min<int64_t>(1000, (n + 2047) / 2048));
    const int64_t chunk = (n + nblk - 1) / nblk;
    k_bsum<<<(unsigned)nblk, 256, 0, s>>>(in, n, chunk, c->blk_tmp);
    k_scan<int64_t><<<1, kScanThreads, 0, s>>>(c->blk_tmp, c->scan_tmp, nblk);
    k_bscan<<<(unsigned)nblk, 256, 0, s>>>(in, n, chunk, c->scan_tmp, nblk, out);
}

// order = interior particles in cell order, multi-block stable compaction: per-block counts, a scan
// of the counts (k_scan), then each block writes its interior ids at its offset in order
__global__ void __launch_bounds__(256) k_compact_count(const int32_t* __restrict__ cell_pts,
                                                       const int8_t* __restrict__ kind, int64_t n, int64_t chunk,
                                                       int32_t* __restrict__ bcnt) {
    __shared__ int wsum[8];
    const int64_t b = blockIdx.x * chunk, e = min(n, b + chunk);
    int cnt = 0;
    for (int64_t i = b + threadIdx.x; i < e; i += 256) cnt += kind[cell_pts[i]] == 0;
    cnt = warp_sum(cnt);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < 8; ++w) t += wsum[w];
        bcnt[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(256) k_compact_write(const int32_t* __restrict__ cell_pts,
                                                       const int8_t* __restrict__ kind, int64_t n, int64_t chunk,
                                                       const int64_t* __restrict__ boff, int32_t* __restrict__ order) {
    __shared__ int wsum[8];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int64_t base = boff[blockIdx.x];
    const int64_t b = blockIdx.x * chunk, e = min(n, b + chunk);
    for (int64_t i0 = b; i0 < e; i0 += 256) {               // 256 ids per round, in order
        const int64_t i = i0 + threadIdx.x;
        const int p = i < e ? cell_pts[i] : 0;
        const bool keep = i < e && kind[p] == 0;
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) wsum[wid] = __popc(bal);
        __syncthreads();
        int before = 0, total = 0;
        for (int w = 0; w < 8; ++w) {
            before += w < wid ? wsum[w] : 0;
            total += wsum[w];
        }
        if (keep) order[base + before + __popc(bal & ((1u << lane) - 1u))] = p;
        base += total;
        __syncthreads();
    }
}


template <int D, bool FILL, bool PAD = false>
__global__ void k_neighbors(const double* __restrict__ x, int64_t N, double h2, const int32_t* __restrict__ cell_of,
                            const int32_t* __restrict__ cell_start, const int32_t* __restrict__ cell_pts, int nc0,
                            int nc1, int nc2, int max_nb, int32_t* __restrict__ nb_cnt,
                            const int64_t* __restrict__ nb_off, int32_t* __restrict__ nb_idx, int64_t cap,
                            int64_t* err) {
    extern __shared__ int32_t sbuf[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + wib;
    if (i >= N) return;
    int32_t* buf = sbuf + wib * max_nb;
    double xi[3];
#pragma unroll
    for (int a = 0; a < D; ++a) xi[a] = x[i * D + a];
    const int cell = cell_of[i];
    int cx, cy, cz;
    cell_decode<D>(cell, cx, cy, cz);
    int m = 0;
    for (int dz = (D == 3 ? -1 : 0); dz <= (D == 3 ? 1 : 0); ++dz) {
        const int z = cz + dz;
        if (z < 0 || z >= nc2) continue;
        for (int dy = -1; dy <= 1; ++dy) {
            const int y = cy + dy;
            if (y < 0 || y >= nc1) continue;
            for (int dx = -1; dx <= 1; ++dx) {
                const int xx = cx + dx;
                if (xx < 0 || xx >= nc0) continue;
                const int c = cell_code<D>(xx, y, z);
                const int cb = cell_start[c], ce = cell_start[c + 1];
                for (int base = cb; base < ce; base += 32) {
                    const int t = base + lane;
                    int j = -1;
                    bool hit = false;
                    if (t < ce) {
                        j = cell_pts[t];
                        if (j != (int)i) {
                            double xj[3];
#pragma unroll
                            for (int a = 0; a < D; ++a) xj[a] = x[(int64_t)j * D + a];
                            hit = dist2_rn<D>(xi, xj) <= h2;
                        }
                    }
                    const unsigned bal = __ballot_sync(0xffffffffu, hit);
                    if (FILL && hit) {
                        const int slot = m + __popc(bal & ((1u << lane) - 1u));
                        if (slot < max_nb) buf[slot] = j;
                    }
                    m += __popc(bal);
                }
            }
        }
    }
    if (!FILL || PAD) {
        if (lane == 0) {            // an overflowing list is left empty: no later kernel reads
            nb_cnt[i] = m > max_nb ? 0 : m;   // past the per-particle capacity (error latched)
            if (m > max_nb) latch_error(err, BGK_E_CAPACITY, i);
        }
        if (!FILL) return;
    }
    __syncwarp();
    // PAD: the sorted list goes to row i of a padded scratch [N][max_nb] (nb_idx is the scratch),
    // compacted into the CSR by k_nb_compact after the scan -- one distance sweep instead of two
    const int64_t off = PAD ? i * (int64_t)max_nb : nb_off[i];
    if (m > max_nb || (!PAD && off + m > cap)) return;   // capacity error already latched / reported
    for (int q = lane; q < m; q += 32) {      // rank sort: lists are short (< max_nb)
        const int v = buf[q];
        int rank = 0;
        for (int r = 0; r < m; ++r) rank += (buf[r] < v);
        nb_idx[off + rank] = v;
    }
}

// padded scratch rows -> CSR (warp per particle, coalesced copies)
__global__ void k_nb_compact(const int32_t* __restrict__ pad, int64_t N, int max_nb,
                             const int32_t* __restrict__ nb_cnt, const int64_t* __restrict__ nb_off,
                             int32_t* __restrict__ nb_idx) {
    const int lane = threadIdx.x & 31;
    const int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= N) return;
    const int m = nb_cnt[i];
    const int64_t off = nb_off[i];
    for (int q = lane; q < m; q += 32) nb_idx[off + q] = pad[i * (int64_t)max_nb + q];
}

}  // namespace

// cells: 7 kernels; neighbours: sweep + scan (1 or 3 kernels) + compaction
int launches_neighbors(const bgk_ctx* c) { return 7 + 2 + (c->N <= 32768 ? 1 : 3); }

void launch_build_neighbors(bgk_ctx* c, cudaStream_t s) {
    const int64_t N = c->N;
    const int tpb = 256;
    const unsigned nb = (unsigned)((N + tpb - 1) / tpb);
    cudaMemsetAsync(c->g.cell_cnt, 0, sizeof(int32_t) * c->ncell, s);
    cudaMemsetAsync(c->g.cell_fill, 0, sizeof(int32_t) * c->ncell, s);
    if (c->d == 3)
        k_cell_assign<3><<<nb, tpb, 0, s>>>(c->x, N, c->cfg.L, 1.0 / c->edge[0], 1.0 / c->edge[1], 1.0 / c->edge[2],
                                           c->nc[0], c->nc[1], c->nc[2], c->g.cell_of, c->g.cell_cnt, c->err);
    else
        k_cell_assign<2><<<nb, tpb, 0, s>>>(c->x, N, c->cfg.L, 1.0 / c->edge[0], 1.0 / c->edge[1], 1.0,
                                           c->nc[0], c->nc[1], 1, c->g.cell_of, c->g.cell_cnt, c->err);
    k_scan<int32_t><<<1, kScanThreads, 0, s>>>(c->g.cell_cnt, c->g.cell_start, c->ncell);
    k_cell_fill<<<nb, tpb, 0, s>>>(N, c->g.cell_of, c->g.cell_start, c->g.cell_fill, c->g.cell_pts);
    k_cell_sort<<<(c->ncell + 3) / 4, 128, 0, s>>>(c->ncell, c->g.cell_start, c->g.cell_pts);
    {
        const int64_t nblk = std::max<int64_t>(1, std::min<int64_t>(1000, (N + 255) / 256));   // 256 ids per block
        const int64_t chunk = (N + nblk - 1) / nblk;
        k_compact_count<<<(unsigned)nblk, 256, 0, s>>>(c->g.cell_pts, c->kind, N, chunk, c->g.nb_cnt);
        k_scan<int64_t><<<1, kScanThreads, 0, s>>>(c->g.nb_cnt, c->scan_tmp, nblk);
        k_compact_write<<<(unsigned)nblk, 256, 0, s>>>(c->g.cell_pts, c->kind, N, chunk, c->scan_tmp, c->g.order);
    }
    const int wpb = 8;
    const unsigned nbw = (unsigned)((N + wpb - 1) / wpb);
    const size_t smem = sizeof(int32_t) * wpb * c->max_nb;
    // one distance sweep: sorted lists into a padded scratch (the WLS pair-record array, rewritten
    // after the neighbours), counts, scan, compaction into the CSR
    int32_t* pad = reinterpret_cast<int32_t*>(c->g.P);
    if (c->d == 3)
        k_neighbors<3, true, true><<<nbw, wpb * 32, smem, s>>>(c->x, N, c->cfg.h2, c->g.cell_of, c->g.cell_start,
                                                              c->g.cell_pts, c->nc[0], c->nc[1], c->nc[2], c->max_nb,
                                                              c->g.nb_cnt, nullptr, pad, c->cap, c->err);
    else
        k_neighbors<2, true, true><<<nbw, wpb * 32, smem, s>>>(c->x, N, c->cfg.h2, c->g.cell_of, c->g.cell_start,
                                                              c->g.cell_pts, c->nc[0], c->nc[1], 1, c->max_nb,
                                                              c->g.nb_cnt, nullptr, pad, c->cap, c->err);
    scan_counts(c, c->g.nb_cnt, c->g.nb_off, N, s);
    k_nb_compact<<<nbw, wpb * 32, 0, s>>>(pad, N, c->max_nb, c->g.nb_cnt, c->g.nb_off, c->g.nb_idx);
}

}  // namespace bgk
