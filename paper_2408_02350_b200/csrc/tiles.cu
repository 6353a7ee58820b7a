// tiles.cu -- fixed-cloud transport of the deep lattice interior as a 3D stencil ("the
// one lever": W = 0 and a cached regular cloud).
//
// On the regular C5-type lattice every interior particle whose whole h-ball lies inside the lattice
// (index 3 .. n-4 on every axis at h = 3.1 dx) has the same neighbour offsets -- the 122 integer
// offsets |delta|^2 <= 9 -- and, with W = 0, the same positive-scheme coefficients (PAPER.md:408-410,
// 476-480 with Z5-Z7):
//     C'_delta(k) = sum_e min(P_delta,e . v_k, 0)   (= C/2, the neg_part form of transport.cu)
// so the transport of those particles is a 122-point stencil with node-dependent coefficients:
//     ftilde_i(k) = f_i(k) - 2 dt (sum_delta C'_delta(k) f_{i+delta}(k) - f_i(k) S(k)),
//     S(k) = sum_delta C'_delta(k).
// k_tile_ctab evaluates C' once per cached geometry from one reference particle's pair records into a
// table [123][Ks] (row 122 = S).  k_transport_tile: block = (8 x 8 x 8 particle tile, range of node
// chunks); per chunk of 4 stored nodes one TMA box brings the tile's halo (15 x 14 x 14 rows: one
// spare x column keeps the y-lines on alternating shared-memory banks) and one the 123 x 4
// coefficients, double-buffered; thread = (node, (y, z) line of the tile) computes the 8 particles of
// its x-line: per run of offsets along x it loads the window once and applies up to 7 offsets to all
// 8 particles (2.4 FMAs per shared-memory load).  Moment partials accumulate in registers over the
// block's chunks and go out in a fixed order (partial slot = the node range).  The pair data differ
// from particle to particle only by rounding (identical offsets): build_rows checks every offset of
// every tile particle against the reference to 1e-12 dx, as for the lattice-row groups.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "async.cuh"
#include "bgk_internal.cuh"

namespace bgk {

namespace {

constexpr int kTN = 4;                   // stored nodes per chunk
constexpr int kTX = 15, kTY = 14, kTZ = 14;   // halo box: 8 + 6 (+ 1 spare in x)
constexpr int kTBox = kTN * kTX * kTY * kTZ;  // doubles
constexpr int kTOff = 122;               // stencil offsets (|delta|^2 <= 9, delta != 0)
constexpr int kTCoef = (kTOff + 1) * kTN;     // coefficient box doubles (+ the S row)
constexpr size_t kTStage = ((size_t)(kTBox + kTCoef) * sizeof(double) + 127) / 128 * 128;
constexpr int kTThreads = kTN * 64;      // node x (y, z) line

struct Run {
    int dz, dy, w, e0;
};
// offsets along x in runs of constant (dz, dy), in ascending neighbour order (dz, dy, dx): e0 = index
// of (dz, dy, -w); the run (0, 0) skips dx = 0 (the particle itself)
constexpr int kTRuns = 29;
__host__ __device__ constexpr Run run_at(int r) {
    constexpr int t[kTRuns][4] = {
        {-3, 0, 0, 0},   {-2, -2, 1, 1},  {-2, -1, 2, 4},  {-2, 0, 2, 9},   {-2, 1, 2, 14},  {-2, 2, 1, 19},
        {-1, -2, 2, 22}, {-1, -1, 2, 27}, {-1, 0, 2, 32},  {-1, 1, 2, 37},  {-1, 2, 2, 42},  {0, -3, 0, 47},
        {0, -2, 2, 48},  {0, -1, 2, 53},  {0, 0, 3, 58},   {0, 1, 2, 64},   {0, 2, 2, 69},   {0, 3, 0, 74},
        {1, -2, 2, 75},  {1, -1, 2, 80},  {1, 0, 2, 85},   {1, 1, 2, 90},   {1, 2, 2, 95},   {2, -2, 1, 100},
        {2, -1, 2, 103}, {2, 0, 2, 108},  {2, 1, 2, 113},  {2, 2, 1, 118},  {3, 0, 0, 121}};
    return Run{t[r][0], t[r][1], t[r][2], t[r][3]};
}

// run R of the stencil for one thread: the window of line (y + dy, z + dz) once, then every offset of
// the run on all 8 particles of the thread's x-line; recurses over the runs at compile time
template <int R>
__device__ __forceinline__ void tile_runs(const double* __restrict__ hs, const double* __restrict__ cs, int yl,
                                          int zl, int n, double (&acc)[8]) {
    constexpr Run rr = run_at(R);
    constexpr int W = rr.w;
    const double* lp = hs + (((zl + 3 + rr.dz) * kTY + (yl + 3 + rr.dy)) * kTX + (3 - W)) * kTN + n;
    double win[2 * W + 8];
#pragma unroll
    for (int i = 0; i < 2 * W + 8; ++i) win[i] = lp[i * kTN];
#pragma unroll
    for (int k = 0; k <= 2 * W; ++k) {
        if (rr.dz == 0 && rr.dy == 0 && k == W) continue;               // the particle itself
        const int e = rr.e0 + k - ((rr.dz == 0 && rr.dy == 0 && k > W) ? 1 : 0);
        const double cc = cs[e * kTN + n];
#pragma unroll
        for (int p = 0; p < 8; ++p) acc[p] = fma(cc, win[p + k], acc[p]);
    }
    if constexpr (R + 1 < kTRuns) tile_runs<R + 1>(hs, cs, yl, zl, n, acc);
}

__device__ __forceinline__ double tile_neg(double t) {   // min(t, 0) on the integer pipe (transport.cu)
    return __hiloint2double(min(__double2hiint(t), 0), __double2loint(t));
}

// C'_e(t) for the reference particle's 122 entries (pair record: dy_e, p_e2, p_e3 per direction),
// W = 0; padding columns 0; row 122 = sum over e in entry order
__global__ void k_tile_ctab(const double* __restrict__ P, int64_t off_ref, double* __restrict__ ctab, int64_t Ks,
                            int n1, int ncol, int ncs, int c0, double vmax, double dv) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= Ks) return;
    const int k1 = (int)(t / ncs), col = (int)(t - (int64_t)k1 * ncs);
    const bool valid = col < ncol;
    const int gc = c0 + (valid ? col : 0);
    const int k2 = gc / n1, k3 = gc - k2 * n1;
    const double c1dv = axis_node(vmax, dv, k1) / dv, v2 = axis_node(vmax, dv, k2), v3 = axis_node(vmax, dv, k3);
    double S = 0.0;
    for (int e = 0; e < kTOff; ++e) {
        const double* pv = P + (off_ref + e) * 10;
        double C = 0.0;
#pragma unroll
        for (int q = 0; q < 3; ++q) C += tile_neg(fma(pv[3 * q], c1dv, fma(pv[3 * q + 1], v2, pv[3 * q + 2] * v3)));
        C = valid ? C : 0.0;
        ctab[(int64_t)e * Ks + t] = C;
        S += C;
    }
    ctab[(int64_t)kTOff * Ks + t] = S;
}

struct TileArgs {
    const int32_t* org;          // [tiles][3] lattice index of the tile's first particle
    double* ft;
    double* partials;
    unsigned long long* stab;
    int64_t Ks;
    int nlat;                    // lattice points per axis (particle = ix + n iy + n^2 iz)
    int nwpp, nq;                // partial slots per particle, node ranges (slot q < nq)
    int nchunk;                  // node chunks (Ks / kTN)
    int n1, ncol, ncs, c0;
    double vmax, dv, dt;
};

__global__ void __launch_bounds__(kTThreads, 1) k_transport_tile(const __grid_constant__ CUtensorMap thalo,
                                                                 const __grid_constant__ CUtensorMap tcoef,
                                                                 const TileArgs A) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + 2 * kTStage);
    const int tid = threadIdx.x;
    const int n = tid & (kTN - 1), line = tid / kTN;           // node of the chunk, (y, z) line
    const int yl = line & 7, zl = line >> 3;
    const int tile = blockIdx.x, q = blockIdx.y;
    const int x0 = A.org[tile * 3], y0 = A.org[tile * 3 + 1], z0 = A.org[tile * 3 + 2];
    const int c_beg = (int)((int64_t)A.nchunk * q / A.nq), c_end = (int)((int64_t)A.nchunk * (q + 1) / A.nq);
    if (tid == 0) {
        mbar_init(full, 1);
        mbar_init(full + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int c, int b) {
        unsigned char* st = smem_raw + (size_t)b * kTStage;
        mbar_expect_tx(full + b, (uint32_t)((kTBox + kTCoef) * sizeof(double)));
        tma_load_4d(st, &thalo, c * kTN, x0 - 3, y0 - 3, z0 - 3, full + b);
        tma_load_2d(st + (size_t)kTBox * sizeof(double), &tcoef, c * kTN, 0, full + b);
    };
    if (tid == 0) {
        if (c_beg < c_end) issue(c_beg, 0);
        if (c_beg + 1 < c_end) issue(c_beg + 1, 1);
    }
    double s[8][kPM];
#pragma unroll
    for (int p = 0; p < 8; ++p)
#pragma unroll
        for (int k = 0; k < kPM; ++k) s[p][k] = 0.0;
    double amax = 0.0;
    const int64_t pbase = (int64_t)x0 + (int64_t)A.nlat * (y0 + yl) + (int64_t)A.nlat * A.nlat * (z0 + zl);
    for (int c = c_beg; c < c_end; ++c) {
        const int b = (c - c_beg) & 1;
        mbar_wait(full + b, (uint32_t)((c - c_beg) >> 1) & 1u);
        const double* hs = reinterpret_cast<const double*>(smem_raw + (size_t)b * kTStage);
        const double* cs = hs + kTBox;
        double acc[8];
#pragma unroll
        for (int p = 0; p < 8; ++p) acc[p] = 0.0;
        tile_runs<0>(hs, cs, yl, zl, n, acc);
        // epilogue of the chunk: ftilde for the 8 particles of the line at this node, moment partials
        const int64_t t = (int64_t)c * kTN + n;
        const int k1 = (int)(t / A.ncs), col = (int)(t - (int64_t)k1 * A.ncs);
        const bool valid = col < A.ncol;
        const double S = cs[kTOff * kTN + n];
        const double* fi = hs + (((zl + 3) * kTY + (yl + 3)) * kTX + 3) * kTN + n;
        const int gc = A.c0 + (valid ? col : 0);
        const int k2 = gc / A.n1, k3 = gc - k2 * A.n1;
        const double v1 = axis_node(A.vmax, A.dv, k1), v2 = axis_node(A.vmax, A.dv, k2),
                     v3 = axis_node(A.vmax, A.dv, k3);
        const double vv = v1 * v1 + v2 * v2 + v3 * v3;
        const double dtq = 2.0 * A.dt;
        if (valid) {
            amax = fmax(amax, -2.0 * S);
#pragma unroll
            for (int p = 0; p < 8; ++p) {
                const double fv = fi[p * kTN];
                const double out = fv - dtq * (acc[p] - fv * S);
                A.ft[(pbase + p) * A.Ks + t] = out;
                s[p][0] += out;
                s[p][1] += v1 * out;
                s[p][2] += v2 * out;
                s[p][3] += v3 * out;
                s[p][4] += vv * out;
            }
        }
        __syncthreads();                                   // every thread is done with stage b
        if (tid == 0 && c + 2 < c_end) issue(c + 2, b);
    }
    // partials: sum over the kTN node lanes of each line (adjacent lanes, fixed order), slot q
#pragma unroll
    for (int p = 0; p < 8; ++p)
#pragma unroll
        for (int k = 0; k < kPM; ++k) {
            double v = s[p][k];
            v += __shfl_xor_sync(0xffffffffu, v, 1);
            v += __shfl_xor_sync(0xffffffffu, v, 2);
            s[p][k] = v;
        }
    if (n == 0) {
#pragma unroll
        for (int p = 0; p < 8; ++p) {
            double* pp = A.partials + ((pbase + p) * A.nwpp + q) * kPM;
#pragma unroll
            for (int k = 0; k < kPM; ++k) pp[k] = s[p][k];
        }
    }
    amax = warp_max(amax);
    if ((tid & 31) == 0) atomicMax(A.stab, (unsigned long long)__double_as_longlong(amax));
}

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult qr;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr) == cudaSuccess &&
            qr == cudaDriverEntryPointSuccess)
            encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    return encode;
}

}  // namespace

// host side of the tiles (build_rows): the reference particle's entries must be exactly the ball in
// (dz, dy, dx) order; every tile particle's stencil equals it (checked by the caller)
bool tile_ball_order(const int64_t* d_off, int m) {
    if (m != kTOff) return false;
    int e = 0;
    for (int ri = 0; ri < kTRuns; ++ri) {
        const Run r = run_at(ri);
        for (int k = -r.w; k <= r.w; ++k) {
            if (r.dz == 0 && r.dy == 0 && k == 0) continue;
            const int64_t* o = d_off + 3 * e++;
            if (o[0] != k || o[1] != r.dy || o[2] != r.dz) return false;
        }
    }
    return e == kTOff;
}

// tensor maps of the tile kernel: f[b] as {Ks, n, n, n} with box {kTN, kTX, kTY, kTZ}; the table as
// {Ks, 123} with box {kTN, 123}
bool make_tile_maps(bgk_ctx* c) {
    PFN_cuTensorMapEncodeTiled_v12000 encode = encoder();
    if (!encode) return false;
    const cuuint64_t n = (cuuint64_t)c->tile_nlat;
    const cuuint64_t dims[4] = {(cuuint64_t)c->Ks, n, n, n};
    const cuuint64_t strides[3] = {(cuuint64_t)c->Ks * sizeof(double), n * c->Ks * sizeof(double),
                                   n * n * c->Ks * sizeof(double)};
    const cuuint32_t box[4] = {kTN, kTX, kTY, kTZ};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    for (int b = 0; b < 2; ++b)
        if (encode(&c->tmap_halo[b], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, c->f[b], dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
    const cuuint64_t cd[2] = {(cuuint64_t)c->Ks, (cuuint64_t)(kTOff + 1)};
    const cuuint64_t cst[1] = {(cuuint64_t)c->Ks * sizeof(double)};
    const cuuint32_t cb[2] = {kTN, kTOff + 1};
    return encode(&c->tmap_ctab, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, c->ctab, cd, cst, cb, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

void launch_tile_ctab(bgk_ctx* c, int64_t off_ref, cudaStream_t s) {
    k_tile_ctab<<<(unsigned)((c->Ks + 255) / 256), 256, 0, s>>>(c->g.P, off_ref, c->ctab, c->Ks, c->n1, c->ncol,
                                                                 c->ncs, c->c0, c->cfg.vmax, c->dv);
}

int tile_particles() { return 512; }
int tile_ranges(const bgk_ctx* c) { return std::min(c->nwpp, 20); }

void launch_transport_tile(bgk_ctx* c, const double* fin, double* fout, cudaStream_t s) {
    if (c->n_tiles == 0) return;
    const size_t smem = 2 * kTStage + 16;
    static bool configured[kMaxDevices] = {};
    if (first_use_on_device(configured))
        cudaFuncSetAttribute(k_transport_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    TileArgs a;
    a.org = c->tile_org;
    a.ft = fout;
    a.partials = c->partials;
    a.stab = c->stab;
    a.Ks = c->Ks;
    a.nlat = c->tile_nlat;
    a.nwpp = c->nwpp;
    a.nq = tile_ranges(c);
    a.nchunk = (int)(c->Ks / kTN);
    a.n1 = c->n1;
    a.ncol = c->ncol;
    a.ncs = c->ncs;
    a.c0 = c->c0;
    a.vmax = c->cfg.vmax;
    a.dv = c->dv;
    a.dt = c->cfg.dt;
    k_transport_tile<<<dim3((unsigned)c->n_tiles, (unsigned)a.nq), kTThreads, smem, s>>>(
        c->tmap_halo[fin == c->f[0] ? 0 : 1], c->tmap_ctab, a);
}

}  // namespace bgk
