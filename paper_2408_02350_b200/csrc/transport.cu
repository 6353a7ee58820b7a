// transport.cu -- the hot loop: positive upwind transport (PAPER.md:163-171,
// 384-481) fused with the per-particle moment partial sums (PAPER.md:185-193,
// 226-255).
//
// For interior particle i and every local velocity node k (c = v_k - W_i,
// W = U^n in ALE mode, 0 on a fixed cloud):
//     C_ijk = sum_{e in n,t[,b]} (P_e.c - |P_e.c|)          (P_e = rot_e * frame_e, wls.cu)
//           = L_j(c) - |y_n| - |y_t| - |y_b|,   L_j(c) = a_j.c = y_n + y_t + y_b
//     ftilde_ik = f_ik - dt * sum_j C_ijk (f_jk - f_ik)     (g1 and g2 share C_ijk in 2D)
//
// Mapping: a warp owns one particle, one chunk of R nodes along v_1
// and a group of 32 velocity columns; each lane owns one column and walks the R
// nodes.  Along v_1 every projection is affine, so y_e and L advance by one add per
// node.  Per (i, j, k) triple: 4 increments, 3 abs-subtracts (free |.| operand
// modifier), 1 FMA (sum C f_j), 1 add (sum C) = 9 DP instructions, plus one LDS.
//
// Neighbour rows are staged by TMA: for each neighbour j one elected lane issues a
// cp.async.bulk.tensor.3d of the box f[j][k1s .. k1s+R)[cols .. cols+32) (6.4 KB in 3D)
// into the warp's NST-deep ring of shared-memory stages, NST-1 neighbours ahead of
// the one being consumed (mbarrier expect_tx / try_wait.parity).  The box's
// out-of-range columns (last column group) are zero-filled by the TMA unit.  Pair
// data P_{j+1} are prefetched into registers one neighbour ahead.  The epilogue
// writes ftilde, reduces the warp's moment partials with shuffles in a fixed order
// (no atomics: bitwise deterministic) and folds max_k sum_j |C_ijk| (stable_dt) into
// one atomicMax.
#include <cudaTypedefs.h>

#include <cstdlib>

#include "bgk_internal.cuh"

namespace bgk {

namespace {

constexpr int kDefaultWarps = 8;   // warps per block (= particles per block); tuned on B200, see DESIGN.md

struct TArgs {
    const double* __restrict__ f;
    double* __restrict__ ft;
    const double* __restrict__ W;
    const int32_t* __restrict__ order;
    const int64_t* __restrict__ nb_off;
    const int32_t* __restrict__ nb_idx;
    const double* __restrict__ P;
    double* __restrict__ partials;
    unsigned long long* stab;
    int64_t n_int;
    int n1, ncol, ncs, c0, ncg, nwpp;
    double vmax, dv, dt;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int c0, int c1, int c2,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// One ring stage: the neighbour's box of f (R rows x 32 columns x nv) and its pair data P_e.
template <int D, int R>
struct Stage {
    static constexpr int NV = (D == 2) ? 2 : 1;
    static constexpr int PD = (D == 2) ? 4 : 10;
    static constexpr int ROW = 32 * NV;                                  // doubles per staged row
    static constexpr uint32_t F_BYTES = R * ROW * sizeof(double);
    static constexpr uint32_t P_BYTES = PD * sizeof(double);
    static constexpr uint32_t BYTES = (F_BYTES + P_BYTES + 127) / 128 * 128;
};

template <int D, int R, int NST, int WPB>
__global__ void __launch_bounds__(WPB * 32, 1) k_transport(const __grid_constant__ CUtensorMap tmap, const TArgs A) {
    using St = Stage<D, R>;
    constexpr int NV = St::NV;
    constexpr int PD = St::PD;
    constexpr int ROW = St::ROW;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    unsigned char* ring = smem_raw + (size_t)wib * NST * St::BYTES;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + (size_t)WPB * NST * St::BYTES) + wib * NST;

    const int64_t pos = (int64_t)blockIdx.x * WPB + wib;
    if (pos >= A.n_int) return;                           // warp-uniform
    const int w = blockIdx.y;
    const int chunk = w / A.ncg, cg = w - chunk * A.ncg;
    const int p = A.order[pos];
    const int col = cg * 32 + lane;
    const bool valid = col < A.ncol;
    const int k1s = chunk * R;
    const int colc = valid ? col : 0;
    const int gc = A.c0 + colc;
    const int64_t off = A.nb_off[p];
    const int m = (int)(A.nb_off[p + 1] - off);
    const int32_t* nbl = A.nb_idx + off;
    const double* Pp = A.P + off * PD;
    // neighbour indices, 32 per register batch: nbA holds [32b, 32b+32), nbB the next batch
    int nbA = lane < m ? __ldg(nbl + lane) : 0;
    int nbB = 32 + lane < m ? __ldg(nbl + 32 + lane) : 0;

    auto issue = [&](int e, int jn) {      // lane 0 only: stage e % NST <- neighbour e
        const int s = e % NST;
        unsigned char* st = ring + s * St::BYTES;
        mbar_expect_tx(bars + s, St::F_BYTES + St::P_BYTES);
        tma_load_3d(st, &tmap, cg * ROW, k1s, jn, bars + s);
        bulk_load(st + St::F_BYTES, Pp + (int64_t)e * PD, St::P_BYTES, bars + s);
    };
    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < NST; ++s) mbar_init(bars + s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncwarp();
#pragma unroll
    for (int s = 0; s < NST; ++s) {
        const int jn = __shfl_sync(0xffffffffu, nbA, s);
        if (lane == 0 && s < m) issue(s, jn);
    }

    // velocity of this lane's column at k1 = k1s, relative to W_p
    double Wp[D];
#pragma unroll
    for (int a = 0; a < D; ++a) Wp[a] = A.W[(int64_t)p * D + a];
    double c0v[D];
    c0v[0] = axis_node(A.vmax, A.dv, k1s) - Wp[0];
    if constexpr (D == 3) {
        const int k2 = gc / A.n1, k3 = gc - k2 * A.n1;
        c0v[1] = axis_node(A.vmax, A.dv, k2) - Wp[1];
        c0v[2] = axis_node(A.vmax, A.dv, k3) - Wp[2];
    } else {
        c0v[1] = axis_node(A.vmax, A.dv, gc) - Wp[1];
    }
    double Qf[R][NV], Sc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        Sc[r] = 0.0;
#pragma unroll
        for (int q = 0; q < NV; ++q) Qf[r][q] = 0.0;
    }
    for (int e = 0; e < m; ++e) {
        const int s = e % NST;
        const uint32_t parity = (uint32_t)(e / NST) & 1u;
        const unsigned char* stb = ring + s * St::BYTES;
        mbar_wait(bars + s, parity);
        double pv[PD];
        const double* ps = reinterpret_cast<const double*>(stb + St::F_BYTES);
#pragma unroll
        for (int q = 0; q < PD; ++q) pv[q] = ps[q];       // broadcast LDS
        double y[D], dy[D];
#pragma unroll
        for (int k = 0; k < D; ++k) {
            double t = pv[k * D] * c0v[0];
#pragma unroll
            for (int a = 1; a < D; ++a) t = fma(pv[k * D + a], c0v[a], t);
            y[k] = t;
            dy[k] = A.dv * pv[k * D];
        }
        double Lc = y[0], dL = dy[0];
#pragma unroll
        for (int k = 1; k < D; ++k) { Lc += y[k]; dL += dy[k]; }
        const double* st = reinterpret_cast<const double*>(stb) + lane * NV;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            // y_e(r) = y_e(0) + r dy_e: one FMA each with r an immediate -> rows are independent
            // (no add chain across r); C = (L - |y_n|) - (|y_t| + |y_b|) keeps the chain 2 deep
            const double rr = (double)r;
            const double Lr = fma(rr, dL, Lc);
            double C;
            if constexpr (D == 3) {
                const double yn = fma(rr, dy[0], y[0]);
                const double yt = fma(rr, dy[1], y[1]);
                const double yb = fma(rr, dy[2], y[2]);
                C = (Lr - fabs(yn)) - (fabs(yt) + fabs(yb));
            } else {
                const double yn = fma(rr, dy[0], y[0]);
                const double yt = fma(rr, dy[1], y[1]);
                C = (Lr - fabs(yn)) - fabs(yt);
            }
            if constexpr (NV == 1) {
                const double v = st[r * ROW];
                Qf[r][0] = fma(C, v, Qf[r][0]);
            } else {
                const double2 v = *reinterpret_cast<const double2*>(st + r * ROW);
                Qf[r][0] = fma(C, v.x, Qf[r][0]);
                Qf[r][1] = fma(C, v.y, Qf[r][1]);
            }
            Sc[r] += C;
        }
        // refill stage s with neighbour e + NST (index from the register batches)
        const int t = e + NST;
        if ((t & 31) == 0) {                               // warp-uniform batch rotation
            nbA = nbB;
            nbB = t + 32 + lane < m ? __ldg(nbl + t + 32 + lane) : 0;
        }
        const int jn = __shfl_sync(0xffffffffu, nbA, t & 31);
        __syncwarp();   // every lane has consumed stage s before it is refilled
        if (lane == 0 && t < m) issue(t, jn);
    }
    // epilogue: ftilde, moment partials, stability bound
    const int64_t rowstride = (int64_t)A.ncs * NV;
    const int64_t lane_off = (int64_t)k1s * rowstride + (int64_t)colc * NV;
    const double* fi = A.f + (int64_t)p * A.n1 * rowstride + lane_off;
    double* fto = A.ft + (int64_t)p * A.n1 * rowstride + lane_off;
    double v2v = 0.0, v3v = 0.0;
    if constexpr (D == 3) {
        const int k2 = gc / A.n1, k3 = gc - k2 * A.n1;
        v2v = axis_node(A.vmax, A.dv, k2);
        v3v = axis_node(A.vmax, A.dv, k3);
    } else {
        v2v = axis_node(A.vmax, A.dv, gc);
    }
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0, sE = 0.0, amax = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const double v1 = axis_node(A.vmax, A.dv, k1s + r);
        const double vv = (D == 3) ? v1 * v1 + v2v * v2v + v3v * v3v : v1 * v1 + v2v * v2v;
        double out[NV];
        if constexpr (NV == 1) {
            const double fv = __ldg(fi + r * rowstride);
            out[0] = fv - A.dt * (Qf[r][0] - fv * Sc[r]);
            if (valid) fto[r * rowstride] = out[0];
        } else {
            const double2 fv = __ldg(reinterpret_cast<const double2*>(fi + r * rowstride));
            out[0] = fv.x - A.dt * (Qf[r][0] - fv.x * Sc[r]);
            out[1] = fv.y - A.dt * (Qf[r][1] - fv.y * Sc[r]);
            if (valid) *reinterpret_cast<double2*>(fto + r * rowstride) = make_double2(out[0], out[1]);
        }
        if (valid) {
            s0 += out[0];
            s1 += v1 * out[0];
            s2 += v2v * out[0];
            if constexpr (D == 3) s3 += v3v * out[0];
            sE += vv * out[0];
            if constexpr (NV == 2) sE += out[1];
            amax = fmax(amax, -Sc[r]);
        }
    }
    s0 = warp_sum(s0);
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    s3 = warp_sum(s3);
    sE = warp_sum(sE);
    amax = warp_max(amax);
    if (lane == 0) {
        double* pp = A.partials + ((int64_t)p * A.nwpp + w) * kPM;
        pp[0] = s0;
        pp[1] = s1;
        pp[2] = s2;
        if constexpr (D == 3) {
            pp[3] = s3;
            pp[4] = sE;
        } else {
            pp[3] = sE;
            pp[4] = 0.0;
        }
        atomicMax(A.stab, (unsigned long long)__double_as_longlong(amax));
    }
}

template <int D, int R, int WPB>
constexpr int stages_for() {
    // ring depth: keep NST-1 neighbour boxes in flight; bounded by 227 KB of shared memory
    constexpr int n = (220 * 1024) / (WPB * Stage<D, R>::BYTES);
    return n > 4 ? 4 : (n < 2 ? 2 : n);
}

template <int D, int R, int WPB>
void launch_one(const CUtensorMap& tm, const TArgs& a, cudaStream_t s) {
    constexpr int NST = stages_for<D, R, WPB>();
    constexpr size_t smem = (size_t)WPB * NST * Stage<D, R>::BYTES + WPB * NST * 8;
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(k_transport<D, R, NST, WPB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = true;
    }
    const unsigned gx = (unsigned)((a.n_int + WPB - 1) / WPB);
    k_transport<D, R, NST, WPB><<<dim3(gx, (unsigned)a.nwpp), WPB * 32, smem, s>>>(tm, a);
}

template <int D, int R>
void launch_wpb(int wpb, const CUtensorMap& tm, const TArgs& a, cudaStream_t s) {
    if constexpr (D == 3 && (R == 25 || R == 17)) {
        if (wpb == 12) return launch_one<D, R, 12>(tm, a, s);
        if (wpb == 16) return launch_one<D, R, 16>(tm, a, s);
        if (wpb == 4) return launch_one<D, R, 4>(tm, a, s);
    }
    launch_one<D, R, kDefaultWarps>(tm, a, s);
}

template <int D>
void dispatch(int R, int wpb, const CUtensorMap& tm, const TArgs& a, cudaStream_t s) {
    if constexpr (D == 3) {
        switch (R) {
            case 25: launch_wpb<D, 25>(wpb, tm, a, s); return;
            case 21: launch_wpb<D, 21>(wpb, tm, a, s); return;
            case 17: launch_wpb<D, 17>(wpb, tm, a, s); return;
            default: break;
        }
    }
    switch (R) {
        case 13: launch_wpb<D, 13>(wpb, tm, a, s); break;
        case 11: launch_wpb<D, 11>(wpb, tm, a, s); break;
        case 9: launch_wpb<D, 9>(wpb, tm, a, s); break;
        case 7: launch_wpb<D, 7>(wpb, tm, a, s); break;
        case 5: launch_wpb<D, 5>(wpb, tm, a, s); break;
        case 3: launch_wpb<D, 3>(wpb, tm, a, s); break;
        default: launch_wpb<D, 1>(wpb, tm, a, s); break;
    }
}

constexpr int kRChoices3[] = {25, 21, 17, 13, 11, 9, 7, 5, 3, 1};
constexpr int kRChoices2[] = {13, 11, 9, 7, 5, 3, 1};

}  // namespace

// rows per thread: the largest divisor of n1 among the instantiated R (2D keeps three
// accumulators per row, so it stops at 13)
int transport_rows_per_thread(int d, int n1) {
    if (d == 3) {
        for (int R : kRChoices3)
            if (n1 % R == 0) return R;
    } else {
        for (int R : kRChoices2)
            if (n1 % R == 0) return R;
    }
    return 1;
}

// TMA descriptors: f[b] viewed as a 3D fp64 tensor {ncs*nv (fastest), n1, N}; box {32*nv, R, 1}.
bool make_tensor_maps(bgk_ctx* c) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return false;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint64_t dims[3] = {(cuuint64_t)c->ncs * c->nv, (cuuint64_t)c->n1, (cuuint64_t)c->N};
    const cuuint64_t strides[2] = {(cuuint64_t)c->ncs * c->nv * sizeof(double),
                                   (cuuint64_t)c->ncs * c->nv * c->n1 * sizeof(double)};
    const cuuint32_t box[3] = {(cuuint32_t)(32 * c->nv), (cuuint32_t)c->R, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    for (int b = 0; b < 2; ++b) {
        CUresult r = encode(&c->tmap[b], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, c->f[b], dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return false;
    }
    return true;
}

void launch_transport(bgk_ctx* c, const double* fin, double* fout, cudaStream_t s) {
    if (c->N_int == 0) return;
    TArgs a;
    a.f = fin;
    a.ft = fout;
    a.W = c->W;
    a.order = c->g.order;
    a.nb_off = c->g.nb_off;
    a.nb_idx = c->g.nb_idx;
    a.P = c->g.P;
    a.partials = c->partials;
    a.stab = c->stab;
    a.n_int = c->N_int;
    a.n1 = c->n1;
    a.ncol = c->ncol;
    a.ncs = c->ncs;
    a.c0 = c->c0;
    a.ncg = c->ncg;
    a.nwpp = c->nwpp;
    a.vmax = c->cfg.vmax;
    a.dv = c->dv;
    a.dt = c->cfg.dt;
    const CUtensorMap& tm = c->tmap[fin == c->f[0] ? 0 : 1];
    static const int wpb = [] {
        const char* e = getenv("BGK_TRANSPORT_WPB");   // tuning knob (4, 8, 12, 16); default 8
        return e ? atoi(e) : kDefaultWarps;
    }();
    if (c->d == 3) dispatch<3>(c->R, wpb, tm, a, s);
    else dispatch<2>(c->R, wpb, tm, a, s);
}

}  // namespace bgk
