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

constexpr int kDefaultWarps = 4;   // warps per block (= particles per block); tuned on B200 (profiles/r01_tuning.md)

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
    unsigned long long* work;          // persistent-warp item counter (zeroed before each launch)
    const int32_t* __restrict__ gU;    // grouped kernel: union neighbour list per particle group
    const int32_t* __restrict__ gUlen; //                 its length
    const uint8_t* __restrict__ gCnt;  //                 users of each union member
    const uint16_t* __restrict__ upos; //                 union position of each CSR entry
    int ucap;                          //                 capacity per group
    bool signed_n;                     // second-order WLS: pair record carries s_n = -sign(abar)
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

// one elected lane of a fully active warp (elect.sync): the TMA operands it uses are warp-uniform,
// so the compiler issues them from uniform registers without a per-lane serialisation loop
__device__ __forceinline__ bool elect_one() {
    uint32_t pred;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "elect.sync _|p, 0xffffffff;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(pred));
    return pred != 0;
}

// non-blocking phase test: 1 if the phase with the given parity has completed
__device__ __forceinline__ uint32_t mbar_test(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok;
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


// Per (neighbour, lane) coefficients at the chunk's first node k1s:
//   y_e = P_e . c0 (c0 = v(k1s, col) - W), dy_e = dv P_e[0] (increment per v_1 node),
//   L = sum_e y_e, dL = sum_e dy_e.
// In 3D the pair record already holds dy_e in slot 3e and dL in slot 9 (k_wls_interior), and
// P_e[0] c1 = dy_e (c1 / dv) with c1dv = c0[0] / dv precomputed per lane.
template <int D>
__device__ __forceinline__ void pair_coeffs(const double* pv, const double (&c0v)[D], double c1dv, double dv,
                                            double (&y)[D], double (&dy)[D], double& Lc, double& dL) {
    if constexpr (D == 3) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            dy[k] = pv[k * 3];
            y[k] = fma(pv[k * 3], c1dv, fma(pv[k * 3 + 1], c0v[1], pv[k * 3 + 2] * c0v[2]));
        }
        Lc = (y[0] + y[1]) + y[2];
        dL = pv[9];
    } else {
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            y[k] = fma(pv[k * 2 + 1], c0v[1], pv[k * 2] * c0v[0]);
            dy[k] = dv * pv[k * 2];
        }
        Lc = y[0] + y[1];
        dL = dy[0] + dy[1];
    }
}

// One ring stage: the neighbour's box of f (R rows x 32 columns x nv) and its pair data P_e.
// SG (second-order WLS): the pair record carries s_n = -sign(abar) after the first-order fields,
// and C's n-term is y_n + s_n |y_n| (abar may be negative; P:408-410 applied literally).
template <int D, int R, bool SG = false>
struct Stage {
    static constexpr int NV = (D == 2) ? 2 : 1;
    static constexpr int PD0 = (D == 2) ? 4 : 10;
    static constexpr int PD = SG ? PD0 + 2 : PD0;
    static constexpr int ROW = 32 * NV;                                  // doubles per staged row
    static constexpr uint32_t F_BYTES = R * ROW * sizeof(double);
    static constexpr uint32_t P_BYTES = PD * sizeof(double);
    static constexpr uint32_t BYTES = (F_BYTES + P_BYTES + 127) / 128 * 128;
};

template <int D, int R, int NST, int WPB, bool SG>
__global__ void __launch_bounds__(WPB * 32, 1) k_transport(const __grid_constant__ CUtensorMap tmap, const TArgs A) {
    using St = Stage<D, R, SG>;
    constexpr int NV = St::NV;
    constexpr int PD = St::PD;
    constexpr int ROW = St::ROW;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    unsigned char* ring = smem_raw + (size_t)wib * NST * St::BYTES;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + (size_t)WPB * NST * St::BYTES) + wib * NST;

    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < NST; ++s) mbar_init(bars + s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncwarp();
    // One (particle, chunk x column group) item per warp; gridDim.y (the column group) is the
    // slowest launch dimension so one group's f slab stays L2-resident.  (A persistent-warp
    // variant pulling items from a global counter measured 8 % slower on C5; the ring
    // indexing below keeps the running stage offset g0 so items could be chained.)
    const uint32_t g0 = 0;
    {
    const int w = blockIdx.y;
    const int64_t pos = (int64_t)blockIdx.x * WPB + wib;
    if (pos >= A.n_int) return;                           // warp-uniform
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

    auto issue = [&](int e, int jn) {      // lane 0 only: ring stage of neighbour e <- its box + pair data
        const int s = (int)((g0 + (uint32_t)e) % NST);
        unsigned char* st = ring + s * St::BYTES;
        mbar_expect_tx(bars + s, St::F_BYTES + St::P_BYTES);
#ifdef BGK_EXP_SAMEBOX
        jn = p;   // timing experiment: always the particle's own (L2-hot) box
#endif
        tma_load_3d(st, &tmap, cg * ROW, k1s, jn, bars + s);
        bulk_load(st + St::F_BYTES, Pp + (int64_t)e * PD, St::P_BYTES, bars + s);
    };
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
    double Qf[R][NV], Sc[R], Sa[SG ? R : 1];   // Sa: sum_j |C| (= -Sc when every C <= 0)
#pragma unroll
    for (int r = 0; r < R; ++r) {
        Sc[r] = 0.0;
        if constexpr (SG) Sa[r] = 0.0;
#pragma unroll
        for (int q = 0; q < NV; ++q) Qf[r][q] = 0.0;
    }
    // per-neighbour coefficients at the chunk's first node: y_e = P_e . c0, dy_e = dv P_e[0],
    // L = sum_e y_e, dL = sum_e dy_e (read from the stage's pair-data slot)
    const double c1dv = c0v[0] / A.dv;
    auto coeffs = [&](int e, double (&y)[D], double (&dy)[D], double& Lc, double& dL, double& sn) {
        const double* ps =
            reinterpret_cast<const double*>(ring + ((g0 + (uint32_t)e) % NST) * St::BYTES + St::F_BYTES);
        double pv[PD];
#pragma unroll
        for (int q = 0; q < PD; ++q) pv[q] = ps[q];       // broadcast LDS
        pair_coeffs<D>(pv, c0v, c1dv, A.dv, y, dy, Lc, dL);
        if constexpr (SG) sn = pv[St::PD0];
    };
    // The readiness of the NEXT stage is tested (non-blocking mbarrier.test_wait) before this
    // neighbour's rows, so the barrier check's latency overlaps the row arithmetic; only if the
    // next box has not landed by the end of the rows does the warp spin on try_wait.
    double y[D], dy[D], Lc = 0.0, dL = 0.0, sn = -1.0;
    if (m > 0) {
        mbar_wait(bars + g0 % NST, (g0 / NST) & 1u);
        coeffs(0, y, dy, Lc, dL, sn);
    }
    for (int e = 0; e < m; ++e) {
        const uint32_t ge = g0 + (uint32_t)e;
        const bool more = e + 1 < m;
        const uint32_t nready = more ? mbar_test(bars + (ge + 1) % NST, ((ge + 1) / NST) & 1u) : 1u;
        const double* st = reinterpret_cast<const double*>(ring + (ge % NST) * St::BYTES) + lane * NV;
        // y_e and L advance by one add per node along v_1 (all DADD: measured ~2 % faster than
        // the independent-FMA form y_e(r) = fma(r, dy_e, y_e(0)))
        double yi[D], Li = Lc;
#pragma unroll
        for (int k = 0; k < D; ++k) yi[k] = y[k];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            double C;
            if constexpr (SG) {
                if constexpr (D == 3) C = fma(fabs(yi[0]), sn, Li) - fabs(yi[1]) - fabs(yi[2]);
                else C = fma(fabs(yi[0]), sn, Li) - fabs(yi[1]);
                Sa[r] += fabs(C);
            } else {
                if constexpr (D == 3) C = Li - fabs(yi[0]) - fabs(yi[1]) - fabs(yi[2]);
                else C = Li - fabs(yi[0]) - fabs(yi[1]);
            }
#pragma unroll
            for (int k = 0; k < D; ++k) yi[k] += dy[k];
            Li += dL;
            if constexpr (NV == 1) {
                Qf[r][0] = fma(C, st[r * ROW], Qf[r][0]);
            } else {
                const double2 v = *reinterpret_cast<const double2*>(st + r * ROW);
                Qf[r][0] = fma(C, v.x, Qf[r][0]);
                Qf[r][1] = fma(C, v.y, Qf[r][1]);
            }
            Sc[r] += C;
        }
        // refill stage of neighbour e with neighbour e + NST (index from the register batches)
        const int t = e + NST;
        if ((t & 31) == 0) {                               // warp-uniform batch rotation
            nbA = nbB;
            nbB = t + 32 + lane < m ? __ldg(nbl + t + 32 + lane) : 0;
        }
        const int jn = __shfl_sync(0xffffffffu, nbA, t & 31);
        __syncwarp();   // every lane has consumed the stage before it is refilled
#ifndef BGK_EXP_NOPIPE   // timing experiment: no refills, no waits (stale data; compute ceiling)
        if (t < m && elect_one()) issue(t, jn);
#endif
        if (more) {
#ifndef BGK_EXP_NOPIPE
            if (!nready) mbar_wait(bars + (ge + 1) % NST, ((ge + 1) / NST) & 1u);
#else
            (void)nready;
#endif
            asm volatile("" ::: "memory");                 // order the stage reads after the test
            coeffs(e + 1, y, dy, Lc, dL, sn);
        }
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
        if (k1s + r >= A.n1) break;                      // ragged last chunk (rows past Nv are TMA zero-fill)
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
            if constexpr (SG) amax = fmax(amax, Sa[r]);
            else amax = fmax(amax, -Sc[r]);
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
}
// ============================================================================
// Grouped transport: one block = G particles (consecutive in the Morton-ordered interior
// list) x one (chunk, column group).  The block walks the sorted UNION of the G neighbour
// lists (precomputed per step by k_group_union); every union neighbour's box is fetched
// ONCE by TMA into a block-shared ring and consumed by every warp whose particle has it.
// On C5 the union of 8 Morton-consecutive particles has ~276 members against 947
// per-particle neighbours, so the L2 -> SM traffic that bounded the per-warp ring
// (~12-13 TB/s, the chip's L2 throughput cap) drops 3.4x.
//   stage fill  : cp.async.bulk.tensor.3d, complete_tx on full[s]
//   stage reuse : each warp, after waiting full[s] and (if the neighbour is its own)
//                 applying it, bumps rel[s]; the G-th release re-arms and refills the stage
//                 NST union members ahead.  Warps may drift up to NST members apart.
//   pair data   : per warp, batches of 8 pair records by cp.async.bulk into a 2-deep ring.
// ============================================================================
constexpr int kGroup = 8;
constexpr int kPBatch = 8;
#ifndef BGK_GRP_MAX_STAGES
#define BGK_GRP_MAX_STAGES 32
#endif
constexpr int kMaxGrpStages = BGK_GRP_MAX_STAGES;   // shared ring depth cap (smem bound: ~30 at R = 25)

template <int D, int R>
struct GStage {
    static constexpr int NV = (D == 2) ? 2 : 1;
    static constexpr int PD = (D == 2) ? 4 : 10;
    static constexpr int ROW = 32 * NV;
    static constexpr uint32_t F_BYTES = R * ROW * sizeof(double);           // multiple of 128 (R*256)
    static constexpr uint32_t PB_BYTES = kPBatch * PD * sizeof(double);    // 640 B (3D) / 256 B (2D)
};

template <int D, int R, int NST>
constexpr size_t grp_smem_bytes(int ucap) {
    using St = GStage<D, R>;
    return (size_t)NST * St::F_BYTES + (size_t)kGroup * 2 * St::PB_BYTES + (size_t)ucap * 5 +
           (NST + 2 * kGroup) * 8 + NST * 8 + 256;
}

template <int D, int R, int NST>
__global__ void __launch_bounds__(kGroup * 32, 1) k_transport_grp(const __grid_constant__ CUtensorMap tmap,
                                                                  const TArgs A) {
    using St = GStage<D, R>;
    constexpr int NV = St::NV;
    constexpr int PD = St::PD;
    constexpr int ROW = St::ROW;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char* ring = smem_raw;
    double* pring = reinterpret_cast<double*>(smem_raw + (size_t)NST * St::F_BYTES);
    int32_t* sU = reinterpret_cast<int32_t*>(smem_raw + (size_t)NST * St::F_BYTES + (size_t)kGroup * 2 * St::PB_BYTES);
    uint64_t* full = reinterpret_cast<uint64_t*>(sU + A.ucap + ((A.ucap & 1) ? 1 : 0));
    uint64_t* pbar = full + NST;                            // [kGroup][2]
    int* rel = reinterpret_cast<int*>(pbar + 2 * kGroup);   // [NST]
    volatile int* smem_member = rel + NST;                  // [NST] union member a stage holds / will hold
    uint8_t* sCnt = reinterpret_cast<uint8_t*>(rel + 2 * NST);  // [ucap]

    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int group = blockIdx.x;
    const int w = blockIdx.y;
    const int chunk = w / A.ncg, cg = w - chunk * A.ncg;
    const int k1s = chunk * R;
    const int ulen = A.gUlen[group];
    const int32_t* gU = A.gU + (int64_t)group * A.ucap;
    for (int q = threadIdx.x; q < ulen; q += blockDim.x) {
        sU[q] = gU[q];
        sCnt[q] = A.gCnt[(int64_t)group * A.ucap + q];
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(full + s, 1);
            rel[s] = 0;
            smem_member[s] = s;
        }
        for (int g = 0; g < 2 * kGroup; ++g) mbar_init(pbar + g, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int s = 0; s < NST && s < ulen; ++s) {
            mbar_expect_tx(full + s, St::F_BYTES);
            tma_load_3d(ring + s * St::F_BYTES, &tmap, cg * ROW, k1s, sU[s], full + s);
        }

    // this warp's particle (an idle warp of a short last group still releases every stage)
    const int64_t pos = (int64_t)group * kGroup + wib;
    const bool active = pos < A.n_int;
    const int p = active ? A.order[pos] : 0;
    const int64_t off = active ? A.nb_off[p] : 0;
    const int m = active ? (int)(A.nb_off[p + 1] - off) : 0;
    const double* Pp = A.P + off * PD;
    const int col = cg * 32 + lane;
    const bool valid = active && col < A.ncol;
    const int colc = col < A.ncol ? col : 0;
    const int gc = A.c0 + colc;
    const uint16_t* upl = A.upos + off;
    int nbA = lane < m ? (int)__ldg(upl + lane) : 0;       // union positions of my neighbours, 32 per batch
    int nbB = 32 + lane < m ? (int)__ldg(upl + 32 + lane) : 0;
    double* myP = pring + (size_t)wib * 2 * kPBatch * PD;
    auto issue_pbatch = [&](int b) {          // lane 0: pair records [8b, 8b+8) -> buffer b & 1
        const int n = min(kPBatch, m - b * kPBatch);
        if (n <= 0) return;
        uint64_t* bar = pbar + wib * 2 + (b & 1);
        mbar_expect_tx(bar, (uint32_t)(n * PD * sizeof(double)));
        bulk_load(myP + (b & 1) * kPBatch * PD, Pp + (int64_t)b * kPBatch * PD, (uint32_t)(n * PD * sizeof(double)),
                  bar);
    };
    if (lane == 0) {
        issue_pbatch(0);
        issue_pbatch(1);
    }

    double Wp[D];
#pragma unroll
    for (int a = 0; a < D; ++a) Wp[a] = active ? A.W[(int64_t)p * D + a] : 0.0;
    double c0v[D];
    c0v[0] = axis_node(A.vmax, A.dv, k1s) - Wp[0];
    if constexpr (D == 3) {
        const int k2 = gc / A.n1, k3 = gc - k2 * A.n1;
        c0v[1] = axis_node(A.vmax, A.dv, k2) - Wp[1];
        c0v[2] = axis_node(A.vmax, A.dv, k3) - Wp[2];
    } else {
        c0v[1] = axis_node(A.vmax, A.dv, gc) - Wp[1];
    }
    const double c1dv = c0v[0] / A.dv;
    double Qf[R][NV], Sc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        Sc[r] = 0.0;
#pragma unroll
        for (int q = 0; q < NV; ++q) Qf[r][q] = 0.0;
    }
    // Each warp visits only its own neighbours; neighbour e sits at union position u.  A
    // member's stage is refilled (NST members ahead) by the last of its sCnt[u] users.
    for (int e = 0; e < m; ++e) {
        const int u = __shfl_sync(0xffffffffu, nbA, e & 31);
        if ((e & 31) == 31) {                               // warp-uniform batch rotation
            nbA = nbB;
            nbB = e + 33 + lane < m ? (int)__ldg(upl + e + 33 + lane) : 0;
        }
        const int s = u % NST;
        const int b = e / kPBatch, eb = e - b * kPBatch;
        if (eb == 0) {
            mbar_wait(pbar + wib * 2 + (b & 1), (uint32_t)(b >> 1) & 1u);
            if (b >= 1 && lane == 0) issue_pbatch(b + 1);  // buffer (b+1)&1 held batch b-1: done
        }
        const double* ps = myP + (b & 1) * kPBatch * PD + eb * PD;
        double pv[PD];
#pragma unroll
        for (int q = 0; q < PD; ++q) pv[q] = ps[q];
        double y[D], dy[D], Lc, dL;
        pair_coeffs<D>(pv, c0v, c1dv, A.dv, y, dy, Lc, dL);
        // a warp may run many members ahead of a slow one: wait until stage s has been armed for
        // member u (parity waits alone cannot tell rounds two phases apart), then for the data
        while (smem_member[s] != u) __nanosleep(64);
        mbar_wait(full + s, (uint32_t)(u / NST) & 1u);
        const double* st = reinterpret_cast<const double*>(ring + s * St::F_BYTES) + lane * NV;
#pragma unroll
        for (int r = 0; r < R; ++r) {
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
                Qf[r][0] = fma(C, st[r * ROW], Qf[r][0]);
            } else {
                const double2 v = *reinterpret_cast<const double2*>(st + r * ROW);
                Qf[r][0] = fma(C, v.x, Qf[r][0]);
                Qf[r][1] = fma(C, v.y, Qf[r][1]);
            }
            Sc[r] += C;
        }
        __syncwarp();
        if (lane == 0) {                                    // release; the member's last user refills
            if (atomicAdd(rel + s, 1) == (int)sCnt[u] - 1) {
                rel[s] = 0;
                if (u + NST < ulen) {
                    smem_member[s] = u + NST;
                    __threadfence_block();
                    mbar_expect_tx(full + s, St::F_BYTES);
                    tma_load_3d(ring + s * St::F_BYTES, &tmap, cg * ROW, k1s, sU[u + NST], full + s);
                }
            }
        }
    }
    if (!active) return;
    // epilogue (as k_transport): ftilde, moment partials, stability bound
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
        if (k1s + r >= A.n1) break;
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

// Union of the neighbour lists of each group of kGroup consecutive particles of `order`:
// bitonic sort of the concatenated lists in shared memory, then drop duplicates.
__global__ void __launch_bounds__(256) k_group_union(const int32_t* __restrict__ order, int64_t n_int,
                                                     const int64_t* __restrict__ nb_off,
                                                     const int32_t* __restrict__ nb_idx, int ucap,
                                                     int32_t* __restrict__ gU, int32_t* __restrict__ gUlen,
                                                     uint8_t* __restrict__ gCnt, uint16_t* __restrict__ upos) {
    extern __shared__ int32_t sa[];                         // [ucap] sort buffer, then [ucap] union
    int32_t* su = sa + ucap;
    __shared__ int s_len[kGroup + 1];
    __shared__ int wsum[8];
    const int group = blockIdx.x;
    if (threadIdx.x == 0) {
        int tot = 0;
        for (int g = 0; g < kGroup; ++g) {
            const int64_t pos = (int64_t)group * kGroup + g;
            s_len[g] = tot;
            if (pos < n_int) {
                const int p = order[pos];
                tot += (int)(nb_off[p + 1] - nb_off[p]);
            }
        }
        s_len[kGroup] = tot;
    }
    __syncthreads();
    const int tot = s_len[kGroup];
    int n2 = 1;
    while (n2 < tot) n2 <<= 1;
    for (int i = threadIdx.x; i < n2; i += blockDim.x) sa[i] = INT_MAX;
    __syncthreads();
    for (int g = 0; g < kGroup; ++g) {
        const int64_t pos = (int64_t)group * kGroup + g;
        if (pos >= n_int) break;
        const int p = order[pos];
        const int64_t off = nb_off[p];
        const int m = (int)(nb_off[p + 1] - off);
        for (int i = threadIdx.x; i < m; i += blockDim.x) sa[s_len[g] + i] = nb_idx[off + i];
    }
    __syncthreads();
    for (int k = 2; k <= n2; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n2; i += blockDim.x) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const int a = sa[i], b = sa[ixj];
                    const bool up = (i & k) == 0;
                    if ((a > b) == up) {
                        sa[i] = b;
                        sa[ixj] = a;
                    }
                }
            }
            __syncthreads();
        }
    // compaction of first occurrences, in order: per-thread contiguous chunk + block scan
    const int per = (n2 + blockDim.x - 1) / blockDim.x;
    const int b0 = threadIdx.x * per, b1 = min(n2, b0 + per);
    int cnt = 0;
    for (int i = b0; i < b1; ++i) cnt += (sa[i] != INT_MAX && (i == 0 || sa[i] != sa[i - 1]));
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int v = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    if (lane == 31) wsum[wid] = v;
    __syncthreads();
    int base = v - cnt;
    for (int q = 0; q < wid; ++q) base += wsum[q];
    int32_t* out = gU + (int64_t)group * ucap;
    uint8_t* cnt_out = gCnt + (int64_t)group * ucap;
    for (int i = b0; i < b1; ++i)
        if (sa[i] != INT_MAX && (i == 0 || sa[i] != sa[i - 1])) {
            int run = 1;                                    // users of this member (<= kGroup)
            while (i + run < n2 && sa[i + run] == sa[i]) ++run;
            su[base] = sa[i];
            out[base] = sa[i];
            cnt_out[base] = (uint8_t)run;
            ++base;
        }
    __shared__ int s_ulen;
    if (threadIdx.x == blockDim.x - 1) {
        gUlen[group] = base;
        s_ulen = base;
    }
    __syncthreads();
    const int ulen = s_ulen;
    // position of every neighbour entry of the group's particles inside the union (binary search)
    for (int g = 0; g < kGroup; ++g) {
        const int64_t pos = (int64_t)group * kGroup + g;
        if (pos >= n_int) break;
        const int p = order[pos];
        const int64_t off = nb_off[p];
        const int m = (int)(nb_off[p + 1] - off);
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
            const int v = nb_idx[off + i];
            int lo = 0, hi = ulen - 1;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (su[mid] < v) lo = mid + 1;
                else hi = mid;
            }
            upos[off + i] = (uint16_t)lo;
        }
    }
}

// ============================================================================
// Warp-specialised transport: the block's last warp is a TMA producer for the other
// kWsConsumers warps (one particle each).  Producer lane c walks consumer c's neighbour
// list, waits for the consumer to release a ring stage (empty[c][s]) and refills it
// (box + pair record on full[c][s]).  Consumers only wait on full, apply the neighbour and
// arrive on empty -- no refill issue, no warp-wide issue path in the hot loop.
// ============================================================================
constexpr int kWsConsumers = 8;
constexpr int kWsThreads = (kWsConsumers + 4) * 32;   // two consumer warpgroups + one producer warpgroup

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int D, int R, int NST>
__global__ void __launch_bounds__(kWsThreads, 1) k_transport_ws(const __grid_constant__ CUtensorMap tmap,
                                                                             const TArgs A) {
    using St = Stage<D, R>;
    constexpr int NV = St::NV;
    constexpr int PD = St::PD;
    constexpr int ROW = St::ROW;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + (size_t)kWsConsumers * NST * St::BYTES);
    uint64_t* empty = full + kWsConsumers * NST;
    const int w = blockIdx.y;
    const int chunk = w / A.ncg, cg = w - chunk * A.ncg;
    const int k1s = chunk * R;
    if (threadIdx.x == 0) {
        for (int q = 0; q < kWsConsumers * NST; ++q) {
            mbar_init(full + q, 1);
            mbar_init(empty + q, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();

    if (wib >= kWsConsumers) {                              // ---------------- producer warpgroup
        // registers move from the producer warpgroup to the consumers (setmaxnreg)
        asm volatile("setmaxnreg.dec.sync.aligned.u32 40;" ::: "memory");
        const int c = lane;
        if (wib != kWsConsumers || c >= kWsConsumers) return;
        const int64_t pos = (int64_t)blockIdx.x * kWsConsumers + c;
        if (pos >= A.n_int) return;
        const int p = A.order[pos];
        const int64_t off = A.nb_off[p];
        const int m = (int)(A.nb_off[p + 1] - off);
        unsigned char* ring = smem_raw + (size_t)c * NST * St::BYTES;
        for (int e = 0; e < m; ++e) {
            const int s = e % NST;
            const int jn = __ldg(A.nb_idx + off + e);
            if (e >= NST) mbar_wait(empty + c * NST + s, (uint32_t)((e / NST) - 1) & 1u);
            unsigned char* st = ring + s * St::BYTES;
            mbar_expect_tx(full + c * NST + s, St::F_BYTES + St::P_BYTES);
            tma_load_3d(st, &tmap, cg * ROW, k1s, jn, full + c * NST + s);
            bulk_load(st + St::F_BYTES, A.P + (off + e) * PD, St::P_BYTES, full + c * NST + s);
        }
        return;
    }
    // ---------------------------------------------------------------- consumer warps
    asm volatile("setmaxnreg.inc.sync.aligned.u32 232;" ::: "memory");
    const int64_t pos = (int64_t)blockIdx.x * kWsConsumers + wib;
    if (pos >= A.n_int) return;
    const int p = A.order[pos];
    const int col = cg * 32 + lane;
    const bool valid = col < A.ncol;
    const int colc = valid ? col : 0;
    const int gc = A.c0 + colc;
    const int64_t off = A.nb_off[p];
    const int m = (int)(A.nb_off[p + 1] - off);
    const unsigned char* ring = smem_raw + (size_t)wib * NST * St::BYTES;
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
    const double c1dv = c0v[0] / A.dv;
    double Qf[R][NV], Sc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        Sc[r] = 0.0;
#pragma unroll
        for (int q = 0; q < NV; ++q) Qf[r][q] = 0.0;
    }
    for (int e = 0; e < m; ++e) {
        const int s = e % NST;
        const unsigned char* stb = ring + s * St::BYTES;
        mbar_wait(full + wib * NST + s, (uint32_t)(e / NST) & 1u);
        const double* ps = reinterpret_cast<const double*>(stb + St::F_BYTES);
        double pv[PD];
#pragma unroll
        for (int q = 0; q < PD; ++q) pv[q] = ps[q];
        double y[D], dy[D], Lc, dL;
        pair_coeffs<D>(pv, c0v, c1dv, A.dv, y, dy, Lc, dL);
        const double* st = reinterpret_cast<const double*>(stb) + lane * NV;
#pragma unroll
        for (int r = 0; r < R; ++r) {
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
                Qf[r][0] = fma(C, st[r * ROW], Qf[r][0]);
            } else {
                const double2 v = *reinterpret_cast<const double2*>(st + r * ROW);
                Qf[r][0] = fma(C, v.x, Qf[r][0]);
                Qf[r][1] = fma(C, v.y, Qf[r][1]);
            }
            Sc[r] += C;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + wib * NST + s);  // stage s free for the producer
    }
    // epilogue (as k_transport)
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
        if (k1s + r >= A.n1) break;
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

template <int D, int R>
void launch_ws_one(const CUtensorMap& tm, const TArgs& a, cudaStream_t s) {
    constexpr int B = Stage<D, R>::BYTES;
    constexpr int NST = []() {
        int n = 2;
        while (n < 8 && (size_t)kWsConsumers * (n + 1) * B + 2 * kWsConsumers * (n + 1) * 8 <= 220 * 1024) ++n;
        return n;
    }();
    constexpr size_t smem = (size_t)kWsConsumers * NST * B + 2 * kWsConsumers * NST * 8;
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(k_transport_ws<D, R, NST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = true;
    }
    const unsigned gx = (unsigned)((a.n_int + kWsConsumers - 1) / kWsConsumers);
    k_transport_ws<D, R, NST><<<dim3(gx, (unsigned)a.nwpp), kWsThreads, smem, s>>>(tm, a);
}

template <int D>
void dispatch_ws(int R, const CUtensorMap& tm, const TArgs& a, cudaStream_t s) {
    if constexpr (D == 3) {
        switch (R) {
            case 25: launch_ws_one<D, 25>(tm, a, s); return;
            case 21: launch_ws_one<D, 21>(tm, a, s); return;
            case 17: launch_ws_one<D, 17>(tm, a, s); return;
            default: break;
        }
    }
    switch (R) {
        case 13: launch_ws_one<D, 13>(tm, a, s); break;
        case 11: launch_ws_one<D, 11>(tm, a, s); break;
        case 9: launch_ws_one<D, 9>(tm, a, s); break;
        case 7: launch_ws_one<D, 7>(tm, a, s); break;
        case 5: launch_ws_one<D, 5>(tm, a, s); break;
        case 3: launch_ws_one<D, 3>(tm, a, s); break;
        default: launch_ws_one<D, 1>(tm, a, s); break;
    }
}

template <int D, int R, int WPB, bool SG>
constexpr int stages_for() {
    // ring depth: keep NST-1 neighbour boxes in flight; bounded by 227 KB of shared memory
    // (sized for 8 resident warps per SM: blocks of WPB warps, 8 / WPB blocks per SM)
    constexpr int blocks = WPB >= 8 ? 1 : 8 / WPB;
    constexpr int n = (220 * 1024) / (blocks * WPB * Stage<D, R, SG>::BYTES);
    return n > 8 ? 8 : (n < 2 ? 2 : n);
}

template <int D, int R, int WPB, bool SG = false>
void launch_one(const CUtensorMap& tm, const TArgs& a, cudaStream_t s) {
    constexpr int NST = stages_for<D, R, WPB, SG>();
    constexpr size_t smem = (size_t)WPB * NST * Stage<D, R, SG>::BYTES + WPB * NST * 8;
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(k_transport<D, R, NST, WPB, SG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = true;
    }
    const unsigned gx = (unsigned)((a.n_int + WPB - 1) / WPB);
    k_transport<D, R, NST, WPB, SG><<<dim3(gx, (unsigned)a.nwpp), WPB * 32, smem, s>>>(tm, a);
}

template <int D, int R>
void launch_wpb(int wpb, const CUtensorMap& tm, const TArgs& a, cudaStream_t s) {
    if (a.signed_n) return launch_one<D, R, kDefaultWarps, true>(tm, a, s);   // second-order WLS
    if constexpr (D == 3 && (R == 25 || R == 17 || R == 13 || R == 9)) {
        if (wpb == 12) return launch_one<D, R, 12>(tm, a, s);
        if (wpb == 16) return launch_one<D, R, 16>(tm, a, s);
        if (wpb == 4) return launch_one<D, R, 4>(tm, a, s);
        if (wpb == 2) return launch_one<D, R, 2>(tm, a, s);
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

template <int D, int R>
void launch_grp_one(const CUtensorMap& tm, const TArgs& a, int n_groups, cudaStream_t s) {
    // ring depth from the shared-memory budget (one block per SM), 4..16 stages
    constexpr int F = GStage<D, R>::F_BYTES;
    constexpr int NST = []() {
        int n = 4;
        while (n < kMaxGrpStages && grp_smem_bytes<D, R, 16>(0) - 16 * F + (n + 1) * F + 16384 <= 225 * 1024) ++n;
        return n;
    }();
    const size_t smem = grp_smem_bytes<D, R, NST>(a.ucap);
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(k_transport_grp<D, R, NST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = true;
    }
    k_transport_grp<D, R, NST><<<dim3((unsigned)n_groups, (unsigned)a.nwpp), kGroup * 32, smem, s>>>(tm, a);
}

template <int D>
void dispatch_grp(int R, const CUtensorMap& tm, const TArgs& a, int n_groups, cudaStream_t s) {
    if constexpr (D == 3) {
        switch (R) {
            case 25: launch_grp_one<D, 25>(tm, a, n_groups, s); return;
            case 21: launch_grp_one<D, 21>(tm, a, n_groups, s); return;
            case 17: launch_grp_one<D, 17>(tm, a, n_groups, s); return;
            default: break;
        }
    }
    switch (R) {
        case 13: launch_grp_one<D, 13>(tm, a, n_groups, s); break;
        case 11: launch_grp_one<D, 11>(tm, a, n_groups, s); break;
        case 9: launch_grp_one<D, 9>(tm, a, n_groups, s); break;
        case 7: launch_grp_one<D, 7>(tm, a, n_groups, s); break;
        case 5: launch_grp_one<D, 5>(tm, a, n_groups, s); break;
        case 3: launch_grp_one<D, 3>(tm, a, n_groups, s); break;
        default: launch_grp_one<D, 1>(tm, a, n_groups, s); break;
    }
}

constexpr int kRChoices3[] = {25, 21, 17, 13, 11, 9, 7, 5, 3, 1};
constexpr int kRChoices2[] = {13, 11, 9, 7, 5, 3, 1};

}  // namespace

int group_size() { return kGroup; }

void launch_group_union(bgk_ctx* c, cudaStream_t s) {
    if (!c->grouped || c->N_int == 0) return;
    const int n_groups = (int)((c->N_int + kGroup - 1) / kGroup);
    k_group_union<<<n_groups, 256, 2 * sizeof(int32_t) * c->ucap, s>>>(c->g.order, c->N_int, c->g.nb_off,
                                                                        c->g.nb_idx, c->ucap, c->gU, c->gUlen,
                                                                        c->gCnt, c->upos);
}

// rows per thread: the largest divisor of n1 among the instantiated R (2D keeps three
// accumulators per row, so it stops at 13)
int transport_rows_per_thread(int d, int n1) {
    if (const char* e = getenv("BGK_TRANSPORT_R")) {    // tuning knob: any instantiated R (ragged chunks OK)
        const int r = atoi(e);
        if (d == 3) {
            for (int R : kRChoices3)
                if (R == r) return R;
        } else {
            for (int R : kRChoices2)
                if (R == r) return R;
        }
    }
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
    a.work = c->work;
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
    a.gU = c->gU;
    a.gUlen = c->gUlen;
    a.gCnt = c->gCnt;
    a.upos = c->upos;
    a.ucap = c->ucap;
    const CUtensorMap& tm = c->tmap[fin == c->f[0] ? 0 : 1];
    static const int variant = [] {     // 0: per-warp ring, 1: warp-specialised producer (tuning knob)
        const char* e = getenv("BGK_TRANSPORT_WS");
        return e ? atoi(e) : 0;
    }();
    a.signed_n = c->wls_order == 2;
    if (variant == 1 && !c->grouped && !a.signed_n) {
        if (c->d == 3) dispatch_ws<3>(c->R, tm, a, s);
        else dispatch_ws<2>(c->R, tm, a, s);
        return;
    }
    if (c->grouped && !a.signed_n) {
        const int n_groups = (int)((c->N_int + kGroup - 1) / kGroup);
        if (c->d == 3) dispatch_grp<3>(c->R, tm, a, n_groups, s);
        else dispatch_grp<2>(c->R, tm, a, n_groups, s);
        return;
    }
    static const int wpb = [] {
        const char* e = getenv("BGK_TRANSPORT_WPB");   // tuning knob (4, 8, 12, 16); default 8
        return e ? atoi(e) : kDefaultWarps;
    }();
    if (c->d == 3) dispatch<3>(c->R, wpb, tm, a, s);
    else dispatch<2>(c->R, wpb, tm, a, s);
}

}  // namespace bgk
