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
// Mapping: a warp owns one particle and 32
// consecutive (chunk, column) slots; each lane walks R consecutive nodes along
// v_1 of its column.  Along v_1 every projection is affine, so y_e and L are
// advanced by one add per node (y += dv * P_e[0]) instead of a 3-term dot
// product.  Per (i, j, k) triple the fp64 work is: 4 increments, 3 abs-subtracts,
// 1 FMA (sum C f_j) and 1 add (sum C) -- 9 DP instructions -- and one coalesced
// 8-B (3D) / 16-B (2D) load of f_jk.  Blocks hold warps of consecutive
// particles of the cell-ordered interior list (shared neighbour rows hit in
// L1); grid.y = warp slot is the slowest launch dimension, so the f slab of one
// column block stays L2-resident while all particles sweep it.
//
// Epilogue: ftilde is written to the next-step buffer; per-warp partial sums
// (sum ft, sum v ft, sum |v|^2 ft (+ g2)) are reduced with shuffles in a fixed
// order and stored per (particle, warp) -- no atomics, deterministic -- and
// max_k sum_j |C_ijk| (for stable_dt) is folded into one atomicMax.
#include "bgk_internal.cuh"

namespace bgk {

namespace {

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
    int n1, ncol, c0, nslots, nwpp;
    double vmax, dv, dt;
};

template <int D, int R>
__global__ void __launch_bounds__(256) k_transport(const TArgs A) {
    constexpr int NV = (D == 2) ? 2 : 1;
    constexpr int PD = (D == 2) ? 4 : 10;
    const int lane = threadIdx.x & 31;
    const int64_t pos = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (pos >= A.n_int) return;                    // warp-uniform
    const int w = blockIdx.y;
    const int p = A.order[pos];
    const int s = w * 32 + lane;
    const bool valid = s < A.nslots;
    const int col = valid ? s % A.ncol : 0;
    const int k1s = valid ? (s / A.ncol) * R : 0;
    const int ncol = A.ncol;
    // velocity of this lane's column at k1 = k1s, relative to W_p
    const int gc = A.c0 + col;
    double Wp[D];
#pragma unroll
    for (int a = 0; a < D; ++a) Wp[a] = A.W[(int64_t)p * D + a];
    double c0v[D];
    c0v[0] = axis_node(A.vmax, A.dv, k1s) - Wp[0];
    if constexpr (D == 3) {
        const int k2 = gc / A.n1, k3 = gc - (gc / A.n1) * A.n1;
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
    const int64_t off = A.nb_off[p];
    const int m = (int)(A.nb_off[p + 1] - off);
    const int64_t rowstride = (int64_t)ncol * NV;        // doubles between consecutive k1
    const int64_t pstride = (int64_t)A.n1 * rowstride;   // doubles between particles
    const int64_t lane_off = (int64_t)k1s * rowstride + (int64_t)col * NV;
    for (int e = 0; e < m; ++e) {
        const int j = __ldg(A.nb_idx + off + e);
        const double* pe = A.P + (off + e) * PD;
        double pv[PD];
#pragma unroll
        for (int q = 0; q < PD; q += 2) {
            const double2 v2 = __ldg(reinterpret_cast<const double2*>(pe + q));
            pv[q] = v2.x;
            pv[q + 1] = v2.y;
        }
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
        const double* fj = A.f + (int64_t)j * pstride + lane_off;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            double C = Lc;
#pragma unroll
            for (int k = 0; k < D; ++k) C -= fabs(y[k]);
            if constexpr (NV == 1) {
                const double v = __ldg(fj + r * rowstride);
                Qf[r][0] = fma(C, v, Qf[r][0]);
            } else {
                const double2 v = __ldg(reinterpret_cast<const double2*>(fj + r * rowstride));
                Qf[r][0] = fma(C, v.x, Qf[r][0]);
                Qf[r][1] = fma(C, v.y, Qf[r][1]);
            }
            Sc[r] += C;
#pragma unroll
            for (int k = 0; k < D; ++k) y[k] += dy[k];
            Lc += dL;
        }
    }
    // epilogue: ftilde, moment partials, stability bound
    const double* fi = A.f + (int64_t)p * pstride + lane_off;
    double* fto = A.ft + (int64_t)p * pstride + lane_off;
    double v2v = 0.0, v3v = 0.0;
    if constexpr (D == 3) {
        const int k2 = gc / A.n1, k3 = gc - (gc / A.n1) * A.n1;
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

constexpr int kRChoices[] = {25, 21, 17, 13, 11, 9, 7, 5, 3, 1};

template <int D, int R>
void launch_one(const TArgs& a, unsigned gx, unsigned gy, cudaStream_t s) {
    k_transport<D, R><<<dim3(gx, gy), 256, 0, s>>>(a);
}

template <int D>
void dispatch(int R, const TArgs& a, unsigned gx, unsigned gy, cudaStream_t s) {
    switch (R) {
        case 25: launch_one<D, 25>(a, gx, gy, s); break;
        case 21: launch_one<D, 21>(a, gx, gy, s); break;
        case 17: launch_one<D, 17>(a, gx, gy, s); break;
        case 13: launch_one<D, 13>(a, gx, gy, s); break;
        case 11: launch_one<D, 11>(a, gx, gy, s); break;
        case 9: launch_one<D, 9>(a, gx, gy, s); break;
        case 7: launch_one<D, 7>(a, gx, gy, s); break;
        case 5: launch_one<D, 5>(a, gx, gy, s); break;
        case 3: launch_one<D, 3>(a, gx, gy, s); break;
        default: launch_one<D, 1>(a, gx, gy, s); break;
    }
}

}  // namespace

// rows per thread: the largest divisor of n1 from the instantiated set (2D caps at 17:
// three accumulators per row there)
int transport_rows_per_thread(int d, int n1) {
    for (int R : kRChoices) {
        if (d == 2 && R > 17) continue;
        if (n1 % R == 0) return R;
    }
    return 1;
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
    a.c0 = c->c0;
    a.nslots = c->nslots;
    a.nwpp = c->nwpp;
    a.vmax = c->cfg.vmax;
    a.dv = c->dv;
    a.dt = c->cfg.dt;
    const unsigned wpb = 8;
    const unsigned gx = (unsigned)((c->N_int + wpb - 1) / wpb);
    const unsigned gy = (unsigned)c->nwpp;
    if (c->d == 3) dispatch<3>(c->R, a, gx, gy, s);
    else dispatch<2>(c->R, a, gx, gy, s);
}

}  // namespace bgk
