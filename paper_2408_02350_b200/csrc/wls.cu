// wls.cu -- batched weighted-least-squares stencil coefficients
// and the rotated upwind coefficients of the positive scheme.
//
// One warp per particle.  Lanes stride over the particle's neighbours to build
// the small normal matrix A = sum_j w_j d_j d_j^T (2x2 / 3x3), a butterfly
// reduction gives every lane the same A, every lane inverts it (Gauss-Jordan,
// partial pivoting) and tests it (Jacobi eigenvalues, lambda_min < 1e-12
// lambda_max -> deficient), then lanes stride over the pairs again
// and write the pair data the transport kernel consumes:
//     a_j = w_j S d_j,  frame (n, t[, b]) of d_j (trig-free form of P:400 / P:420-431,
//     with (cos phi, sin phi) = (1, 0) when dx = dy = 0, Z10),
//     rot = (a.n, a.t[, a.b])  (Z8),
//     P[e] = (abar n, bbar t[, gbar b])   -- so the flux coefficient is
//     C = sum_e (P_e.c - |P_e.c|)  (abar > 0; P:408-410, P:476-480 with Z5-Z7).
// Offsets are scaled by 1/h inside the solve so the matrices are O(1).
// Boundary particles get linear-WLS interpolation weights over their interior
// neighbours (Z19): c_bj = w_j e0^T B^{-1} (1, d_j/h), B = sum w (1, d/h)(1, d/h)^T.
#include "bgk_internal.cuh"
#include "linalg.cuh"

namespace bgk {

namespace {

// frame rows of direction d (any scale): F[0] = n, F[1] = t, F[2] = b
template <int D>
__device__ __forceinline__ void frame_of(const double (&d)[D], double (&F)[D][D]) {
    if constexpr (D == 2) {
        const double r = sqrt(d[0] * d[0] + d[1] * d[1]);
        const double cp = d[0] / r, sp = d[1] / r;
        F[0][0] = cp;  F[0][1] = sp;
        F[1][0] = -sp; F[1][1] = cp;
    } else {
        const double rxy2 = d[0] * d[0] + d[1] * d[1];
        const double rxy = sqrt(rxy2);
        const double r = sqrt(rxy2 + d[D - 1] * d[D - 1]);
        double cp = 1.0, sp = 0.0;                  // Z10 / Z26: phi = 0 for a pair vertical to rounding
        if (rxy2 > 1e-16 * (rxy2 + d[D - 1] * d[D - 1])) { cp = d[0] / rxy; sp = d[1] / rxy; }
        const double ct = d[D - 1] / r, st = rxy / r;
        double* f = &F[0][0];
        f[0] = st * cp; f[1] = st * sp; f[2] = ct;       // n
        f[3] = ct * cp; f[4] = ct * sp; f[5] = -st;      // t
        f[6] = -sp;     f[7] = cp;      f[8] = 0.0;      // b
    }
}

// Taylor monomials of the scaled offset q = d/h: order 1 -> q; order 2 -> (q, q_a^2/2, q_a q_b (a<b))
// (the second-order expansion adds the Hessian; same ordering as the oracle's)
template <int D, int ORDER>
struct Taylor {
    static constexpr int NU = ORDER == 1 ? D : (D == 2 ? 5 : 9);
    __device__ static __forceinline__ void mono(const double (&q)[D], double (&mv)[NU]) {
#pragma unroll
        for (int a = 0; a < D; ++a) mv[a] = q[a];
        if constexpr (ORDER == 2) {
#pragma unroll
            for (int a = 0; a < D; ++a) mv[D + a] = 0.5 * q[a] * q[a];
            int k = 2 * D;
#pragma unroll
            for (int a = 0; a < D; ++a)
#pragma unroll
                for (int b = a + 1; b < D; ++b) mv[k++] = q[a] * q[b];
        }
    }
};

template <int D, int ORDER>
__global__ void k_wls_interior(const double* __restrict__ x, const int32_t* __restrict__ ids, int64_t n_ids,
                               const int64_t* __restrict__ nb_off, const int32_t* __restrict__ nb_idx, double h,
                               double h2, double alpha, double dv, double* __restrict__ S_out, double* __restrict__ P,
                               double* __restrict__ cw, double* __restrict__ rot_out, double* __restrict__ frame_out,
                               int64_t* err) {
    // pair record: 2D (pn, pt) [+ (s_n, 0)], 3D (dy_n, pn1, pn2, dy_t, pt1, pt2, dy_b, pb1, pb2, dL) [+ (s_n, 0)]
    // -- the signed tail only for second order, where abar may be negative (s_n = -sign(abar))
    constexpr int PD0 = (D == 2) ? 4 : 10;
    constexpr int PD = ORDER == 2 ? PD0 + 2 : PD0;
    using T = Taylor<D, ORDER>;
    constexpr int NU = T::NU;
    const int lane = threadIdx.x & 31;
    const int64_t w = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
    if (w >= n_ids) return;
    const int p = ids[w];
    const int64_t off = nb_off[p];
    const int m = (int)(nb_off[p + 1] - off);
    const double inv_h = 1.0 / h;
    double xi[D];
#pragma unroll
    for (int a = 0; a < D; ++a) xi[a] = x[(int64_t)p * D + a];
    constexpr int NT = NU * (NU + 1) / 2;      // upper triangle of the normal matrix
    double At[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) At[t] = 0.0;
    for (int e = lane; e < m; e += 32) {
        const int j = nb_idx[off + e];
        double xj[D], dd[D], mv[NU];
#pragma unroll
        for (int a = 0; a < D; ++a) { xj[a] = x[(int64_t)j * D + a]; dd[a] = (xj[a] - xi[a]) * inv_h; }
        T::mono(dd, mv);
        const double wgt = exp(-alpha * dist2_rn<D>(xi, xj) / h2);
        int t = 0;
#pragma unroll
        for (int r = 0; r < NU; ++r)
#pragma unroll
            for (int q = r; q < NU; ++q) At[t++] += wgt * mv[r] * mv[q];
    }
    double A[NU][NU];
    {
        int t = 0;
#pragma unroll
        for (int r = 0; r < NU; ++r)
#pragma unroll
            for (int q = r; q < NU; ++q) {
                const double v = warp_sum(At[t++]);
                A[r][q] = v;
                A[q][r] = v;
            }
    }
    double Si[NU][NU];
    const int m_min = ORDER == 1 ? D + 2 : NU + 1;
    bool ok = (m >= m_min) && small_inverse<NU>(A, Si) && rank_test<NU>(A, Si);
    if (!ok) {
        if (lane == 0) latch_error(err, BGK_E_DEFICIENT_STENCIL, p);
        return;
    }
    if (lane == 0 && S_out) {
#pragma unroll
        for (int r = 0; r < D; ++r)
#pragma unroll
            for (int q = 0; q < D; ++q) S_out[(int64_t)p * D * D + r * D + q] = Si[r][q] * inv_h * inv_h;
    }
    for (int e = lane; e < m; e += 32) {
        const int j = nb_idx[off + e];
        double xj[D], dd[D], mv[NU];
#pragma unroll
        for (int a = 0; a < D; ++a) { xj[a] = x[(int64_t)j * D + a]; dd[a] = (xj[a] - xi[a]) * inv_h; }
        T::mono(dd, mv);
        const double wgt = exp(-alpha * dist2_rn<D>(xi, xj) / h2);
        double av[D];   // a_j = w_j [(M^T W M)^{-1} m_j]_{0:d} / h, physical units 1/m
#pragma unroll
        for (int r = 0; r < D; ++r) {
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < NU; ++q) s += Si[r][q] * mv[q];
            av[r] = wgt * s * inv_h;
        }
        double F[D][D];
        frame_of<D>(dd, F);
        double rot[D];
#pragma unroll
        for (int k = 0; k < D; ++k) {
            double s = 0.0;
#pragma unroll
            for (int a = 0; a < D; ++a) s += av[a] * F[k][a];
            rot[k] = s;
        }
        cw[off + e] = 0.0;     // boundary-interpolation weights are defined on boundary rows only
        double* pe = P + (off + e) * PD;
#pragma unroll
        for (int k = 0; k < D; ++k)
#pragma unroll
            for (int a = 0; a < D; ++a) pe[k * D + a] = rot[k] * F[k][a];
        if constexpr (D == 3) {
            // transport walks v_1 in steps of dv: store dy_e = dv * P_e[0] in place of P_e[0]
            // and dL = sum_e dy_e in the pad slot (lane-independent, saves 5 DP per neighbour)
            double dl = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) {
                pe[k * D] = dv * pe[k * D];
                dl += pe[k * D];
            }
            pe[PD0 - 1] = dl;
        }
        if constexpr (ORDER == 2) {
            pe[PD0] = rot[0] > 0.0 ? -1.0 : 1.0;   // C's n-term = y_n - sign(abar)|y_n| (P:408-410 literal)
            pe[PD0 + 1] = 0.0;
        }
        if (rot_out) {
#pragma unroll
            for (int k = 0; k < D; ++k) rot_out[(off + e) * D + k] = rot[k];
#pragma unroll
            for (int k = 0; k < D; ++k)
#pragma unroll
                for (int a = 0; a < D; ++a) frame_out[(off + e) * D * D + k * D + a] = F[k][a];
        }
    }
}

template <int D>
__global__ void k_wls_boundary(const double* __restrict__ x, const int8_t* __restrict__ kind,
                               const int32_t* __restrict__ ids, int64_t n_ids, const int64_t* __restrict__ nb_off,
                               const int32_t* __restrict__ nb_idx, double h, double h2, double alpha,
                               double* __restrict__ cw, int32_t* __restrict__ bidx, double* __restrict__ bcw,
                               int32_t* __restrict__ bcnt, int64_t* err) {
    constexpr int n = D + 1;
    const int lane = threadIdx.x & 31;
    const int64_t w = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
    if (w >= n_ids) return;
    const int b = ids[w];
    const int64_t off = nb_off[b];
    const int m = (int)(nb_off[b + 1] - off);
    const double inv_h = 1.0 / h;
    double xb[D];
#pragma unroll
    for (int a = 0; a < D; ++a) xb[a] = x[(int64_t)b * D + a];
    double B[n][n];
#pragma unroll
    for (int r = 0; r < n; ++r)
#pragma unroll
        for (int q = 0; q < n; ++q) B[r][q] = 0.0;
    int mi = 0;
    for (int e = lane; e < m; e += 32) {
        const int j = nb_idx[off + e];
        if (kind[j] != 0) continue;
        ++mi;
        double xj[D], Pv[n];
        Pv[0] = 1.0;
#pragma unroll
        for (int a = 0; a < D; ++a) { xj[a] = x[(int64_t)j * D + a]; Pv[1 + a] = (xj[a] - xb[a]) * inv_h; }
        const double wgt = exp(-alpha * dist2_rn<D>(xb, xj) / h2);
#pragma unroll
        for (int r = 0; r < n; ++r)
#pragma unroll
            for (int q = 0; q < n; ++q) B[r][q] += wgt * Pv[r] * Pv[q];
    }
    mi = warp_sum(mi);
#pragma unroll
    for (int r = 0; r < n; ++r)
#pragma unroll
        for (int q = 0; q < n; ++q) B[r][q] = warp_sum(B[r][q]);
    double Bi[n][n];
    const bool ok = (mi >= D + 2) && small_inverse<n>(B, Bi) && rank_test<n>(B, Bi);
    if (!ok) {
        if (lane == 0) {
            latch_error(err, BGK_E_DEFICIENT_STENCIL, b);
            bcnt[b] = 0;   // keep the interpolation kernel in bounds until the error is reported
        }
        return;
    }
    int base = 0;   // compacted (interior neighbour, weight) list for the interpolation kernel
    for (int e0 = 0; e0 < m; e0 += 32) {
        const int e = e0 + lane;
        const int j = e < m ? nb_idx[off + e] : 0;
        double c = 0.0;
        const bool inter = e < m && kind[j] == 0;
        if (inter) {
            double xj[D], Pv[n];
            Pv[0] = 1.0;
#pragma unroll
            for (int a = 0; a < D; ++a) { xj[a] = x[(int64_t)j * D + a]; Pv[1 + a] = (xj[a] - xb[a]) * inv_h; }
            const double wgt = exp(-alpha * dist2_rn<D>(xb, xj) / h2);
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < n; ++q) s += Bi[0][q] * Pv[q];
            c = wgt * s;
        }
        if (e < m) cw[off + e] = c;
        const unsigned bal = __ballot_sync(0xffffffffu, inter);
        if (inter) {
            const int slot = base + __popc(bal & ((1u << lane) - 1u));
            bidx[off + slot] = j;
            bcw[off + slot] = c;
        }
        base += __popc(bal);
    }
    if (lane == 0) bcnt[b] = base;
}

}  // namespace

int launches_wls() { return 2; }

template <int D>
static void launch_interior(bgk_ctx* c, unsigned gi, int wpb, double* rot, double* frames, cudaStream_t s) {
    const double h = c->cfg.h, h2 = c->cfg.h2, al = c->cfg.alpha_w;
    if (c->wls_order == 2)
        k_wls_interior<D, 2><<<gi, wpb * 32, 0, s>>>(c->x, c->interior, c->N_int, c->g.nb_off, c->g.nb_idx, h, h2, al,
                                                     c->dv, c->g.S, c->g.P, c->g.cw, rot, frames, c->err);
    else
        k_wls_interior<D, 1><<<gi, wpb * 32, 0, s>>>(c->x, c->interior, c->N_int, c->g.nb_off, c->g.nb_idx, h, h2, al,
                                                     c->dv, c->g.S, c->g.P, c->g.cw, rot, frames, c->err);
}

static void run_wls(bgk_ctx* c, double* rot, double* frames, cudaStream_t s) {
    const int wpb = 4;
    const unsigned gi = (unsigned)((c->N_int + wpb - 1) / wpb);
    const unsigned gb = (unsigned)((c->N_b + wpb - 1) / wpb);
    const double h = c->cfg.h, h2 = c->cfg.h2, al = c->cfg.alpha_w;
    if (c->d == 3) {
        if (gi) launch_interior<3>(c, gi, wpb, rot, frames, s);
        if (gb && !rot)
            k_wls_boundary<3><<<gb, wpb * 32, 0, s>>>(c->x, c->kind, c->boundary, c->N_b, c->g.nb_off, c->g.nb_idx, h,
                                                     h2, al, c->g.cw, c->g.bidx, c->g.bcw, c->g.bcnt, c->err);
    } else {
        if (gi) launch_interior<2>(c, gi, wpb, rot, frames, s);
        if (gb && !rot)
            k_wls_boundary<2><<<gb, wpb * 32, 0, s>>>(c->x, c->kind, c->boundary, c->N_b, c->g.nb_off, c->g.nb_idx, h,
                                                     h2, al, c->g.cw, c->g.bidx, c->g.bcw, c->g.bcnt, c->err);
    }
}

void launch_wls(bgk_ctx* c, cudaStream_t s) { run_wls(c, nullptr, nullptr, s); }

// the two halves of launch_wls on separate streams (graph.cu forks them: they write disjoint rows)
void launch_wls_interior(bgk_ctx* c, cudaStream_t s) {
    const int wpb = 4;
    const unsigned gi = (unsigned)((c->N_int + wpb - 1) / wpb);
    if (!gi) return;
    if (c->d == 3) launch_interior<3>(c, gi, wpb, nullptr, nullptr, s);
    else launch_interior<2>(c, gi, wpb, nullptr, nullptr, s);
}

void launch_wls_boundary(bgk_ctx* c, cudaStream_t s) {
    const int wpb = 4;
    const unsigned gb = (unsigned)((c->N_b + wpb - 1) / wpb);
    if (!gb) return;
    const double h = c->cfg.h, h2 = c->cfg.h2, al = c->cfg.alpha_w;
    if (c->d == 3)
        k_wls_boundary<3><<<gb, wpb * 32, 0, s>>>(c->x, c->kind, c->boundary, c->N_b, c->g.nb_off, c->g.nb_idx, h, h2,
                                                 al, c->g.cw, c->g.bidx, c->g.bcw, c->g.bcnt, c->err);
    else
        k_wls_boundary<2><<<gb, wpb * 32, 0, s>>>(c->x, c->kind, c->boundary, c->N_b, c->g.nb_off, c->g.nb_idx, h, h2,
                                                 al, c->g.cw, c->g.bidx, c->g.bcw, c->g.bcnt, c->err);
}

void launch_wls_export(bgk_ctx* c, double* rot, double* frames, cudaStream_t s) { run_wls(c, rot, frames, s); }

}  // namespace bgk
