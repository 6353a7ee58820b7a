// manage.cu -- particle management: "Adding and removing points" (
// the algorithm and its readings are DESIGN.md Z28).  One pass, on the step-start cloud of an ALE
// step, right after the neighbour search:
//   1. merge -- interior i ascending: the first neighbour j > i (ascending) that is interior,
//      unprocessed and closer than r_merge pairs with i; both become processed.  The pair becomes
//      ONE particle at (x_i + x_j) * 0.5 in slot i (slot j is removed), interpolated from every
//      other particle within h of the midpoint; a deficient stencil keeps the pair.
//   2. fill  -- interior i ascending, not processed, with |N(i)| < m_min: candidates
//      x_i + s (0.5 h) e_a (a ascending, s = + then -) strictly inside (0, L)^d and farther than
//      0.45 dx from every particle of the current cloud (removed slots excluded, merged particles
//      at their midpoints, inserts so far included) are appended, interpolated from the old cloud
//      within h; deficient candidates are skipped; inserts stop at the capacity.
//   3. compaction -- surviving slots in ascending old order, then the inserts.
// Interpolation (the value at p of the linear WLS fit with a constant term, the
// boundary-interpolation construction of Z19): c_s = w_s e0^T B^{-1} P_s, P_s = (1, (x_s - p)/h),
// w_s = exp(-alpha |x_s - p|^2 / h^2), B = sum_s w_s P_s P_s^T; applied to every f node, to W and to
// the macro state.
//
// Kernels: k_mg_detect_w (warp per particle: merge-candidate / deficient flags), k_mg_decide (ONE
// warp: the greedy, order-dependent decisions -- merges and inserts are rare, the warp
// parallelises only the inner scans), k_mg_interp (new rows), k_mg_gather (row compaction into
// the idle f buffer), k_mg_small (positions, W, macro, kinds).  The host reads the decision
// counts once (the pass synchronises the stream) and, if the cloud changed, re-installs the
// interior / boundary lists and the TMA maps for the new N.
#include <vector>

#include "bgk_internal.cuh"
#include "cells.cuh"
#include "linalg.cuh"

namespace bgk {

namespace {

constexpr uint8_t kMergeCand = 1, kDeficient = 2, kProcessed = 0x80;

// flags from the fresh neighbour lists: merge candidate (an interior j > i closer than r_merge) and
// deficient (|N(i)| < m_min); a warp per particle, lanes over the list (a thread per particle walked
// ~28-120 dependent loads each in one wave: 12 us on C2, 64 us on C5)
template <int D>
__global__ void __launch_bounds__(256) k_mg_detect_w(const double* __restrict__ x, const int8_t* __restrict__ kind,
                                                     int64_t N, const int64_t* __restrict__ nb_off,
                                                     const int32_t* __restrict__ nb_idx, double rm2, int m_min,
                                                     uint8_t* __restrict__ flag, int32_t* __restrict__ counts) {
    const int lane = threadIdx.x & 31;
    const int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= N) return;
    uint8_t fl = 0;
    const int64_t off = nb_off[i];
    const int m = (int)(nb_off[i + 1] - off);
    if (kind[i] == 0) {
        if (m < m_min) fl |= kDeficient;
        double xi[3];
#pragma unroll
        for (int a = 0; a < D; ++a) xi[a] = x[i * D + a];
        bool close = false;
        for (int e = lane; e < m; e += 32) {
            const int j = nb_idx[off + e];
            if (j <= i || kind[j] != 0) continue;
            double xj[3];
#pragma unroll
            for (int a = 0; a < D; ++a) xj[a] = x[(int64_t)j * D + a];
            close = close || dist2_rn<D>(xi, xj) < rm2;
        }
        if (__any_sync(0xffffffffu, close)) fl |= kMergeCand;
    }
    if (lane == 0) {
        flag[i] = fl;
        if (fl) atomicAdd(counts, 1);
    }
}


// wall particles (the boundary list): Z30's deficiency of the interpolation system, in a kernel of
// its own so that the interior flags keep their lean register budget
template <int D>
__global__ void __launch_bounds__(256) k_mg_detect_wall(const double* __restrict__ x, const int8_t* __restrict__ kind,
                                                        const int32_t* __restrict__ bids, int64_t nb,
                                                        const int64_t* __restrict__ nb_off,
                                                        const int32_t* __restrict__ nb_idx, double inv_h, double h2,
                                                        double alpha, uint8_t* __restrict__ flag,
                                                        int32_t* __restrict__ counts) {
    const int lane = threadIdx.x & 31;
    const int64_t w = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
    if (w >= nb) return;
    const int64_t i = bids[w];
    const int64_t off = nb_off[i];
    const int m = (int)(nb_off[i + 1] - off);
    uint8_t fl = 0;
    // a wall particle whose interpolation system (Z19: linear WLS with a constant term over its
    // interior neighbours, offsets in units of h) is deficient -- fewer than d + 2 members, or,
    // for fewer than 3 (d + 1) members, lambda_min < 1e-12 lambda_max or a zero pivot (the test of
    // k_wls_boundary): the fill pass proposes points inward of it (Z30)
    constexpr int n = D + 1;
    int n_int = 0;
    for (int e = lane; e < m; e += 32) n_int += kind[nb_idx[off + e]] == 0;
    n_int = warp_sum(n_int);
    if (n_int < D + 2) {
        fl |= kDeficient;
    } else if (n_int < 3 * n) {               // small stencils: the full test of the boundary WLS
        double xb[3];
#pragma unroll
        for (int a = 0; a < D; ++a) xb[a] = x[i * D + a];
        double B[n][n];
#pragma unroll
        for (int r = 0; r < n; ++r)
#pragma unroll
            for (int q = 0; q < n; ++q) B[r][q] = 0.0;
        for (int e = lane; e < m; e += 32) {
            const int j = nb_idx[off + e];
            if (kind[j] != 0) continue;
            double xj[3], Pv[n];
            Pv[0] = 1.0;
#pragma unroll
            for (int a = 0; a < D; ++a) { xj[a] = x[(int64_t)j * D + a]; Pv[1 + a] = (xj[a] - xb[a]) * inv_h; }
            const double w = exp(-alpha * dist2_rn<D>(xb, xj) / h2);
#pragma unroll
            for (int r = 0; r < n; ++r)
#pragma unroll
                for (int q = 0; q < n; ++q) B[r][q] += w * Pv[r] * Pv[q];
        }
#pragma unroll
        for (int r = 0; r < n; ++r)
#pragma unroll
            for (int q = 0; q < n; ++q) B[r][q] = warp_sum(B[r][q]);
        double Bi[n][n];
        if (!(well_conditioned<n>(B) && small_inverse<n>(B, Bi))) fl |= kDeficient;
    }
    if (lane == 0 && fl) {
        flag[i] = fl;
        atomicAdd(counts, 1);
    }
}

struct MgArgs {
    const double* x;
    const int8_t* kind;
    const double* W;
    const double* macro;
    int64_t N, Ncap;
    const int64_t* nb_off;
    const int32_t* nb_idx;
    const int32_t* cell_start;
    const int32_t* cell_pts;
    int nc[3];
    double inv_e[3];
    double L, h, h2, alpha, rm2, hh, thr2;
    int max_nb;
    Manage m;
};

// every particle within h of p (closed ball, the O2 distance with p as the centre), except ex0 /
// ex1, into out[0 .. cap); returns the count (may exceed cap).  Warp-cooperative, uniform result.
template <int D>
__device__ int mg_stencil(const MgArgs& A, const double (&p)[3], int64_t ex0, int64_t ex1, int32_t* out, int cap) {
    const int lane = threadIdx.x & 31;
    int ci[3] = {0, 0, 0};
#pragma unroll
    for (int a = 0; a < D; ++a) ci[a] = min(max((int)floor(p[a] * A.inv_e[a]), 0), A.nc[a] - 1);
    int m = 0;
    for (int dz = (D == 3 ? -1 : 0); dz <= (D == 3 ? 1 : 0); ++dz)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                const int cx = ci[0] + dx, cy = ci[1] + dy, cz = ci[2] + dz;
                if (cx < 0 || cx >= A.nc[0] || cy < 0 || cy >= A.nc[1] || cz < 0 || cz >= A.nc[2]) continue;
                const int c = cell_code<D>(cx, cy, cz);
                const int cb = A.cell_start[c], ce = A.cell_start[c + 1];
                for (int b = cb; b < ce; b += 32) {
                    const int t = b + lane;
                    int k = -1;
                    bool hit = false;
                    if (t < ce) {
                        k = A.cell_pts[t];
                        if (k != ex0 && k != ex1) {
                            double xk[3];
#pragma unroll
                            for (int a = 0; a < D; ++a) xk[a] = A.x[(int64_t)k * D + a];
                            hit = dist2_rn<D>(p, xk) <= A.h2;
                        }
                    }
                    const unsigned bal = __ballot_sync(0xffffffffu, hit);
                    const int slot = m + __popc(bal & ((1u << lane) - 1u));
                    if (hit && slot < cap) out[slot] = k;
                    m += __popc(bal);
                }
            }
    return m;
}

// interpolation weights of p from the stencil (linear WLS with a constant term) into sc[0 .. m),
// and the interpolated W / macro into nW / nM.  Returns false if the stencil is deficient
// (m < d + 2 or lambda_min(B) < 1e-12 lambda_max(B) or a zero pivot).
template <int D>
__device__ bool mg_weights(const MgArgs& A, const double (&p)[3], const int32_t* sidx, int m, double* sc,
                           double* nW, double* nM) {
    constexpr int n = D + 1;
    const int lane = threadIdx.x & 31;
    const double inv_h = 1.0 / A.h;
    double B[n][n];
#pragma unroll
    for (int r = 0; r < n; ++r)
#pragma unroll
        for (int q = 0; q < n; ++q) B[r][q] = 0.0;
    for (int s = lane; s < m; s += 32) {
        const int k = sidx[s];
        double xk[3], Pv[n];
        Pv[0] = 1.0;
#pragma unroll
        for (int a = 0; a < D; ++a) { xk[a] = A.x[(int64_t)k * D + a]; Pv[1 + a] = (xk[a] - p[a]) * inv_h; }
        const double w = exp(-A.alpha * dist2_rn<D>(p, xk) / A.h2);
#pragma unroll
        for (int r = 0; r < n; ++r)
#pragma unroll
            for (int q = 0; q < n; ++q) B[r][q] += w * Pv[r] * Pv[q];
    }
#pragma unroll
    for (int r = 0; r < n; ++r)
#pragma unroll
        for (int q = 0; q < n; ++q) B[r][q] = warp_sum(B[r][q]);
    double Bi[n][n];
    if (!(m >= D + 2 && well_conditioned<n>(B) && small_inverse<n>(B, Bi))) return false;
    double aW[3] = {0.0, 0.0, 0.0}, aM[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int s = lane; s < m; s += 32) {
        const int k = sidx[s];
        double xk[3], Pv[n];
        Pv[0] = 1.0;
#pragma unroll
        for (int a = 0; a < D; ++a) { xk[a] = A.x[(int64_t)k * D + a]; Pv[1 + a] = (xk[a] - p[a]) * inv_h; }
        const double w = exp(-A.alpha * dist2_rn<D>(p, xk) / A.h2);
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < n; ++q) acc += Bi[0][q] * Pv[q];
        const double c = w * acc;
        sc[s] = c;
#pragma unroll
        for (int a = 0; a < D; ++a) aW[a] += c * A.W[(int64_t)k * D + a];
#pragma unroll
        for (int a = 0; a < D + 2; ++a) aM[a] += c * A.macro[(int64_t)k * (D + 2) + a];
    }
#pragma unroll
    for (int a = 0; a < D; ++a) aW[a] = warp_sum(aW[a]);
#pragma unroll
    for (int a = 0; a < D + 2; ++a) aM[a] = warp_sum(aM[a]);
    if (lane == 0) {
#pragma unroll
        for (int a = 0; a < D; ++a) nW[a] = aW[a];
#pragma unroll
        for (int a = 0; a < D + 2; ++a) nM[a] = aM[a];
    }
    return true;
}

// p farther than 0.45 dx from every particle of the current cloud: old particles that are not
// removed (merged ones at their midpoints) and the inserts [q0, q1)
template <int D>
__device__ bool mg_clear(const MgArgs& A, const double (&p)[3], int q0, int q1) {
    const int lane = threadIdx.x & 31;
    int ci[3] = {0, 0, 0};
#pragma unroll
    for (int a = 0; a < D; ++a) ci[a] = min(max((int)floor(p[a] * A.inv_e[a]), 0), A.nc[a] - 1);
    bool close = false;
    for (int dz = (D == 3 ? -1 : 0); dz <= (D == 3 ? 1 : 0); ++dz)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                const int cx = ci[0] + dx, cy = ci[1] + dy, cz = ci[2] + dz;
                if (cx < 0 || cx >= A.nc[0] || cy < 0 || cy >= A.nc[1] || cz < 0 || cz >= A.nc[2]) continue;
                const int c = cell_code<D>(cx, cy, cz);
                for (int t = A.cell_start[c] + lane; t < A.cell_start[c + 1]; t += 32) {
                    const int k = A.cell_pts[t];
                    const int st = A.m.status[k];
                    if (st < 0) continue;
                    double xk[3];
#pragma unroll
                    for (int a = 0; a < D; ++a) xk[a] = st > 0 ? A.m.pos[(int64_t)(st - 1) * D + a] : A.x[(int64_t)k * D + a];
                    if (!(dist2_rn<D>(p, xk) > A.thr2)) close = true;
                }
            }
    for (int q = q0 + lane; q < q1; q += 32) {
        double xq[3];
#pragma unroll
        for (int a = 0; a < D; ++a) xq[a] = A.m.pos[(int64_t)q * D + a];
        if (!(dist2_rn<D>(p, xq) > A.thr2)) close = true;
    }
    return !__any_sync(0xffffffffu, close);
}

// one warp: the greedy decisions (merges, inserts) and the compaction map
template <int D>
__global__ void __launch_bounds__(32) k_mg_decide(const MgArgs A, int64_t fill_cap) {
    const int lane = threadIdx.x & 31;
    Manage m = A.m;
    int64_t rep[8] = {0, 0, 0, 0, 0, A.N, 0, 0};
    if (m.counts[0] == 0) {
        if (lane == 0)
            for (int r = 0; r < 8; ++r) m.rep[r] = rep[r];
        return;
    }
    int q = 0;   // new particles so far
    // 1. merges (flag bit 0), ascending i
    for (int64_t base = 0; base < A.N; base += 32) {
        const int64_t ii = base + lane;
        unsigned bal = __ballot_sync(0xffffffffu, ii < A.N && (m.flag[ii] & kMergeCand));
        while (bal) {
            const int64_t i = base + __ffs(bal) - 1;
            bal &= bal - 1;
            __syncwarp();
            if (m.flag[i] & kProcessed) continue;
            double xi[3];
#pragma unroll
            for (int a = 0; a < D; ++a) xi[a] = A.x[i * D + a];
            const int64_t off = A.nb_off[i];
            const int mi = (int)(A.nb_off[i + 1] - off);
            int64_t j = -1;
            for (int e0 = 0; e0 < mi && j < 0; e0 += 32) {
                const int e = e0 + lane;
                bool ok = false;
                int k = -1;
                if (e < mi) {
                    k = A.nb_idx[off + e];
                    if (k > i && A.kind[k] == 0 && !(m.flag[k] & kProcessed)) {
                        double xk[3];
#pragma unroll
                        for (int a = 0; a < D; ++a) xk[a] = A.x[(int64_t)k * D + a];
                        ok = dist2_rn<D>(xi, xk) < A.rm2;
                    }
                }
                const unsigned b2 = __ballot_sync(0xffffffffu, ok);
                if (b2) j = __shfl_sync(0xffffffffu, k, __ffs(b2) - 1);
            }
            if (j < 0) continue;
            __syncwarp();
            if (lane == 0) {
                m.flag[i] |= kProcessed;
                m.flag[j] |= kProcessed;
            }
            __syncwarp();
            double p[3] = {0.0, 0.0, 0.0};
#pragma unroll
            for (int a = 0; a < D; ++a) p[a] = __dmul_rn(__dadd_rn(xi[a], A.x[j * D + a]), 0.5);
            if (q >= kManageMaxNew) {
                ++rep[1];
                continue;
            }
            int32_t* sidx = m.sidx + (int64_t)q * A.max_nb;
            const int ms = mg_stencil<D>(A, p, i, j, sidx, A.max_nb);
            __syncwarp();
            if (ms > A.max_nb ||
                !mg_weights<D>(A, p, sidx, ms, m.sc + (int64_t)q * A.max_nb, m.nW + (int64_t)q * D,
                               m.nM + (int64_t)q * (D + 2))) {
                ++rep[1];
                continue;
            }
            if (lane == 0) {
                for (int a = 0; a < D; ++a) m.pos[(int64_t)q * D + a] = p[a];
                m.sm[q] = ms;
                m.status[i] = q + 1;
                m.status[j] = -1;
            }
            __syncwarp();
            ++rep[0];
            ++q;
        }
    }
    // 2. inserts (flag bit 1), ascending i, candidates x_i +- 0.5 h e_a
    const int q_fill0 = q;
    const int64_t cap_ins = fill_cap - (A.N - rep[0]);
    int64_t nf = 0;
    for (int64_t base = 0; base < A.N; base += 32) {
        const int64_t ii = base + lane;
        unsigned bal = __ballot_sync(0xffffffffu, ii < A.N && (m.flag[ii] & kDeficient));
        while (bal) {
            const int64_t i = base + __ffs(bal) - 1;
            bal &= bal - 1;
            __syncwarp();
            if (m.flag[i] & kProcessed) continue;
            // candidates in proposal order: interior x_i +- 0.5 h e_a (a ascending, + before -);
            // wall particle (Z30): x_i + s h N, N = sum of its inward wall normals, s = 1/2, 1/4, 3/4,
            // the first accepted one only
            double cand[2 * D > 3 ? 2 * D : 3][3];
            int nc = 0;
            if (A.kind[i] == 0) {
                for (int a = 0; a < D; ++a)
                    for (int sgn = 0; sgn < 2; ++sgn) {
#pragma unroll
                        for (int b = 0; b < D; ++b) cand[nc][b] = A.x[i * D + b];
                        cand[nc][a] = sgn == 0 ? __dadd_rn(cand[nc][a], A.hh) : __dsub_rn(cand[nc][a], A.hh);
                        ++nc;
                    }
            } else {
                double nrm[3] = {0.0, 0.0, 0.0};    // sum of the inward normals of its walls
                for (int a = 0; a < D; ++a) {
                    const double v = A.x[i * D + a];
                    if (v == 0.0) nrm[a] = 1.0;
                    else if (v == A.L) nrm[a] = -1.0;
                }
                const double hs[3] = {0.5 * A.h, 0.25 * A.h, 0.75 * A.h};
                for (int k = 0; k < 3; ++k, ++nc)
                    for (int b = 0; b < D; ++b) cand[nc][b] = __dadd_rn(A.x[i * D + b], __dmul_rn(hs[k], nrm[b]));
            }
            const bool wall = A.kind[i] != 0;       // a wall particle takes its first accepted candidate
            for (int k = 0; k < nc; ++k) {
                    double p[3] = {0.0, 0.0, 0.0};
#pragma unroll
                    for (int b = 0; b < D; ++b) p[b] = cand[k][b];
                    bool inside = true;
#pragma unroll
                    for (int b = 0; b < D; ++b)
                        if (!(p[b] > 0.0 && p[b] < A.L)) inside = false;
                    if (!inside) continue;
                    if (!mg_clear<D>(A, p, q_fill0, q)) continue;
                    if (nf >= cap_ins || q >= kManageMaxNew) {
                        ++rep[4];
                        continue;
                    }
                    int32_t* sidx = m.sidx + (int64_t)q * A.max_nb;
                    const int ms = mg_stencil<D>(A, p, -1, -1, sidx, A.max_nb);
                    __syncwarp();
                    if (ms > A.max_nb ||
                        !mg_weights<D>(A, p, sidx, ms, m.sc + (int64_t)q * A.max_nb, m.nW + (int64_t)q * D,
                                       m.nM + (int64_t)q * (D + 2))) {
                        ++rep[3];
                        continue;
                    }
                    if (lane == 0) {
                        for (int b = 0; b < D; ++b) m.pos[(int64_t)q * D + b] = p[b];
                        m.sm[q] = ms;
                    }
                    __syncwarp();
                    ++q;
                    ++nf;
                    if (wall) break;
            }
        }
    }
    rep[2] = nf;
    // 3. compaction map: surviving slots ascending, then the inserts
    int64_t t = 0;
    for (int64_t base = 0; base < A.N; base += 32) {
        const int64_t i = base + lane;
        const int st = i < A.N ? m.status[i] : -1;
        const bool alive = i < A.N && st >= 0;
        const unsigned bal = __ballot_sync(0xffffffffu, alive);
        if (alive) {
            const int64_t ti = t + __popc(bal & ((1u << lane) - 1u));
            m.map[ti] = st > 0 ? -st : (int32_t)i;
            if (st > 0) m.dst[st - 1] = (int32_t)ti;
        }
        t += __popc(bal);
    }
    for (int qq = q_fill0 + lane; qq < q; qq += 32) {
        const int64_t ti = t + (qq - q_fill0);
        m.map[ti] = -(qq + 1);
        m.dst[qq] = (int32_t)ti;
    }
    t += q - q_fill0;
    rep[5] = t;
    rep[6] = q;
    rep[7] = (rep[0] > 0 || nf > 0) ? 1 : 0;
    if (lane == 0)
        for (int r = 0; r < 8; ++r) m.rep[r] = rep[r];
}

// new rows: f_new[dst[q]] = sum_s c_s f_old[s] over the row (padding columns interpolate zeros)
__global__ void __launch_bounds__(256) k_mg_interp(const double* __restrict__ fold, double* __restrict__ fnew,
                                                   int64_t RS, Manage m, int max_nb) {
    extern __shared__ double sc[];                          // [max_nb] weights, then [max_nb] indices
    int32_t* si = reinterpret_cast<int32_t*>(sc + max_nb);
    const int q = blockIdx.x;
    const int ms = m.sm[q];
    for (int s = threadIdx.x; s < ms; s += blockDim.x) {
        si[s] = m.sidx[(int64_t)q * max_nb + s];
        sc[s] = m.sc[(int64_t)q * max_nb + s];
    }
    __syncthreads();
    const int64_t e = blockIdx.y * (int64_t)blockDim.x + threadIdx.x;
    if (e >= RS) return;
    double acc = 0.0;
    for (int s = 0; s < ms; ++s) acc = fma(sc[s], fold[(int64_t)si[s] * RS + e], acc);
    fnew[(int64_t)m.dst[q] * RS + e] = acc;
}

// surviving rows move to their new index (16-byte copies; RS is even)
__global__ void __launch_bounds__(256) k_mg_gather(const double* __restrict__ fold, double* __restrict__ fnew,
                                                   int64_t RS, const int32_t* __restrict__ map) {
    const int64_t t = blockIdx.x;
    const int src = map[t];
    if (src < 0) return;
    const double2* a = reinterpret_cast<const double2*>(fold + (int64_t)src * RS);
    double2* b = reinterpret_cast<double2*>(fnew + t * RS);
    for (int64_t e = blockIdx.y * (int64_t)blockDim.x + threadIdx.x; e < RS / 2; e += (int64_t)gridDim.y * blockDim.x)
        b[e] = a[e];
}

template <int D>
__global__ void k_mg_small(const double* __restrict__ x, const int8_t* __restrict__ kind, const double* __restrict__ W,
                           const double* __restrict__ macro, int64_t n_out, Manage m) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n_out) return;
    const int src = m.map[t];
    if (src >= 0) {
#pragma unroll
        for (int a = 0; a < D; ++a) {
            m.x[t * D + a] = x[(int64_t)src * D + a];
            m.W[t * D + a] = W[(int64_t)src * D + a];
        }
#pragma unroll
        for (int a = 0; a < D + 2; ++a) m.macro[t * (D + 2) + a] = macro[(int64_t)src * (D + 2) + a];
        m.kind[t] = kind[src];
    } else {
        const int q = -src - 1;
#pragma unroll
        for (int a = 0; a < D; ++a) {
            m.x[t * D + a] = m.pos[(int64_t)q * D + a];
            m.W[t * D + a] = m.nW[(int64_t)q * D + a];
        }
#pragma unroll
        for (int a = 0; a < D + 2; ++a) m.macro[t * (D + 2) + a] = m.nM[(int64_t)q * (D + 2) + a];
        m.kind[t] = 0;
    }
}

// detect + decide (device only): the decisions and the 8-word report m.rep, rep[7] = cloud changed
template <int D>
void decide_pass(bgk_ctx* c, cudaStream_t s) {
    const int64_t N = c->N;
    const bgk_config& cf = c->cfg;
    const double rm = cf.r_merge > 0.0 ? cf.r_merge : 0.2 * cf.dx;
    const int m_min = cf.m_min > 0 ? cf.m_min : D + 3;
    Manage& m = c->mg;
    cudaMemsetAsync(m.counts, 0, 4 * sizeof(int32_t), s);
    cudaMemsetAsync(m.status, 0, sizeof(int32_t) * N, s);
    k_mg_detect_w<D><<<(unsigned)((N + 7) / 8), 256, 0, s>>>(c->x, c->kind, N, c->g.nb_off, c->g.nb_idx, rm * rm,
                                                             m_min, m.flag, m.counts);
    if (c->N_b)
        k_mg_detect_wall<D><<<(unsigned)((c->N_b + 7) / 8), 256, 0, s>>>(c->x, c->kind, c->boundary, c->N_b,
                                                                          c->g.nb_off, c->g.nb_idx, 1.0 / cf.h, cf.h2,
                                                                          cf.alpha_w, m.flag, m.counts);
    MgArgs A;
    A.x = c->x;
    A.kind = c->kind;
    A.W = c->W;
    A.macro = c->macro;
    A.N = N;
    A.Ncap = c->Ncap;
    A.nb_off = c->g.nb_off;
    A.nb_idx = c->g.nb_idx;
    A.cell_start = c->g.cell_start;
    A.cell_pts = c->g.cell_pts;
    for (int a = 0; a < 3; ++a) {
        A.nc[a] = c->nc[a];
        A.inv_e[a] = 1.0 / c->edge[a];
    }
    A.L = cf.L;
    A.h = cf.h;
    A.h2 = cf.h2;
    A.alpha = cf.alpha_w;
    A.rm2 = rm * rm;
    A.hh = 0.5 * cf.h;
    A.thr2 = (0.45 * cf.dx) * (0.45 * cf.dx);
    A.max_nb = c->max_nb;
    A.m = m;
    k_mg_decide<D><<<1, 32, 0, s>>>(A, c->Ncap);
}

// read the report back (one stream synchronisation) and, if the cloud changed, apply the decisions
template <int D>
bgk_status apply_pass(bgk_ctx* c, cudaStream_t s, bool* changed) {
    Manage& m = c->mg;
    int64_t rep[8];
    cudaError_t e = cudaMemcpyAsync(rep, m.rep, sizeof(rep), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return BGK_E_CUDA;
    for (int r = 0; r < 6; ++r) c->mg_report[r] = rep[r];
    *changed = rep[7] != 0;
    if (!*changed) return BGK_OK;
    const int64_t n_out = rep[5], n_new = rep[6];
    double* fold = c->f[c->fcur];
    double* fnew = c->f[1 - c->fcur];
    const unsigned chunks = (unsigned)((c->RS + 255) / 256);
    if (n_new > 0)
        k_mg_interp<<<dim3((unsigned)n_new, chunks), 256, (size_t)c->max_nb * (sizeof(double) + sizeof(int32_t)), s>>>(
            fold, fnew, c->RS, m, c->max_nb);
    k_mg_gather<<<dim3((unsigned)n_out, (unsigned)std::min<int64_t>(8, (c->RS / 2 + 255) / 256)), 256, 0, s>>>(
        fold, fnew, c->RS, m.map);
    k_mg_small<D><<<(unsigned)((n_out + 255) / 256), 256, 0, s>>>(c->x, c->kind, c->W, c->macro, n_out, m);
    cudaMemcpyAsync(c->x, m.x, sizeof(double) * n_out * D, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(c->W, m.W, sizeof(double) * n_out * D, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(c->macro, m.macro, sizeof(double) * n_out * (D + 2), cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(c->kind, m.kind, (size_t)n_out, cudaMemcpyDeviceToDevice, s);
    c->fcur = 1 - c->fcur;
    c->N = n_out;
    ++c->cloud_gen;                     // rows renumbered: a pending staged input is stale
    std::vector<int8_t> hk(n_out);
    std::vector<double> hx(n_out * D);
    e = cudaMemcpyAsync(hk.data(), c->kind, (size_t)n_out, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hx.data(), c->x, sizeof(double) * n_out * D, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return BGK_E_CUDA;
    c->geometry_valid = false;
    return install_lists(c, hk.data(), hx.data(), s);
}

}  // namespace

void manage_decide(bgk_ctx* c, cudaStream_t s) {
    if (!c->cfg.manage || c->N == 0) return;
    if (c->d == 3) decide_pass<3>(c, s);
    else decide_pass<2>(c, s);
}

bgk_status manage_apply(bgk_ctx* c, cudaStream_t s, bool* changed) {
    *changed = false;
    if (!c->cfg.manage || c->N == 0) return BGK_OK;
    const bgk_status st = c->d == 3 ? apply_pass<3>(c, s, changed) : apply_pass<2>(c, s, changed);
    if (st != BGK_OK) return st;
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? BGK_OK : BGK_E_CUDA;
}

bgk_status manage_pass(bgk_ctx* c, cudaStream_t s, bool* changed) {
    *changed = false;
    if (!c->cfg.manage || c->N == 0) return BGK_OK;
    manage_decide(c, s);
    const bgk_status st = manage_apply(c, s, changed);
    if (st != BGK_OK) return st;
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? BGK_OK : BGK_E_CUDA;
}

}  // namespace bgk
