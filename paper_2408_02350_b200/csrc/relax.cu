// relax.cu -- moment recovery, local Maxwellian, implicit BGK relaxation, ALE
// motion, diffuse-reflection walls, initial state and diagnostics moments.
//
//  k_moment_reduce : per-particle sum of the transport warps' partials (fixed order)
//  k_relax(_w2)    : rho, U, T from the (all-reduced) sums,
//                    tau, M^{n+1} inline as a product of three 1D Gaussian
//                    factors (P:46-49 / P:98-105 with Z1, Z2),
//                    f^{n+1} = (tau ftilde + dt M)/(tau + dt),
//                    W <- U^{n+1}, x += dt U^{n+1} clamped
//  k_bnd_union     : per geometry build, the union of a boundary group's interior neighbours
//                    and its dense weight matrix (3D: face tiles of <= 16 members; 2D: 4)
//  k_bnd_interp_s  : 3D incoming half of each boundary row by WLS interpolation of the
//                    interior f^{n+1} (Z17, Z19) on the FP64 tensor cores + flux partials
//  k_bnd_interp_t  : the same in 2D (ring-staged union rows, FMA)
//  k_wall_reduce   : per boundary particle, fixed-order sum of the flux partials
//  k_bnd_fill      : rho_w = -flux_in / sum_{v.n>0}(v.n) M_w ; outgoing half = rho_w M_w
#include "async.cuh"
#include "bgk_internal.cuh"
#include "relax_params.cuh"

namespace bgk {

namespace {


template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int q = 0; q < NT / 32; ++q) t += sh[q];   // fixed order
    return t;                                            // valid in thread 0
}

// node velocity components of local node t = k1 * ncol + col
template <int D>
__device__ __forceinline__ void node_vel(int t, int ncol, int c0, int n1, double vmax, double dv, double (&v)[3],
                                         int (&kk)[3]) {
    const int k1 = t / ncol, col = t - k1 * ncol, gc = c0 + col;
    kk[0] = k1;
    if constexpr (D == 3) {
        kk[1] = gc / n1;
        kk[2] = gc - kk[1] * n1;
    } else {
        kk[1] = gc;
        kk[2] = 0;
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) v[a] = (a < D) ? axis_node(vmax, dv, kk[a]) : 0.0;
}

// velocity of STORED node ts = k1 * ncs + col; false for the padding column (col >= ncol)
template <int D>
__device__ __forceinline__ bool node_vel_s(int64_t ts, int ncs, int ncol, int c0, int n1, double vmax, double dv,
                                           double (&v)[3]) {
    const int k1 = (int)(ts / ncs), col = (int)(ts - (int64_t)k1 * ncs);
    if (col >= ncol) return false;
    int kk[3];
    node_vel<D>(k1 * ncol + col, ncol, c0, n1, vmax, dv, v, kk);
    return true;
}

__global__ void k_moment_reduce(const int32_t* __restrict__ ids, int64_t n, const double* __restrict__ partials,
                                int nwpp, double* __restrict__ sums) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int p = ids[t];
    double acc[kPM] = {0, 0, 0, 0, 0};
    for (int w = 0; w < nwpp; ++w)
#pragma unroll
        for (int q = 0; q < kPM; ++q) acc[q] += partials[((int64_t)p * nwpp + w) * kPM + q];
#pragma unroll
    for (int q = 0; q < kPM; ++q) sums[(int64_t)p * kPM + q] = acc[q];
}

template <int D>
__global__ void __launch_bounds__(256) k_relax(const RelaxArgs A) {
    constexpr int NV = (D == 2) ? 2 : 1;
    __shared__ double e[D][64];
    __shared__ double par[8];
    extern __shared__ double colf[];            // [ncs] per stored column (dynamic)
    const int64_t bi = blockIdx.x;
    if (bi >= A.n) return;
    const int p = A.ids[bi];
    // 16-byte accesses: in 3D two adjacent columns (ncs is even), in 2D the (g1, g2) pair of a node.
    // The first round of each thread's loads is issued before the moment recovery and the
    // exponentials below, so its latency overlaps them (short 2D rows: one round per thread).
    double2* fp2 = reinterpret_cast<double2*>(A.f + (int64_t)p * A.Ks * NV);
    const int P = (D == 3) ? A.ncs / 2 : A.ncs;              // 16-B elements per stored row
    const int n2 = P * A.n1;
    constexpr int U = 4;
    double2 g[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
        const int u = threadIdx.x + q * blockDim.x;
        if (u < n2) g[q] = fp2[u];
    }
    if (threadIdx.x == 0) relax_params<D>(A, A.sums + (int64_t)p * kPM, p, par);
    __syncthreads();
    const double inv2RT = par[4];
    for (int t = threadIdx.x; t < D * A.n1; t += blockDim.x) {
        const int a = t / A.n1, j = t - a * A.n1;
        const double dvel = axis_node(A.vmax, A.dv, j) - par[5 + a];
        e[a][j] = exp(-dvel * dvel * inv2RT);
    }
    __syncthreads();
    const double a1 = par[0], a2 = par[1], pref = par[2], RT = par[3];
    // per stored column: the v_2 (and v_3) factor of the separable Maxwellian, 0 on padding columns
    for (int c = threadIdx.x; c < A.ncs; c += blockDim.x) {
        double cf = 0.0;
        if (c < A.ncol) {
            const int gc = A.c0 + c;
            if constexpr (D == 3) cf = e[1][gc / A.n1] * e[2][gc - (gc / A.n1) * A.n1];
            else cf = e[1][gc];
        }
        colf[c] = cf;
    }
    __syncthreads();
    // Four independent loads in flight per thread; (row, column) of each advance incrementally
    // (no integer division in the streaming loop).
    const int stride = U * blockDim.x;
    const int dk = stride / P, dc = stride - dk * P;
    int kr[U], cq[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
        const int u = threadIdx.x + q * blockDim.x;
        kr[q] = u / P;
        cq[q] = u - kr[q] * P;
    }
    for (int u0 = threadIdx.x; u0 < n2; u0 += stride) {
        if (u0 != (int)threadIdx.x) {
#pragma unroll
            for (int q = 0; q < U; ++q) {
                const int u = u0 + q * blockDim.x;
                if (u < n2) g[q] = fp2[u];
            }
        }
#pragma unroll
        for (int q = 0; q < U; ++q) {
            const int u = u0 + q * blockDim.x;
            if (u < n2) {
                const double rowf = pref * e[0][kr[q]];
                if constexpr (D == 3) {
                    const int col = 2 * cq[q];
                    g[q].x = a1 * g[q].x + a2 * (rowf * colf[col]);
                    g[q].y = col + 1 < A.ncol ? a1 * g[q].y + a2 * (rowf * colf[col + 1]) : 0.0;
                } else {
                    const double M = rowf * colf[cq[q]];
                    g[q].x = a1 * g[q].x + a2 * M;
                    g[q].y = a1 * g[q].y + a2 * (RT * M);
                }
                fp2[u] = g[q];
            }
            cq[q] += dc;
            kr[q] += dk;
            if (cq[q] >= P) {
                cq[q] -= P;
                ++kr[q];
            }
        }
    }
}

// 2D relaxation, one warp per particle: a 2D row is short (C2/C3: 1089 nodes, 17 KB), so a
// 256-thread block per particle spent its time in the block-wide prologue (moments -> tau, the
// 2 x (Nv+1) exponentials, three __syncthreads) with one round of loads per thread; here the lanes
// share the prologue and each streams ~34 (g1, g2) pairs with four loads in flight.
__global__ void __launch_bounds__(256) k_relax_w2(const RelaxArgs A) {
    __shared__ double e[8][2][64];
    __shared__ double par[8][8];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t bi = (int64_t)blockIdx.x * 8 + wib;
    if (bi >= A.n) return;
    const int p = A.ids[bi];
    double2* fp2 = reinterpret_cast<double2*>(A.f + (int64_t)p * A.Ks * 2);
    const int n2 = A.ncs * A.n1;                      // 16-B (g1, g2) pairs of the stored row
    constexpr int U = 4;
    double2 g[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
        const int u = lane + 32 * q;
        if (u < n2) g[q] = fp2[u];
    }
    if (lane == 0) relax_params<2>(A, A.sums + (int64_t)p * kPM, p, par[wib]);
    __syncwarp();
    const double inv2RT = par[wib][4];
    for (int t = lane; t < 2 * A.n1; t += 32) {
        const int a = t / A.n1, j = t - a * A.n1;
        const double dvel = axis_node(A.vmax, A.dv, j) - par[wib][5 + a];
        e[wib][a][j] = exp(-dvel * dvel * inv2RT);
    }
    __syncwarp();
    const double a1 = par[wib][0], a2 = par[wib][1], pref = par[wib][2], RT = par[wib][3];
    const double* e0 = e[wib][0];
    const double* e1 = e[wib][1] + A.c0;
    // (row, column) of element u = lane + 32 (q + U k) advance incrementally
    int kr[U], cq[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
        const int u = lane + 32 * q;
        kr[q] = u / A.ncs;
        cq[q] = u - kr[q] * A.ncs;
    }
    const int stride = 32 * U, dk = stride / A.ncs, dc = stride - dk * A.ncs;
    for (int u0 = lane; u0 < n2; u0 += stride) {
        if (u0 != lane) {
#pragma unroll
            for (int q = 0; q < U; ++q) {
                const int u = u0 + 32 * q;
                if (u < n2) g[q] = fp2[u];
            }
        }
#pragma unroll
        for (int q = 0; q < U; ++q) {
            const int u = u0 + 32 * q;
            if (u < n2) {
                const double M = pref * e0[kr[q]] * e1[cq[q]];
                g[q].x = a1 * g[q].x + a2 * M;
                g[q].y = a1 * g[q].y + a2 * (RT * M);
                fp2[u] = g[q];
            }
            cq[q] += dc;
            kr[q] += dk;
            if (cq[q] >= A.ncs) {
                cq[q] -= A.ncs;
                ++kr[q];
            }
        }
    }
}

// Maxwellian M(rho, U, T) (2D: (G1, G2)) at node velocity v
template <int D>
__device__ __forceinline__ void maxwellian_at(double rho, const double* U, double T, double R, const double (&v)[3],
                                              double (&out)[2]) {
    const double RT = R * T;
    double q = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) q += (v[a] - U[a]) * (v[a] - U[a]);
    const double twoPiRT = 2.0 * kPi * RT;
    const double pref = (D == 3) ? rho / (twoPiRT * sqrt(twoPiRT)) : rho / twoPiRT;
    out[0] = pref * exp(-q / (2.0 * RT));
    out[1] = RT * out[0];
}

template <int D>
__global__ void k_init_f(const double* __restrict__ macro0, int64_t N, double* __restrict__ f,
                         double* __restrict__ macro, double* __restrict__ W, int ale, int n1, int ncol, int ncs,
                         int c0, int64_t Ks, double vmax, double dv, double R, double Twall) {
    constexpr int NV = (D == 2) ? 2 : 1;
    const int64_t p = blockIdx.x;
    if (p >= N) return;
    double rho = 1.0, U[3] = {0, 0, 0}, T = Twall;
    if (macro0) {
        rho = macro0[p * (D + 2)];
#pragma unroll
        for (int a = 0; a < D; ++a) U[a] = macro0[p * (D + 2) + 1 + a];
        T = macro0[p * (D + 2) + 1 + D];
    }
    if (threadIdx.x == 0) {
        macro[p * (D + 2)] = rho;
#pragma unroll
        for (int a = 0; a < D; ++a) {
            macro[p * (D + 2) + 1 + a] = U[a];
            W[p * D + a] = ale ? U[a] : 0.0;
        }
        macro[p * (D + 2) + 1 + D] = T;
    }
    for (int64_t t = threadIdx.x; t < Ks; t += blockDim.x) {
        double v[3];
        if (!node_vel_s<D>(t, ncs, ncol, c0, n1, vmax, dv, v)) continue;
        double M[2];
        maxwellian_at<D>(rho, U, T, R, v, M);
#pragma unroll
        for (int q = 0; q < NV; ++q) f[(p * Ks + t) * NV + q] = M[q];
    }
}

// wall tables: Mw[w][local node] = M(1, U_w, T_w); den[w] = sum over the GLOBAL grid of
// (v.n)^+ M_w (2D: G1), identical on every rank.
template <int D>
__global__ void k_wall_M(double* __restrict__ Mw, int n1, int ncol, int ncs, int c0, int64_t Ks, double vmax,
                         double dv, double R, double Twall, double lid0, double lid1, double lid2) {
    constexpr int NV = (D == 2) ? 2 : 1;
    const int wid = blockIdx.y + 1;
    const int axis = (wid - 1) / 2;
    const double sgn = ((wid - 1) % 2 == 0) ? 1.0 : -1.0;
    const double U[3] = {wid == 2 * D ? lid0 : 0.0, wid == 2 * D ? lid1 : 0.0, wid == 2 * D ? lid2 : 0.0};
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < Ks; t += (int64_t)gridDim.x * blockDim.x) {
        double v[3];
        double M[2] = {-1.0, -1.0};    // -1: not an outgoing node of this wall (k_bnd_fill skips it)
        if (node_vel_s<D>(t, ncs, ncol, c0, n1, vmax, dv, v) && sgn * v[axis] > 0.0)
            maxwellian_at<D>(1.0, U, Twall, R, v, M);
#pragma unroll
        for (int q = 0; q < NV; ++q) Mw[((int64_t)blockIdx.y * Ks + t) * NV + q] = M[q];
    }
}

template <int D>
__global__ void __launch_bounds__(256) k_wall_den(double* __restrict__ den, int n1, int ncol_g, double vmax,
                                                  double dv, double R, double Twall, double lid0, double lid1,
                                                  double lid2, int64_t* err) {
    __shared__ double sh[32];
    const int wid = blockIdx.x + 1;
    const int axis = (wid - 1) / 2;
    const double sgn = ((wid - 1) % 2 == 0) ? 1.0 : -1.0;
    const double U[3] = {wid == 2 * D ? lid0 : 0.0, wid == 2 * D ? lid1 : 0.0, wid == 2 * D ? lid2 : 0.0};
    const int64_t K = (int64_t)n1 * ncol_g;
    double acc = 0.0;
    for (int64_t t = threadIdx.x; t < K; t += blockDim.x) {
        double v[3];
        int kk[3];
        node_vel<D>((int)t, ncol_g, 0, n1, vmax, dv, v, kk);
        const double vn = sgn * v[axis];
        if (vn > 0.0) {
            double M[2];
            maxwellian_at<D>(1.0, U, Twall, R, v, M);
            acc += vn * M[0];
        }
    }
    const double tot = block_sum<256>(acc, sh);
    if (threadIdx.x == 0) {
        den[blockIdx.x] = tot;
        if (!(tot > 0.0)) latch_error(err, BGK_E_WALL, -1);
    }
}

constexpr int kBndChunk = 256;

// ---------------------------------------------------------------------------------------------
// Boundary interpolation by groups of G consecutive particles of the face-sorted boundary list
// (G = 8 in 3D, 4 in 2D; BGK_BND_G = 4 or 8 overrides).  k_bnd_union (per geometry build) merges
// their compacted (neighbour, weight) lists into one union with a dense G-column weight matrix;
// k_bnd_interp_t loads each union row's chunk ONCE for the group and applies it to every member
// (weight 0 if not its neighbour): fewer row loads for more FMAs.  Round 1 measured the per-particle
// form at 3.20 ms on C5 and an __ldg union of 4 at 2.83-2.89 ms (both removed in round 2).
// ---------------------------------------------------------------------------------------------
// TILE (3D): group g is the member range bg_off[g] .. bg_off[g+1] of the boundary list (face tiles,
// install_lists).
template <int G, bool TILE = false>
__global__ void __launch_bounds__(256) k_bnd_union(const int32_t* __restrict__ bids, int64_t nb,
                                                   const int32_t* __restrict__ bg_off,
                                                   const int64_t* __restrict__ nb_off,
                                                   const int32_t* __restrict__ bidx, const double* __restrict__ bcw,
                                                   const int32_t* __restrict__ bcnt, int cap,
                                                   int32_t* __restrict__ bu_j, double* __restrict__ bu_w,
                                                   int32_t* __restrict__ bu_n,
                                                   int64_t* err) {
    constexpr int QB = G > 8 ? 4 : 3;                       // member bits of a key
    constexpr int QM = (1 << QB) - 1;
    extern __shared__ int32_t keys[];                       // [2 n2]: sorted (j << QB | q), then union slots
    __shared__ int s_len[G + 1];
    __shared__ int s_n;
    const int64_t g = blockIdx.x;
    const int64_t gb = TILE ? bg_off[g] : g * G;            // first member's position in the list
    const int64_t ge = TILE ? bg_off[g + 1] : min(gb + G, nb);
    if (threadIdx.x == 0) {
        int tot = 0;
        for (int q = 0; q < G; ++q) {
            s_len[q] = tot;
            const int64_t bi = gb + q;
            if (bi < ge) tot += bcnt[bids[bi]];
        }
        s_len[G] = tot;
    }
    __syncthreads();
    const int tot = s_len[G];
    int n2 = 1;
    while (n2 < tot) n2 <<= 1;
    for (int i = threadIdx.x; i < n2; i += blockDim.x) keys[i] = INT_MAX;
    __syncthreads();
    for (int q = 0; q < G; ++q) {
        const int64_t bi = gb + q;
        if (bi >= ge) break;
        const int b = bids[bi];
        const int64_t off = nb_off[b];
        for (int i = threadIdx.x; i < bcnt[b]; i += blockDim.x) keys[s_len[q] + i] = (bidx[off + i] << QB) | q;
    }
    __syncthreads();
    for (int k = 2; k <= n2; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n2; i += blockDim.x) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const int a = keys[i], b = keys[ixj];
                    if ((a > b) == ((i & k) == 0)) {
                        keys[i] = b;
                        keys[ixj] = a;
                    }
                }
            }
            __syncthreads();
        }
    int32_t* upos = keys + n2;
    // union slot of every sorted entry: a block-wide scan of "first of its j" flags, 256 at a time
    // (a serial walk by one thread was the kernel's latency on the 2D workloads)
    __shared__ int wcnt[8];
    int ubase = 0;
    for (int i0 = 0; i0 < tot; i0 += 256) {
        const int i = i0 + threadIdx.x;
        const int j = i < tot ? keys[i] >> QB : -1;
        const bool first = i < tot && (i == 0 || (keys[i - 1] >> QB) != j);
        const unsigned bal = __ballot_sync(0xffffffffu, first);
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        if (lane == 0) wcnt[wid] = __popc(bal);
        __syncthreads();
        int before = ubase, total = 0;
        for (int w = 0; w < 8; ++w) {
            before += w < wid ? wcnt[w] : 0;
            total += wcnt[w];
        }
        const int u = before + __popc(bal & ((1u << lane) - 1u)) + (first ? 0 : -1);   // slot of entry i
        if (i < tot) {
            upos[i] = u;
            if (first && u < cap) bu_j[g * cap + u] = j;
        }
        ubase += total;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        s_n = ubase;
        if (ubase > cap) latch_error(err, BGK_E_CAPACITY, bids[gb]);
        bu_n[g] = ubase > cap ? 0 : ubase;
    }
    __syncthreads();
    if (s_n > cap) return;
    double* W = bu_w + g * cap * G;
    for (int i = threadIdx.x; i < s_n * G; i += blockDim.x) W[i] = 0.0;
    __syncthreads();
    for (int i = threadIdx.x; i < tot; i += blockDim.x) {
        const int j = keys[i] >> QB, q = keys[i] & QM;
        const int b = bids[gb + q];
        const int64_t off = nb_off[b];
        int lo = 0, hi = bcnt[b] - 1;                       // compacted lists are ascending in j
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (bidx[off + mid] < j) lo = mid + 1;
            else hi = mid;
        }
        W[upos[i] * G + q] = bcw[off + lo];
    }
}

// ---------------------------------------------------------------------------------------------
// Boundary interpolation with the union rows staged by bulk copies (k_bnd_interp_t).  Block =
// (group of G face-consecutive boundary particles, chunk of 256*NPT stored nodes).  The group's
// union rows (k_bnd_union) stream through an NS-deep shared-memory ring, one contiguous
// cp.async.bulk per (row, chunk) on a "full" mbarrier; the ring is refilled half by half: after
// the block has consumed the NS/2 rows of one half (__syncthreads), thread 0 issues the next NS/2
// rows into it while the other half is applied -- the row traffic is in flight asynchronously
// instead of waiting on each thread's loads (the __ldg form of k_bnd_interp_u sat at ~4 TB/s of
// useful L2 traffic, latency-bound).  Each thread applies a staged row to its NPT nodes for all G
// members (dense G-column weights).  A chunk with no incoming node for any member (walls normal to
// v_1: half the rows) only writes zero flux partials.
// ---------------------------------------------------------------------------------------------
template <int D, int G, int NPT, int NS, int MINB = 2>
__global__ void __launch_bounds__(256, MINB) k_bnd_interp_t(const int32_t* __restrict__ bids, int64_t nb,
                                                      const int8_t* __restrict__ kind,
                                                      const int32_t* __restrict__ bu_j,
                                                      const double* __restrict__ bu_w,
                                                      const int32_t* __restrict__ bu_n, int cap,
                                                      double* __restrict__ f, double* __restrict__ wallpart,
                                                      int nch, int n1, int ncol, int ncs, int c0, int64_t Kloc,
                                                      double vmax, double dv) {
    constexpr int NV = (D == 2) ? 2 : 1;
    constexpr int CH = 256 * NPT;                             // stored nodes per chunk
    constexpr uint32_t SB = CH * NV * sizeof(double);         // bytes per ring stage
    extern __shared__ __align__(128) unsigned char sm[];
    double* ring = reinterpret_cast<double*>(sm);
    static_assert(NS % 2 == 0, "the ring is refilled half by half");
    constexpr int NH = NS / 2;
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + NS * SB);
    double* sW = reinterpret_cast<double*>(full + 2 * NS);    // [U][G] (2 NS words reserved)
    int32_t* sJ = reinterpret_cast<int32_t*>(sW + (size_t)cap * G);
    __shared__ double sh[32];
    const int64_t g = blockIdx.x;
    const int tid = threadIdx.x;
    const int U = bu_n[g];
    int b[G], axis[G];
    bool live[G];
    double sgn[G];
#pragma unroll
    for (int q = 0; q < G; ++q) {
        const int64_t bi = g * G + q;
        live[q] = bi < nb;
        b[q] = live[q] ? bids[bi] : 0;
        const int wid = live[q] ? kind[b[q]] : 1;
        axis[q] = (wid - 1) / 2;
        sgn[q] = ((wid - 1) % 2 == 0) ? 1.0 : -1.0;
    }
    int64_t t[NPT];
    double v[NPT][3];
    bool inc[G][NPT];
    bool any = false;
#pragma unroll
    for (int n = 0; n < NPT; ++n) {
        t[n] = (int64_t)blockIdx.y * CH + n * 256 + tid;
        v[n][0] = v[n][1] = v[n][2] = 0.0;
        const bool in_range = t[n] < Kloc && node_vel_s<D>(t[n], ncs, ncol, c0, n1, vmax, dv, v[n]);
#pragma unroll
        for (int q = 0; q < G; ++q) {
            inc[q][n] = live[q] && in_range && sgn[q] * v[n][axis[q]] <= 0.0;
            any = any || inc[q][n];
        }
    }
    if (!__syncthreads_or(any) || U == 0) {                   // nothing incoming in this chunk
        if (tid < G && g * G + tid < nb) wallpart[(g * G + tid) * nch + blockIdx.y] = 0.0;
        return;
    }
    for (int i = tid; i < U * G; i += blockDim.x) sW[i] = bu_w[g * cap * G + i];
    for (int i = tid; i < U; i += blockDim.x) sJ[i] = bu_j[g * cap + i];
    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < NS; ++s) mbar_init(full + s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    const int64_t c0n = (int64_t)blockIdx.y * CH;
    const uint32_t bytes = (uint32_t)(min((int64_t)CH, Kloc - c0n) * NV * sizeof(double));
    auto issue = [&](int u) {                                 // thread 0: row u's chunk into stage u % NS
        const int s = u % NS;
        mbar_expect_tx(full + s, bytes);
        bulk_load(ring + (size_t)s * CH * NV, f + ((int64_t)sJ[u] * Kloc + c0n) * NV, bytes, full + s);
    };
    // rows are issued by parallel threads (one row each): one thread issuing a ring's rows in sequence
    // holds ~800 cycles per row (tools/probe/bulk_probe.cu)
    if (tid < NS && tid < U) issue(tid);
    double acc[G][NPT][NV];
#pragma unroll
    for (int q = 0; q < G; ++q)
#pragma unroll
        for (int n = 0; n < NPT; ++n)
#pragma unroll
            for (int c = 0; c < NV; ++c) acc[q][n][c] = 0.0;
    for (int u = 0; u < U; ++u) {
        const int s = u % NS;
        const uint32_t ph = (uint32_t)(u / NS) & 1u;
        mbar_wait(full + s, ph);
        const double* st = ring + (size_t)s * CH * NV;
        double fv[NPT][NV];
#pragma unroll
        for (int n = 0; n < NPT; ++n) {
            if constexpr (NV == 1) {
                fv[n][0] = st[n * 256 + tid];
            } else {
                const double2 gv = reinterpret_cast<const double2*>(st)[n * 256 + tid];
                fv[n][0] = gv.x;
                fv[n][1] = gv.y;
            }
        }
        const double* wu = sW + u * G;
#pragma unroll
        for (int q = 0; q < G; ++q) {
            const double w = wu[q];
#pragma unroll
            for (int n = 0; n < NPT; ++n)
#pragma unroll
                for (int c = 0; c < NV; ++c) acc[q][n][c] = fma(w, fv[n][c], acc[q][n][c]);
        }
        if (u % NH == NH - 1 && u + 1 < U) {                  // a half consumed by every warp:
            __syncthreads();                                  // refill it NS rows ahead
            const int q = u + 1 - NH + NS + tid;
            if (tid < NH && q < U) issue(q);
        }
    }
#pragma unroll
    for (int q = 0; q < G; ++q) {
        double flux = 0.0;
#pragma unroll
        for (int n = 0; n < NPT; ++n) {
            if (!inc[q][n]) continue;
            if constexpr (NV == 1) f[(int64_t)b[q] * Kloc + t[n]] = acc[q][n][0];
            else reinterpret_cast<double2*>(f)[(int64_t)b[q] * Kloc + t[n]] = make_double2(acc[q][n][0], acc[q][n][1]);
            const double vn = sgn[q] * v[n][axis[q]];
            if (vn < 0.0) flux += vn * acc[q][n][0];
        }
        const double tot = block_sum<256>(flux, sh);
        if (threadIdx.x == 0 && live[q]) wallpart[(g * G + q) * nch + blockIdx.y] = tot;
    }
}

// ---------------------------------------------------------------------------------------------
// 3D boundary interpolation over face tiles (k_bnd_interp_s), on the FP64 tensor cores.  Block =
// (tile group g of up to G = 16 members of ONE wall, chunk ch of that wall's plan).  The plan
// (bnd_plan, host, once per context) lists for each wall the velocity nodes that can be incoming
// (v.n <= 0) and cuts them into chunks of at most kBndAct nodes whose stored positions fit in
// kBndSeg contiguous segments of at most kBndStage nodes -- only incoming nodes are computed and,
// where they are contiguous runs (walls normal to v_1 or v_2), only their bytes are staged.
// For the chunk the block computes the dense product
//     F_b[member m][node n] = sum_u W[u][m] F[u][n]      (u = the group's union rows)
// with mma.sync m16n8k4 f64: A = W^T (16 members x 4 union rows), B = 4 union rows x 8 listed nodes,
// the 16 x 8 accumulator tile in registers; each of the 12 consumer warps owns 64 listed nodes
// (8 tiles).  The ~70 % zero weights of a 4 x 4 tile's union cost tensor-pipe slots, not issue slots:
// per 4 union rows a warp issues 8 MMAs against 4 x 64 predicated DFMAs + weight loads of the
// DFMA form (2.1 ms on C5, latency-bound on the shared-memory loads feeding it).
// The union rows (the chunk's segments + the row's 16 weights) stream through a ring of as many
// stages as 192 KB holds (at most 32; the staged bytes per row differ 2x between walls): a producer
// warp (warp 12) waits for a stage's "empty" mbarrier (one arrival per consumer warp) and its lanes
// issue 6 rows' bulk copies at once on the stages' "full" mbarriers.  In a k-step lane l reads the
// stage of union row u0 + (l & 3) only.  The flux partials reduce in a fixed order.
// Measured on C5 (tools/phase_times.py; the line-group kernel k_bnd_interp_t took 2.44 ms): one lane
// issuing the copies row after row ran ~800 cycles per row whatever the ring depth (2.1-2.5 ms; the
// same per-thread issue limit shows in tools/probe/bulk_probe.cu), lanes issuing 6 rows at once
// 1.61 ms with 32 stages -- copies alone 1.47 ms, the MMAs alone 1.27 ms.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ void mma_f64_16x8x4(double (&c)[4], double a0, double a1, double b) {
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0, %1, %2, %3}, {%4, %5}, {%6}, "
                 "{%0, %1, %2, %3};"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                 : "d"(a0), "d"(a1), "d"(b));
}

constexpr int kBndWarps = 12;                                // consumer warps of k_bnd_interp_s
static_assert(kBndWarps * 64 == kBndAct, "64 listed nodes per consumer warp");

constexpr int kBndRing = 192 * 1024;                        // ring bytes of k_bnd_interp_s
constexpr int kBndPR = 6;                                    // rows issued per producer iteration
constexpr int kBndNSMax = 32;                                // ring stages at most

__global__ void __launch_bounds__((kBndWarps + 1) * 32, 1) k_bnd_interp_s(const int32_t* __restrict__ bids,
                                                         const int32_t* __restrict__ bg_off,
                                                         const int8_t* __restrict__ kind,
                                                         const int32_t* __restrict__ bu_j,
                                                         const double* __restrict__ bu_w,
                                                         const int32_t* __restrict__ bu_n, int cap,
                                                         const BndChunk* __restrict__ chunks,
                                                         const int32_t* __restrict__ act_t,
                                                         const int32_t* __restrict__ act_s, double* __restrict__ f,
                                                         double* __restrict__ wallpart, int nch, int n1, int ncol,
                                                         int ncs, int c0, int64_t Ks, double vmax, double dv,
                                                         int nsmax) {
    constexpr int G = kBndTile;
    static_assert(G == 16, "one m16 tile of members");
    constexpr int NTILE = 8;                                  // 8-node MMA tiles per consumer warp
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + kBndRing);
    uint64_t* empty = full + kBndNSMax;
    int32_t* sJ = reinterpret_cast<int32_t*>(empty + kBndNSMax);   // [cap] union rows
    __shared__ double red[kBndWarps][G];
    const int64_t g = blockIdx.x;
    const int ch = blockIdx.y, tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
    const int b0 = bg_off[g], nm = bg_off[g + 1] - b0;
    const int w = kind[bids[b0]] - 1;                          // every member lies on this wall
    const int axis = w / 2;
    const double sgn = (w % 2 == 0) ? 1.0 : -1.0;
    const int U = bu_n[g];
    const int64_t cix = (int64_t)w * nch + ch;
    const int nact = chunks[cix].nact;
    // stage = the chunk's staged nodes + the row's weights; as many stages as the ring holds (the
    // staged bytes per row differ 2x between walls: the ring keeps ~190 KB in flight for all)
    const int FB = (chunks[cix].slen * (int)sizeof(double) + 127) / 128 * 128;
    // stage stride = 64 (mod 128) bytes: the 4 stages a k-step reads (lanes with tig 0..3 at the same
    // node offsets) fall on alternating bank halves -- 2 wavefronts per warp load instead of 4
    const int SB = (FB + G * (int)sizeof(double) + 127) / 128 * 128 + 64;
    const int NS = min(nsmax, kBndRing / SB);
    if (U == 0 || nact == 0) {
        if (tid < nm) wallpart[(int64_t)(b0 + tid) * nch + ch] = 0.0;
        return;
    }
    for (int i = tid; i < U; i += blockDim.x) sJ[i] = bu_j[g * cap + i];
    if (tid == 0) {
#pragma unroll
        for (int q = 0; q < NS; ++q) {
            mbar_init(full + q, 1);
            mbar_init(empty + q, kBndWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (wp == kBndWarps) {                                    // producer warp
        // kBndPR rows per iteration, one lane per (row, piece): pieces 0 .. nseg-1 are the chunk's
        // segments, piece kBndSeg the row's weights.  Issuing from many lanes at once matters: one
        // lane issuing expect_tx + bulk copies row after row managed ~800 cycles per row whatever the
        // size or ring depth (tools/probe/bulk_probe.cu: 3.0 TB/s at 8 KB per row), 4+ rows issued by
        // parallel lanes stream at the DRAM rate (6.7-7.0 TB/s)
        constexpr int PC = kBndSeg + 1;                       // pieces per row
        const BndChunk* C = chunks + cix;
        const int nseg = C->nseg;
        const uint32_t txb = (uint32_t)C->slen * 8u + G * 8u;
        const int pr = lane / PC, pc = lane - pr * PC;        // this lane's row in the batch, piece
        const int sk = min(pc, kBndSeg - 1);
        const int ssrc = C->src[sk], sdst = C->dst[sk];
        const uint32_t slen = (uint32_t)C->len[sk] * 8u;
        const bool active = pr < kBndPR && (pc < nseg || pc == kBndSeg);
        for (int u0 = 0; u0 < U; u0 += kBndPR) {
            const int u = u0 + pr;
            const bool mine = active && u < U;
            const int q = u % NS;
            if (mine && u >= NS) mbar_wait_sleep(empty + q, (uint32_t)(u / NS - 1) & 1u);
            if (mine && pc == 0) mbar_expect_tx(full + q, txb);
            __syncwarp();
            if (mine) {
                unsigned char* st = sm + (size_t)q * SB;
                if (pc < kBndSeg) bulk_load(st + (size_t)sdst * 8, f + (int64_t)sJ[u] * Ks + ssrc, slen, full + q);
                else bulk_load(st + FB, bu_w + (g * cap + u) * G, G * 8u, full + q);
            }
            __syncwarp();
        }
    } else {
        const int gq = lane >> 2, tig = lane & 3;
        const int abase = wp * 64;                            // this warp's listed nodes
        const int ntile = max(0, min(NTILE, (nact - abase + 7) / 8));   // tiles holding listed nodes
        int so[NTILE];
#pragma unroll
        for (int j = 0; j < NTILE; ++j) {
            const int a = abase + j * 8 + gq;
            so[j] = a < nact ? act_s[cix * kBndAct + a] : 0;  // unlisted columns read a staged node
        }
        double acc[NTILE][4];
#pragma unroll
        for (int j = 0; j < NTILE; ++j)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[j][e] = 0.0;
        for (int u0 = 0; u0 < U; u0 += 4) {
            const int r = u0 + tig;                           // this lane's union row in the k-step
            const bool live = r < U;
            const double* st = reinterpret_cast<const double*>(sm + (size_t)(r % NS) * SB);
            double a0 = 0.0, a1 = 0.0;
            if (live) {
                mbar_wait_sleep(full + r % NS, (uint32_t)(r / NS) & 1u);
                a0 = st[FB / 8 + gq];
                a1 = st[FB / 8 + gq + 8];
            }
            if (ntile == NTILE) {
#pragma unroll
                for (int j = 0; j < NTILE; ++j) mma_f64_16x8x4(acc[j], a0, a1, live ? st[so[j]] : 0.0);
            } else {
#pragma unroll
                for (int j = 0; j < NTILE; ++j)
                    if (j < ntile) mma_f64_16x8x4(acc[j], a0, a1, live ? st[so[j]] : 0.0);
            }
            __syncwarp();                                     // the warp is done with the 4 stages
            if (lane < 4 && u0 + lane < U) mbar_arrive(empty + (u0 + lane) % NS);
        }
        // epilogue: acc[j] = members (gq, gq + 8) x listed nodes abase + 8 j + 2 tig + (0, 1)
        double flux[2] = {0.0, 0.0};
        const int64_t fm0 = gq < nm ? (int64_t)bids[b0 + gq] * Ks : -1;
        const int64_t fm1 = gq + 8 < nm ? (int64_t)bids[b0 + gq + 8] * Ks : -1;
#pragma unroll
        for (int j = 0; j < NTILE; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int a = abase + j * 8 + 2 * tig + e;
                if (a >= nact) continue;
                const int64_t t = act_t[cix * kBndAct + a];
                double v[3];
                // the plan is a superset near v.n = 0; the device decides with the same expression as
                // k_wall_M (incoming = not outgoing)
                if (!node_vel_s<3>(t, ncs, ncol, c0, n1, vmax, dv, v) || !(sgn * v[axis] <= 0.0)) continue;
                const double vn = sgn * v[axis];
                if (fm0 >= 0) {
                    f[fm0 + t] = acc[j][e];
                    if (vn < 0.0) flux[0] += vn * acc[j][e];
                }
                if (fm1 >= 0) {
                    f[fm1 + t] = acc[j][2 + e];
                    if (vn < 0.0) flux[1] += vn * acc[j][2 + e];
                }
            }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            flux[h] += __shfl_xor_sync(0xffffffffu, flux[h], 1);
            flux[h] += __shfl_xor_sync(0xffffffffu, flux[h], 2);
        }
        if (tig == 0) {
            red[wp][gq] = flux[0];
            red[wp][gq + 8] = flux[1];
        }
    }
    __syncthreads();
    if (tid < nm) {
        double tot = 0.0;
#pragma unroll
        for (int k = 0; k < kBndWarps; ++k) tot += red[k][tid];
        wallpart[(int64_t)(b0 + tid) * nch + ch] = tot;
    }
}

__global__ void k_wall_reduce(const int32_t* __restrict__ bids, int64_t nb, const double* __restrict__ wallpart,
                              int nch, double* __restrict__ wallnum) {
    const int64_t bi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (bi >= nb) return;
    double s = 0.0;
    for (int q = 0; q < nch; ++q) s += wallpart[bi * nch + q];
    wallnum[bids[bi]] = s;
}

template <int D>
__global__ void __launch_bounds__(kBndChunk) k_bnd_fill(const int32_t* __restrict__ bids, const int8_t* __restrict__ kind,
                                                        const double* __restrict__ wallnum,
                                                        const double* __restrict__ den, const double* __restrict__ Mw,
                                                        double* __restrict__ f, int n1, int ncol, int ncs, int c0,
                                                        int64_t Kloc, double vmax, double dv) {
    constexpr int NV = (D == 2) ? 2 : 1;
    // block per boundary particle, threads stride over the stored nodes of its row
    const int b = bids[blockIdx.x];
    const int wid = kind[b];
    const int axis = (wid - 1) / 2;
    const double sgn = ((wid - 1) % 2 == 0) ? 1.0 : -1.0;
    const double rho_w = -wallnum[b] / den[wid - 1];
    const double* Mrow = Mw + (int64_t)(wid - 1) * Kloc * NV;
    double* frow = f + (int64_t)b * Kloc * NV;
    // the wall table holds M(1, U_w, T_w) on the wall's outgoing nodes and -1 elsewhere (k_wall_M)
    (void)axis;
    (void)sgn;
    if constexpr (NV == 1) {
        // 16-B pairs of stored nodes (Ks is even in 3D), four in flight per thread; a pair with one
        // outgoing node writes that node alone
        const double2* M2 = reinterpret_cast<const double2*>(Mrow);
        double2* f2 = reinterpret_cast<double2*>(frow);
        const int64_t np = Kloc / 2;
        for (int64_t t0 = threadIdx.x; t0 < np; t0 += 4 * (int64_t)blockDim.x) {
            double2 m[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t t = t0 + u * (int64_t)blockDim.x;
                m[u] = t < np ? __ldg(M2 + t) : make_double2(-1.0, -1.0);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t t = t0 + u * (int64_t)blockDim.x;
                if (m[u].x >= 0.0 && m[u].y >= 0.0) f2[t] = make_double2(rho_w * m[u].x, rho_w * m[u].y);
                else if (m[u].x >= 0.0) frow[2 * t] = rho_w * m[u].x;
                else if (m[u].y >= 0.0) frow[2 * t + 1] = rho_w * m[u].y;
            }
        }
    } else {
        for (int64_t t = threadIdx.x; t < Kloc; t += blockDim.x) {
            const double m0 = Mrow[t * NV];
            if (m0 < 0.0) continue;
#pragma unroll
            for (int q = 0; q < NV; ++q) frow[t * NV + q] = rho_w * Mrow[t * NV + q];
        }
    }
}

// moments of every row (diagnostics, bgk_moments): sums[p] = (s0, s_v, s_E[+g2])
template <int D>
__global__ void __launch_bounds__(256) k_row_moments(const double* __restrict__ f, int64_t N, double* __restrict__ sums,
                                                     int n1, int ncol, int ncs, int c0, int64_t Kloc, double vmax,
                                                     double dv) {
    // Kloc = STORED nodes per row (n1 * ncs)
    constexpr int NV = (D == 2) ? 2 : 1;
    __shared__ double sh[32];
    const int64_t p = blockIdx.x;
    if (p >= N) return;
    double s[kPM] = {0, 0, 0, 0, 0};
    for (int64_t t = threadIdx.x; t < Kloc; t += blockDim.x) {
        double v[3];
        if (!node_vel_s<D>(t, ncs, ncol, c0, n1, vmax, dv, v)) continue;
        const double g = f[(p * Kloc + t) * NV];
        s[0] += g;
#pragma unroll
        for (int a = 0; a < D; ++a) s[1 + a] += v[a] * g;
        double vv = 0.0;
#pragma unroll
        for (int a = 0; a < D; ++a) vv += v[a] * v[a];
        s[1 + D] += vv * g;
        if constexpr (NV == 2) s[1 + D] += f[(p * Kloc + t) * NV + 1];
    }
#pragma unroll
    for (int q = 0; q < kPM; ++q) {
        const double tot = block_sum<256>(s[q], sh);
        if (threadIdx.x == 0) sums[p * kPM + q] = tot;
    }
}

template <int D>
__global__ void k_moments_finalize(const double* __restrict__ sums, int64_t N, double dv, double R,
                                   double* __restrict__ out, int64_t* err) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= N) return;
    const double* s = sums + p * kPM;
    double dvd = dv * dv;
    if (D == 3) dvd *= dv;
    const double rho = s[0] * dvd;
    double uu = 0.0;
    double* o = out + p * (D + 2);
    o[0] = rho;
#pragma unroll
    for (int a = 0; a < D; ++a) {
        const double u = s[1 + a] / s[0];
        o[1 + a] = u;
        uu += u * u;
    }
    const double T = (s[1 + D] * dvd - rho * uu) / (3.0 * rho * R);
    o[1 + D] = T;
    if (!(rho > 0.0) || !(T > 1e-12)) latch_error(err, BGK_E_DEGENERATE_STATE, p);
}

// internal [p][k1][col (stride ncs)][q]  <->  canonical [p][q][k1][col (ncol)]
template <bool TO_CANON>
__global__ void k_transpose(const double* __restrict__ in, double* __restrict__ out, int64_t N, int nv, int n1,
                            int ncol, int ncs) {
    const int64_t Kc = (int64_t)n1 * ncol, total = N * nv * Kc;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = t / (nv * Kc);
        const int64_t r = t - p * nv * Kc;
        const int q = (int)(r / Kc);
        const int64_t k = r - (int64_t)q * Kc;
        const int64_t k1 = k / ncol, col = k - k1 * ncol;
        const int64_t si = ((p * n1 + k1) * ncs + col) * nv + q;
        if (TO_CANON) out[t] = in[si];
        else out[si] = in[t];
    }
}

template <int D>
__global__ void k_check_domain(const double* __restrict__ x, int64_t N, double L, int64_t* err) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
#pragma unroll
    for (int a = 0; a < D; ++a) {
        const double v = x[i * D + a];
        if (!(v >= 0.0 && v <= L)) latch_error(err, BGK_E_OUT_OF_DOMAIN, i);
    }
}

}  // namespace

void launch_moment_reduce(bgk_ctx* c, cudaStream_t s) {
    if (!c->N_int) return;
    k_moment_reduce<<<(unsigned)((c->N_int + 255) / 256), 256, 0, s>>>(c->interior, c->N_int, c->partials, c->nwpp,
                                                                        c->sums);
}

void launch_relax(bgk_ctx* c, double* fnew, cudaStream_t s) {
    if (!c->N_int) return;
    RelaxArgs a;
    a.ids = c->interior;
    a.sums = c->sums;
    a.f = fnew;
    a.macro = c->macro;
    a.W = c->W;
    a.x = c->x;
    a.err = c->err;
    a.n = c->N_int;
    a.n1 = c->n1;
    a.ncol = c->ncol;
    a.ncs = c->ncs;
    a.c0 = c->c0;
    a.Ks = (int)c->Ks;
    a.ale = c->cfg.ale;
    a.vmax = c->cfg.vmax;
    a.dv = c->dv;
    a.dt = c->cfg.dt;
    a.R = c->cfg.R;
    a.kb = c->cfg.kb;
    a.dmol = c->cfg.dmol;
    a.L = c->cfg.L;
    a.clamp_eps = 1e-3 * c->cfg.dx;
    const size_t smem = sizeof(double) * c->ncs;   // column factors of the separable Maxwellian
    if (c->d == 3) k_relax<3><<<(unsigned)c->N_int, 256, smem, s>>>(a);
    else if (c->n1 <= 64) k_relax_w2<<<(unsigned)((c->N_int + 7) / 8), 256, 0, s>>>(a);
    else k_relax<2><<<(unsigned)c->N_int, 256, smem, s>>>(a);
}

template <int G, bool TILE>
void bnd_union_g(bgk_ctx* c, cudaStream_t s) {
    const unsigned ng = TILE ? (unsigned)c->n_bg : (unsigned)((c->N_b + G - 1) / G);
    int n2 = 1;
    while (n2 < G * c->max_nb) n2 <<= 1;
    const size_t smem = sizeof(int32_t) * 2 * n2;
    static bool configured[kMaxDevices] = {};
    if (smem > 48 * 1024 && first_use_on_device(configured))
        cudaFuncSetAttribute(k_bnd_union<G, TILE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    k_bnd_union<G, TILE><<<ng, 256, smem, s>>>(c->boundary, c->N_b, c->bg_off, c->g.nb_off, c->g.bidx, c->g.bcw,
                                              c->g.bcnt, c->bu_cap, c->bu_j, c->bu_w, c->bu_n, c->err);
}

void launch_bnd_union(bgk_ctx* c, cudaStream_t s) {
    if (!c->N_b) return;
    if (c->d == 3) bnd_union_g<kBndTile, true>(c, s);
    else bnd_union_g<4, false>(c, s);
}

template <int D, int G, int NPT, int NS, int MINB = 2>
void bnd_interp_t(bgk_ctx* c, double* fnew, cudaStream_t s) {
    constexpr int CH = 256 * NPT;
    constexpr int NV = D == 2 ? 2 : 1;
    const size_t smem = (size_t)NS * CH * NV * sizeof(double) + 2 * NS * sizeof(uint64_t) +
                        (size_t)c->bu_cap * (G * sizeof(double) + sizeof(int32_t));
    static bool configured[kMaxDevices] = {};
    if (first_use_on_device(configured))
        cudaFuncSetAttribute(k_bnd_interp_t<D, G, NPT, NS, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             200 * 1024);
    const int nch = c->bnd_nch;                              // = ceil(Ks / CH) (api.cu derive)
    dim3 gg((unsigned)((c->N_b + G - 1) / G), (unsigned)nch);
    k_bnd_interp_t<D, G, NPT, NS, MINB><<<gg, 256, smem, s>>>(c->boundary, c->N_b, c->kind, c->bu_j, c->bu_w, c->bu_n,
                                                        c->bu_cap, fnew, c->wallpart, nch, c->n1, c->ncol, c->ncs,
                                                        c->c0, c->Ks, c->cfg.vmax, c->dv);
    k_wall_reduce<<<(unsigned)((c->N_b + 255) / 256), 256, 0, s>>>(c->boundary, c->N_b, c->wallpart, nch,
                                                                    c->wallnum);
}

// 3D: tiles of kBndTile members on the FP64 tensor cores, a 192 KB ring (one block of 12 consumer
// warps + 1 producer warp per SM)
void bnd_interp_s(bgk_ctx* c, double* fnew, cudaStream_t s) {
    const size_t smem = kBndRing + 2 * kBndNSMax * sizeof(uint64_t) + (size_t)c->bu_cap * sizeof(int32_t);
    static bool configured[kMaxDevices] = {};
    if (first_use_on_device(configured))      // opt in once for the largest union capacity (512 rows)
        cudaFuncSetAttribute(k_bnd_interp_s, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(kBndRing + 2 * kBndNSMax * sizeof(uint64_t) + 512 * sizeof(int32_t)));
    const int nch = c->bnd_nch;
    // ring stages at most (BGK_BND_NS, 8 .. 32; C5: 12 stages 2.12 ms, 32 stages 1.61 ms)
    static const int nsmax = [] {
        const char* e = getenv("BGK_BND_NS");
        const int v = e ? atoi(e) : kBndNSMax;
        return v >= 8 && v <= kBndNSMax ? v : kBndNSMax;
    }();
    dim3 gg((unsigned)c->n_bg, (unsigned)nch);
    k_bnd_interp_s<<<gg, (kBndWarps + 1) * 32, smem, s>>>(c->boundary, c->bg_off, c->kind, c->bu_j, c->bu_w,
                                                            c->bu_n, c->bu_cap, c->bnd_chunks, c->bnd_act_t,
                                                            c->bnd_act_s, fnew, c->wallpart, nch, c->n1, c->ncol,
                                                            c->ncs, c->c0, c->Ks, c->cfg.vmax, c->dv, nsmax);
    k_wall_reduce<<<(unsigned)((c->N_b + 255) / 256), 256, 0, s>>>(c->boundary, c->N_b, c->wallpart, nch,
                                                                    c->wallnum);
}

void launch_boundary_interp(bgk_ctx* c, double* fnew, cudaStream_t s) {
    if (!c->N_b) return;
    if (c->d == 3) bnd_interp_s(c, fnew, s);
    else (c->bnd_g == 4 ? bnd_interp_t<2, 4, 2, 6>(c, fnew, s) : bnd_interp_t<2, 8, 2, 6>(c, fnew, s));
}

// The per-wall plan of the tile kernel's velocity chunks.  A node is listed for wall w if it is a
// valid local node whose v.n is <= 0 up to 1e-9 dv (a superset of the device's incoming test, which
// the kernel re-applies).  Listed nodes are taken in stored order; a listed node within kBndGap of
// the current segment's end extends it (the gap is staged, not computed), otherwise it opens a new
// segment; a chunk closes when it holds kBndAct nodes, kBndSeg segments or kBndStage staged nodes.
// Segment starts and lengths are even (16-B bulk copies of fp64 rows whose stride Ks is even).
int bnd_plan(const bgk_ctx* c, std::vector<BndChunk>* chunks, std::vector<int32_t>* act_t,
             std::vector<int32_t>* act_s, int* nchw) {
    const int nw = 2 * c->d;
    const int64_t kA = 16;                      // segment alignment in nodes (128 B: whole L2 lines)
    std::vector<std::vector<BndChunk>> per(nw);
    std::vector<std::vector<int32_t>> pt(nw), ps(nw);
    int mx = 0;
    for (int w = 0; w < nw; ++w) {
        const int axis = w / 2;
        const double sgn = (w % 2 == 0) ? 1.0 : -1.0;
        BndChunk cur{};
        int64_t seg_end = -1;                   // stored end (exclusive, unrounded) of the open segment
        auto close = [&]() {
            if (cur.nact == 0) return;
            const int k = cur.nseg - 1;
            cur.len[k] = (int32_t)std::min<int64_t>(((seg_end - cur.src[k]) + kA - 1) / kA * kA, c->Ks - cur.src[k]);
            cur.slen = cur.dst[k] + cur.len[k];
            per[w].push_back(cur);
            while ((int)pt[w].size() < (int)per[w].size() * kBndAct) {
                pt[w].push_back(0);
                ps[w].push_back(0);
            }
            cur = BndChunk{};
            seg_end = -1;
        };
        for (int64_t t = 0; t < c->Ks; ++t) {
            const int k1 = (int)(t / c->ncs), col = (int)(t - (int64_t)k1 * c->ncs);
            if (col >= c->ncol) continue;
            const int gc = c->c0 + col;
            const int kk[3] = {k1, gc / c->n1, gc - (gc / c->n1) * c->n1};
            const double va = -c->cfg.vmax + (double)kk[axis] * c->dv;
            if (!(sgn * va <= 1e-9 * c->dv)) continue;
            for (int pass = 0; pass < 2; ++pass) {
                const bool extend = cur.nseg > 0 && t - seg_end < kBndGap;
                const int64_t src = extend ? cur.src[cur.nseg - 1] : (t / kA * kA);
                const int64_t dst = extend ? cur.dst[cur.nseg - 1]
                                           : (cur.nseg > 0 ? cur.dst[cur.nseg - 1] +
                                                                 ((seg_end - cur.src[cur.nseg - 1]) + kA - 1) / kA * kA
                                                           : 0);
                const int64_t stage_end = dst + (t + 1 - src) + kA - 1;   // + kA - 1: the round-up
                const bool fits = cur.nact < kBndAct && stage_end <= kBndStage && (extend || cur.nseg < kBndSeg);
                if (!fits) {
                    close();
                    continue;                       // second pass: a fresh chunk always fits
                }
                if (!extend) {
                    if (cur.nseg > 0) cur.len[cur.nseg - 1] = (int32_t)(dst - cur.dst[cur.nseg - 1]);
                    cur.src[cur.nseg] = (int32_t)src;
                    cur.dst[cur.nseg] = (int32_t)dst;
                    ++cur.nseg;
                }
                seg_end = t + 1;
                pt[w].push_back((int32_t)t);
                ps[w].push_back((int32_t)(dst + (t - src)));
                ++cur.nact;
                break;
            }
        }
        close();
        if (nchw) nchw[w] = (int)per[w].size();
        mx = std::max(mx, (int)per[w].size());
    }
    if (chunks) {
        const int nch = std::max(1, mx);
        chunks->assign((size_t)nw * nch, BndChunk{});
        act_t->assign((size_t)nw * nch * kBndAct, 0);
        act_s->assign((size_t)nw * nch * kBndAct, 0);
        for (int w = 0; w < nw; ++w)
            for (size_t k = 0; k < per[w].size(); ++k) {
                (*chunks)[(size_t)w * nch + k] = per[w][k];
                for (int a = 0; a < per[w][k].nact; ++a) {
                    (*act_t)[((size_t)w * nch + k) * kBndAct + a] = pt[w][k * kBndAct + a];
                    (*act_s)[((size_t)w * nch + k) * kBndAct + a] = ps[w][k * kBndAct + a];
                }
            }
    }
    return mx;
}

bgk_status upload_bnd_plan(bgk_ctx* c, cudaStream_t s) {
    if (c->d != 3) return BGK_OK;
    std::vector<BndChunk> ch;
    std::vector<int32_t> at, as;
    bnd_plan(c, &ch, &at, &as, c->bnd_nchw);
    if ((int64_t)ch.size() != (int64_t)2 * c->d * c->bnd_nch) return BGK_E_INVALID_ARG;
    cudaError_t e = cudaMemcpyAsync(c->bnd_chunks, ch.data(), sizeof(BndChunk) * ch.size(), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(c->bnd_act_t, at.data(), sizeof(int32_t) * at.size(), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(c->bnd_act_s, as.data(), sizeof(int32_t) * as.size(), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    return e == cudaSuccess ? BGK_OK : BGK_E_CUDA;
}

void launch_boundary_fill(bgk_ctx* c, double* fnew, cudaStream_t s) {
    if (!c->N_b) return;
    const unsigned g = (unsigned)c->N_b;
    if (c->d == 3)
        k_bnd_fill<3><<<g, kBndChunk, 0, s>>>(c->boundary, c->kind, c->wallnum, c->wall_den, c->Mw, fnew, c->n1,
                                              c->ncol, c->ncs, c->c0, c->Ks, c->cfg.vmax, c->dv);
    else
        k_bnd_fill<2><<<g, kBndChunk, 0, s>>>(c->boundary, c->kind, c->wallnum, c->wall_den, c->Mw, fnew, c->n1,
                                              c->ncol, c->ncs, c->c0, c->Ks, c->cfg.vmax, c->dv);
}

void launch_wall_tables(bgk_ctx* c, cudaStream_t s) {
    const bgk_config& k = c->cfg;
    const int nw = 2 * c->d;
    dim3 g((unsigned)std::min<int64_t>((c->Ks + 255) / 256, 4096), (unsigned)nw);
    if (c->d == 3) {
        k_wall_M<3><<<g, 256, 0, s>>>(c->Mw, c->n1, c->ncol, c->ncs, c->c0, c->Ks, k.vmax, c->dv, k.R, k.T_wall,
                                      k.U_lid[0], k.U_lid[1], k.U_lid[2]);
        k_wall_den<3><<<nw, 256, 0, s>>>(c->wall_den, c->n1, c->ncol_g, k.vmax, c->dv, k.R, k.T_wall, k.U_lid[0],
                                         k.U_lid[1], k.U_lid[2], c->err);
    } else {
        k_wall_M<2><<<g, 256, 0, s>>>(c->Mw, c->n1, c->ncol, c->ncs, c->c0, c->Ks, k.vmax, c->dv, k.R, k.T_wall,
                                      k.U_lid[0], k.U_lid[1], k.U_lid[2]);
        k_wall_den<2><<<nw, 256, 0, s>>>(c->wall_den, c->n1, c->ncol_g, k.vmax, c->dv, k.R, k.T_wall, k.U_lid[0],
                                         k.U_lid[1], k.U_lid[2], c->err);
    }
}

void launch_init_f(bgk_ctx* c, const double* macro0, cudaStream_t s) {
    const bgk_config& k = c->cfg;
    if (c->d == 3)
        k_init_f<3><<<(unsigned)c->N, 256, 0, s>>>(macro0, c->N, c->f[c->fcur], c->macro, c->W, k.ale, c->n1, c->ncol,
                                                   c->ncs, c->c0, c->Ks, k.vmax, c->dv, k.R, k.T_wall);
    else
        k_init_f<2><<<(unsigned)c->N, 256, 0, s>>>(macro0, c->N, c->f[c->fcur], c->macro, c->W, k.ale, c->n1, c->ncol,
                                                   c->ncs, c->c0, c->Ks, k.vmax, c->dv, k.R, k.T_wall);
}

void launch_row_moments(bgk_ctx* c, const double* f, cudaStream_t s) {
    if (c->d == 3)
        k_row_moments<3><<<(unsigned)c->N, 256, 0, s>>>(f, c->N, c->sums, c->n1, c->ncol, c->ncs, c->c0, c->Ks, c->cfg.vmax,
                                                        c->dv);
    else
        k_row_moments<2><<<(unsigned)c->N, 256, 0, s>>>(f, c->N, c->sums, c->n1, c->ncol, c->ncs, c->c0, c->Ks, c->cfg.vmax,
                                                        c->dv);
}

void launch_moments_finalize(bgk_ctx* c, double* out, cudaStream_t s) {
    const unsigned g = (unsigned)((c->N + 255) / 256);
    if (c->d == 3) k_moments_finalize<3><<<g, 256, 0, s>>>(c->sums, c->N, c->dv, c->cfg.R, out, c->err);
    else k_moments_finalize<2><<<g, 256, 0, s>>>(c->sums, c->N, c->dv, c->cfg.R, out, c->err);
}

void launch_to_canonical(bgk_ctx* c, const double* fin, double* fout, cudaStream_t s) {
    if (c->nv == 1 && c->ncs == c->ncol) {
        cudaMemcpyAsync(fout, fin, sizeof(double) * c->N * c->RS, cudaMemcpyDeviceToDevice, s);
        return;
    }
    k_transpose<true><<<4096, 256, 0, s>>>(fin, fout, c->N, c->nv, c->n1, c->ncol, c->ncs);
}

void launch_from_canonical(bgk_ctx* c, const double* fin, double* fout, cudaStream_t s) {
    if (c->nv == 1 && c->ncs == c->ncol) {
        cudaMemcpyAsync(fout, fin, sizeof(double) * c->N * c->RS, cudaMemcpyDeviceToDevice, s);
        return;
    }
    k_transpose<false><<<4096, 256, 0, s>>>(fin, fout, c->N, c->nv, c->n1, c->ncol, c->ncs);
}

void launch_check_domain(bgk_ctx* c, cudaStream_t s) {
    const unsigned g = (unsigned)((c->N + 255) / 256);
    if (c->d == 3) k_check_domain<3><<<g, 256, 0, s>>>(c->x, c->N, c->cfg.L, c->err);
    else k_check_domain<2><<<g, 256, 0, s>>>(c->x, c->N, c->cfg.L, c->err);
}

}  // namespace bgk
