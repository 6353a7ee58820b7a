// bgk_internal.cuh -- internal state and device helpers of the B200 BGK step.
//
// Internal distribution layout:
//   f[p][k1][col][q], p = particle, k1 = 0..n1-1 index along v_1 (n1 = Nv+1),
//   col = local velocity column (nodes sharing (j2[, j3])), q = value (g1, g2 in
//   2D; f in 3D).  A warp's 32 lanes own 32 consecutive (chunk, column) slots
//   of one particle and walk k1 sequentially, so every load of a neighbour row
//   at fixed k1 is one coalesced 256-B (3D) / 512-B (2D) transaction.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "../../include/bgk.h"

namespace bgk {

constexpr int kPM = 5;          // moment partials per particle: s0, s_v (d), s_E  (2D: s0, s1, s2, sE, 0)
constexpr int kMaxCellsPerAxis = 4096;

struct Geo {                    // per-step geometry arrays (device)
    int32_t* cell_of;           // [N]
    int32_t* cell_cnt;          // [ncell]
    int32_t* cell_start;        // [ncell+1]
    int32_t* cell_fill;         // [ncell]
    int32_t* cell_pts;          // [N] particles grouped by cell, ascending inside a cell
    int32_t* nb_cnt;            // [N]
    int64_t* nb_off;            // [N+1]
    int32_t* nb_idx;            // [cap]
    double* S;                  // [N][d*d]
    double* P;                  // [cap][PD] pair data p_n, p_t[, p_b] = abar n, bbar t[, gbar b]
    double* cw;                 // [cap] boundary interpolation weights (aligned with the CSR)
    int32_t* bidx;              // [cap] per boundary particle: its interior neighbours, compacted at the row start
    double* bcw;                // [cap]   and their weights
    int32_t* bcnt;              // [N]     count
    int32_t* order;             // [N_int] interior particles in cell order (transport processing order)
};

// particle management (manage.cu, Z28)
constexpr int kManageMaxNew = 4096;   // new particles (merges + inserts) per pass
#ifndef BGK_ROWS_R
#define BGK_ROWS_R 5
#endif
constexpr int kRowsG = 8;            // particles per lattice-row group (fixed-cloud transport)
constexpr int kRowsR = BGK_ROWS_R;   // velocity nodes per lane along v_1 in the lattice-row kernel
constexpr int kFoldR = 13;           // rows per lane of a folded column group (2 kFoldR >= n1)

// 3D boundary interpolation over face tiles (relax.cu k_bnd_interp_s): a block stages one union row's
// incoming nodes of a velocity chunk -- up to kBndSeg contiguous bulk-copy segments, at most
// kBndStage stored nodes -- and applies it to up to kBndTile members; the chunk's incoming nodes
// (at most kBndAct = 12 consumer warps x 64) are listed per wall by the host (bnd_plan)
constexpr int kBndTile = 16;         // members per tile group (4 x 4 face-lattice points)
constexpr int kBndSeg = 4;
constexpr int kBndStage = 2048;
constexpr int kBndAct = 768;
constexpr int kBndGap = 64;          // an inactive run shorter than this stays inside a segment
struct BndChunk {
    int32_t nseg, slen, nact, pad;   // segments, staged nodes, listed nodes
    int32_t src[kBndSeg], dst[kBndSeg], len[kBndSeg];   // stored node -> stage offset, node count (even)
};
struct Manage {
    uint8_t* flag;      // [Ncap] bit0: merge candidate (a j > i closer than r_merge), bit1: < m_min neighbours
    int32_t* status;    // [Ncap] 0 live, -1 removed (merged into its partner), q+1: slot holds merged particle q
    int32_t* map;       // [Ncap] new index t -> old index (>= 0) or -(q+1) for new particle q
    double* x;          // [Ncap][d]   gathered arrays (copied back after the pass)
    double* W;          // [Ncap][d]
    double* macro;      // [Ncap][d+2]
    int8_t* kind;       // [Ncap]
    double* pos;        // [kManageMaxNew][d] new particles: position
    double* nW;         // [kManageMaxNew][d]            interpolated transport velocity
    double* nM;         // [kManageMaxNew][d+2]          interpolated macro state
    int32_t* dst;       // [kManageMaxNew]               final index
    int32_t* sm;        // [kManageMaxNew]               stencil size
    int32_t* sidx;      // [kManageMaxNew][max_nb]       stencil (old indices)
    double* sc;         // [kManageMaxNew][max_nb]       interpolation weights
    int64_t* rep;       // [8] merges, kept, inserts, deficient, capacity, N_out, n_new, changed
    int32_t* counts;    // [4] flagged particles
};

}  // namespace bgk

struct bgk_ctx {
    bgk_config cfg;
    int d, nv, n1, ncol_g, c0, c1, ncol;
    int ncs;                           // stored column stride: ncol rounded up to a multiple of 16 in 3D (128-B rows)
    int64_t N, N_int, N_b, Kloc, Ks, RS;   // Kloc = n1*ncol logical nodes, Ks = n1*ncs stored, RS = Ks*nv doubles
    int64_t Ncap;                      // particle capacity of the workspace (>= N; management inserts)
    int ncg;                           // 32-column groups per chunk (transport)
    int xc;                            // 2D, 33 columns: column 32 rides in the group's box (k_transport XC)
    int fuse2;                         // 2D XC, single rank: bgk_step runs transport + relaxation fused
    CUtensorMap tmap[2];               // TMA descriptors of f[0], f[1] viewed as [N][n1][ncs*nv] fp64
    CUtensorMap tmap_rows[2];          //   the same with the lattice-row kernel's box {32, kRowsR, 1}
    CUtensorMap tmap_fold[2];          //   the folded last group's box {16, 2 kFoldR, 1} (fold)
    int fold;                          // 3D: the last column group (<= 16 columns) runs folded (FD = 1)
    int max_nb;
    int64_t cap;
    int nc[3];
    int ncell;
    double edge[3];
    double dv, vmin;
    int PD;                     // doubles of pair data per CSR entry
    int wls_order;              // 1 or 2 (second order adds the signed tail to the pair record)
    int R, nchunk, nslots, nwpp; // transport mapping
    int bnd_chunk, bnd_nch;     // boundary node chunking (3D: chunks per wall of the tile kernel, max)
    bool geometry_valid;
    int fcur;
    // device buffers (carved from the caller's workspace)
    double* x;          // [N][d]
    int8_t* kind;       // [N]
    int32_t* interior;  // [N_int] static list of interior particles
    int32_t* boundary;  // [N_b] static list of boundary particles
    double* W;          // [N][d] transport velocity of the next step
    double* macro;      // [N][d+2] recovered (rho, U, T)
    double* f[2];       // [N][RS] double buffer
    double* partials;   // [N][nwpp][kPM]
    double* sums;       // [N][kPM] rank-local (then all-reduced) moment sums
    double* wallpart;   // [N_b][bnd_nch]
    double* wallnum;    // [N] rank-local (then all-reduced) incoming wall flux
    double* Mw;         // [2d][RS] wall Maxwellians M(1, U_w, T_w) on the outgoing nodes of each wall, -1 elsewhere
    double* wall_den;   // [2d] sum_{v.n>0} (v.n) M_w over the GLOBAL grid
    double* outbuf;     // [N][d+2] scratch for moments / copies
    int64_t* err;       // [4] packed (code << 56 | particle) word (latch_error), spare
    unsigned long long* stab;  // [1] max_{i,k} sum_j |C_ijk| as ordered bits
    bgk::Manage mg;     // particle-management scratch (cfg.manage)
    double* stage;      // [Ncap][nv*Kloc] canonical input staging buffer (cfg.staging)
    // grouped boundary interpolation (relax.cu): union of a group's interior neighbours and the dense
    // weight matrix, rebuilt with the geometry.  2D: bnd_g = 4 consecutive boundary particles of the
    // (wall, y, x) order.  3D: face tiles of up to kBndTile members of one wall (install_lists), member
    // range bg_off[g] .. bg_off[g+1] of the boundary list
    int bnd_g;          // members per group (2D 4; 3D kBndTile)
    int bu_cap;
    int64_t bg_max;     // group capacity of the carved arrays
    int64_t n_bg;       // groups (3D tiles)
    int32_t* bg_off;    // [bg_max + 1] 3D: group g = boundary list positions bg_off[g] .. bg_off[g+1]-1
    int32_t* bu_j;      // [groups][bu_cap]
    double* bu_w;       // [groups][bu_cap][bnd_g]
    int32_t* bu_n;      // [groups]
    int bnd_nchw[6];    // 3D: chunks of each wall (bnd_plan)
    bgk::BndChunk* bnd_chunks;   // [2d][bnd_nch]
    int32_t* bnd_act_t;          // [2d][bnd_nch][kBndAct] listed node: stored index
    int32_t* bnd_act_s;          //                         and its stage offset
    cudaEvent_t ev_staged, ev_consumed;
    bool stage_pending;
    int64_t stage_N;        // N when the staged copy was enqueued
    uint64_t stage_gen;     //   and the cloud generation (bgk_use_staged_f refuses a changed cloud)
    uint64_t cloud_gen;     // incremented whenever particle management changes N or the row numbering
    int64_t mg_report[6];   // host copy of the last pass's report
    // fixed-cloud lattice rows (transport_rows.cu): groups of kRowsG consecutive particles along x
    // with identical neighbour offsets share the pair coefficients and every neighbour box
    bool rows_on;       // possible for this configuration (fixed cloud, 3D, first order, one particle per warp)
    bool rows_built;    // groups detected for the cached geometry
    int64_t n_rows;     // groups
    int64_t n_rest;     // interior particles left to the general kernel
    int32_t* rows_p0;   // [Ncap / kRowsG] first particle of each group
    int32_t* rows_stride;   // [Ncap / kRowsG] index step between the group's particles (x, y or z line)
    int16_t* rows_perm;     // [Ncap / kRowsG][256] p0's neighbour entries in run order
    int32_t* order_rest;// [Ncap] the rest, in cell order
    // fixed cloud, deep lattice interior as a 3D stencil (tiles.cu): 8 x 8 x 8 tiles of particles whose
    // stencil is the 122-offset ball; C'_delta(k) tabulated once per cached geometry
    int n_tiles;        // tiles in use (0: none)
    int tile_nlat;      // lattice points per axis (particle = ix + n iy + n^2 iz)
    int32_t* tile_org;  // [Ncap / 512 + 1][3] lattice index of each tile's first particle
    double* ctab;       // [123][Ks] C'_delta(k) of the 122 offsets, then S(k)
    CUtensorMap tmap_halo[2];   // f[b] as {Ks, n, n, n}, box {4, 15, 14, 14}
    CUtensorMap tmap_ctab;      // ctab as {Ks, 123}, box {4, 123}
    int rows_nchunk;    // velocity chunks of kRowsR nodes along v_1
    // whole-step CUDA graphs (graph.cu): one executable per buffer parity, rebuilt when the key changes
    bool graph_ok;                 // graphs usable (BGK_GRAPH != 0, conditional nodes available)
    int eager_steps;               // steps run eagerly since the last key change (capture after one)
    cudaStream_t cap_stream, cap_stream2, cap_stream3;   // private capture streams (step, bodies, fork)
    cudaEvent_t cap_fork, cap_join;    // fork / join of the boundary half of the WLS inside a capture
    cudaStream_t gstream;          // stream of the last graph launch (reconcile of stream-less calls)
    uint64_t eager_key;            // key of the last eager step
    int force_eager;               // steps that must run eagerly (a management change to apply)
    cudaGraphExec_t gexec[2];
    uint64_t gkey[2];
    int64_t* gflag;                // [4] device: [0] a management change skipped the rest, [1] bodies run,
                                   // [2] bodies in total, [3] test hook fired (graph.cu)
    int64_t gsteps;                // graph steps enqueued since the last reconcile (managed mode)
    int gfcur0;                    // fcur before the first of them
    int64_t gstat[3];              // graph launches, captures, re-run steps (bgk_graph_info)
    int64_t* scan_tmp;  // [1024]
    int32_t* blk_tmp;   // [1024] per-block partial counts of the multi-block scans
    bgk::Geo g;
    // host-side error state
    char msg[256];
    int64_t bad;
    int64_t nnz_last;
};

namespace bgk {

// ------------------------------------------------------------ device helpers
__device__ __forceinline__ double axis_node(double vmax, double dv, int j) {
    return -vmax + (double)j * dv;
}

// squared distance with every operation rounded, no contraction (Z22)
template <int D>
__device__ __forceinline__ double dist2_rn(const double* xi, const double* xj) {
    double s = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
        double t = __dsub_rn(xj[a], xi[a]);
        s = __dadd_rn(s, __dmul_rn(t, t));
    }
    return s;
}

// The device error word err[0]: error code in the top byte, offending particle in the low 56 bits
// (kErrNoParticle: none).  The first code latched wins; later errors of the same code lower the
// particle to the smallest index (deterministic), so code and particle always belong together.
constexpr unsigned long long kErrNoParticle = 0x00FFFFFFFFFFFFFFull;

__device__ __forceinline__ void latch_error(int64_t* err, int code, int64_t particle) {
    unsigned long long* e = reinterpret_cast<unsigned long long*>(err);
    const unsigned long long pk = particle >= 0 ? (unsigned long long)particle & kErrNoParticle : kErrNoParticle;
    const unsigned long long want = ((unsigned long long)code << 56) | pk;
    unsigned long long old = atomicCAS(e, 0ull, want);
    while (old != 0ull && (old >> 56) == (unsigned long long)code && (old & kErrNoParticle) > pk) {
        const unsigned long long prev = atomicCAS(e, old, want);
        if (prev == old) break;
        old = prev;
    }
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Kernel attributes (cudaFuncSetAttribute: the dynamic shared-memory opt-in) are per device: a
// launcher keeps one flag per device and sets the attribute the first time it runs on each.
constexpr int kMaxDevices = 64;
inline bool first_use_on_device(bool (&done)[kMaxDevices]) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return true;
    if (done[dev]) return false;
    done[dev] = true;
    return true;
}

// ---------------------------------------------------------------- launchers
void launch_build_neighbors(bgk_ctx* c, cudaStream_t s);
void launch_wls(bgk_ctx* c, cudaStream_t s);
void launch_wls_export(bgk_ctx* c, double* rot, double* frames, cudaStream_t s);
void launch_wls_interior(bgk_ctx* c, cudaStream_t s);
void launch_wls_boundary(bgk_ctx* c, cudaStream_t s);
void launch_transport(bgk_ctx* c, const double* fin, double* fout, cudaStream_t s);
// 2D, 33 columns, single rank (c->fuse2): transport + moments + relaxation in one kernel
void launch_transport_fused(bgk_ctx* c, const double* fin, double* fout, cudaStream_t s);
void launch_moment_reduce(bgk_ctx* c, cudaStream_t s);
void launch_relax(bgk_ctx* c, double* fnew, cudaStream_t s);
void launch_boundary_interp(bgk_ctx* c, double* fnew, cudaStream_t s);
void launch_bnd_union(bgk_ctx* c, cudaStream_t s);
void launch_boundary_fill(bgk_ctx* c, double* fnew, cudaStream_t s);
void launch_wall_tables(bgk_ctx* c, cudaStream_t s);
void launch_init_f(bgk_ctx* c, const double* macro0, cudaStream_t s);
void launch_row_moments(bgk_ctx* c, const double* f, cudaStream_t s);
void launch_moments_finalize(bgk_ctx* c, double* out, cudaStream_t s);
void launch_to_canonical(bgk_ctx* c, const double* fin, double* fout, cudaStream_t s);
void launch_from_canonical(bgk_ctx* c, const double* fin, double* fout, cudaStream_t s);
void launch_check_domain(bgk_ctx* c, cudaStream_t s);
int transport_rows_per_thread(int d, int n1);

bool make_tensor_maps(bgk_ctx* c);
// 3D boundary tiles: the per-wall chunk plan of the incoming velocity nodes (host; returns the largest
// chunk count, fills the tables when the vectors are given) and its upload
int bnd_plan(const bgk_ctx* c, std::vector<BndChunk>* chunks, std::vector<int32_t>* act_t,
             std::vector<int32_t>* act_s, int* nchw);
bgk_status upload_bnd_plan(bgk_ctx* c, cudaStream_t s);
// fixed-cloud lattice rows: host-side group detection on the cached geometry, and the kernel
bgk_status build_rows(bgk_ctx* c, cudaStream_t s);
void launch_transport_rows(bgk_ctx* c, const double* fin, double* fout, cudaStream_t s);
// tiles.cu: the deep-interior stencil of a fixed lattice cloud
bool tile_ball_order(const int64_t* offsets_dxdydz, int m);
bool make_tile_maps(bgk_ctx* c);
void launch_tile_ctab(bgk_ctx* c, int64_t off_ref, cudaStream_t s);
void launch_transport_tile(bgk_ctx* c, const double* fin, double* fout, cudaStream_t s);
int tile_particles();
int tile_ranges(const bgk_ctx* c);
// storage index of local node t = k1*ncol + col  ->  k1*ncs + col
__host__ __device__ __forceinline__ int64_t stored_node(int64_t t, int ncol, int ncs) {
    const int64_t k1 = t / ncol;
    return k1 * ncs + (t - k1 * ncol);
}
int launches_neighbors(const bgk_ctx* c);
int launches_wls();
// particle management: one pass (synchronises the stream); *changed = N or indices changed.
// manage_decide enqueues detect + decide only (device report mg.rep, rep[7] = changed);
// manage_apply reads the report back and applies a change.
bgk_status manage_pass(bgk_ctx* c, cudaStream_t s, bool* changed);
void manage_decide(bgk_ctx* c, cudaStream_t s);
bgk_status manage_apply(bgk_ctx* c, cudaStream_t s, bool* changed);
// whole-step CUDA graphs (graph.cu): graph_step enqueues one step as a graph launch (false: not
// possible now -- run the step eagerly); graph_reconcile settles steps a management change skipped;
// graph_release frees the graphs
bool graph_step(bgk_ctx* c, cudaStream_t s);
bgk_status graph_reconcile(bgk_ctx* c, cudaStream_t s);
void graph_release(bgk_ctx* c);
void launch_step_eager_body(bgk_ctx* c, cudaStream_t s);
// kinds/positions on the host -> interior / boundary / order lists, counts, TMA maps
bgk_status install_lists(bgk_ctx* c, const int8_t* hk, const double* hx, cudaStream_t s);

}  // namespace bgk
