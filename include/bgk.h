/*
 * bgk.h -- C ABI of the B200-native time step of the meshfree ALE scheme for
 * the BGK equation (arXiv 2408.02350, "PAPER.md" below; line numbers P:n).
 *
 * One step covers, for every particle and every discrete velocity
 * (P:163-199 full model, P:202-262 Chu-reduced 2D model):
 *   neighbour search, weighted-least-squares stencil coefficients
 *   (P:290-365), positive upwind transport, moments (P:185-193,
 *   P:226-255), local Maxwellian, implicit relaxation
 *   (P:196-199), ALE motion and diffuse-reflection walls
 *   (construction in DESIGN.md reading Z17).
 *
 * Conventions
 *  - All floating point is IEEE fp64.  Particles are indexed 0..N-1 in the
 *    order the caller passes them.  kind[i] = 0 for interior particles and
 *    1..2*dims for boundary particles on wall id kind[i]
 *    (1: x=0, 2: x=L, 3: y=0, 4: y=L, 5: z=0, 6: z=L; the lid is wall 2*dims).
 *  - Velocity grid: per axis v_j = -vmax + j*dv, j = 0..Nv,
 *    dv = 2 vmax / Nv; node k = ((j1*(Nv+1)) + j2)*(Nv+1) + j3 (last axis
 *    fastest).  A "column" is the set of nodes sharing (j2[, j3]); there are
 *    (Nv+1)^(dims-1) columns, each holding Nv+1 nodes along v_1.  A rank owns
 *    the columns [col_begin, col_end) of the grid (velocity sharding across
 *    GPUs, one process per GPU).
 *  - Canonical distribution layout at the ABI (bgk_get_f / bgk_set_f):
 *    f[N][nval][Nv+1][ncol_local] row-major, nval = 2 (g1, g2) in 2D
 *    and 1 (f) in 3D.  With one rank and all columns this is f[N][nval][K].
 *  - Device memory is owned by the caller (PyTorch allocates it): the library
 *    carves its buffers out of one caller-provided device workspace and never
 *    allocates device memory itself.  The context object is a small host
 *    struct owned by the library (bgk_destroy frees it).
 *  - Pointers documented "host or device" may be either (unified addressing);
 *    the call copies with cudaMemcpyAsync(cudaMemcpyDefault) on the given
 *    stream and synchronises that stream before returning.
 *  - Every call returns a bgk_status and never throws.  Kernel-side failures
 *    (deficient stencil, degenerate state, capacity, out-of-domain) are
 *    latched in a device error word and reported by the next synchronising
 *    call (bgk_sync, bgk_wls_coeffs, bgk_build_neighbors, bgk_moments,
 *    bgk_get_f).  bgk_last_error gives the message and the particle index.
 *  - All work is enqueued on the caller's stream; bgk_step enqueues no host
 *    synchronisation and is CUDA-graph capturable -- unless particle management is on
 *    (cfg.manage = 1), which reads its decision counts back once per ALE step.
 */
#ifndef BGK_B200_H
#define BGK_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bgk_ctx bgk_ctx;
typedef void* bgk_stream; /* a cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream); NULL = legacy default stream */

typedef enum {
    BGK_OK = 0,
    BGK_E_INVALID_ARG = 1,      /* bad configuration or argument */
    BGK_E_CAPACITY = 2,         /* neighbour storage too small (needed count reported) */
    BGK_E_DEFICIENT_STENCIL = 3,/* < dims+2 neighbours or lambda_min < 1e-12 lambda_max */
    BGK_E_DEGENERATE_STATE = 4, /* rho <= 0 or T <= 1e-12 K after moment recovery */
    BGK_E_OUT_OF_DOMAIN = 5,    /* a particle outside [0, L]^dims */
    BGK_E_CUDA = 6,             /* a CUDA runtime error (message in bgk_last_error) */
    BGK_E_WALL = 7              /* diffuse-reflection denominator <= 0 */
} bgk_status;

typedef struct bgk_config {
    int32_t dims;        /* 2 = Chu-reduced 2D model (values g1, g2), 3 = full 3D model */
    int32_t Nv;          /* velocity cells per axis, 2..63: Nv+1 nodes per axis; odd Nv
                          * (no zero node) as in the paper's Figs. 6-7 (Nv = 15) */
    double vmax;         /* velocity bound; <= 0: |U_lid| + 4 sqrt(R T_wall) (Z4) */
    double L;            /* cavity edge [m] */
    double h;            /* neighbour radius [m], h = 3.1 dx */
    double h2;           /* h*h exactly as the caller computed it; neighbour test d2 <= h2 */
    double alpha_w;      /* Gaussian weight exponent, 6 */
    double dt;           /* time step [s] */
    double R;            /* specific gas constant */
    double kb;           /* Boltzmann constant */
    double dmol;         /* molecular diameter [m] */
    double T_wall;       /* wall temperature [K] */
    double U_lid[3];     /* lid velocity [m/s]; other walls at rest */
    double dx;           /* nominal particle spacing [m]; ALE clamp margin = 1e-3 dx */
    int32_t ale;         /* 1: ALE, W = U^n, particles move, geometry rebuilt every step;
                            0: fixed cloud, W = 0, geometry built once and cached */
    int32_t col_begin;   /* first velocity column owned by this rank */
    int32_t col_end;     /* one past the last owned column; col_begin = col_end = 0 means all */
    int32_t max_neighbors; /* per-particle neighbour capacity (0: 96 in 2D, 256 in 3D) */
    int32_t wls_order;   /* Taylor order of the WLS derivative: 0 or 1 = first order (the paper's
                            scheme); 2 = second order, Hessian terms added to the
                            least-squares fit: nu = 5 (2D) / 9 (3D) unknowns, deficient
                            below nu+1 neighbours.  abar may then be negative; the transport applies
                            the flux formula literally, abar (c.n - |c.n|). */
    int32_t manage;      /* particle management (Z28): 1 = a merge/fill pass at
                            the start of every ALE step (bgk_step / bgk_step_transport then
                            synchronise the stream once per step and may change N); 0 = off */
    int32_t m_min;       /* fill threshold: interior particles with fewer neighbours get candidates
                            (<= 0: dims + 3) */
    double r_merge;      /* merge radius [m]: interior pairs closer than this are merged
                            (<= 0: 0.2 dx) */
    int64_t max_particles; /* particle capacity of the workspace (<= 0: N); management inserts
                            stop there (reported) */
    int32_t staging;     /* 1: the workspace also holds an input staging buffer for bgk_stage_f /
                            bgk_use_staged_f (host -> device copies overlapped with steps); 0: none */
} bgk_config;

/* Bytes of device workspace bgk_init_cloud needs for N particles (sized for
 * max(N, cfg->max_particles) particles). */
bgk_status bgk_workspace_size(const bgk_config* cfg, int64_t N, size_t* bytes);

/* Create a context and fill the initial state.
 *   x      : host or device, N*dims fp64 positions (row-major [N][dims]), inside [0, L]^dims;
 *            or NULL (with kind NULL) for the regular cavity lattice of n = L/dx + 1 points per
 *            axis (N must be n^dims): index ix + n iy (+ n^2 iz), coordinates i dx (the last one
 *            exactly L), face points are boundary particles of the lowest wall id they lie on.
 *   kind   : host or device, N int8 (0 interior, 1..2*dims wall id), or NULL with x.
 *   macro0 : host or device, N*(dims+2) fp64 initial (rho, U[dims], T) per particle, or NULL for
 *            the uniform state (rho, U, T) = (1, 0, T_wall).  f^0 = M(rho^0, U^0, T^0) at every
 *            particle; the transport velocity W^0 = U^0 (ALE) or 0 (fixed cloud).
 *   workspace, ws_bytes : caller-owned device memory of at least bgk_workspace_size bytes,
 *            16-byte aligned; it must outlive the context.
 * Errors: BGK_E_INVALID_ARG (dims not 2/3, Nv < 2 or > 63, vmax NaN, N < 1, bad column
 * range, workspace too small, x == NULL with N not a lattice size), BGK_E_OUT_OF_DOMAIN.
 * Synchronises the stream. */
bgk_status bgk_init_cloud(const bgk_config* cfg, const double* x, const int8_t* kind,
                          const double* macro0, int64_t N, void* workspace, size_t ws_bytes,
                          bgk_stream stream, bgk_ctx** out);

/* Cell-linked-list neighbour search on the current positions:
 * N(i) = { j != i : ((x_j-x_i)^2 + (y_j-y_i)^2) + (z_j-z_i)^2 <= h2 }, each operation rounded
 * (no FMA), ascending j.  Also refreshes the context's internal lists.
 * If offsets/idx are non-NULL (device), writes the CSR copy there: offsets[N+1] int64,
 * idx[offsets[N]] int32; cap = capacity of idx.  *needed (host, may be NULL) receives offsets[N].
 * Errors: BGK_E_CAPACITY if offsets[N] > cap or any particle exceeds max_neighbors (such a
 * particle's internal list is left empty, so no later kernel reads past the per-particle
 * capacity; bgk_last_error reports the smallest such particle).
 * Synchronises the stream. */
bgk_status bgk_build_neighbors(bgk_ctx* ctx, int64_t* offsets, int32_t* idx, int64_t cap,
                               int64_t* needed, bgk_stream stream);

/* Batched WLS stencil coefficients on the current neighbour lists:
 * interior particles: S = (M^T W M)^{-1}, a_j = w_j S d_j, frame (n, t[, b]) of each pair,
 * rotated coefficients (abar, bbar[, gbar]) = (a.n, a.t[, a.b]); boundary particles: linear
 * WLS interpolation weights c_bj over interior neighbours (Z19).
 * Errors: BGK_E_DEFICIENT_STENCIL with the first offending particle.  Synchronises. */
bgk_status bgk_wls_coeffs(bgk_ctx* ctx, bgk_stream stream);

/* Copy WLS results out (device or host pointers, NULL to skip):
 *   S[N][dims][dims] (interior rows), rot[nnz][dims] = (abar, bbar[, gbar]),
 *   frames[nnz][dims][dims] = rows n, t[, b], cw[nnz] = boundary weights (0 elsewhere).
 * nnz = offsets[N] of the last neighbour build.  rot/frames are assembled in the idle f buffer,
 * or -- when that is smaller than nnz*(dims+dims^2) doubles (tiny velocity grids) -- in a
 * temporary stream-ordered device allocation freed before return.  Synchronises. */
bgk_status bgk_get_wls(bgk_ctx* ctx, double* S, double* rot, double* frames, double* cw,
                       bgk_stream stream);

/* n_steps time steps n -> n+1 (S:414 order): [ALE: neighbours + WLS on x^n],
 * transport, moment recovery, relaxation, [ALE: move], diffuse reflection.  Single rank
 * only (col range = all columns); multi-rank runs use the split-phase calls below.
 * Asynchronous; errors are latched (see conventions).  From the second step with unchanged
 * counts each step is replayed as one CUDA graph (BGK_GRAPH=0 disables; not while the caller's
 * stream is being captured).  With particle management the graph decides on the device: a pass
 * that changes the cloud skips the rest of that step and of every graph step queued after it,
 * and the next call that reads or changes the state (any call taking the context except
 * bgk_step, bgk_destroy, bgk_last_error, bgk_launches_per_step, bgk_transport_info,
 * bgk_graph_info) synchronises and re-runs the skipped steps, the first one eagerly, so results
 * are those of the eager path. */
bgk_status bgk_step(bgk_ctx* ctx, int n_steps, bgk_stream stream);

/* Split phases of one step, for velocity-sharded runs (one rank per GPU):
 *   bgk_step_transport: [ALE: neighbours + WLS], transport of the local columns, and the
 *        rank-local moment sums written to bgk_buffer(BGK_BUF_MOMENT_SUMS) ([N][5] fp64);
 *   -- caller: all_reduce(SUM) of that buffer across ranks --
 *   bgk_step_relax: moments -> (rho, U, T, tau), relaxation of the local columns, ALE move,
 *        boundary interpolation of the local columns and the rank-local incoming wall flux in
 *        bgk_buffer(BGK_BUF_WALL_FLUX) ([N] fp64);
 *   -- caller: all_reduce(SUM) of that buffer --
 *   bgk_step_boundary: rho_w and the outgoing half of every boundary row.
 * Asynchronous. */
bgk_status bgk_step_transport(bgk_ctx* ctx, bgk_stream stream);
bgk_status bgk_step_relax(bgk_ctx* ctx, bgk_stream stream);
bgk_status bgk_step_boundary(bgk_ctx* ctx, bgk_stream stream);

/* Finer phases of one step, in order, for per-phase timing (the paper's Table 3 breakdown):
 * bgk_step_transport = GEOMETRY + TRANSPORT + MOMENT_SUMS, bgk_step_relax = RELAX +
 * BOUNDARY_INTERP, bgk_step_boundary = BOUNDARY_FILL (which also makes f^{n+1} current).
 * GEOMETRY rebuilds neighbours + WLS only in ALE mode or when the cached geometry is stale.
 * Asynchronous. */
typedef enum {
    BGK_PHASE_GEOMETRY = 0,        /* cell-list neighbour search + WLS coefficients */
    BGK_PHASE_TRANSPORT = 1,       /* positive upwind transport + moment partials */
    BGK_PHASE_MOMENT_SUMS = 2,     /* per-particle reduction of the partials */
    BGK_PHASE_RELAX = 3,           /* moments -> tau -> Maxwellian -> relaxation, ALE move */
    BGK_PHASE_BOUNDARY_INTERP = 4, /* incoming half of boundary rows + wall flux (Z17, Z19) */
    BGK_PHASE_BOUNDARY_FILL = 5    /* outgoing half = rho_w M_w; swap buffers */
} bgk_phase;

bgk_status bgk_run_phase(bgk_ctx* ctx, bgk_phase phase, bgk_stream stream);

typedef enum {
    BGK_BUF_MOMENT_SUMS = 0, /* [N][5] fp64 rank-local sums (sum f, sum v f, sum |v|^2 f (+g2)) */
    BGK_BUF_WALL_FLUX = 1,   /* [N] fp64 rank-local sum_{v.n<0} (v.n) f_b (boundary rows) */
    BGK_BUF_F = 2            /* the current distribution, internal layout f[N][Nv+1][ncs][nval] fp64 where
                                ncs = local column count rounded up to a multiple of 16 in 3D (128-B
                                rows; BGK_NCS_ALIGN = 2, 4, 8 overrides), equal in 2D; read ncs off
                                the buffer size (bytes / (8 N (Nv+1) nval)); padding columns are zero */
} bgk_buffer_id;

/* Device pointer and byte size of an internal buffer (inside the caller's workspace). */
bgk_status bgk_buffer(bgk_ctx* ctx, bgk_buffer_id id, void** ptr, size_t* bytes);

/* Moments of the current distribution at every particle:
 * rho = dv^d sum f, U = dv^d sum v f / rho, 3 rho R T = dv^d sum |v-U|^2 f (+ dv^2 sum g2 in 2D).
 * rho[N], U[N][dims], T[N]: host or device, any may be NULL.  Single rank; for sharded runs use
 * bgk_moments_partial + all_reduce + bgk_moments_finalize.  Synchronises. */
bgk_status bgk_moments(bgk_ctx* ctx, double* rho, double* U, double* T, bgk_stream stream);
bgk_status bgk_moments_partial(bgk_ctx* ctx, bgk_stream stream); /* into BGK_BUF_MOMENT_SUMS */
bgk_status bgk_moments_finalize(bgk_ctx* ctx, double* rho, double* U, double* T, bgk_stream stream);

/* Recovered state (rho, U, T) of the last step at interior particles: macro[N][dims+2].
 * Host or device.  Synchronises. */
bgk_status bgk_get_macro(bgk_ctx* ctx, double* macro, bgk_stream stream);

/* Distribution in the canonical layout (see conventions), host or device.  Synchronises. */
bgk_status bgk_get_f(bgk_ctx* ctx, double* f, bgk_stream stream);
bgk_status bgk_set_f(bgk_ctx* ctx, const double* f, bgk_stream stream);

/* Positions x[N][dims] (host or device).  Synchronises. */
bgk_status bgk_get_positions(bgk_ctx* ctx, double* x, bgk_stream stream);

/* Neighbour lists of the last build: offsets[N+1], idx[nnz] (host or device; NULL idx to read
 * the count only via *nnz).  Synchronises. */
bgk_status bgk_get_neighbors(bgk_ctx* ctx, int64_t* offsets, int32_t* idx, int64_t* nnz,
                             bgk_stream stream);

/* Largest explicit-stable dt on the current geometry and W:
 * 1 / max_{i,k} sum_j |C_ijk| over local columns.  Synchronises. */
bgk_status bgk_stable_dt(bgk_ctx* ctx, double* dt_out, bgk_stream stream);

/* Number of CUDA kernels one bgk_step(ctx, 1) launches (for launch accounting). */
bgk_status bgk_launches_per_step(bgk_ctx* ctx, int64_t* n);

/* Wait for the stream and report any latched device error. */
bgk_status bgk_sync(bgk_ctx* ctx, bgk_stream stream);

/* Message of the last error and the offending particle index (-1 if none). */
const char* bgk_last_error(bgk_ctx* ctx, int64_t* particle);

/* Free the host context (the workspace stays owned by the caller). */
bgk_status bgk_destroy(bgk_ctx* ctx);

/* Library version string. */
const char* bgk_version(void);

/* Overlapped host input (cfg.staging = 1).  bgk_stage_f enqueues the host -> device copy of a
 * canonical-layout f (as bgk_set_f: host or device, N*nval*K_local doubles) into the staging
 * buffer on copy_stream, after the previously staged input has been consumed; it returns
 * without synchronising.  bgk_use_staged_f makes `stream` wait for that copy and converts the
 * staged state into the current f (the state the next bgk_step advances).  A user loop
 *   stage(f_0); for n: { use_staged(); stage(f_{n+1}); step(); read results; }
 * moves step n+1's input while step n computes.  Size contract: bgk_stage_f copies
 * N*nval*K_local doubles for the N current when it is called (the caller's buffer must hold that
 * many) and records N and the cloud generation; bgk_use_staged_f refuses (BGK_E_INVALID_ARG,
 * nothing converted, the staged input dropped) if particle management changed N or renumbered the
 * rows in between -- stage again for the new cloud.  Errors: BGK_E_INVALID_ARG (no staging buffer,
 * nothing staged, stale staged input), BGK_E_CUDA. */
bgk_status bgk_stage_f(bgk_ctx* ctx, const double* f, bgk_stream copy_stream);
bgk_status bgk_use_staged_f(bgk_ctx* ctx, bgk_stream stream);

/* Particle management pass ("Adding and removing points"; SPEC.md:316-358;
 * DESIGN.md reading Z28) on the current state, with the thresholds of the configuration:
 *  1. merge: interior pairs closer than r_merge (greedy, ascending index) become ONE particle at
 *     the midpoint (slot of the smaller index), its f row, transport velocity W and macro state
 *     interpolated (linear WLS with a constant term, the boundary-interpolation construction of
 *     Z19) from every other particle within h of the midpoint;
 *  2. fill: interior particles with fewer than m_min neighbours propose x +- 0.5 h e_a, and wall
 *     particles whose interpolation stencil has fewer than dims + 2 interior members propose
 *     x + 0.5 h (sum of their inward wall normals) and x + 0.5 h n_a per wall (Z30);
 *     proposals inside the open box and farther than 0.45 dx from every particle are inserted
 *     (appended), interpolated the same way;
 *  3. the surviving particles keep their relative order, inserted ones follow.
 * Deficient interpolation stencils keep the pair / skip the proposal; inserts stop at the
 * capacity.  One pass creates at most 4096 new particles (merged + inserted): pairs past that
 * are kept (counted with the deficient ones) and proposals past it are counted as capacity
 * skips; the next pass takes them up (the oracle has no such limit).  report (host, may be NULL) receives int64[6] = {merges, merges kept (deficient),
 * inserts, inserts skipped (deficient), inserts skipped (capacity), N after the pass}.
 * Runs on the caller's stream and synchronises it; invalidates cached geometry; the next
 * bgk_step rebuilds it.  Particle indices change when anything was merged or inserted:
 * re-query bgk_count and re-read arrays.  Errors: BGK_E_CUDA. */
bgk_status bgk_manage(bgk_ctx* ctx, int64_t* report, bgk_stream stream);

/* Current particle counts (they change only through particle management): N, interior,
 * boundary (host pointers, each may be NULL), and the capacity. */
bgk_status bgk_count(bgk_ctx* ctx, int64_t* N, int64_t* n_interior, int64_t* n_boundary, int64_t* capacity);

/* Transport mapping in use (diagnostics; info holds 5 values): info[0] particles per warp, info[1]
 * rows per lane R of the general kernel, info[2] fixed-cloud lattice-row groups (8 particles each,
 * 0 if the lattice-row kernel is not used), info[3] interior particles left to the general kernel,
 * info[4] fixed-cloud deep-interior tiles (8 x 8 x 8 particles each, tiles.cu). */
bgk_status bgk_transport_info(bgk_ctx* ctx, int64_t* info);

/* Whole-step graph use (diagnostics, host int64[4]): info[0] 1 if graphs are enabled and usable,
 * info[1] steps launched as graphs, info[2] graph captures, info[3] steps re-run after a
 * management change skipped them. */
bgk_status bgk_graph_info(bgk_ctx* ctx, int64_t* info);

/* Kinds of the current particles (host or device int8[N]); synchronises. */
bgk_status bgk_get_kind(bgk_ctx* ctx, int8_t* kind, bgk_stream stream);

/* Report of the last management pass (int64[6] as bgk_manage), zeros if none ran. */
bgk_status bgk_manage_report(bgk_ctx* ctx, int64_t* report);

#ifdef __cplusplus
}
#endif
#endif /* BGK_B200_H */
