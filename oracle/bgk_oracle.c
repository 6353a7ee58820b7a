/*
 * bgk_oracle.c -- CPU ORACLE for one time step of the meshfree ALE BGK scheme
 * of arXiv 2408.02350 (PAPER.md in the reference mount).
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path may load, link or
 * call this file.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs use it.  It shares no code, header,
 * table or constant generator with the CUDA path (paper_2408_02350_b200/).
 *
 * Plain, slow, obviously correct fp64 loops, in the paper's order and
 * notation.  Compiled with -O2 -ffp-contract=off (no FMA contraction), so
 * every expression is evaluated as written with round-to-nearest.  OpenMP
 * (optional) only parallelises the outer loop over particles; every
 * per-particle sum runs in fixed ascending order, so results do not depend on
 * the thread count.
 *
 * Citations "P:n" are PAPER.md line numbers; "Zn" are the readings of the
 * garbled/silent passages listed in SURVEY.md §8(c) and DESIGN.md.
 *
 * Conventions
 *   d      = dims (2: Chu-reduced, 3: full); nval = 2 (g1, g2) in 2D, 1 in 3D.
 *   nodes  : per axis v_j = -vmax + j*dv, j = 0..Nv, dv = 2 vmax/Nv
 *            (P:266-269 with the paper's j-1 written as j), K = (Nv+1)^d,
 *            flattened k = ((j1*(Nv+1)) + j2)*(Nv+1) + j3, last axis fastest.
 *   f row  : nval*K doubles, [g1(0..K-1) | g2(0..K-1)] in 2D, f(0..K-1) in 3D.
 *   kind   : 0 interior, 1..2d wall id (1: x=0, 2: x=L, 3: y=0, 4: y=L,
 *            5: z=0, 6: z=L); the lid is wall 2d.
 *
 * Every function that has no independent pin says so; see DESIGN.md
 * "Oracle pins" for the list (all functions below are pinned).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_E_INVALID 1
#define OR_E_CAPACITY 2
#define OR_E_DEFICIENT 3
#define OR_E_DEGENERATE 4
#define OR_E_WALL 5

typedef struct {
    int32_t dims;     /* 2 or 3 */
    int32_t Nv;       /* velocity cells per axis: Nv+1 nodes per axis (Z3) */
    double vmax;      /* Z4 */
    double L;         /* cavity edge */
    double h;         /* neighbour radius h = 3.1 dx */
    double h2;        /* h*h, computed once by the harness (Z11, Z22) */
    double alpha_w;   /* Gaussian weight constant, 6 */
    double dt;        /* time step */
    double R, kb, dmol; /* gas constant, Boltzmann constant, molecular diameter */
    double Twall;     /* wall temperature T0 */
    double Ulid[3];   /* lid velocity */
    double dx;        /* nominal spacing, for the ALE clamp */
    int32_t ale;      /* 1: ALE (W = U^n, particles move), 0: fixed cloud (W = 0, Z21) */
    int32_t wls_order;/* 1 (or 0): first-order Taylor WLS; 2: second order */
} or_cfg;

/* ------------------------------------------------------------------ O1 --- */
/* Velocity grid: dv = 2 vmax / Nv, v_j = -vmax + (j-1) dv, j=1..Nv+1. */
double or_dv(const or_cfg* c) { return 2.0 * c->vmax / (double)c->Nv; }

double or_axis_node(const or_cfg* c, int j) { return -c->vmax + (double)j * or_dv(c); }

int64_t or_num_nodes(const or_cfg* c) {
    int64_t n = c->Nv + 1, K = 1;
    for (int a = 0; a < c->dims; ++a) K *= n;
    return K;
}

/* velocity vector of flattened node k (last axis fastest) */
void or_node_velocity(const or_cfg* c, int64_t k, double* v) {
    int n = c->Nv + 1;
    for (int a = c->dims - 1; a >= 0; --a) {
        v[a] = or_axis_node(c, (int)(k % n));
        k /= n;
    }
}

static int nval_of(const or_cfg* c) { return c->dims == 2 ? 2 : 1; }

/* ------------------------------------------------------------------ O2 --- */
/* Squared distance ((x_j-x_i)^2 + (y_j-y_i)^2) + (z_j-z_i)^2, each op rounded
 * (Z22).  Neighbour set N(i) = { j != i : d2 <= h^2 }, ascending j
 * ("inside the disc of radius h", closed ball per the weight
 * support "<= 1" of P:299, Z11). */
static double dist2(int d, const double* xi, const double* xj) {
    double s = 0.0;
    for (int a = 0; a < d; ++a) {
        double t = xj[a] - xi[a];
        s = s + t * t;
    }
    return s;
}

/* Neighbours of one particle by brute force over all N (O(N)). Returns count,
 * writes up to cap indices. */
int64_t or_neighbors_of(int d, const double* x, int64_t N, double h2, int64_t i,
                        int32_t* out, int64_t cap) {
    int64_t m = 0;
    for (int64_t j = 0; j < N; ++j) {
        if (j == i) continue;
        if (dist2(d, x + i * d, x + j * d) <= h2) {
            if (m < cap) out[m] = (int32_t)j;
            ++m;
        }
    }
    return m;
}

/* CSR neighbour lists for all particles, O(N^2). offsets[N+1]; returns OR_OK or
 * OR_E_CAPACITY with *needed = total entries. */
int or_neighbors(int d, const double* x, int64_t N, double h2, int64_t* offsets,
                 int32_t* idx, int64_t cap, int64_t* needed) {
    int64_t* cnt = (int64_t*)malloc(sizeof(int64_t) * (size_t)(N > 0 ? N : 1));
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t i = 0; i < N; ++i) cnt[i] = or_neighbors_of(d, x, N, h2, i, NULL, 0);
    offsets[0] = 0;
    for (int64_t i = 0; i < N; ++i) offsets[i + 1] = offsets[i] + cnt[i];
    free(cnt);
    *needed = offsets[N];
    if (offsets[N] > cap) return OR_E_CAPACITY;
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t i = 0; i < N; ++i)
        or_neighbors_of(d, x, N, h2, i, idx + offsets[i], offsets[i + 1] - offsets[i]);
    return OR_OK;
}

/* ------------------------------------------------------------ linear algebra */
/* Gauss-Jordan inverse with partial pivoting of an n x n matrix (n <= 9).
 * Returns 0 on success, 1 if a pivot is exactly zero. */
static int inverse(int n, const double* A, double* Ainv) {
    double M[9][18];
    for (int r = 0; r < n; ++r)
        for (int c = 0; c < 2 * n; ++c)
            M[r][c] = c < n ? A[r * n + c] : (c - n == r ? 1.0 : 0.0);
    for (int col = 0; col < n; ++col) {
        int piv = col;
        for (int r = col + 1; r < n; ++r)
            if (fabs(M[r][col]) > fabs(M[piv][col])) piv = r;
        if (M[piv][col] == 0.0) return 1;
        if (piv != col)
            for (int c = 0; c < 2 * n; ++c) {
                double t = M[col][c]; M[col][c] = M[piv][c]; M[piv][c] = t;
            }
        double p = M[col][col];
        for (int c = 0; c < 2 * n; ++c) M[col][c] = M[col][c] / p;
        for (int r = 0; r < n; ++r) {
            if (r == col) continue;
            double fct = M[r][col];
            for (int c = 0; c < 2 * n; ++c) M[r][c] = M[r][c] - fct * M[col][c];
        }
    }
    for (int r = 0; r < n; ++r)
        for (int c = 0; c < n; ++c) Ainv[r * n + c] = M[r][n + c];
    return 0;
}

/* Eigenvalues of a symmetric n x n matrix by cyclic Jacobi rotations. */
void or_sym_eigenvalues(int n, const double* A, double* lam) {
    double a[9][9];
    for (int r = 0; r < n; ++r)
        for (int c = 0; c < n; ++c) a[r][c] = A[r * n + c];
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0, diag = 0.0;
        for (int r = 0; r < n; ++r)
            for (int c = 0; c < n; ++c) {
                if (r != c) off += a[r][c] * a[r][c];
                else diag += a[r][c] * a[r][c];
            }
        if (off <= 1e-60 * diag) break;
        for (int p = 0; p < n; ++p)
            for (int q = p + 1; q < n; ++q) {
                if (a[p][q] == 0.0) continue;
                double theta = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
                double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                double cs = 1.0 / sqrt(t * t + 1.0), sn = t * cs;
                for (int k = 0; k < n; ++k) { /* rotate columns p,q */
                    double akp = a[k][p], akq = a[k][q];
                    a[k][p] = cs * akp - sn * akq;
                    a[k][q] = sn * akp + cs * akq;
                }
                for (int k = 0; k < n; ++k) { /* rotate rows p,q */
                    double apk = a[p][k], aqk = a[q][k];
                    a[p][k] = cs * apk - sn * aqk;
                    a[q][k] = sn * apk + cs * aqk;
                }
            }
    }
    for (int r = 0; r < n; ++r) lam[r] = a[r][r];
}

/* Deficiency test of S:253/S:303: m < d+2, or lambda_min < 1e-12 lambda_max. */
static int deficient(int n_unknown_dim, int m, int n, const double* A) {
    if (m < n_unknown_dim + 2) return 1;
    double lam[9];
    or_sym_eigenvalues(n, A, lam);
    double lo = lam[0], hi = lam[0];
    for (int r = 1; r < n; ++r) {
        if (lam[r] < lo) lo = lam[r];
        if (lam[r] > hi) hi = lam[r];
    }
    return !(hi > 0.0) || lo < 1e-12 * hi;
}

/* ------------------------------------------------------------------ O3 --- */
/* Truncated Gaussian weight: w = exp(-alpha |x_j - x_i|^2 / h^2)
 * if |x_j - x_i| / h <= 1, else 0. */
double or_weight(double r2, double h2, double alpha) {
    if (r2 <= h2) return exp(-alpha * r2 / h2);
    return 0.0;
}

/* WLS derivative coefficients for one particle.
 * M rows d_j = x_j - x_i, W = diag(w_j); S = (M^T W M)^{-1};
 * (alpha_ij, beta_ij, gamma_ij) = w_j S d_j.
 * Outputs: S[d*d], a[m*d]. Returns OR_OK or OR_E_DEFICIENT. */
/* Second-order Taylor WLS ("higher-order approximations are obtained by using
 * higher-order Taylor's expansion in (taylor)"): per neighbour
 *   f_j - f_i = g . d_j + 1/2 d_j^T H d_j + e_j,
 * unknowns (g, H_11, H_22[, H_33], H_12[, H_13, H_23]) -- nu = 5 (2D) / 9 (3D) -- solved by
 * weighted least squares with the same Gaussian weights.  Offsets are written in units of h
 * (dimensionless, O(1) matrix; the rank test is then meaningful) and the gradient rows are
 * scaled back: a_j = w_j (S^ m^_j)[0:d] / h.  S (output) = leading d x d block / h^2.
 * Deficient when m < nu + 1 or lambda_min < 1e-12 lambda_max. */
static int wls_one_order2(int d, const double* x, int64_t i, int m, const int32_t* nb, double h2,
                          double alpha_w, double* S, double* a) {
    const int nu = d == 2 ? 5 : 9;
    const double h = sqrt(h2);
    double A[81] = {0}, Ai[81];
    for (int jj = 0; jj < m; ++jj) {
        const double* xj = x + (int64_t)nb[jj] * d;
        double q[3], mv[9];
        for (int r = 0; r < d; ++r) q[r] = (xj[r] - x[i * d + r]) / h;
        int k = 0;
        for (int r = 0; r < d; ++r) mv[k++] = q[r];
        for (int r = 0; r < d; ++r) mv[k++] = 0.5 * q[r] * q[r];
        for (int r = 0; r < d; ++r)
            for (int c = r + 1; c < d; ++c) mv[k++] = q[r] * q[c];
        double w = or_weight(dist2(d, x + i * d, xj), h2, alpha_w);
        for (int r = 0; r < nu; ++r)
            for (int c = 0; c < nu; ++c) A[r * nu + c] = A[r * nu + c] + w * mv[r] * mv[c];
    }
    if (m < nu + 1) return OR_E_DEFICIENT;
    if (deficient(0, 2, nu, A)) return OR_E_DEFICIENT;
    if (inverse(nu, A, Ai)) return OR_E_DEFICIENT;
    for (int r = 0; r < d; ++r)
        for (int c = 0; c < d; ++c) S[r * d + c] = Ai[r * nu + c] / h2;
    for (int jj = 0; jj < m; ++jj) {
        const double* xj = x + (int64_t)nb[jj] * d;
        double q[3], mv[9];
        for (int r = 0; r < d; ++r) q[r] = (xj[r] - x[i * d + r]) / h;
        int k = 0;
        for (int r = 0; r < d; ++r) mv[k++] = q[r];
        for (int r = 0; r < d; ++r) mv[k++] = 0.5 * q[r] * q[r];
        for (int r = 0; r < d; ++r)
            for (int c = r + 1; c < d; ++c) mv[k++] = q[r] * q[c];
        double w = or_weight(dist2(d, x + i * d, xj), h2, alpha_w);
        for (int r = 0; r < d; ++r) {
            double s = 0.0;
            for (int c = 0; c < nu; ++c) s = s + Ai[r * nu + c] * mv[c];
            a[jj * d + r] = w * s / h;
        }
    }
    return OR_OK;
}

int or_wls_one_order(int d, const double* x, int64_t i, int m, const int32_t* nb, double h2,
                     double alpha_w, int order, double* S, double* a);

int or_wls_one(int d, const double* x, int64_t i, int m, const int32_t* nb,
               double h2, double alpha_w, double* S, double* a) {
    double A[9] = {0};
    for (int jj = 0; jj < m; ++jj) {
        const double* xj = x + (int64_t)nb[jj] * d;
        double dj[3];
        for (int r = 0; r < d; ++r) dj[r] = xj[r] - x[i * d + r];
        double w = or_weight(dist2(d, x + i * d, xj), h2, alpha_w);
        for (int r = 0; r < d; ++r)
            for (int c = 0; c < d; ++c) A[r * d + c] = A[r * d + c] + w * dj[r] * dj[c];
    }
    if (deficient(d, m, d, A)) return OR_E_DEFICIENT;
    if (inverse(d, A, S)) return OR_E_DEFICIENT;
    for (int jj = 0; jj < m; ++jj) {
        const double* xj = x + (int64_t)nb[jj] * d;
        double dj[3];
        for (int r = 0; r < d; ++r) dj[r] = xj[r] - x[i * d + r];
        double w = or_weight(dist2(d, x + i * d, xj), h2, alpha_w);
        for (int r = 0; r < d; ++r) {
            double s = 0.0;
            for (int c = 0; c < d; ++c) s = s + S[r * d + c] * dj[c];
            a[jj * d + r] = w * s;
        }
    }
    return OR_OK;
}

/* WLS of the requested Taylor order (1 or 0: first order; 2: second order). */
int or_wls_one_order(int d, const double* x, int64_t i, int m, const int32_t* nb, double h2,
                     double alpha_w, int order, double* S, double* a) {
    if (order == 2) return wls_one_order2(d, x, i, m, nb, h2, alpha_w, S, a);
    return or_wls_one(d, x, i, m, nb, h2, alpha_w, S, a);
}

/* ------------------------------------------------------------------ O4 --- */
/* Frame of the pair (i, j).
 * 2D: phi = atan2(dy, dx), n = (cos phi, sin phi), t = (-sin phi, cos phi).
 * 3D: phi = atan2(dy, dx) (atan2(+0,+0) = 0, Z10; phi = 0 also when the pair is
 *   vertical to rounding, dx^2 + dy^2 <= 1e-16 r^2, Z26),
 *   theta = arccos(dz / r) (argument clamped to [-1, 1]),
 *   rows of A: n = (sin th cos ph, sin th sin ph, cos th),
 *              t = (cos th cos ph, cos th sin ph, -sin th),
 *              b = (-sin ph, cos ph, 0).
 * frame[0..d-1] = n, [d..2d-1] = t, [2d..3d-1] = b (3D). */
void or_frame(int d, const double* dj, double* frame) {
    double phi = atan2(dj[1], dj[0]);
    if (d == 3) {
        double rxy2 = dj[0] * dj[0] + dj[1] * dj[1];
        if (rxy2 <= 1e-16 * (rxy2 + dj[2] * dj[2])) phi = 0.0;   /* Z26 */
    }
    if (d == 2) {
        frame[0] = cos(phi); frame[1] = sin(phi);
        frame[2] = -sin(phi); frame[3] = cos(phi);
        return;
    }
    double r = sqrt(dj[0] * dj[0] + dj[1] * dj[1] + dj[2] * dj[2]);
    double ct = dj[2] / r;
    if (ct > 1.0) ct = 1.0;
    if (ct < -1.0) ct = -1.0;
    double th = acos(ct);
    frame[0] = sin(th) * cos(phi); frame[1] = sin(th) * sin(phi); frame[2] = cos(th);
    frame[3] = cos(th) * cos(phi); frame[4] = cos(th) * sin(phi); frame[5] = -sin(th);
    frame[6] = -sin(phi);          frame[7] = cos(phi);          frame[8] = 0.0;
}

/* Rotated coefficients, P:413-416 (2D) and P:461-473 read as A (alpha, beta,
 * gamma)^T (Z8): abar = a . n, bbar = a . t, gbar = a . b. */
void or_rotate(int d, const double* a, const double* frame, double* rot) {
    for (int e = 0; e < d; ++e) {
        double s = 0.0;
        for (int r = 0; r < d; ++r) s = s + a[r] * frame[e * d + r];
        rot[e] = s;
    }
}

/* Full WLS + frames + rotation for every interior particle of a CSR cloud.
 * S[N*d*d] (interior rows), a/rot[nnz*d], frames[nnz*d*d] (interior rows).
 * Returns OR_OK or OR_E_DEFICIENT with *bad = first offending particle. */
int or_wls_all(int d, const double* x, int64_t N, const int8_t* kind, const int64_t* off,
               const int32_t* idx, double h2, double alpha_w, int order, double* S, double* a,
               double* frames, double* rot, int64_t* bad) {
    int64_t first_bad = -1;
    for (int64_t i = 0; i < N; ++i) {
        if (kind[i] != 0) continue;
        int m = (int)(off[i + 1] - off[i]);
        int st = or_wls_one_order(d, x, i, m, idx + off[i], h2, alpha_w, order, S + i * d * d, a + off[i] * d);
        if (st != OR_OK) {
            if (first_bad < 0) first_bad = i;
            continue;
        }
        for (int jj = 0; jj < m; ++jj) {
            int64_t e = off[i] + jj;
            double dj[3];
            for (int r = 0; r < d; ++r) dj[r] = x[(int64_t)idx[e] * d + r] - x[i * d + r];
            or_frame(d, dj, frames + e * d * d);
            or_rotate(d, a + e * d, frames + e * d * d, rot + e * d);
        }
    }
    *bad = first_bad;
    return first_bad < 0 ? OR_OK : OR_E_DEFICIENT;
}

/* ------------------------------------------------------------------ O5 --- */
/* Positive upwind flux and explicit transport for one interior particle
 * (P:163-171 explicit step; P:406-416 2D flux; P:474-481 3D flux, with the
 * readings Z5-Z7: beta in the y-sum, b in the third sum, sign(bbar)|c.t|):
 *   c = v_k - W_i  (W = U^n in ALE mode, 0 on a fixed cloud; Z15, Z21)
 *   Q_ik = sum_j [ abar (c.n - |c.n|) + bbar (c.t) - |bbar| |c.t|
 *                 (+ gbar (c.b) - |gbar| |c.b|) ] (f_jk - f_ik)
 *   ftilde_ik = f_ik - dt Q_ik      (each of g1, g2 in 2D)
 * rot[m*d] = (abar, bbar[, gbar]) per neighbour, frames[m*d*d],
 * fnb[m] = pointers to the neighbour rows, fi = own row, fti = output row.
 * Nodes [k_begin, k_end) only (used for sampled checks). */
void or_transport_one(const or_cfg* c, const double* W, int m, const double* rot,
                      const double* frames, const double* const* fnb, const double* fi,
                      double* fti, int64_t k_begin, int64_t k_end) {
    int d = c->dims, nv = nval_of(c);
    int64_t K = or_num_nodes(c);
    for (int64_t k = k_begin; k < k_end; ++k) {
        double v[3], cv[3];
        or_node_velocity(c, k, v);
        for (int a = 0; a < d; ++a) cv[a] = v[a] - W[a];
        for (int q = 0; q < nv; ++q) {
            double Q = 0.0;
            for (int jj = 0; jj < m; ++jj) {
                const double* fr = frames + jj * d * d;
                const double* rt = rot + jj * d;
                double coef = 0.0;
                for (int e = 0; e < d; ++e) {
                    double proj = 0.0;
                    for (int a = 0; a < d; ++a) proj = proj + cv[a] * fr[e * d + a];
                    if (e == 0) coef = coef + rt[0] * (proj - fabs(proj));
                    else coef = coef + (rt[e] * proj - fabs(rt[e]) * fabs(proj));
                }
                Q = Q + coef * (fnb[jj][q * K + k] - fi[q * K + k]);
            }
            fti[q * K + k] = fi[q * K + k] - c->dt * Q;
        }
    }
}

/* Largest explicit-stable step: 1 / max_{i,k} sum_j |C_ijk|,
 * C_ijk the coefficient multiplying (f_jk - f_ik) above.  Returns the max of
 * sum_j |C_ijk| over nodes for one particle. */
double or_coef_absmax_one(const or_cfg* c, const double* W, int m, const double* rot,
                          const double* frames) {
    int d = c->dims;
    int64_t K = or_num_nodes(c);
    double best = 0.0;
    for (int64_t k = 0; k < K; ++k) {
        double v[3], cv[3];
        or_node_velocity(c, k, v);
        for (int a = 0; a < d; ++a) cv[a] = v[a] - W[a];
        double s = 0.0;
        for (int jj = 0; jj < m; ++jj) {
            const double* fr = frames + jj * d * d;
            const double* rt = rot + jj * d;
            double coef = 0.0;
            for (int e = 0; e < d; ++e) {
                double proj = 0.0;
                for (int a = 0; a < d; ++a) proj = proj + cv[a] * fr[e * d + a];
                if (e == 0) coef = coef + rt[0] * (proj - fabs(proj));
                else coef = coef + (rt[e] * proj - fabs(rt[e]) * fabs(proj));
            }
            s = s + fabs(coef);
        }
        if (s > best) best = s;
    }
    return best;
}

/* ------------------------------------------------------------- O6, O7, O8 --- */
/* Moments of one row, fixed ascending k.
 * 3D, P:52-60 / P:189-190: rho = sum f dv^3, rho U = sum v f dv^3,
 *     3 rho R T = sum |v - U|^2 f dv^3.
 * 2D (Chu), P:112-115 / P:229 / P:253: rho = sum g1 dv^2, rho U = sum v g1 dv^2,
 *     3 rho R T = sum |v - U|^2 g1 dv^2 + sum g2 dv^2.
 * out = (rho, U[d], T). Returns OR_E_DEGENERATE if rho <= 0 or T <= 1e-12. */
int or_moments_row(const or_cfg* c, const double* f, double* out) {
    int d = c->dims;
    int64_t K = or_num_nodes(c);
    double dv = or_dv(c), w = 1.0;
    for (int a = 0; a < d; ++a) w = w * dv;
    double s0 = 0.0, s1[3] = {0, 0, 0};
    for (int64_t k = 0; k < K; ++k) {
        double v[3];
        or_node_velocity(c, k, v);
        s0 = s0 + f[k];
        for (int a = 0; a < d; ++a) s1[a] = s1[a] + v[a] * f[k];
    }
    double rho = s0 * w, U[3];
    for (int a = 0; a < d; ++a) U[a] = s1[a] * w / rho;
    double s2 = 0.0;
    for (int64_t k = 0; k < K; ++k) {
        double v[3], q = 0.0;
        or_node_velocity(c, k, v);
        for (int a = 0; a < d; ++a) q = q + (v[a] - U[a]) * (v[a] - U[a]);
        s2 = s2 + q * f[k];
    }
    if (d == 2)
        for (int64_t k = 0; k < K; ++k) s2 = s2 + f[K + k];
    double T = s2 * w / (3.0 * rho * c->R);
    out[0] = rho;
    for (int a = 0; a < d; ++a) out[1 + a] = U[a];
    out[1 + d] = T;
    if (!(rho > 0.0) || !(T > 1e-12)) return OR_E_DEGENERATE;
    return OR_OK;
}

/* Relaxation time: Cbar = sqrt(8RT/pi), lambda = k_b/(sqrt(2) pi rho R d^2),
 * tau = 4 lambda / (pi Cbar).  Also returns lambda. */
double or_tau(const or_cfg* c, double rho, double T, double* lambda_out) {
    double pi = 3.14159265358979323846;
    double Cbar = sqrt(8.0 * c->R * T / pi);
    double lambda = c->kb / (sqrt(2.0) * pi * rho * c->R * c->dmol * c->dmol);
    if (lambda_out) *lambda_out = lambda;
    return 4.0 * lambda / (pi * Cbar);
}

/* Local Maxwellian on the grid.
 * 3D, P:46-49 (exponent sign restored, Z1): M = rho/(2 pi R T)^{3/2} exp(-|v-U|^2/(2RT)).
 * 2D, P:98-105 (pi and sign restored, Z1/Z2): G1 = rho/(2 pi R T) exp(-|v-U|^2/(2RT)),
 *     G2 = R T G1.  Row layout as f. */
void or_maxwellian_row(const or_cfg* c, double rho, const double* U, double T, double* M) {
    int d = c->dims;
    int64_t K = or_num_nodes(c);
    double pi = 3.14159265358979323846;
    double RT = c->R * T;
    double pref = d == 3 ? rho / pow(2.0 * pi * RT, 1.5) : rho / (2.0 * pi * RT);
    for (int64_t k = 0; k < K; ++k) {
        double v[3], q = 0.0;
        or_node_velocity(c, k, v);
        for (int a = 0; a < d; ++a) q = q + (v[a] - U[a]) * (v[a] - U[a]);
        M[k] = pref * exp(-q / (2.0 * RT));
        if (d == 2) M[K + k] = RT * M[k];
    }
}

/* Implicit relaxation in closed form, P:196-199 / P:259-262:
 * f^{n+1} = (tau ftilde + dt M) / (tau + dt), nodewise. */
void or_relax_row(int64_t n, double tau, double dt, const double* ft, const double* M,
                  double* fnew) {
    for (int64_t k = 0; k < n; ++k) fnew[k] = (tau * ft[k] + dt * M[k]) / (tau + dt);
}

/* ----------------------------------------------------------------- O10 --- */
/* Inward unit normal of a wall id (1: x=0 -> +x, 2: x=L -> -x, ...). */
void or_wall_normal(int d, int wid, double* n) {
    for (int a = 0; a < d; ++a) n[a] = 0.0;
    int a = (wid - 1) / 2;
    n[a] = ((wid - 1) % 2 == 0) ? 1.0 : -1.0;
}

/* Wall velocity: the lid (wall 2d) moves with Ulid, the other walls are at rest. */
void or_wall_velocity(const or_cfg* c, int wid, double* Uw) {
    for (int a = 0; a < c->dims; ++a) Uw[a] = (wid == 2 * c->dims) ? c->Ulid[a] : 0.0;
}

/* Boundary interpolation weights ("with the help of the least squares
 * method"; Z19: linear WLS with a constant term).  For boundary
 * particle b and its interior neighbours j (members of N(b) with kind 0):
 * P_j = (1, d_j), B = sum_j w_j P_j P_j^T, c_bj = w_j e0^T B^{-1} P_j.
 * c[m] aligned with nb[m]; non-interior neighbours get 0.
 * The offsets are written in units of h, P_j = (1, d_j / h), so that B is
 * dimensionless and the scale-free rank test below is meaningful; c_bj does
 * not depend on that scaling (e0^T B^{-1} P_j is invariant).
 * Returns OR_OK or OR_E_DEFICIENT (fewer than d+2 interior neighbours or
 * lambda_min(B) < 1e-12 lambda_max(B)). */
int or_boundary_weights_one(int d, const double* x, const int8_t* kind, int64_t b, int m,
                            const int32_t* nb, double h2, double alpha_w, double* cw) {
    int n = d + 1, mi = 0;
    double h = sqrt(h2);
    double B[16] = {0}, Binv[16];
    for (int jj = 0; jj < m; ++jj) {
        int64_t j = nb[jj];
        if (kind[j] != 0) continue;
        ++mi;
        double P[4];
        P[0] = 1.0;
        for (int r = 0; r < d; ++r) P[1 + r] = (x[j * d + r] - x[b * d + r]) / h;
        double w = or_weight(dist2(d, x + b * d, x + j * d), h2, alpha_w);
        for (int r = 0; r < n; ++r)
            for (int q = 0; q < n; ++q) B[r * n + q] = B[r * n + q] + w * P[r] * P[q];
    }
    if (deficient(d, mi, n, B)) return OR_E_DEFICIENT;
    if (inverse(n, B, Binv)) return OR_E_DEFICIENT;
    for (int jj = 0; jj < m; ++jj) {
        int64_t j = nb[jj];
        if (kind[j] != 0) { cw[jj] = 0.0; continue; }
        double P[4];
        P[0] = 1.0;
        for (int r = 0; r < d; ++r) P[1 + r] = (x[j * d + r] - x[b * d + r]) / h;
        double w = or_weight(dist2(d, x + b * d, x + j * d), h2, alpha_w);
        double s = 0.0;
        for (int q = 0; q < n; ++q) s = s + Binv[0 * n + q] * P[q];
        cw[jj] = w * s;
    }
    return OR_OK;
}

/* Diffuse reflection at one boundary particle (Z17):
 *   nodes with v.n <= 0 (towards the wall or tangential): f_bk = sum_j c_bj f_jk
 *     (each value; interior rows fnb[], weights cw[]);
 *   rho_w = - sum_{v.n<0} (v.n) f_bk / sum_{v.n>0} (v.n) M_w,k,
 *     M_w = M(1, U_wall, T_wall) (2D: the flux uses g1 and G1);
 *   nodes with v.n > 0 (leaving the wall): f_bk = rho_w M_w,k (2D: G1 and G2).
 * (v - U_wall).n = v.n because U_wall is tangential.  fb = output row.
 * Returns OR_OK or OR_E_WALL if the outgoing denominator is <= 0; *rho_w out. */
int or_diffuse_one(const or_cfg* c, int wid, int m, const double* cw,
                   const double* const* fnb, double* fb, double* rho_w_out) {
    int d = c->dims, nv = nval_of(c);
    int64_t K = or_num_nodes(c);
    double n[3], Uw[3];
    or_wall_normal(d, wid, n);
    or_wall_velocity(c, wid, Uw);
    double* Mw = (double*)malloc(sizeof(double) * (size_t)(nv * K));
    or_maxwellian_row(c, 1.0, Uw, c->Twall, Mw);
    double flux_in = 0.0, den = 0.0;
    for (int64_t k = 0; k < K; ++k) {
        double v[3], vn = 0.0;
        or_node_velocity(c, k, v);
        for (int a = 0; a < d; ++a) vn = vn + v[a] * n[a];
        if (vn <= 0.0) {
            for (int q = 0; q < nv; ++q) {
                double s = 0.0;
                for (int jj = 0; jj < m; ++jj)
                    if (fnb[jj]) s = s + cw[jj] * fnb[jj][q * K + k];
                fb[q * K + k] = s;
            }
            if (vn < 0.0) flux_in = flux_in + vn * fb[k];
        } else {
            den = den + vn * Mw[k];
        }
    }
    if (!(den > 0.0)) { free(Mw); return OR_E_WALL; }
    double rho_w = -flux_in / den;
    for (int64_t k = 0; k < K; ++k) {
        double v[3], vn = 0.0;
        or_node_velocity(c, k, v);
        for (int a = 0; a < d; ++a) vn = vn + v[a] * n[a];
        if (vn > 0.0)
            for (int q = 0; q < nv; ++q) fb[q * K + k] = rho_w * Mw[q * K + k];
    }
    free(Mw);
    *rho_w_out = rho_w;
    return OR_OK;
}

/* ----------------------------------------------------------- initial state */
/* f^0 = M(rho^0, U^0, T^0) at every particle (boundary too), W^0 = U^0. */
void or_init_f(const or_cfg* c, int64_t N, const double* rho, const double* U,
               const double* T, double* f) {
    int d = c->dims, nv = nval_of(c);
    int64_t K = or_num_nodes(c);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; ++i) or_maxwellian_row(c, rho[i], U + i * d, T[i], f + i * nv * K);
}

/* ------------------------------------------------------- one full step --- */
/* One time step n -> n+1 in the order of S:414 / SURVEY §8(c) O1-O11:
 *   geometry from x^n: neighbours (O2), WLS + frames (O3, O4), boundary weights;
 *   transport (O5) -> ftilde at interior particles;
 *   moments of ftilde (O6) -> rho, U, T; tau (O7); relaxation (O8) -> f^{n+1};
 *   ALE: x^{n+1} = x^n + dt U^{n+1}, clamped to [eps, L - eps], eps = 1e-3 dx (P:177-180,
 *        S:440); W <- U^{n+1} (O9, O11);
 *   diffuse reflection at boundary particles from the interior f^{n+1} with the
 *        step-start weights (O10).
 * In/out: x[N*d], f[N*nval*K], W[N*d]; out: macro[N*(d+2)] (rho, U, T) of the
 * recovered state at interior particles, moments of the new row at boundary ones;
 * rho_w[N] (boundary particles).  Returns OR_OK or an error code with *bad. */
int or_step(const or_cfg* c, int64_t N, double* x, const int8_t* kind, double* f, double* W,
            double* macro, double* rho_w, int64_t* bad) {
    int d = c->dims, nv = nval_of(c);
    int64_t K = or_num_nodes(c), RK = (int64_t)nv * K;
    *bad = -1;
    /* O2 */
    int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(N + 1));
    int64_t need = 0;
    or_neighbors(d, x, N, c->h2, off, NULL, 0, &need);
    int32_t* idx = (int32_t*)malloc(sizeof(int32_t) * (size_t)(need > 0 ? need : 1));
    or_neighbors(d, x, N, c->h2, off, idx, need, &need);
    /* O3, O4 */
    double* S = (double*)calloc((size_t)(N * d * d), sizeof(double));
    double* a = (double*)calloc((size_t)(need * d + 1), sizeof(double));
    double* fr = (double*)calloc((size_t)(need * d * d + 1), sizeof(double));
    double* rot = (double*)calloc((size_t)(need * d + 1), sizeof(double));
    double* cw = (double*)calloc((size_t)(need + 1), sizeof(double));
    int st = or_wls_all(d, x, N, kind, off, idx, c->h2, c->alpha_w, c->wls_order, S, a, fr, rot, bad);
    if (st == OR_OK)
        for (int64_t b = 0; b < N; ++b) {
            if (kind[b] == 0) continue;
            if (or_boundary_weights_one(d, x, kind, b, (int)(off[b + 1] - off[b]), idx + off[b],
                                        c->h2, c->alpha_w, cw + off[b]) != OR_OK) {
                *bad = b;
                st = OR_E_DEFICIENT;
                break;
            }
        }
    double* ft = NULL;
    if (st == OR_OK) ft = (double*)malloc(sizeof(double) * (size_t)(N * RK));
    /* O5 */
    if (st == OR_OK) {
#pragma omp parallel for schedule(dynamic, 4)
        for (int64_t i = 0; i < N; ++i) {
            if (kind[i] != 0) continue;
            int m = (int)(off[i + 1] - off[i]);
            const double** fnb = (const double**)malloc(sizeof(double*) * (size_t)(m > 0 ? m : 1));
            for (int jj = 0; jj < m; ++jj) fnb[jj] = f + (int64_t)idx[off[i] + jj] * RK;
            double Wi[3] = {0, 0, 0};
            if (c->ale)
                for (int q = 0; q < d; ++q) Wi[q] = W[i * d + q];
            or_transport_one(c, Wi, m, rot + off[i] * d, fr + off[i] * d * d, fnb, f + i * RK,
                             ft + i * RK, 0, K);
            free(fnb);
        }
    }
    /* O6, O7, O8 */
    int64_t first_degenerate = -1;
    if (st == OR_OK) {
        for (int64_t i = 0; i < N; ++i) {
            if (kind[i] != 0) continue;
            double* mo = macro + i * (d + 2);
            if (or_moments_row(c, ft + i * RK, mo) != OR_OK) {
                if (first_degenerate < 0) first_degenerate = i;
                continue;
            }
            double tau = or_tau(c, mo[0], mo[1 + d], NULL);
            double* M = (double*)malloc(sizeof(double) * (size_t)RK);
            or_maxwellian_row(c, mo[0], mo + 1, mo[1 + d], M);
            or_relax_row(RK, tau, c->dt, ft + i * RK, M, f + i * RK);
            free(M);
        }
        if (first_degenerate >= 0) {
            *bad = first_degenerate;
            st = OR_E_DEGENERATE;
        }
    }
    /* O9, O11 */
    if (st == OR_OK && c->ale) {
        double eps = 1e-3 * c->dx;
        for (int64_t i = 0; i < N; ++i) {
            if (kind[i] != 0) continue;
            for (int q = 0; q < d; ++q) {
                double u = macro[i * (d + 2) + 1 + q];
                double xn = x[i * d + q] + c->dt * u;
                if (xn < eps) xn = eps;
                if (xn > c->L - eps) xn = c->L - eps;
                x[i * d + q] = xn;
                W[i * d + q] = u;
            }
        }
    }
    /* O10 */
    if (st == OR_OK) {
        for (int64_t b = 0; b < N; ++b) {
            if (kind[b] == 0) continue;
            int m = (int)(off[b + 1] - off[b]);
            const double** fnb = (const double**)malloc(sizeof(double*) * (size_t)(m > 0 ? m : 1));
            for (int jj = 0; jj < m; ++jj) {
                int64_t j = idx[off[b] + jj];
                fnb[jj] = kind[j] == 0 ? f + j * RK : NULL;
            }
            double rw = 0.0;
            int s2 = or_diffuse_one(c, kind[b], m, cw + off[b], fnb, f + b * RK, &rw);
            free(fnb);
            if (s2 != OR_OK) {
                *bad = b;
                st = s2;
                break;
            }
            if (rho_w) rho_w[b] = rw;
            or_moments_row(c, f + b * RK, macro + b * (d + 2));
        }
    }
    free(off); free(idx); free(S); free(a); free(fr); free(rot); free(cw); free(ft);
    return st;
}

/* ------------------------------------------------- particle management --- */
/* Interpolation weights of a new point p from the particles S[0..m) ("update the
 * distribution function on these new grid points with the help of the least squares
 * method"; S:283-287 interpolate_value): linear WLS with a constant term, f ~ a0 + a.(x - p),
 * w_s = exp(-alpha |x_s - p|^2 / h^2), P_s = (1, (x_s - p) / h), B = sum_s w_s P_s P_s^T,
 * c_s = w_s e0^T B^{-1} P_s (the value at p is sum_s c_s f_s).  Same construction as the
 * boundary weights (Z19) with every stencil member used.  Deficient: m < d+2 or
 * lambda_min(B) < 1e-12 lambda_max(B) -> OR_E_DEFICIENT. */
int or_interp_weights(int d, const double* x, const int32_t* S, int m, const double* p,
                      double h2, double alpha_w, double* cw) {
    int n = d + 1;
    double h = sqrt(h2);
    double B[16] = {0}, Binv[16];
    for (int s = 0; s < m; ++s) {
        const double* xs = x + (int64_t)S[s] * d;
        double P[4];
        P[0] = 1.0;
        for (int r = 0; r < d; ++r) P[1 + r] = (xs[r] - p[r]) / h;
        double w = or_weight(dist2(d, p, xs), h2, alpha_w);
        for (int r = 0; r < n; ++r)
            for (int q = 0; q < n; ++q) B[r * n + q] = B[r * n + q] + w * P[r] * P[q];
    }
    if (deficient(d, m, n, B)) return OR_E_DEFICIENT;
    if (inverse(n, B, Binv)) return OR_E_DEFICIENT;
    for (int s = 0; s < m; ++s) {
        const double* xs = x + (int64_t)S[s] * d;
        double P[4];
        P[0] = 1.0;
        for (int r = 0; r < d; ++r) P[1 + r] = (xs[r] - p[r]) / h;
        double w = or_weight(dist2(d, p, xs), h2, alpha_w);
        double acc = 0.0;
        for (int q = 0; q < n; ++q) acc = acc + Binv[0 * n + q] * P[q];
        cw[s] = w * acc;
    }
    return OR_OK;
}

/* Stencil of a new point p: every particle of the cloud (x, N) within h of p (closed ball,
 * the O2 distance), ascending, except ex0 / ex1.  Returns the count (writes <= cap). */
static int stencil_of(int d, const double* x, int64_t N, double h2, const double* p, int64_t ex0,
                      int64_t ex1, int32_t* S, int cap) {
    int m = 0;
    for (int64_t k = 0; k < N; ++k) {
        if (k == ex0 || k == ex1) continue;
        if (dist2(d, p, x + k * d) <= h2) {
            if (m < cap) S[m] = (int32_t)k;
            ++m;
        }
    }
    return m;
}

/* Interpolate one new particle at p from the OLD state: f row, W, macro.  Returns status. */
static int interp_new(const or_cfg* c, int64_t N, const double* x, const double* f, const double* W,
                      const double* macro, const double* p, int64_t ex0, int64_t ex1, double* f_row,
                      double* W_row, double* macro_row) {
    int d = c->dims, nv = nval_of(c);
    int64_t RK = (int64_t)nv * or_num_nodes(c);
    int cap = 4096;
    int32_t* S = (int32_t*)malloc(sizeof(int32_t) * (size_t)cap);
    int m = stencil_of(d, x, N, c->h2, p, ex0, ex1, S, cap);
    if (m > cap) { free(S); return OR_E_CAPACITY; }
    double* cw = (double*)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
    int st = or_interp_weights(d, x, S, m, p, c->h2, c->alpha_w, cw);
    if (st == OR_OK) {
        for (int64_t k = 0; k < RK; ++k) {
            double acc = 0.0;
            for (int s = 0; s < m; ++s) acc = acc + cw[s] * f[(int64_t)S[s] * RK + k];
            f_row[k] = acc;
        }
        for (int q = 0; q < d; ++q) {
            double acc = 0.0;
            for (int s = 0; s < m; ++s) acc = acc + cw[s] * W[(int64_t)S[s] * d + q];
            W_row[q] = acc;
        }
        for (int q = 0; q < d + 2; ++q) {
            double acc = 0.0;
            for (int s = 0; s < m; ++s) acc = acc + cw[s] * macro[(int64_t)S[s] * (d + 2) + q];
            macro_row[q] = acc;
        }
    }
    free(S);
    free(cw);
    return st;
}

/* Particle management pass ("if two points are close to each other, we remove both
 * of them and introduce a new grid in the mid-point ... when they scatter ... one has to add
 * new particles"; Z28), at the start of an ALE step, on the state
 * (x, kind, f, W, macro) of N particles:
 *  1. merge: for interior i ascending, unprocessed: the first j of N(i) (ascending) with j > i,
 *     interior, unprocessed and d2(i, j) < r_merge^2 pairs with i; both become processed.  The
 *     pair is replaced by ONE particle at m = (x_i + x_j) * 0.5 in slot i (slot j is removed);
 *     its f row, W and macro are interpolated from every other particle of the OLD cloud
 *     within h of m.  A deficient stencil keeps the pair (reported).
 *  2. fill: for i ascending, not processed in 1, either interior with |N(i)| < m_min -- the
 *     candidates p = x_i + s (0.5 h) e_a (a = 0..d-1; s = +1, then -1) -- or a boundary particle
 *     whose interpolation system (its interior neighbours, Z19) is deficient -- fewer than d + 2
 *     members, or (for fewer than 3 (d + 1) members) lambda_min < 1e-12 lambda_max or a zero pivot,
 *     the test of or_boundary_weights_one -- the
 *     candidates x_i + s h N, N = sum of the inward normals of the walls it lies on, s = 1/2, 1/4,
 *     3/4 in that order, of which it takes the first accepted one (Z30) --
 *     those strictly inside (0, L)^d and farther than 0.45 dx from every particle of the CURRENT
 *     cloud (old particles minus the removed slots, merged particles at their midpoints,
 *     candidates inserted so far) are appended, interpolated from the OLD cloud within h of p.
 *     Deficient candidates are skipped; insertion stops at the capacity cap (both reported).
 *  3. compaction: the surviving slots in ascending old order, then the appended particles.
 * Outputs (capacity cap): x_out, kind_out, f_out, W_out, macro_out;
 * report[6] = {merges, merges kept (deficient), fills, fills skipped (deficient),
 * fills skipped (capacity), N_out}. */
int or_manage(const or_cfg* c, int64_t N, const double* x, const int8_t* kind, const double* f,
              const double* W, const double* macro, double r_merge, int m_min, int64_t cap,
              double* x_out, int8_t* kind_out, double* f_out, double* W_out, double* macro_out,
              int64_t* report) {
    int d = c->dims, nv = nval_of(c);
    int64_t RK = (int64_t)nv * or_num_nodes(c);
    double rm2 = r_merge * r_merge;
    double hh = 0.5 * c->h;
    double thr2 = (0.45 * c->dx) * (0.45 * c->dx);
    for (int q = 0; q < 6; ++q) report[q] = 0;
    int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(N + 1));
    int64_t need = 0;
    or_neighbors(d, x, N, c->h2, off, NULL, 0, &need);
    int32_t* idx = (int32_t*)malloc(sizeof(int32_t) * (size_t)(need > 0 ? need : 1));
    or_neighbors(d, x, N, c->h2, off, idx, need, &need);
    char* processed = (char*)calloc((size_t)N + 1, 1);
    char* removed = (char*)calloc((size_t)N + 1, 1);
    int64_t* partner = (int64_t*)malloc(sizeof(int64_t) * (size_t)(N + 1));
    double* cur = (double*)malloc(sizeof(double) * (size_t)(N * d + 1));   /* current positions */
    memcpy(cur, x, sizeof(double) * (size_t)(N * d));
    double* mf = (double*)malloc(sizeof(double) * (size_t)(N * RK + 1)); /* merged rows (slot i) */
    double* mW = (double*)malloc(sizeof(double) * (size_t)(N * d + 1));
    double* mM = (double*)malloc(sizeof(double) * (size_t)(N * (d + 2) + 1));
    for (int64_t i = 0; i < N; ++i) partner[i] = -1;
    /* 1. merge */
    for (int64_t i = 0; i < N; ++i) {
        if (kind[i] != 0 || processed[i]) continue;
        int64_t j = -1;
        for (int64_t e = off[i]; e < off[i + 1]; ++e) {
            int64_t k = idx[e];
            if (k > i && kind[k] == 0 && !processed[k] && dist2(d, x + i * d, x + k * d) < rm2) {
                j = k;
                break;
            }
        }
        if (j < 0) continue;
        processed[i] = processed[j] = 1;
        double mp[3];
        for (int a = 0; a < d; ++a) mp[a] = (x[i * d + a] + x[j * d + a]) * 0.5;
        if (interp_new(c, N, x, f, W, macro, mp, i, j, mf + i * RK, mW + i * d, mM + i * (d + 2)) != OR_OK) {
            ++report[1];
            continue;
        }
        ++report[0];
        partner[i] = j;
        removed[j] = 1;
        for (int a = 0; a < d; ++a) cur[i * d + a] = mp[a];
    }
    /* 2. fill */
    int64_t n_live = N - report[0];
    int64_t nf = 0, fcap = cap - n_live > 0 ? cap - n_live : 0;
    double* fx = (double*)malloc(sizeof(double) * (size_t)((fcap > 0 ? fcap : 1) * d));
    double* ff = (double*)malloc(sizeof(double) * (size_t)((fcap > 0 ? fcap : 1) * RK));
    double* fW = (double*)malloc(sizeof(double) * (size_t)((fcap > 0 ? fcap : 1) * d));
    double* fM = (double*)malloc(sizeof(double) * (size_t)((fcap > 0 ? fcap : 1) * (d + 2)));
    for (int64_t i = 0; i < N; ++i) {
        if (processed[i]) continue;
        double cand[6][3];                        /* the candidates of i, in proposal order */
        int nc = 0;
        if (kind[i] == 0) {
            if (off[i + 1] - off[i] >= m_min) continue;
            for (int a = 0; a < d; ++a)
                for (int sgn = 0; sgn < 2; ++sgn) {
                    for (int q = 0; q < d; ++q) cand[nc][q] = x[i * d + q];
                    cand[nc][a] = sgn == 0 ? x[i * d + a] + hh : x[i * d + a] - hh;
                    ++nc;
                }
        } else {
            /* a wall particle whose interpolation system (Z19: its interior neighbours) is
             * deficient -- fewer than d + 2 members or lambda_min < 1e-12 lambda_max (Z30) */
            int mb = (int)(off[i + 1] - off[i]), n_int = 0;
            for (int64_t e = off[i]; e < off[i + 1]; ++e) n_int += kind[idx[e]] == 0;
            if (n_int >= 3 * (d + 1)) continue;   /* the conditioning test only on small stencils */
            double* cwt = (double*)malloc(sizeof(double) * (size_t)(mb > 0 ? mb : 1));
            int st_b = or_boundary_weights_one(d, x, kind, i, mb, idx + off[i], c->h2, c->alpha_w, cwt);
            free(cwt);
            if (st_b == OR_OK) continue;
            double nrm[3] = {0.0, 0.0, 0.0};      /* sum of the inward normals of its walls */
            for (int a = 0; a < d; ++a) {
                if (x[i * d + a] == 0.0) nrm[a] = 1.0;
                else if (x[i * d + a] == c->L) nrm[a] = -1.0;
            }
            const double hs[3] = {0.5 * c->h, 0.25 * c->h, 0.75 * c->h};
            for (int k = 0; k < 3; ++k, ++nc)
                for (int q = 0; q < d; ++q) cand[nc][q] = x[i * d + q] + hs[k] * nrm[q];
        }
        const int wall = kind[i] != 0;            /* a wall particle takes its first accepted candidate */
        for (int k = 0; k < nc && k < 2 * d; ++k) {
                double p[3];
                for (int q = 0; q < d; ++q) p[q] = cand[k][q];
                int inside = 1;
                for (int q = 0; q < d; ++q)
                    if (!(p[q] > 0.0 && p[q] < c->L)) inside = 0;
                if (!inside) continue;
                int clear = 1;
                for (int64_t k2 = 0; k2 < N && clear; ++k2)
                    if (!removed[k2] && !(dist2(d, p, cur + k2 * d) > thr2)) clear = 0;
                for (int64_t k2 = 0; k2 < nf && clear; ++k2)
                    if (!(dist2(d, p, fx + k2 * d) > thr2)) clear = 0;
                if (!clear) continue;
                if (nf >= fcap) { ++report[4]; continue; }
                if (interp_new(c, N, x, f, W, macro, p, -1, -1, ff + nf * RK, fW + nf * d,
                               fM + nf * (d + 2)) != OR_OK) {
                    ++report[3];
                    continue;
                }
                for (int q = 0; q < d; ++q) fx[nf * d + q] = p[q];
                ++nf;
                if (wall) break;
        }
    }
    report[2] = nf;
    /* 3. compaction */
    int64_t t = 0;
    for (int64_t i = 0; i < N; ++i) {
        if (removed[i]) continue;
        int merged = partner[i] >= 0;
        for (int q = 0; q < d; ++q) x_out[t * d + q] = cur[i * d + q];
        kind_out[t] = kind[i];
        memcpy(f_out + t * RK, merged ? mf + i * RK : f + i * RK, sizeof(double) * (size_t)RK);
        memcpy(W_out + t * d, merged ? mW + i * d : W + i * d, sizeof(double) * (size_t)d);
        memcpy(macro_out + t * (d + 2), merged ? mM + i * (d + 2) : macro + i * (d + 2),
               sizeof(double) * (size_t)(d + 2));
        ++t;
    }
    for (int64_t k = 0; k < nf; ++k, ++t) {
        for (int q = 0; q < d; ++q) x_out[t * d + q] = fx[k * d + q];
        kind_out[t] = 0;
        memcpy(f_out + t * RK, ff + k * RK, sizeof(double) * (size_t)RK);
        memcpy(W_out + t * d, fW + k * d, sizeof(double) * (size_t)d);
        memcpy(macro_out + t * (d + 2), fM + k * (d + 2), sizeof(double) * (size_t)(d + 2));
    }
    report[5] = t;
    free(off); free(idx); free(processed); free(removed); free(partner); free(cur);
    free(mf); free(mW); free(mM); free(fx); free(ff); free(fW); free(fM);
    return OR_OK;
}

/* Moments of every row of f, interior and boundary. */
int or_moments_all(const or_cfg* c, int64_t N, const double* f, double* macro, int64_t* bad) {
    int d = c->dims, nv = nval_of(c);
    int64_t RK = (int64_t)nv * or_num_nodes(c);
    *bad = -1;
    for (int64_t i = 0; i < N; ++i)
        if (or_moments_row(c, f + i * RK, macro + i * (d + 2)) != OR_OK && *bad < 0) *bad = i;
    return *bad < 0 ? OR_OK : OR_E_DEGENERATE;
}

#ifdef _OPENMP
#include <omp.h>
#endif
int or_omp_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void or_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
