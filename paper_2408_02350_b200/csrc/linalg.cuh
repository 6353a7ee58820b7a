// linalg.cuh -- small dense fp64 helpers shared by the WLS (wls.cu) and particle-management
// (manage.cu) kernels: Gauss-Jordan inverse with partial pivoting and the scale-free rank test
// lambda_min >= 1e-12 lambda_max by cyclic Jacobi sweeps (Z24).
#pragma once

namespace bgk {

template <int n>
__device__ inline bool small_inverse(const double (&A)[n][n], double (&Ai)[n][n]) {
    double M[n][2 * n];
#pragma unroll
    for (int r = 0; r < n; ++r)
#pragma unroll
        for (int q = 0; q < 2 * n; ++q) M[r][q] = q < n ? A[r][q] : (q - n == r ? 1.0 : 0.0);
#pragma unroll
    for (int col = 0; col < n; ++col) {
        int piv = col;
        double best = fabs(M[col][col]);
#pragma unroll
        for (int r = col + 1; r < n; ++r)
            if (fabs(M[r][col]) > best) { best = fabs(M[r][col]); piv = r; }
        if (best == 0.0) return false;
        if (piv != col) {
#pragma unroll
            for (int r = col + 1; r < n; ++r)
                if (r == piv)
#pragma unroll
                    for (int q = 0; q < 2 * n; ++q) { double t = M[col][q]; M[col][q] = M[r][q]; M[r][q] = t; }
        }
        const double ip = 1.0 / M[col][col];
#pragma unroll
        for (int q = 0; q < 2 * n; ++q) M[col][q] *= ip;
#pragma unroll
        for (int r = 0; r < n; ++r) {
            if (r == col) continue;
            const double fct = M[r][col];
#pragma unroll
            for (int q = 0; q < 2 * n; ++q) M[r][q] -= fct * M[col][q];
        }
    }
#pragma unroll
    for (int r = 0; r < n; ++r)
#pragma unroll
        for (int q = 0; q < n; ++q) Ai[r][q] = M[r][n + q];
    return true;
}

// lambda_min / lambda_max of a symmetric n x n matrix by cyclic Jacobi sweeps
template <int n>
__device__ inline bool well_conditioned(const double (&A)[n][n]) {
    double a[n][n];
#pragma unroll
    for (int r = 0; r < n; ++r)
#pragma unroll
        for (int q = 0; q < n; ++q) a[r][q] = A[r][q];
    for (int sweep = 0; sweep < 12; ++sweep) {
        double off = 0.0, dia = 0.0;
#pragma unroll
        for (int r = 0; r < n; ++r)
#pragma unroll
            for (int q = 0; q < n; ++q) (r == q ? dia : off) += a[r][q] * a[r][q];
        if (off <= 1e-40 * dia) break;
#pragma unroll
        for (int p = 0; p < n; ++p)
#pragma unroll
            for (int q = p + 1; q < n; ++q) {
                if (a[p][q] == 0.0) continue;
                const double th = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
                const double t = copysign(1.0, th) / (fabs(th) + sqrt(th * th + 1.0));
                const double cs = rsqrt(t * t + 1.0), sn = t * cs;
#pragma unroll
                for (int k = 0; k < n; ++k) {
                    const double akp = a[k][p], akq = a[k][q];
                    a[k][p] = cs * akp - sn * akq;
                    a[k][q] = sn * akp + cs * akq;
                }
#pragma unroll
                for (int k = 0; k < n; ++k) {
                    const double apk = a[p][k], aqk = a[q][k];
                    a[p][k] = cs * apk - sn * aqk;
                    a[q][k] = sn * apk + cs * aqk;
                }
            }
    }
    double lo = a[0][0], hi = a[0][0];
#pragma unroll
    for (int r = 1; r < n; ++r) { lo = fmin(lo, a[r][r]); hi = fmax(hi, a[r][r]); }
    return hi > 0.0 && lo >= 1e-12 * hi;
}

// The rank test without the sweeps where it cannot fail: lambda_max <= ||A||_F and 1 / lambda_min =
// ||A^-1||_2 <= ||A^-1||_F, so ||A||_F ||A^-1||_F <= 1e10 proves lambda_min >= 1e-10 lambda_max -- a
// factor 100 above the 1e-12 threshold, far beyond the sweeps' rounding, so the decision is the one
// well_conditioned takes.  Only stencils the bound cannot clear pay for the Jacobi sweeps.
template <int n>
__device__ inline bool rank_test(const double (&A)[n][n], const double (&Ai)[n][n]) {
    double fa = 0.0, fi = 0.0;
#pragma unroll
    for (int r = 0; r < n; ++r)
#pragma unroll
        for (int q = 0; q < n; ++q) {
            fa += A[r][q] * A[r][q];
            fi += Ai[r][q] * Ai[r][q];
        }
    if (fa * fi <= 1e20) return true;
    return well_conditioned<n>(A);
}

}  // namespace bgk
