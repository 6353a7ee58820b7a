// relax_params.cuh -- the relaxation step's per-particle parameters (relax.cu k_relax / k_relax_w2,
// and the fused 2D transport + relaxation of transport.cu): rho, U, T from the moment sums, tau,
// the implicit-relaxation weights and the Maxwellian prefactor; ALE move.
#pragma once
#include "bgk_internal.cuh"

namespace bgk {

constexpr double kPi = 3.14159265358979323846;

struct RelaxArgs {
    const int32_t* ids;
    const double* sums;
    double* f;       // ftilde in, f^{n+1} out (in place)
    double* macro;
    double* W;
    double* x;
    int64_t* err;
    int64_t n;
    int n1, ncol, ncs, c0, Ks, ale;
    double vmax, dv, dt, R, kb, dmol, L, clamp_eps;
};

// rho, U, T from the all-reduced sums (single pass, Z25), tau,
// the relaxation weights and the Maxwellian's prefactor into par[0 .. 4+D] (par[5..] = U), the
// recovered macro state, and in ALE mode W <- U and the clamped move x += dt U
template <int D>
__device__ __forceinline__ void relax_params(const RelaxArgs& A, const double* s, int p, double* par) {
    double dvd = A.dv * A.dv;
    if (D == 3) dvd *= A.dv;
    const double rho = s[0] * dvd;
    double U[D], uu = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) { U[a] = s[1 + a] / s[0]; uu += U[a] * U[a]; }
    const double e3 = s[1 + D] * dvd - rho * uu;          // 3 rho R T
    const double T = e3 / (3.0 * rho * A.R);
    bool bad = !(rho > 0.0) || !(T > 1e-12);
    if (bad) latch_error(A.err, BGK_E_DEGENERATE_STATE, p);
    const double RT = A.R * T;
    const double lambda = A.kb / (sqrt(2.0) * kPi * rho * A.R * A.dmol * A.dmol);
    const double Cbar = sqrt(8.0 * RT / kPi);
    const double tau = 4.0 * lambda / (kPi * Cbar);
    const double inv = 1.0 / (tau + A.dt);
    const double twoPiRT = 2.0 * kPi * RT;
    const double pref = (D == 3) ? rho / (twoPiRT * sqrt(twoPiRT)) : rho / twoPiRT;
    par[0] = bad ? 1.0 : tau * inv;   // a1: degenerate rows are left as ftilde
    par[1] = bad ? 0.0 : A.dt * inv;  // a2
    par[2] = pref;
    par[3] = RT;
    par[4] = 1.0 / (2.0 * RT);
#pragma unroll
    for (int a = 0; a < D; ++a) par[5 + a] = U[a];
    double* mo = A.macro + (int64_t)p * (D + 2);
    mo[0] = rho;
#pragma unroll
    for (int a = 0; a < D; ++a) mo[1 + a] = U[a];
    mo[1 + D] = T;
    if (A.ale && !bad) {
#pragma unroll
        for (int a = 0; a < D; ++a) {
            A.W[(int64_t)p * D + a] = U[a];
            double xn = A.x[(int64_t)p * D + a] + A.dt * U[a];
            xn = fmin(fmax(xn, A.clamp_eps), A.L - A.clamp_eps);
            A.x[(int64_t)p * D + a] = xn;
        }
    }
}


}  // namespace bgk
