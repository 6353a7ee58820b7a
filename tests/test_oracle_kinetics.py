"""Oracle pins: Maxwellian (A2/A8), moments (O6), tau (O7), relaxation (O8).  CPU only."""
import math
import os

import numpy as np
import pytest

import bgk_inputs as bi

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SIG = math.sqrt(bi.R_GAS * bi.T0)


def _paper():
    out = {}
    for line in open(os.path.join(GOLD, "paper_values.txt")):
        if line.startswith("#") or not line.strip():
            continue
        p = [s.strip() for s in line.split("|")]
        out[p[0]] = p[1:]
    return out


def cfg(dims, Nv, vmax):
    return bi.CavityConfig("t", dims, 5, Nv, vmax=vmax)


def test_tau_paper_values(oracle_lib):
    g = _paper()
    c = oracle_lib.make_cfg(bi.C1)
    for key, rho in (("tau_rho1_T270", 1.0), ("tau_rho0.1_T270", 0.1)):
        val, tol = float(g[key][0]), float(g[key][1])
        t, _ = oracle_lib.tau(c, rho, 270.0)
        assert abs(t / val - 1.0) < tol, (key, t)


def test_rho0_matches_knudsen(oracle_lib):
    """The literal rho0 values of bgk_inputs give lambda/L = Kn (Z13)."""
    c = oracle_lib.make_cfg(bi.C1)
    for Kn, rho0 in bi.RHO0_BY_KN.items():
        _, lam = oracle_lib.tau(c, rho0, 270.0)
        assert abs(lam / bi.L_CAVITY / Kn - 1.0) < 1e-14
    # tau scales as 1/rho and as 1/sqrt(T)
    t1, _ = oracle_lib.tau(c, 1.0, 270.0)
    t2, _ = oracle_lib.tau(c, 0.5, 270.0)
    t3, _ = oracle_lib.tau(c, 1.0, 4 * 270.0)
    assert abs(t2 / t1 - 2.0) < 1e-14 and abs(t1 / t3 - 2.0) < 1e-14


def _center(Nv, d):
    n = Nv + 1
    k = 0
    for _ in range(d):
        k = k * n + Nv // 2
    return k


def test_maxwellian_peak_symmetry_and_G2(oracle_lib):
    rho, T = 0.7, 300.0
    for d in (2, 3):
        c = oracle_lib.make_cfg(cfg(d, 12, bi.VMAX_DEFAULT))
        K = oracle_lib.num_nodes(c)
        M = oracle_lib.maxwellian_row(c, rho, np.zeros(d), T)
        peak = rho / (2 * math.pi * bi.R_GAS * T) ** (d / 2.0 if d == 3 else 1.0)
        assert abs(M[_center(12, d)] / peak - 1.0) < 1e-15
        np.testing.assert_allclose(M[:K], M[:K][::-1], rtol=1e-13)   # M(v) = M(-v) at U = 0
        assert np.all(M[:K] > 0) and M[:K].max() == M[_center(12, d)]
        if d == 2:
            np.testing.assert_allclose(M[K:] / M[:K], bi.R_GAS * T, rtol=1e-15)
    # rho = 1, 2RT = 1, U = 0 -> G1(0) = 1/pi
    c = oracle_lib.make_cfg(cfg(2, 2, 1.0))
    c.R = 1.0
    G = oracle_lib.maxwellian_row(c, 1.0, np.zeros(2), 0.5)
    assert abs(G[4] - 1.0 / math.pi) < 1e-16


def test_maxwellian_one_axis_decay(oracle_lib):
    """Along an axis through U the ratio to the peak is exp(-(v-U)^2/(2RT)) (Z1)."""
    c = oracle_lib.make_cfg(cfg(3, 12, bi.VMAX_DEFAULT))
    U = np.zeros(3)
    M = oracle_lib.maxwellian_row(c, 1.0, U, 270.0)
    ax = oracle_lib.axis_nodes(c)
    n = 13
    for j in range(n):
        k = (6 * n + 6) * n + j
        assert abs(M[k] / M[_center(12, 3)] - math.exp(-ax[j] ** 2 / (2 * bi.R_GAS * 270.0))) < 1e-15


@pytest.mark.parametrize("d,Nv", [(3, 24), (2, 32), (3, 23), (2, 31)])
def test_moment_quadrature_wide_grid_exact(oracle_lib, d, Nv):
    """On a wide fine grid the rectangle rule of a Gaussian is exact to ~1e-15
    (SURVEY appendix), so moments(M(rho,U,T)) returns (rho,U,T).  Odd Nv (no zero node, the
    paper's Nv = 15 grids of Figs. 6-7): the trapezoid/rectangle rule of a Gaussian
    with dv < sigma is exact to exp(-2 pi^2 sigma^2/dv^2) for any grid offset."""
    c = oracle_lib.make_cfg(cfg(d, Nv, 8 * SIG + 1))
    rng = np.random.default_rng(d)
    for _ in range(5):
        rho = rng.uniform(0.01, 2.0)
        T = rng.uniform(230, 310)
        U = rng.uniform(-20, 20, size=d)
        r, u, t = oracle_lib.moments_row(c, oracle_lib.maxwellian_row(c, rho, U, T))
        # tail truncation at vmax = 8 sigma0 + 1 for T up to 310 K is ~1e-13
        assert abs(r / rho - 1) < 1e-12
        assert np.abs(u - U).max() / SIG < 1e-12
        assert abs(t / T - 1) < 1e-12


@pytest.mark.parametrize("d,Nv", [(3, 24), (3, 16), (2, 12), (2, 32)])
def test_moment_quadrature_workload_grid_separable(oracle_lib, d, Nv):
    """Workload grid (vmax = 4 sigma + 1): the d-dimensional node sum equals the
    product of 1D sums of the separable Gaussian; the defect is within the
    SPEC round-trip tolerance 1e-3."""
    c = oracle_lib.make_cfg(cfg(d, Nv, bi.VMAX_DEFAULT))
    ax = oracle_lib.axis_nodes(c)
    dv = oracle_lib.dv(c)
    rho, T = 1.0, 270.0
    U = np.array([1.0, 0.0, 0.0])[:d]
    r, u, t = oracle_lib.moments_row(c, oracle_lib.maxwellian_row(c, rho, U, T))
    s2 = 2 * bi.R_GAS * T
    one = [np.exp(-(ax - U[a]) ** 2 / s2) for a in range(d)]
    pref = rho / (math.pi * s2) ** (d / 2.0)
    r_sep = pref * np.prod([o.sum() * dv for o in one])
    assert abs(r / r_sep - 1) < 1e-13
    assert abs(r / rho - 1) < 1e-3 and abs(t / T - 1) < 1e-3
    assert abs(r / rho - 1) > 1e-7   # the truncation defect is real on this grid (SURVEY §0 finding 5)


def test_moments_homogeneity_and_g2(oracle_lib):
    c3 = oracle_lib.make_cfg(cfg(3, 12, bi.VMAX_DEFAULT))
    f = oracle_lib.maxwellian_row(c3, 0.4, np.array([5.0, -3.0, 2.0]), 280.0)
    r1, u1, t1 = oracle_lib.moments_row(c3, f)
    r2, u2, t2 = oracle_lib.moments_row(c3, 2 * f)
    assert r2 == 2 * r1 and np.allclose(u1, u2, rtol=1e-15) and abs(t2 / t1 - 1) < 1e-15
    c2 = oracle_lib.make_cfg(cfg(2, 12, bi.VMAX_DEFAULT))
    K = oracle_lib.num_nodes(c2)
    g = oracle_lib.maxwellian_row(c2, 0.4, np.array([5.0, -3.0]), 280.0)
    r1, u1, t1 = oracle_lib.moments_row(c2, g)
    g2 = g.copy()
    g2[K:] *= 2
    r2, u2, t2 = oracle_lib.moments_row(c2, g2)
    dv = oracle_lib.dv(c2)
    assert r1 == r2 and np.array_equal(u1, u2)
    expect = t1 + g[K:].sum() * dv * dv / (3 * r1 * bi.R_GAS)
    assert abs(t2 / expect - 1) < 1e-13 and t2 > t1
    with pytest.raises(oracle_lib.OracleError):
        oracle_lib.moments_row(c3, np.zeros_like(f))


def test_chu_marginal_consistency(oracle_lib):
    """G1 = int M dv3, G2 = int v3^2 M dv3: marginalise the 3D
    Maxwellian numerically on a wide fine grid and compare with the 2D pair."""
    Nv, vmax = 32, 8 * SIG + 1
    c3 = oracle_lib.make_cfg(cfg(3, Nv, vmax))
    c2 = oracle_lib.make_cfg(cfg(2, Nv, vmax))
    rho, T = 0.3, 260.0
    U3 = np.array([12.0, -7.0, 0.0])
    M = oracle_lib.maxwellian_row(c3, rho, U3, T).reshape(Nv + 1, Nv + 1, Nv + 1)
    G = oracle_lib.maxwellian_row(c2, rho, U3[:2], T)
    K2 = (Nv + 1) ** 2
    ax = oracle_lib.axis_nodes(c3)
    dv = oracle_lib.dv(c3)
    g1 = (M.sum(axis=2) * dv).reshape(-1)
    g2 = ((M * ax[None, None, :] ** 2).sum(axis=2) * dv).reshape(-1)
    np.testing.assert_allclose(g1, G[:K2], rtol=1e-12, atol=1e-14 * G[:K2].max())
    np.testing.assert_allclose(g2, G[K2:], rtol=1e-12, atol=1e-14 * G[K2:].max())
    # and the reduced moments equal the 3D moments
    r3, u3, t3 = oracle_lib.moments_row(c3, M.reshape(-1))
    r2, u2, t2 = oracle_lib.moments_row(c2, np.concatenate([g1, g2]))
    assert abs(r2 / r3 - 1) < 1e-13 and np.abs(u2 - u3[:2]).max() < 1e-10 and abs(t2 / t3 - 1) < 1e-13


def test_relax_identities(oracle_lib):
    rng = np.random.default_rng(0)
    ft = rng.uniform(0, 1, 1000)
    M = rng.uniform(0, 1, 1000)
    out = oracle_lib.relax_row(3e-10, 1e-11, M, M)
    np.testing.assert_allclose(out, M, rtol=5e-16)
    out = oracle_lib.relax_row(1e-11, 1e-11, ft, M)
    np.testing.assert_allclose(out, (ft + M) / 2, rtol=5e-16)
    out = oracle_lib.relax_row(3e-10, 1e-11, ft, M)
    assert np.all(out >= np.minimum(ft, M) * (1 - 1e-15)) and np.all(out <= np.maximum(ft, M) * (1 + 1e-15))
    out = oracle_lib.relax_row(3e-10, 0.0, ft, M)
    np.testing.assert_allclose(out, ft, rtol=5e-16)


@pytest.mark.parametrize("d,Nv", [(3, 24), (2, 32)])
def test_relaxation_conserves_on_wide_grid(oracle_lib, d, Nv):
    """mom(f^{n+1}) = (tau mom(ft) + dt mom(M))/(tau + dt) and mom(M) = mom(ft)
    on the wide grid -> mass, momentum, energy conserved to 1e-12."""
    c = oracle_lib.make_cfg(cfg(d, Nv, 8 * SIG + 1))
    # a non-Maxwellian ft: sum of two shifted Maxwellians
    ft = oracle_lib.maxwellian_row(c, 0.5, np.full(d, 40.0), 250.0) + \
        oracle_lib.maxwellian_row(c, 0.3, np.full(d, -60.0), 320.0)
    r, u, t = oracle_lib.moments_row(c, ft)
    tau_, _ = oracle_lib.tau(c, r, t)
    M = oracle_lib.maxwellian_row(c, r, u, t)
    f1 = oracle_lib.relax_row(tau_, 1e-11, ft, M)
    r1, u1, t1 = oracle_lib.moments_row(c, f1)
    assert abs(r1 / r - 1) < 1e-12 and np.abs(u1 - u).max() / SIG < 1e-12 and abs(t1 / t - 1) < 1e-12
    assert abs(f1 - ft).max() > 1e-6 * ft.max()   # the relaxation did move f
