"""Oracle pins for the whole step (O1-O11) and the diffuse-reflection wall.  CPU only."""
import math

import numpy as np
import pytest

import bgk_inputs as bi
import oracle

SIG = math.sqrt(bi.R_GAS * bi.T0)


def _state(cfg, **kw):
    cloud = bi.make_cloud(cfg)
    for k, v in kw.items():
        cloud[k] = v
    return oracle.State(oracle.make_cfg(cfg), cloud)


def _wall_flux(c, s):
    """sum_k (v.n) f_bk for each boundary particle, and the scale sum |v.n| f."""
    V = oracle.node_velocities(c)
    K = oracle.num_nodes(c)
    out = []
    for b in np.nonzero(s.kind != 0)[0]:
        n = oracle.wall_normal(c.dims, int(s.kind[b]))
        vn = V @ n
        f = s.f[b, :K]
        out.append(((vn * f).sum(), (np.abs(vn) * f).sum()))
    return np.array(out)


@pytest.mark.parametrize("cfg", [bi.C1, bi.CavityConfig("c4small", 3, 7, 8)])
def test_zero_wall_mass_flux_every_step(oracle_lib, cfg):
    s = _state(cfg)
    for _ in range(3):
        s.step(1)
        fl = _wall_flux(s.c, s)
        assert np.all(np.abs(fl[:, 0]) <= 1e-12 * fl[:, 1])


def test_diffuse_equilibrium_reproduces_wall_maxwellian(oracle_lib):
    """Interior at the wall Maxwellian (rho, U_w, T_w) -> boundary row = rho M_w and
    rho_w = rho; checked on the moving lid (wall 4, 2D) and a side wall."""
    c = oracle.make_cfg(bi.C1)
    x, kind = bi.lattice(bi.C1)
    off, idx = oracle.neighbors(x, c.h2)
    cw = oracle.boundary_weights(x, kind, off, idx, c.h2)
    for wid in (4, 1):
        b = int(np.nonzero(kind == wid)[0][5])
        Uw = np.array([1.0, 0.0]) if wid == 4 else np.zeros(2)
        Mw = oracle.maxwellian_row(c, 0.37, Uw, bi.T0)
        nb = idx[off[b]:off[b + 1]]
        rows = [Mw if kind[j] == 0 else None for j in nb]
        fb, rw = oracle.diffuse_one(c, wid, cw[off[b]:off[b + 1]], rows)
        assert abs(rw / 0.37 - 1) < 1e-13
        np.testing.assert_allclose(fb, Mw, rtol=1e-12, atol=1e-14 * Mw.max())


def test_single_node_beam_balanced(oracle_lib):
    """Stationary wall, incoming beam at one node: outgoing half is M_w scaled to
    cancel the beam's flux exactly."""
    c = oracle.make_cfg(bi.C1)
    K = oracle.num_nodes(c)
    V = oracle.node_velocities(c)
    n = oracle.wall_normal(2, 1)               # wall x = 0, normal +x
    kin = int(np.nonzero((V @ n) < 0)[0][7])
    beam = np.zeros(2 * K)
    beam[kin] = 2.5
    fb, rw = oracle.diffuse_one(c, 1, np.array([1.0]), [beam])
    Mw = oracle.maxwellian_row(c, 1.0, np.zeros(2), bi.T0)
    vn = V @ n
    out = vn > 0
    assert abs(rw - (-(vn[kin] * 2.5) / (vn[out] * Mw[:K][out]).sum())) < 1e-15 * abs(rw)
    assert abs((vn * fb[:K]).sum()) < 1e-13 * 2.5 * abs(vn[kin])


def test_dt_zero_is_identity_on_interior(oracle_lib):
    cfg = bi.C1.replace(dt=0.0)
    s = _state(cfg)
    f0, x0 = s.f.copy(), s.x.copy()
    s.step(1)
    inter = s.kind == 0
    np.testing.assert_allclose(s.f[inter], f0[inter], rtol=4e-16, atol=0)
    assert np.array_equal(s.x, x0)


@pytest.mark.parametrize("cfg,steps", [
    (bi.CavityConfig("eq2", 2, 15, 32, vmax=8 * SIG + 1, lid=0.0, init="equilibrium"), 10),
    (bi.CavityConfig("eq3", 3, 6, 24, vmax=8 * SIG + 1, lid=0.0, init="equilibrium"), 2),
])
def test_equilibrium_fixed_point_wide_grid(oracle_lib, cfg, steps):
    """A uniform Maxwellian at rest with stationary walls at T0 stays put to 1e-12
    on a wide grid (SURVEY §8(c) whole-step pin)."""
    s = _state(cfg)
    r0, u0, t0 = s.moments()
    s.step(steps)
    r, u, t = s.moments()
    assert np.abs(r / r0 - 1).max() < 1e-12
    assert np.abs(u).max() / SIG < 1e-12
    assert np.abs(t / t0 - 1).max() < 1e-12
    assert np.abs(s.x - bi.lattice(cfg)[0]).max() < 1e-12 * cfg.dx


def test_equilibrium_drift_on_workload_grid(oracle_lib):
    """On the narrow workload grid the drift is bounded by n dt/(tau+dt) x the grid
    defect: 10 steps of C1 at rest stay within 1e-5."""
    cfg = bi.C1.replace(lid=0.0, init="equilibrium")
    s = _state(cfg)
    r0, u0, t0 = s.moments()
    s.step(10)
    r, u, t = s.moments()
    assert np.abs(r / r0 - 1).max() < 1e-5 and np.abs(t / t0 - 1).max() < 1e-5


def test_interior_positivity_and_ale_motion(oracle_lib):
    cfg = bi.C1
    s = _state(cfg)
    x0 = s.x.copy()
    s.step(1)
    inter = s.kind == 0
    assert s.f[inter].min() >= 0.0
    U = s.macro[:, 1:3]
    np.testing.assert_allclose(s.x[inter], x0[inter] + cfg.dt * U[inter], rtol=0, atol=1e-22)
    assert np.array_equal(s.W[inter], U[inter])
    assert np.array_equal(s.x[~inter], x0[~inter])


def test_fixed_cloud_mode_keeps_positions(oracle_lib):
    cfg = bi.C1.replace(ale=0)
    s = _state(cfg)
    x0 = s.x.copy()
    s.step(2)
    assert np.array_equal(s.x, x0) and np.all(s.W == 0.0)


def test_thread_count_does_not_change_results(oracle_lib):
    cfg = bi.C1
    n = oracle.omp_threads()
    oracle.set_threads(1)
    a = _state(cfg).step(2)
    oracle.set_threads(max(n, 4))
    b = _state(cfg).step(2)
    oracle.set_threads(n)
    assert np.array_equal(a.f, b.f) and np.array_equal(a.x, b.x)


def test_sampled_step_matches_full_step(oracle_lib):
    """The sampled driver (used at full size) reproduces the whole-cloud step."""
    cfg = bi.CavityConfig("s3", 3, 8, 6)
    cloud = bi.make_cloud(cfg)
    full = oracle.State(oracle.make_cfg(cfg), cloud).step(1)
    sample = [0, 9, 73, 200, 511, int(np.nonzero(cloud["kind"] == 6)[0][4])]
    got = oracle.sampled_first_step(cfg, cloud, sample)
    for i in sample:
        np.testing.assert_array_equal(got[i]["f"], full.f[i])
        np.testing.assert_array_equal(got[i]["x"], full.x[i])
