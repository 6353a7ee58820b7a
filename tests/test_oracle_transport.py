"""Oracle pins: positive upwind transport (O5) and stable_dt.  CPU only."""
import numpy as np
import pytest

import bgk_inputs as bi


def _cfg(d, Nv=8, dt=1e-11, vmax=bi.VMAX_DEFAULT):
    return bi.CavityConfig("t", d, 5, Nv, dt=dt, vmax=vmax)


def _stencil_geometry(oracle_lib, x, i, nb, h2):
    S, a = oracle_lib.wls_one(x, i, nb, h2)
    frs = np.stack([oracle_lib.frame(x[j] - x[i]) for j in nb])
    rot = np.stack([oracle_lib.rotate(a[q], frs[q]) for q in range(len(nb))])
    return rot, frs


@pytest.mark.parametrize("d", [2, 3])
def test_cross_stencil_is_first_order_upwind(oracle_lib, d):
    """4-/6-neighbour cross stencil: the scheme reduces to the textbook
    first-order upwind difference  Q = sum_a [c_a^+ (f_i - f_{-a})/dx_a + c_a^- (f_{+a} - f_i)/dx_a]
    (SPEC.md:275, 281)."""
    hx = np.array([2e-8, 3e-8, 2.5e-8])[:d]
    pts = [np.zeros(d)]
    for a in range(d):
        for s in (+1, -1):
            p = np.zeros(d)
            p[a] = s * hx[a]
            pts.append(p)
    x = np.array(pts)
    nb = np.arange(1, 2 * d + 1, dtype=np.int32)
    h2 = (1.01 * hx.max()) ** 2
    rot, frs = _stencil_geometry(oracle_lib, x, 0, nb, h2)
    c = oracle_lib.make_cfg(_cfg(d))
    K = oracle_lib.num_nodes(c)
    nv = 2 if d == 2 else 1
    rng = np.random.default_rng(d)
    rows = [rng.uniform(0.5, 1.5, nv * K) for _ in range(2 * d + 1)]
    W = rng.uniform(-30, 30, d)
    ft = oracle_lib.transport_one(c, W, rot, frs, rows[1:], rows[0])
    V = oracle_lib.node_velocities(c)
    for q in range(nv):
        sl = slice(q * K, (q + 1) * K)
        fi = rows[0][sl]
        Q = np.zeros(K)
        for a in range(d):
            cv = V[:, a] - W[a]
            fp, fm = rows[1 + 2 * a][sl], rows[2 + 2 * a][sl]
            Q += np.maximum(cv, 0) * (fi - fm) / hx[a] + np.minimum(cv, 0) * (fp - fi) / hx[a]
        np.testing.assert_allclose(ft[sl], fi - c.dt * Q, rtol=1e-13, atol=1e-15)


def _lattice_setup(oracle_lib, cfg):
    x, kind = bi.lattice(cfg)
    off, idx = oracle_lib.neighbors(x, cfg.h2)
    S, a, fr, rot = oracle_lib.wls_all(x, kind, off, idx, cfg.h2)
    return x, kind, off, idx, fr, rot


@pytest.mark.parametrize("d,n", [(2, 15), (3, 9)])
def test_uniform_and_zero_velocity(oracle_lib, d, n):
    cfg = bi.CavityConfig("t", d, n, 8)
    x, kind, off, idx, fr, rot = _lattice_setup(oracle_lib, cfg)
    c = oracle_lib.make_cfg(cfg)
    K = oracle_lib.num_nodes(c)
    nv = 2 if d == 2 else 1
    i = int(np.nonzero(kind == 0)[0][3])
    s, e = off[i], off[i + 1]
    rng = np.random.default_rng(1)
    row = rng.uniform(0, 1, nv * K)
    ft = oracle_lib.transport_one(c, np.full(d, 7.0), rot[s:e], fr[s:e], [row] * (e - s), row)
    assert np.array_equal(ft, row)            # f uniform in space -> Q = 0 exactly
    rows = [rng.uniform(0, 1, nv * K) for _ in range(e - s)]
    V = oracle_lib.node_velocities(c)
    k0 = 17
    ft = oracle_lib.transport_one(c, V[k0], rot[s:e], fr[s:e], rows, row)
    for q in range(nv):
        assert ft[q * K + k0] == row[q * K + k0]   # c = v - W = 0 -> Q = 0 exactly
    assert np.abs(ft - row).max() > 0


@pytest.mark.parametrize("d,n", [(2, 15), (3, 10)])
def test_linear_field_exact_on_symmetric_stencils(oracle_lib, d, n):
    """Linear f: on centrally symmetric stencils the dissipation cancels and
    Q = c . grad f (SURVEY §8(c) O5 pin); one-sided wall stencils are not exact."""
    cfg = bi.CavityConfig("t", d, n, 6)
    x, kind, off, idx, fr, rot = _lattice_setup(oracle_lib, cfg)
    c = oracle_lib.make_cfg(cfg)
    K = oracle_lib.num_nodes(c)
    nv = 2 if d == 2 else 1
    V = oracle_lib.node_velocities(c)
    g = np.array([3.0, -2.0, 1.5])[:d] / cfg.dx
    W = np.array([4.0, -6.0, 2.0])[:d]
    ii = np.rint(x / cfg.dx).astype(int)
    errs_sym, errs_wall = [], []
    for i in np.nonzero(kind == 0)[0][::3]:
        s, e = off[i], off[i + 1]
        val = lambda p: np.tile(np.full(K, 10.0 + g @ x[p]), nv)
        ft = oracle_lib.transport_one(c, W, rot[s:e], fr[s:e], [val(j) for j in idx[s:e]], val(i))
        Q = -(ft[:K] - val(i)[:K]) / c.dt
        exact = (V - W) @ g
        err = np.abs(Q - exact).max() / np.abs(exact).max()
        (errs_sym if np.all((ii[i] >= 3) & (ii[i] <= n - 4)) else errs_wall).append(err)
    assert max(errs_sym) < 1e-11
    assert max(errs_wall) > 1e-2


@pytest.mark.parametrize("d,n", [(2, 13), (3, 8)])
def test_coefficients_nonpositive_and_max_principle(oracle_lib, d, n):
    cfg = bi.CavityConfig("t", d, n, 6, jitter=0.25)
    x, kind, off, idx, fr, rot = _lattice_setup(oracle_lib, cfg)
    c = oracle_lib.make_cfg(cfg)
    K = oracle_lib.num_nodes(c)
    nv = 2 if d == 2 else 1
    rng = np.random.default_rng(5)
    W = rng.uniform(-10, 10, d)
    inter = np.nonzero(kind == 0)[0]
    i = int(inter[len(inter) // 2])
    s, e = off[i], off[i + 1]
    m = e - s
    # probe C_ijk: neighbour row j = 1, all else 0 -> ft_i = -dt C_ijk
    zero = np.zeros(nv * K)
    for jj in range(0, m, max(1, m // 6)):
        rows = [zero] * m
        rows = rows[:jj] + [np.ones(nv * K)] + rows[jj + 1:]
        ft = oracle_lib.transport_one(c, W, rot[s:e], fr[s:e], rows, zero)
        Cjk = -ft / c.dt
        assert np.all(Cjk <= 0.0)
    # max principle under dt <= stable_dt (acceptance 4)
    amax = oracle_lib.coef_absmax_one(c, W, rot[s:e], fr[s:e])
    c.dt = 0.95 / amax
    rows = [rng.uniform(0, 1, nv * K) for _ in range(m)]
    fi = rng.uniform(0, 1, nv * K)
    ft = oracle_lib.transport_one(c, W, rot[s:e], fr[s:e], rows, fi)
    lo = np.minimum(fi, np.min(rows, axis=0))
    hi = np.maximum(fi, np.max(rows, axis=0))
    assert np.all(ft >= lo - 1e-14) and np.all(ft <= hi + 1e-14)
    c.dt = 3.0 / amax    # beyond the bound positivity is lost somewhere
    ft = oracle_lib.transport_one(c, W, rot[s:e], fr[s:e], rows, fi)
    assert np.any(ft < lo - 1e-9) or np.any(ft > hi + 1e-9)


def test_stable_dt_c1_regression(oracle_lib):
    """stable_dt of the regular 21^2 cloud at W = 0 (3.38e-11)."""
    cfg = bi.C1
    x, kind, off, idx, fr, rot = _lattice_setup(oracle_lib, cfg)
    c = oracle_lib.make_cfg(cfg)
    amax = max(oracle_lib.coef_absmax_one(c, np.zeros(2), rot[off[i]:off[i + 1]], fr[off[i]:off[i + 1]])
               for i in np.nonzero(kind == 0)[0])
    assert abs(1.0 / amax / 3.38e-11 - 1) < 0.01


@pytest.mark.parametrize("cfg", [bi.C2, bi.C3])
def test_config_dt_within_positivity_cfl(oracle_lib, cfg):
    """The fixed dt of C2/C3 is <= 0.9 stable_dt of the initial (stress) cloud (Z12)."""
    cloud = bi.make_cloud(cfg)
    x, kind = cloud["x"], cloud["kind"]
    off, idx = oracle_lib.neighbors(x, cfg.h2)
    S, a, fr, rot = oracle_lib.wls_all(x, kind, off, idx, cfg.h2)
    c = oracle_lib.make_cfg(cfg)
    amax = max(oracle_lib.coef_absmax_one(c, cloud["U"][i], rot[off[i]:off[i + 1]], fr[off[i]:off[i + 1]])
               for i in np.nonzero(kind == 0)[0])
    assert cfg.dt <= 0.9 / amax
