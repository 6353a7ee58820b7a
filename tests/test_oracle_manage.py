"""Oracle pins for particle management ("Adding and removing points"; SPEC.md:283-358;
DESIGN.md Z28): the WLS interpolation of a new point, the greedy merge, the hole fill and the
compaction order.  CPU only.

What pins what (none of these re-types the oracle's arithmetic):
  * interpolation -- constants and linear fields reproduced (the fit's definition), a0 equal to an
    independent dense weighted least-squares solve (numpy lstsq), deficiency on collinear /
    too-small stencils;
  * merge -- closed-form geometry (exact midpoint in the smaller slot, every other particle
    unchanged and in order), constant fields stay constant, greedy ascending pairing;
  * fill -- the rules checked directly on the output (offset +-0.5h from a deficient particle,
    inside the box, farther than 0.45 dx from every particle) and linear fields reproduced;
  * whole steps -- the equilibrium fixed point survives managed steps.
"""
import math

import numpy as np
import pytest

import bgk_inputs as bi
import oracle

SIG = math.sqrt(bi.R_GAS * bi.T0)


def _state(cfg, cloud=None):
    cloud = cloud if cloud is not None else bi.make_cloud(cfg)
    return oracle.State(oracle.make_cfg(cfg), cloud), cloud


# ------------------------------------------------------------ interpolation
@pytest.mark.parametrize("d,seed", [(2, 1), (3, 2)])
def test_interp_reproduces_constants_and_linears(oracle_lib, d, seed):
    rng = np.random.default_rng(seed)
    h = 0.31
    x = rng.uniform(-0.3, 0.3, size=(60, d))
    p = rng.uniform(-0.05, 0.05, size=d)
    S = np.nonzero(((x - p) ** 2).sum(1) <= h * h)[0]
    st, c = oracle.interp_weights(x, S, p, h * h, bi.ALPHA_W)
    assert st == 0
    assert abs(c.sum() - 1.0) < 1e-13
    np.testing.assert_allclose(c @ x[S], p, rtol=0, atol=1e-13)
    a, b = 0.7, rng.normal(size=d)
    f = a + x[S] @ b
    assert abs(c @ f - (a + p @ b)) < 1e-13


def test_interp_matches_dense_weighted_lstsq(oracle_lib):
    """a0 of the weighted fit f ~ a0 + a.(x - p), solved independently with lstsq."""
    rng = np.random.default_rng(5)
    d, h = 3, 0.3
    x = rng.uniform(-0.25, 0.25, size=(80, d))
    p = np.array([0.01, -0.02, 0.015])
    S = np.nonzero(((x - p) ** 2).sum(1) <= h * h)[0]
    f = np.sin(3 * x[S, 0]) + x[S, 1] ** 2 - 0.5 * x[S, 2] * x[S, 0]
    st, c = oracle.interp_weights(x, S, p, h * h, bi.ALPHA_W)
    assert st == 0
    w = np.exp(-bi.ALPHA_W * ((x[S] - p) ** 2).sum(1) / (h * h))
    M = np.column_stack([np.ones(len(S)), (x[S] - p) / h])
    sol, *_ = np.linalg.lstsq(M * np.sqrt(w)[:, None], f * np.sqrt(w), rcond=None)
    assert abs(c @ f - sol[0]) < 1e-12 * max(1.0, abs(sol[0]))


def test_interp_deficient_stencils(oracle_lib):
    # collinear points in 2D: the fit (1, x, y) is rank deficient
    t = np.linspace(-0.2, 0.2, 9)
    x = np.column_stack([t, 2 * t])
    st, _ = oracle.interp_weights(x, np.arange(9), np.zeros(2), 0.3 ** 2, bi.ALPHA_W)
    assert st == 3
    # fewer than d + 2 members
    x = np.array([[0.1, 0.0], [0.0, 0.1], [-0.1, -0.1]])
    st, _ = oracle.interp_weights(x, np.arange(3), np.zeros(2), 0.3 ** 2, bi.ALPHA_W)
    assert st == 3


# ---------------------------------------------------------------- merging
def _pair_cloud(cfg, shift=0.95):
    """Regular lattice with one interior particle moved `shift` dx towards its +x neighbour."""
    cloud = bi.make_cloud(cfg)
    n = cfg.n_per_axis
    i = (n // 2) + n * (n // 2) + (n * n * (n // 2) if cfg.dims == 3 else 0)
    assert cloud["kind"][i] == 0 and cloud["kind"][i + 1] == 0
    cloud["x"] = cloud["x"].copy()
    cloud["x"][i, 0] += shift * cfg.dx
    return cloud, i


@pytest.mark.parametrize("dims,n", [(2, 15), (3, 9)])
def test_merge_pair_to_midpoint(oracle_lib, dims, n):
    cfg = bi.CavityConfig("mp", dims, n, 6, init="equilibrium", manage=1)
    cloud, i = _pair_cloud(cfg)
    s, _ = _state(cfg, cloud)
    x0, f0 = s.x.copy(), s.f.copy()
    rep = s.manage(cfg.merge_radius, cfg.min_neighbors, cfg.capacity)
    N = len(x0)
    assert rep == (1, 0, 0, 0, 0, N - 1)
    mid = (x0[i] + x0[i + 1]) * 0.5
    assert np.array_equal(s.x[i], mid)
    keep = np.r_[0:i, i + 2:N]
    out = np.r_[0:i, i + 1:N - 1]
    assert np.array_equal(s.x[out], x0[keep])
    assert np.array_equal(s.f[out], f0[keep])
    # uniform Maxwellian everywhere: the interpolated row is that row (sum c = 1)
    assert np.abs(s.f[i] - f0[0]).max() <= 1e-13 * np.abs(f0[0]).max()
    assert s.kind[i] == 0 and len(s.kind) == N - 1


def test_no_change_on_regular_lattice(oracle_lib):
    cfg = bi.C1.replace(manage=1)
    s, _ = _state(cfg)
    x0, f0 = s.x.copy(), s.f.copy()
    rep = s.manage(cfg.merge_radius, cfg.min_neighbors, cfg.capacity)
    assert rep == (0, 0, 0, 0, 0, len(x0))
    assert np.array_equal(s.x, x0) and np.array_equal(s.f, f0)


def test_merge_is_greedy_in_index_order(oracle_lib):
    """Three interior particles pairwise closer than r_merge: the smallest index pairs with the
    next one; the third stays (SPEC.md:324 greedy ascending pass)."""
    cfg = bi.CavityConfig("g3", 2, 15, 6, init="equilibrium", manage=1)
    cloud = bi.make_cloud(cfg)
    n, dx = cfg.n_per_axis, cfg.dx
    i = 7 + 7 * n
    cloud["x"] = cloud["x"].copy()
    cloud["x"][i + 1] = cloud["x"][i] + [0.05 * dx, 0.0]
    cloud["x"][i + n] = cloud["x"][i] + [0.0, 0.08 * dx]
    s, _ = _state(cfg, cloud)
    x0 = s.x.copy()
    rep = s.manage(cfg.merge_radius, cfg.min_neighbors, cfg.capacity)
    assert rep[0] == 1
    assert np.array_equal(s.x[i], (x0[i] + x0[i + 1]) * 0.5)
    assert np.array_equal(s.x[i + n - 1], x0[i + n])        # survived, shifted down by one slot


# ------------------------------------------------------------------ filling
@pytest.mark.parametrize("dims,n,m_min", [(2, 17, 27), (3, 10, 118)])
def test_fill_rules_and_linear_reproduction(oracle_lib, dims, n, m_min):
    cfg = bi.CavityConfig("fh", dims, n, 4, init="equilibrium", manage=1, m_min=m_min, jitter=0.05)
    cloud = bi.make_cloud(cfg)
    # cut a 2^d hole in the middle
    c0 = n // 2
    offs = np.array(np.meshgrid(*([[0, 1]] * dims), indexing="ij")).reshape(dims, -1).T
    stride = np.array([n ** a for a in range(dims)])
    hole = (c0 + offs) @ stride
    keep = np.setdiff1d(np.arange(len(cloud["x"])), hole)
    for k in ("x", "kind", "rho", "U", "T"):
        cloud[k] = cloud[k][keep]
    s, _ = _state(cfg, cloud)
    x0 = s.x.copy()
    N = len(x0)
    # a linear field in every node: f_k(x) = 1 + (k + 1) x.b / L
    b = np.linspace(0.3, 0.9, dims)
    s.f[:] = 1.0 + np.outer(x0 @ b / cfg.L, np.arange(1, s.f.shape[1] + 1))
    off, idx = oracle.neighbors(x0, cfg.h2)
    cnt = np.diff(off)
    rep = s.manage(cfg.merge_radius, cfg.min_neighbors, cfg.capacity)
    assert rep[0] == 0 and rep[2] > 0 and rep[5] == N + rep[2]
    assert np.array_equal(s.x[:N], x0)
    new = s.x[N:]
    assert np.all(s.kind[N:] == 0)
    assert np.all((new > 0) & (new < cfg.L))
    hh = 0.5 * cfg.h
    deficient = np.nonzero((cloud["kind"] == 0) & (cnt < m_min))[0]
    for p in new:
        # an axis offset +-0.5 h of a deficient particle
        dpos = p[None, :] - x0[deficient]
        ok = [(np.sum(np.abs(dd) > 0) == 1 and np.isclose(np.abs(dd).max(), hh, rtol=0, atol=1e-12 * cfg.L))
              for dd in dpos]
        assert any(ok)
        # farther than 0.45 dx from every other particle of the output cloud
        d2 = ((s.x - p) ** 2).sum(1)
        assert np.sort(d2)[1] > (0.45 * cfg.dx) ** 2
    expect = 1.0 + np.outer(new @ b / cfg.L, np.arange(1, s.f.shape[1] + 1))
    assert np.abs(s.f[N:] - expect).max() <= 1e-12 * np.abs(expect).max()


def test_fill_capacity_is_reported(oracle_lib):
    cfg = bi.CavityConfig("fc", 2, 17, 4, init="equilibrium", manage=1, m_min=27, jitter=0.05)
    s, cloud = _state(cfg)
    N = len(s.x)
    big = oracle.State(oracle.make_cfg(cfg), cloud)
    full = big.manage(cfg.merge_radius, cfg.min_neighbors, 10 * N)
    rep = s.manage(cfg.merge_radius, cfg.min_neighbors, N + 3)
    assert full[2] > 3
    # the first three inserts are those of the unbounded pass; every later accepted candidate
    # (at least the unbounded pass's remaining inserts) is reported as over capacity
    assert rep[2] == 3 and rep[5] == N + 3 and rep[4] >= full[2] - 3
    assert np.array_equal(s.x[N:], big.x[N:N + 3])


# --------------------------------------------------------------- whole steps
def test_equilibrium_fixed_point_with_management(oracle_lib):
    """Resting equilibrium (lid off) on a cloud with close pairs and holes: the merges
    interpolate the uniform state exactly (sum c = 1), so managed steps stay at the fixed point."""
    cfg = bi.CavityConfig("eq", 2, 21, 32, init="equilibrium", lid=0.0, manage=1, defects=2, m_min=21,
                          vmax=8 * SIG + 1, jitter=0.05)
    s, _ = _state(cfg)
    s.manage_params = oracle.manage_params(cfg)
    r0, _, t0 = s.moments()
    s.step(3)
    assert s.reports[0][0] >= 1 and s.reports[0][2] >= 1
    rho, U, T = s.moments()
    assert np.abs(rho / r0[0] - 1).max() < 1e-12
    assert np.abs(U).max() / SIG < 1e-12
    assert np.abs(T / t0[0] - 1).max() < 1e-12


# ------------------------------------------------------------ wall fills (Z30)
def _depleted_corner(dims, n):
    """A lattice whose corner x = 0, y = L (2D) / origin (3D) has lost interior neighbours: the
    interior lattice points nearest to it are removed, leaving its interpolation stencil with
    fewer than d + 2 members (the lattice corner has 4 in 2D and 7 in 3D)."""
    cfg = bi.CavityConfig("wc", dims, n, 4, init="equilibrium", manage=1)
    cloud = bi.make_cloud(cfg)
    x, dx, L = cloud["x"], cfg.dx, cfg.L
    corner = np.zeros(dims)
    if dims == 2:
        corner[1] = L
    ii = np.rint(np.abs(x - corner) / dx).astype(int)            # lattice offsets from the corner
    # 2D: the nearest interior point (4 -> 3 left); 3D: (1,1,1), (1,1,2), (1,2,1) (7 -> 4 left)
    gone = [(1, 1)] if dims == 2 else [(1, 1, 1), (1, 1, 2), (1, 2, 1)]
    drop = np.nonzero((cloud["kind"] == 0) & np.any(np.all(ii[:, None, :] == np.array(gone)[None], axis=2),
                                                      axis=1))[0]
    keep = np.setdiff1d(np.arange(len(x)), drop)
    for k in ("x", "kind", "rho", "U", "T"):
        cloud[k] = cloud[k][keep]
    return cfg, cloud, corner


@pytest.mark.parametrize("dims,n", [(2, 15), (3, 9)])
def test_wall_fill_at_a_depleted_corner(oracle_lib, dims, n):
    """Z30: a wall particle whose interpolation system is deficient (here: fewer than d + 2 interior
    neighbours) proposes x_b + 0.5 h (sum of the inward normals); on the depleted corner that point is
    inside the box and clear of every particle (> 0.45 dx), so it is inserted and the corner's
    stencil has d + 2 members again."""
    cfg, cloud, corner = _depleted_corner(dims, n)
    s, _ = _state(cfg, cloud)
    x0 = s.x.copy()
    N = len(x0)
    b = int(np.nonzero(np.all(x0 == corner, axis=1))[0][0])
    off, idx = oracle.neighbors(x0, cfg.h2)
    n_int = int((cloud["kind"][idx[off[b]:off[b + 1]]] == 0).sum())
    assert n_int < dims + 2
    rep = s.manage(cfg.merge_radius, cfg.min_neighbors, cfg.capacity)
    assert rep[0] == 0 and rep[2] >= 1
    inward = np.where(corner == 0.0, 1.0, -1.0)
    want = corner + 0.5 * cfg.h * inward
    new = s.x[N:]
    assert np.any(np.all(new == want, axis=1)), (new, want)
    assert np.all(s.kind[N:] == 0) and np.all((new > 0) & (new < cfg.L))
    assert np.array_equal(s.x[:N], x0)
    off2, idx2 = oracle.neighbors(s.x, cfg.h2)
    n_int2 = int((s.kind[idx2[off2[b]:off2[b + 1]]] == 0).sum())
    assert n_int2 == n_int + 1 == dims + 2
    # the inserted rows are WLS interpolations: an equilibrium field stays the same Maxwellian row
    assert np.abs(s.f[N:] - s.f[0]).max() <= 1e-10 * np.abs(s.f[0]).max()
