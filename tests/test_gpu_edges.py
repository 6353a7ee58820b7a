"""GPU edge cases against the oracle: the smallest velocity grids, clouds of a few particles,
a partial second 32-column group in 3D, neighbour-capacity overflow, and a coarse grid that
drives the state degenerate (the error surfaces at the same step and particle as the oracle's).

Bars as in test_gpu_parity.py (BASELINE.json north_star): f, rho, U, T within 1e-10 after 5 steps;
error codes and the reported particle exact.
"""
import math

import numpy as np
import pytest

import bgk_inputs as bi
import oracle

pytestmark = pytest.mark.gpu

TOL = 1e-10
SIG = math.sqrt(bi.R_GAS * bi.T0)


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    oracle.build()
    return torch


def gpu(cfg, cloud, **kw):
    from paper_2408_02350_b200 import Bgk
    return Bgk(cfg, cloud, device="cuda:0", **kw)


def rel(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


SMALL = [
    bi.CavityConfig("nv2_2d", 2, 15, 2, dt=4e-12),                # 3 nodes per axis (2D: 3 columns)
    bi.CavityConfig("nv3_3d", 3, 8, 3, dt=4e-12),                 # 16 of 32 lanes in the only group
    bi.CavityConfig("nv5_3d", 3, 8, 5, jitter=0.1, dt=4e-12),     # 36 columns: a 4-column second group
    bi.CavityConfig("small2d", 2, 6, 10, dt=4e-12),               # 16 interior particles
    bi.CavityConfig("small3d", 3, 5, 4, dt=4e-12),                # 27 interior particles
]


@pytest.mark.parametrize("cfg", SMALL, ids=[c.name for c in SMALL])
def test_small_grids_and_clouds(torch_cuda, cfg):
    cloud = bi.make_cloud(cfg)
    g = gpu(cfg, cloud)
    g.step(5)
    g.sync()
    ref = oracle.run_steps(cfg, 5, cloud)
    assert rel(g.get_f().reshape(g.N, -1), ref.f) <= TOL
    assert np.abs(g.positions() - ref.x).max() <= 1e-12 * cfg.dx
    rho, U, T = g.moments()
    r0, u0, t0 = ref.moments()
    assert np.abs(rho / r0 - 1).max() <= TOL
    assert np.abs(U - u0).max() / SIG <= TOL
    assert np.abs(T / t0 - 1).max() <= TOL


def test_neighbor_capacity_reported(torch_cuda):
    """max_neighbors below the stencil size (~29 in 2D at h = 3.1 dx): BGK_E_CAPACITY, not a
    truncated list."""
    from paper_2408_02350_b200 import BgkError
    cfg = bi.C1
    cloud = bi.make_cloud(cfg)
    with pytest.raises(BgkError) as ei:
        g = gpu(cfg, cloud, max_neighbors=8)
        g.step(1)
        g.sync()
    assert ei.value.status == 2
    off, _ = oracle.neighbors(cloud["x"], cfg.h2)
    assert ei.value.particle == int(np.nonzero(np.diff(off) > 8)[0][0])
    # the context stays usable: a fresh one with the default capacity steps normally
    g = gpu(cfg, cloud)
    g.step(1)
    g.sync()


def test_coarse_grid_degenerate_state_matches_oracle(torch_cuda):
    """N_v = 2 in 3D (3 nodes per axis): the lid-driven state turns degenerate (T <= 1e-12 K or
    rho <= 0).  Both sides stop at the same step with the same (smallest)
    particle."""
    from paper_2408_02350_b200 import BgkError
    cfg = bi.CavityConfig("nv2_3d", 3, 8, 2, dt=4e-12)
    cloud = bi.make_cloud(cfg)
    s = oracle.State(oracle.make_cfg(cfg), cloud)
    ref_step = ref_bad = None
    for k in range(8):
        try:
            s.step(1)
        except oracle.OracleError as e:
            ref_step, ref_bad = k, e.bad
            assert e.code == 4
            break
    assert ref_step is not None
    g = gpu(cfg, cloud)
    for k in range(ref_step):
        g.step(1)
        g.sync()
    with pytest.raises(BgkError) as ei:
        g.step(1)
        g.sync()
    assert ei.value.status == 4 and ei.value.particle == ref_bad


@pytest.mark.parametrize("n, nv", [(10, 8), (9, 24)])
def test_offlattice_wall_points_and_ragged_tiles(torch_cuda, n, nv):
    """3D boundary interpolation on face tiles (k_bnd_interp_s): wall points moved along their face
    (seeded, up to 0.3 dx; edges and corners stay) so no face row holds more than one point and every
    tile is a ragged column of rows; n = 9 gives 7-wide faces (tiles of 4 and 3).  N_v = 24 is C5's
    velocity grid (per-wall chunk plans of 11 chunks).  Five ALE steps against the oracle."""
    cfg = bi.CavityConfig(f"offlat{n}_{nv}", 3, n, nv, dt=5e-12)
    cloud = bi.make_cloud(cfg)
    x, kind = cloud["x"].copy(), cloud["kind"]
    rng = np.random.Generator(np.random.PCG64(2408023511))
    dx = cfg.dx
    on = np.stack([(np.abs(x[:, a]) < 1e-12 * cfg.L) | (np.abs(x[:, a] - cfg.L) < 1e-12 * cfg.L)
                   for a in range(3)], axis=1)
    face = (kind > 0) & (on.sum(axis=1) == 1)
    for a in range(3):
        sel = face & ~on[:, a]
        x[sel, a] += rng.uniform(-0.3, 0.3, size=int(sel.sum())) * dx
    cloud = dict(cloud, x=x)
    cloud.update(zip(("rho", "U", "T"), bi.initial_fields(cfg, x)))
    g = gpu(cfg, cloud)
    g.step(5)
    g.sync()
    ref = oracle.run_steps(cfg, 5, cloud)
    f = g.get_f().reshape(g.N, -1)
    assert rel(f, ref.f) <= TOL, rel(f, ref.f)
    rho, U, T = g.moments()
    r0, u0, t0 = ref.moments()
    assert np.abs(rho / r0 - 1).max() <= TOL
    assert np.abs(U - u0).max() / SIG <= TOL
    assert np.abs(T / t0 - 1).max() <= TOL
    g.close()
