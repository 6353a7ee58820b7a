"""Particle management on the GPU (Z28) against the oracle.

Bars: the decisions (which pairs merge, which candidates are inserted, the compaction order) are
integer outcomes of the same rounded distance tests on both sides -> reports, kinds and positions
bit-exact after one pass; interpolated rows within 1e-12 of the oracle's (one weighted sum);
after managed ALE steps the usual 1e-10 bar of the step parity tests.
"""
import math

import numpy as np
import pytest

import bgk_inputs as bi
import oracle

pytestmark = pytest.mark.gpu

TOL = 1e-10
SIG = math.sqrt(bi.R_GAS * bi.T0)

M2 = bi.CavityConfig("M2", 2, 21, 12, manage=1, defects=2, m_min=21, jitter=0.05, dt=5e-12)
M3 = bi.CavityConfig("M3", 3, 12, 6, manage=1, defects=2, m_min=84, jitter=0.05, dt=5e-12)


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    oracle.build()
    return torch


def gpu(cfg, cloud):
    from paper_2408_02350_b200 import Bgk
    return Bgk(cfg, cloud, device="cuda:0")


def rel(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


@pytest.mark.parametrize("cfg", [M2, M3])
def test_one_pass_matches_oracle(torch_cuda, cfg):
    cloud = bi.make_cloud(cfg)
    g = gpu(cfg, cloud)
    rep = g.manage()
    s = oracle.State(oracle.make_cfg(cfg), cloud)
    ref = s.manage(*oracle.manage_params(cfg))
    assert rep == ref
    assert rep[0] >= 1 and rep[2] >= 1
    N = rep[5]
    assert g.N == N
    assert np.array_equal(g.positions(), s.x)
    assert np.array_equal(g.kinds(), s.kind)
    f = g.get_f().reshape(N, -1)
    assert rel(f, s.f) <= 1e-12
    n_int = int((s.kind == 0).sum())
    assert g.counts()[:3] == (N, n_int, N - n_int)


def test_capacity_limit_reported(torch_cuda):
    cfg = M2.replace(max_particles=0)
    cloud = bi.make_cloud(cfg)
    cap = len(cloud["x"]) + 2
    cfg = cfg.replace(max_particles=cap)
    g = gpu(cfg, cloud)
    rep = g.manage()
    ref = oracle.State(oracle.make_cfg(cfg), cloud).manage(*oracle.manage_params(cfg))
    assert rep == ref and rep[4] > 0 and rep[5] <= cap


@pytest.mark.parametrize("cfg", [M2, M3])
def test_managed_steps_match_oracle(torch_cuda, cfg):
    cloud = bi.make_cloud(cfg)
    g = gpu(cfg, cloud)
    g.step(5)
    g.sync()
    ref = oracle.run_steps(cfg, 5, cloud)
    assert g.manage_report() == ref.reports[-1]
    N = len(ref.x)
    assert g.N == N
    assert np.array_equal(g.kinds(), ref.kind)
    assert np.abs(g.positions() - ref.x).max() <= 1e-12 * cfg.dx
    f = g.get_f().reshape(N, -1)
    assert rel(f, ref.f) <= TOL
    rho, U, T = g.moments()
    r0, u0, t0 = ref.moments()
    assert np.abs(rho / r0 - 1).max() <= TOL
    assert np.abs(U - u0).max() / SIG <= TOL
    assert np.abs(T / t0 - 1).max() <= TOL


def test_management_is_a_noop_on_regular_lattice(torch_cuda):
    """C4 with management on: nothing merges or fills, so the run is bitwise the unmanaged one."""
    a = gpu(bi.C4.replace(manage=1), bi.make_cloud(bi.C4))
    b = gpu(bi.C4, bi.make_cloud(bi.C4))
    a.step(3)
    b.step(3)
    assert a.manage_report() == (0, 0, 0, 0, 0, bi.C4.n_particles)
    assert np.array_equal(a.get_f(), b.get_f())


def test_managed_column_sharded_steps(torch_cuda):
    """Velocity-sharded run with management on: every rank takes the same decisions (they
    depend on positions only), interpolates its own columns, and the ranks exchange only the
    two summed buffers -- the gathered result equals the oracle's managed run."""
    import torch
    cfg = M2
    cloud = bi.make_cloud(cfg)
    ncol = (cfg.Nv + 1) ** (cfg.dims - 1)
    shards = bi.column_shards(ncol, 3)
    from paper_2408_02350_b200 import Bgk
    ranks = [Bgk(cfg, cloud, col_range=s, device="cuda:0") for s in shards]
    steps = 4
    for _ in range(steps):
        for r in ranks:
            r.step_transport()
        tot = sum(r.buffer(0).clone() for r in ranks)
        for r in ranks:
            r.buffer(0).copy_(tot)
            r.step_relax()
        tot = sum(r.buffer(1).clone() for r in ranks)
        for r in ranks:
            r.buffer(1).copy_(tot)
            r.step_boundary()
    torch.cuda.synchronize()
    ref = oracle.run_steps(cfg, steps, cloud)
    N = len(ref.x)
    assert all(r.N == N for r in ranks)
    for r in ranks:
        assert np.array_equal(r.kinds(), ref.kind)
    n1 = cfg.Nv + 1
    full = np.zeros((N, 2, n1, ncol))
    for r, (c0, c1) in zip(ranks, shards):
        full[:, :, :, c0:c1] = r.get_f().reshape(N, -1, n1, c1 - c0)
    assert rel(full.reshape(N, -1), ref.f) <= TOL


@pytest.mark.parametrize("dims,n", [(2, 15), (3, 9)])
def test_wall_fill_matches_oracle(torch_cuda, dims, n):
    """Z30 wall fills: a corner whose interpolation stencil lost its interior neighbours triggers an
    insert inward of it -- one pass bit-exact against the oracle (report, positions, kinds; rows
    1e-12), then three managed ALE steps at the step parity bar."""
    from test_oracle_manage import _depleted_corner
    cfg, cloud, corner = _depleted_corner(dims, n)
    cfg = cfg.replace(init="stress", dt=5e-12)
    cloud.update({k: v for k, v in zip(("rho", "U", "T"), bi.initial_fields(cfg, cloud["x"]))})
    g = gpu(cfg, cloud)
    rep = g.manage()
    s = oracle.State(oracle.make_cfg(cfg), cloud)
    ref = s.manage(*oracle.manage_params(cfg))
    assert rep == ref and rep[2] >= 1
    assert np.array_equal(g.positions(), s.x)
    assert np.array_equal(g.kinds(), s.kind)
    assert rel(g.get_f().reshape(g.N, -1), s.f) <= 1e-12
    g2 = gpu(cfg, cloud)
    g2.step(3)
    g2.sync()
    ref = oracle.run_steps(cfg, 3, cloud)
    assert g2.N == ref.x.shape[0]
    assert np.abs(g2.positions() - ref.x).max() <= 1e-12 * cfg.dx
    assert rel(g2.get_f().reshape(g2.N, -1), ref.f) <= TOL
