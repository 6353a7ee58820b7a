"""2D particle-set transport (k_transport2s) against the CPU oracle.

A warp owns P cell-consecutive interior particles and walks the union of their neighbour lists;
each lane owns QC nodes of a 32*QC-node chunk.  Every instantiated (P, QC), the N_v = 32 velocity
grid of C2/C3 (33 x 33 nodes: chunks end mid-row, the last one ragged), a jittered cloud (ragged
lists, 16-35 neighbours), column shards (ncol = 11 per rank) and the second-order WLS variant are
replayed for ten steps and compared element by element at the north-star bar (1e-10 relative
max-norm on f; rho, T relative; U / sqrt(R T0)).  Citations: PAPER.md:163-171, 384-481
(transport), 185-199 (moments, relaxation), 177-180 (ALE); SURVEY.md §8(d) C2/C3.
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
    return torch


def rel(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


def check(g, ref, cfg):
    f = g.get_f().reshape(g.N, -1)
    assert rel(f, ref.f) <= TOL, rel(f, ref.f)
    rho, U, T = g.moments()
    r0, u0, t0 = ref.moments()
    assert np.abs(rho / r0 - 1).max() <= TOL
    assert np.abs(U - u0).max() / SIG <= TOL
    assert np.abs(T / t0 - 1).max() <= TOL
    assert np.abs(g.positions() - ref.x).max() <= 1e-12 * cfg.dx


@pytest.mark.parametrize("P,QC", [(8, 2), (4, 2), (4, 4), (8, 3)])
@pytest.mark.parametrize("cfg", [
    bi.CavityConfig("C2grid_15", 2, 15, 32, dt=4e-12),
    bi.CavityConfig("C3grid_21j", 2, 21, 32, jitter=0.3, dt=2e-12),
])
def test_set_kernel_ten_steps(torch_cuda, monkeypatch, cfg, P, QC):
    from paper_2408_02350_b200 import Bgk
    monkeypatch.setenv("BGK_SET_P", str(P))
    monkeypatch.setenv("BGK_SET_QC", str(QC))
    cloud = bi.make_cloud(cfg)
    g = Bgk(cfg, cloud, device="cuda:0")
    assert tuple(g.transport_info()[:2]) == (P, QC)
    g.step(10)
    g.sync()
    check(g, oracle.run_steps(cfg, 10, cloud), cfg)
    g.close()


def test_set_kernel_fixed_cloud_and_managed(torch_cuda):
    from paper_2408_02350_b200 import Bgk
    for cfg in (bi.CavityConfig("C2fix", 2, 17, 32, ale=0, dt=4e-12),
                bi.CavityConfig("C2man", 2, 19, 32, manage=1, defects=2, m_min=21, jitter=0.05, dt=3e-12)):
        cloud = bi.make_cloud(cfg)
        g = Bgk(cfg, cloud, device="cuda:0")
        g.step(10)
        g.sync()
        ref = oracle.run_steps(cfg, 10, cloud)
        assert g.N == ref.x.shape[0]
        check(g, ref, cfg)
        g.close()


def test_set_kernel_column_shards(torch_cuda):
    """ncol = 11 per rank (three column shards of the 33 columns): chunks wrap several rows."""
    import torch
    from paper_2408_02350_b200 import Bgk
    cfg = bi.CavityConfig("C2sh", 2, 13, 32, dt=4e-12)
    cloud = bi.make_cloud(cfg)
    shards = bi.column_shards(cfg.Nv + 1, 3)
    ranks = [Bgk(cfg, cloud, col_range=s, device="cuda:0") for s in shards]
    for _ in range(10):
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
    ref = oracle.run_steps(cfg, 10, cloud)
    K1 = cfg.Nv + 1
    fr = ref.f.reshape(len(cloud["x"]), 2, K1, K1)      # [N][g][k1][col] canonical 2D layout
    for (c0, c1), r in zip(shards, ranks):
        f = r.get_f().reshape(r.N, 2, K1, c1 - c0)
        assert rel(f, fr[:, :, :, c0:c1]) <= TOL
    m = ranks[0].macro()
    inter = ref.kind == 0
    assert np.abs(m[inter, 0] / ref.macro[inter, 0] - 1).max() <= TOL
    for r in ranks:
        r.close()


def test_set_kernel_second_order(torch_cuda):
    from paper_2408_02350_b200 import Bgk
    cfg = bi.CavityConfig("C2o2", 2, 15, 32, wls_order=2, jitter=0.1, dt=3e-12)
    cloud = bi.make_cloud(cfg)
    g = Bgk(cfg, cloud, device="cuda:0")
    assert tuple(g.transport_info()[:2]) == (4, 2)
    g.step(10)
    g.sync()
    check(g, oracle.run_steps(cfg, 10, cloud), cfg)
    g.close()
