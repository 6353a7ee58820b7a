"""Second-order WLS on the GPU against the oracle.

The GPU solves the nu x nu (5 in 2D, 9 in 3D) normal equations per particle; on jittered
clouds some abar come out negative and the transport applies P:408-410 literally (signed
n-term).  Checked: coefficients against the oracle, quadratic exactness of the GPU's own
coefficients on wall and jittered stencils, 10-step parity (f, rho, U, T within 1e-10), the
stability bound.
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


def gpu(cfg):
    from paper_2408_02350_b200 import Bgk
    cloud = bi.make_cloud(cfg)
    return Bgk(cfg, cloud, device="cuda:0"), cloud


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


C1q = bi.C1.replace(wls_order=2)
C3q = bi.C3.replace(n_per_axis=41, wls_order=2, dt=4.0e-12)       # jittered: some abar < 0
C4q = bi.C4.replace(wls_order=2)
C4jq = bi.CavityConfig("C4j", 3, 20, 4, jitter=0.3, wls_order=2)


@pytest.mark.parametrize("cfg", [C1q, C3q, C4q, C4jq])
def test_wls2_coefficients(torch_cuda, cfg):
    g, cloud = gpu(cfg)
    g.build_neighbors()
    g.wls_coeffs()
    S, rot, fr, cw = g.wls()
    x, kind = cloud["x"], cloud["kind"]
    off, idx = oracle.neighbors(x, cfg.h2)
    rS, ra, rfr, rrot = oracle.wls_all(x, kind, off, idx, cfg.h2, order=2)
    inter = kind == 0
    erow = np.repeat(inter, np.diff(off))
    assert rel(S[inter], rS[inter]) < 1e-11
    assert rel(rot[erow], rrot[erow]) < 1e-11
    # The oracle's theta = arccos(dz/r) carries an error u/sin(theta) near the pole
    # (d arccos(c)/dc = -1/sin(theta)); jittered 3D clouds have pairs with sin(theta) ~ 1e-3.
    # Tolerance per pair: 1e-14 + 8u/sin(theta).
    rows = np.repeat(np.arange(len(x)), np.diff(off))
    dvec = x[idx] - x[rows]
    r = np.linalg.norm(dvec, axis=1)
    sin_t = np.hypot(dvec[:, 0], dvec[:, 1]) / r if cfg.dims == 3 else np.ones_like(r)
    tol = 1e-14 + 8 * np.finfo(float).eps / np.maximum(sin_t, 1e-300)
    ferr = np.abs(fr - rfr).reshape(len(r), -1).max(axis=1)
    assert np.all(ferr[erow] <= tol[erow])
    if cfg.jitter > 0:
        assert (rrot[erow, 0] < 0).any()          # the signed transport path is exercised


@pytest.mark.parametrize("cfg", [C1q, C4jq])
def test_wls2_gpu_coefficients_reproduce_quadratics(torch_cuda, cfg):
    g, cloud = gpu(cfg)
    g.build_neighbors()
    g.wls_coeffs()
    S, rot, fr, cw = g.wls()
    off, idx = g.neighbors()
    x, kind = cloud["x"], cloud["kind"]
    d = cfg.dims
    xs = x / cfg.dx
    rng = np.random.default_rng(5)
    gv = rng.normal(size=d)
    H = rng.normal(size=(d, d))
    H = H + H.T
    f = 1.0 + xs @ gv + 0.5 * np.einsum("ni,ij,nj->n", xs, H, xs)
    a = np.einsum("ek,eka->ea", rot, fr.reshape(-1, d, d))     # a_j = sum_e rot_e F_e (F orthonormal)
    worst = 0.0
    for i in np.nonzero(kind == 0)[0]:
        nb = idx[off[i]:off[i + 1]]
        grad = (a[off[i]:off[i + 1]] * (f[nb] - f[i])[:, None]).sum(0) * cfg.dx
        exact = gv + H @ xs[i]
        worst = max(worst, np.abs(grad - exact).max() / np.abs(exact).max())
    assert worst < 1e-10


@pytest.mark.parametrize("cfg", [C1q, C1q.replace(ale=0), C3q, C4q, C4jq])
def test_wls2_ten_steps(torch_cuda, cfg):
    g, _ = gpu(cfg)
    g.step(10)
    g.sync()
    ref = oracle.run_steps(cfg, 10)
    f = g.get_f().reshape(g.N, -1)
    assert rel(f, ref.f) <= TOL, rel(f, ref.f)
    rho, U, T = g.moments()
    r0, u0, t0 = ref.moments()
    assert np.abs(rho / r0 - 1).max() <= TOL
    assert np.abs(U - u0).max() / SIG <= TOL
    assert np.abs(T / t0 - 1).max() <= TOL
    assert np.abs(g.positions() - ref.x).max() <= 1e-12 * cfg.dx


def test_wls2_stable_dt(torch_cuda):
    cfg = C3q
    g, cloud = gpu(cfg)
    dt = g.stable_dt()
    x, kind = cloud["x"], cloud["kind"]
    off, idx = oracle.neighbors(x, cfg.h2)
    S, a, fr, rot = oracle.wls_all(x, kind, off, idx, cfg.h2, order=2)
    c = oracle.make_cfg(cfg)
    amax = max(oracle.coef_absmax_one(c, cloud["U"][i], rot[off[i]:off[i + 1]], fr[off[i]:off[i + 1]])
               for i in np.nonzero(kind == 0)[0])
    assert abs(dt * amax - 1) < 1e-12
