"""GPU parity: the CUDA path through the C ABI against the CPU oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star):
  neighbour lists: bit-exact (same rounded arithmetic, ascending order);
  f: ||f_gpu - f_ref||_inf / ||f_ref||_inf <= 1e-10 after 10 steps;
  rho, T: max relative error <= 1e-10;  U: ||dU||_inf / sqrt(R T0) <= 1e-10;
  WLS coefficients (a single solve, no time stepping): 1e-12 relative to the array's max.
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


def gpu(cfg, cloud=None, **kw):
    from paper_2408_02350_b200 import Bgk
    cloud = cloud if cloud is not None else bi.make_cloud(cfg)
    return Bgk(cfg, cloud, device="cuda:0", **kw), cloud


def rel(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


# ------------------------------------------------------------------ neighbours
@pytest.mark.parametrize("cfg", [bi.C1, bi.C3, bi.C4, bi.CavityConfig("C4j", 3, 20, 4, jitter=0.3)])
def test_neighbors_bit_exact_cavity(torch_cuda, cfg):
    g, cloud = gpu(cfg)
    g.build_neighbors()
    off, idx = g.neighbors()
    roff, ridx = oracle.neighbors(cloud["x"], cfg.h2)
    assert np.array_equal(off, roff)
    assert np.array_equal(idx, ridx)


@pytest.mark.parametrize("dims,N,n_axis,seed", [(2, 3000, 30, 11), (3, 6000, 14, 12), (3, 257, 5, 13)])
def test_neighbors_bit_exact_random_cloud(torch_cuda, dims, N, n_axis, seed):
    """Uniform random points (not a lattice): irregular counts, ties decided by the same
    rounded d^2 on both sides."""
    cfg = bi.CavityConfig("rand", dims, n_axis, 4)
    x = bi.random_cloud(N, dims, seed, L=cfg.L)
    cloud = {"x": x, "kind": np.zeros(N, dtype=np.int8)}
    g, _ = gpu(cfg, cloud, max_neighbors=512)
    g.build_neighbors()
    off, idx = g.neighbors()
    roff, ridx = oracle.neighbors(x, cfg.h2)
    assert np.array_equal(off, roff) and np.array_equal(idx, ridx)


def test_neighbors_ties_exactly_h(torch_cuda):
    """Closed ball (Z11): a pair exactly h apart is a neighbour (d2 == h2 bit for bit),
    a pair h(1+1e-9) apart is not."""
    cfg = bi.CavityConfig("tie", 2, 5, 4, L=1.0)
    h = cfg.h
    x = np.array([[0.0, 0.0], [h, 0.0], [0.0, h * (1 + 1e-9)], [0.9, 0.9]])
    assert (x[1, 0] - x[0, 0]) ** 2 == cfg.h2
    cloud = {"x": x, "kind": np.zeros(4, dtype=np.int8)}
    g, _ = gpu(cfg, cloud)
    g.build_neighbors()
    off, idx = g.neighbors()
    assert list(idx[off[0]:off[1]]) == [1] and list(idx[off[1]:off[2]]) == [0]
    roff, ridx = oracle.neighbors(x, cfg.h2)
    assert np.array_equal(off, roff) and np.array_equal(idx, ridx)


# ------------------------------------------------------------------------ WLS
@pytest.mark.parametrize("cfg", [bi.C1, bi.C3, bi.C4])
def test_wls_coefficients(torch_cuda, cfg):
    g, cloud = gpu(cfg)
    g.build_neighbors()
    g.wls_coeffs()
    S, rot, fr, cw = g.wls()
    x, kind = cloud["x"], cloud["kind"]
    off, idx = oracle.neighbors(x, cfg.h2)
    rS, ra, rfr, rrot = oracle.wls_all(x, kind, off, idx, cfg.h2)
    rcw = oracle.boundary_weights(x, kind, off, idx, cfg.h2)
    inter = kind == 0
    assert rel(S[inter], rS[inter]) < 1e-12
    erow = np.repeat(inter, np.diff(off))
    assert rel(rot[erow], rrot[erow]) < 1e-12
    assert np.abs(fr[erow] - rfr[erow]).max() < 1e-14
    assert np.abs(cw - rcw).max() < 1e-12
    assert np.all(cw[erow] == 0)


# -------------------------------------------------------------- whole steps
_ref_cache = {}


def oracle_run(cfg, steps):
    key = (cfg, steps)
    if key not in _ref_cache:
        _ref_cache[key] = oracle.run_steps(cfg, steps)
    return _ref_cache[key]


def check_state(g, ref, cfg):
    f = g.get_f().reshape(g.N, -1)
    assert rel(f, ref.f) <= TOL, rel(f, ref.f)
    rho, U, T = g.moments()
    r0, u0, t0 = ref.moments()
    assert np.abs(rho / r0 - 1).max() <= TOL
    assert np.abs(U - u0).max() / SIG <= TOL
    assert np.abs(T / t0 - 1).max() <= TOL
    m = g.macro()
    inter = ref.kind == 0
    assert np.abs(m[inter, 0] / ref.macro[inter, 0] - 1).max() <= TOL
    assert np.abs(m[inter, 1:1 + cfg.dims] - ref.macro[inter, 1:1 + cfg.dims]).max() / SIG <= TOL
    assert np.abs(m[inter, -1] / ref.macro[inter, -1] - 1).max() <= TOL
    x = g.positions()
    assert np.abs(x - ref.x).max() <= 1e-12 * cfg.dx


@pytest.mark.parametrize("cfg", [bi.C1, bi.C4])
def test_one_step(torch_cuda, cfg):
    g, _ = gpu(cfg)
    g.step(1)
    g.sync()
    check_state(g, oracle_run(cfg, 1), cfg)


@pytest.mark.parametrize("cfg", [bi.C1, bi.C1.replace(ale=0), bi.C1.replace(init="equilibrium"),
                                 bi.C2, bi.C2.replace(Kn=0.1), bi.C2.replace(Kn=10.0), bi.C3, bi.C4,
                                 bi.C1.replace(Nv=11), bi.CavityConfig("C4odd", 3, 14, 15)])
def test_ten_steps(torch_cuda, cfg):
    g, _ = gpu(cfg)
    g.step(10)
    g.sync()
    check_state(g, oracle_run(cfg, 10), cfg)


def test_deterministic(torch_cuda):
    cfg = bi.C4
    a, _ = gpu(cfg)
    b, _ = gpu(cfg)
    a.step(3)
    b.step(3)
    assert np.array_equal(a.get_f(), b.get_f())


def test_stable_dt(torch_cuda):
    cfg = bi.C1
    g, cloud = gpu(cfg)
    dt = g.stable_dt()
    x, kind = cloud["x"], cloud["kind"]
    off, idx = oracle.neighbors(x, cfg.h2)
    S, a, fr, rot = oracle.wls_all(x, kind, off, idx, cfg.h2)
    c = oracle.make_cfg(cfg)
    amax = max(oracle.coef_absmax_one(c, cloud["U"][i], rot[off[i]:off[i + 1]], fr[off[i]:off[i + 1]])
               for i in np.nonzero(kind == 0)[0])
    assert abs(dt * amax - 1) < 1e-12


# --------------------------------------------- velocity sharding on one device
@pytest.mark.parametrize("cfg,P", [(bi.C1, 3), (bi.CavityConfig("C4s", 3, 12, 8), 4),
                                   (bi.CavityConfig("C5s8", 3, 8, 24), 8)])   # 78/79 columns: folded last group
def test_column_sharded_step_matches(torch_cuda, cfg, P):
    """P contexts, each owning a column shard, exchanging only the two summed buffers
    (what the NCCL all-reduce does across GPUs) reproduce the single-context run."""
    import torch
    cloud = bi.make_cloud(cfg)
    ncol = (cfg.Nv + 1) ** (cfg.dims - 1)
    shards = bi.column_shards(ncol, P)
    ranks = [gpu(cfg, cloud, col_range=s)[0] for s in shards]
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
    ref = oracle_run(cfg, steps)
    n1 = cfg.Nv + 1
    full = np.zeros((len(cloud["x"]), 2 if cfg.dims == 2 else 1, n1, ncol))
    for r, (c0, c1) in zip(ranks, shards):
        full[:, :, :, c0:c1] = r.get_f().reshape(r.N, -1, n1, c1 - c0)
    assert rel(full.reshape(len(cloud["x"]), -1), ref.f) <= TOL
    # sharded moments via partial sums
    for r in ranks:
        r.L.bgk_moments_partial(r.ctx, r.stream)
    tot = sum(r.buffer(0).clone() for r in ranks)
    ranks[0].buffer(0).copy_(tot)
    import ctypes as C
    rho = np.zeros(ranks[0].N)
    st = ranks[0].L.bgk_moments_finalize(ranks[0].ctx, rho.ctypes.data, None, None, ranks[0].stream)
    assert st == 0
    r0, _, _ = ref.moments()
    assert np.abs(rho / r0 - 1).max() <= TOL


# ------------------------------------------------------- full size, sampled
def test_c5_full_size_sampled(torch_cuda):
    """BASELINE config C5 (40^3 particles x 25^3 velocities) in the launch configuration
    bench.py times: one GPU step vs the oracle evaluated one particle at a time."""
    import torch
    from paper_2408_02350_b200 import _lib
    cfg = bi.C5
    g, cloud = gpu(cfg)
    g.step(1)
    g.sync()
    kind = cloud["kind"]
    inter = np.nonzero(kind == 0)[0]
    rng = np.random.default_rng(5)
    sample = list(rng.choice(inter, 4, replace=False)) + [int(inter[0]), int(inter[-1])]
    sample += [int(np.nonzero(kind == 6)[0][700]), int(np.nonzero(kind == 1)[0][0])]  # lid, corner
    ref = oracle.sampled_first_step(cfg, cloud, sample)
    fbuf = g.f_internal()
    rows = fbuf[torch.tensor(sample, device=fbuf.device)].reshape(len(sample), -1).cpu().numpy()
    macro = g.macro()
    x = g.positions()
    for q, i in enumerate(sample):
        r = ref[i]
        assert rel(rows[q], r["f"]) <= TOL, (i, rel(rows[q], r["f"]))
        assert np.abs(x[i] - r["x"]).max() <= 1e-12 * cfg.dx
        if kind[i] == 0:
            assert abs(macro[i, 0] / r["rho"] - 1) <= TOL
            assert np.abs(macro[i, 1:4] - r["U"]).max() / SIG <= TOL
            assert abs(macro[i, 4] / r["T"] - 1) <= TOL


# ---------------------------------------------------------------- edge cases
def test_deficient_boundary_stencil_reported(torch_cuda):
    from paper_2408_02350_b200 import BgkError
    cfg = bi.CavityConfig("tiny", 2, 3, 4, L=1e-6)
    g, _ = gpu(cfg)
    with pytest.raises(BgkError) as ei:
        g.build_neighbors()
        g.wls_coeffs()
    assert ei.value.status == 3 and ei.value.particle >= 0


def test_degenerate_state_reported(torch_cuda):
    from paper_2408_02350_b200 import BgkError
    cfg = bi.C1
    g, _ = gpu(cfg)
    g.set_f(np.zeros((g.N, 2, g.Kloc)))
    g.step(1)
    with pytest.raises(BgkError) as ei:
        g.sync()
    assert ei.value.status == 4 and ei.value.particle >= 0


def test_out_of_domain_rejected(torch_cuda):
    from paper_2408_02350_b200 import BgkError
    cfg = bi.C1
    cloud = bi.make_cloud(cfg)
    cloud["x"] = cloud["x"].copy()
    cloud["x"][7, 0] = 1.5 * cfg.L
    with pytest.raises(BgkError) as ei:
        gpu(cfg, cloud)
    assert ei.value.status == 5


def test_set_get_f_roundtrip(torch_cuda):
    for cfg in (bi.C1, bi.CavityConfig("t3", 3, 6, 6)):
        g, _ = gpu(cfg)
        f = np.random.default_rng(0).uniform(size=(g.N, g.nval, g.Kloc))
        g.set_f(f)
        assert np.array_equal(g.get_f(), f)


def test_cuda_graph_capture_matches_eager(torch_cuda):
    """bgk_step enqueues no host synchronisation: three steps captured in a CUDA graph and
    replayed give the bitwise result of three eager steps."""
    import torch
    cfg = bi.C4
    eager, cloud = gpu(cfg)
    eager.step(1)                       # warm-up (one-time kernel attribute setup) outside capture
    eager.step(3)
    g, _ = gpu(cfg, cloud)
    g.step(1)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            g.step(3)
    graph.replay()
    torch.cuda.synchronize()
    assert np.array_equal(g.get_f(), eager.get_f())


def test_c5_ten_steps_invariants(torch_cuda):
    """Full-size C5, 10 ALE steps (beyond what the oracle can replay): properties that hold at
    any size -- zero net mass flux through every wall particle (diffuse reflection, Z17),
    nonnegative interior f (positive scheme under dt < stable_dt), finite moments and
    particles inside the box."""
    import torch
    cfg = bi.C5
    g, cloud = gpu(cfg)
    assert g.stable_dt() > cfg.dt
    g.step(10)
    g.sync()
    f = g.f_internal()[..., 0]                          # [N, n1, ncol] on the device
    kind = torch.as_tensor(cloud["kind"], device=f.device)
    n1 = cfg.Nv + 1
    ax = torch.tensor([-cfg.vmax + j * (2 * cfg.vmax / cfg.Nv) for j in range(n1)], dtype=torch.float64,
                      device=f.device)
    v1 = ax.view(n1, 1, 1).expand(n1, n1, n1).reshape(n1, n1 * n1)
    v2 = ax.view(1, n1, 1).expand(n1, n1, n1).reshape(n1, n1 * n1)
    v3 = ax.view(1, 1, n1).expand(n1, n1, n1).reshape(n1, n1 * n1)
    vel = (v1, v2, v3)
    for wid in range(1, 7):
        rows = torch.nonzero(kind == wid).flatten()
        if rows.numel() == 0:
            continue
        a, sgn = (wid - 1) // 2, (1.0 if (wid - 1) % 2 == 0 else -1.0)
        vn = sgn * vel[a]
        fb = f[rows]
        flux = (fb * vn).sum(dim=(1, 2))
        scale = (fb * vn.abs()).sum(dim=(1, 2))
        assert torch.all(flux.abs() <= 1e-12 * scale), wid
    assert f[kind == 0].min().item() >= 0.0
    rho, U, T = g.moments()
    assert np.all(np.isfinite(rho)) and np.all(rho > 0) and np.all(T > 0)
    x = g.positions()
    assert np.all(x >= 0) and np.all(x <= cfg.L)


# -------------------------------------------------- degenerate cloud shapes
@pytest.mark.parametrize("cfg", [bi.CavityConfig("open2d", 2, 17, 10, jitter=0.2, dt=4e-12),
                                 bi.CavityConfig("open3d", 3, 9, 6, jitter=0.2, dt=4e-12)])
def test_all_interior_cloud_no_walls(torch_cuda, cfg):
    """No boundary particles at all (N_b = 0): every particle is transported with one-sided
    stencils at the edges, the boundary phases are empty; 5 ALE steps against the oracle."""
    cloud = bi.make_cloud(cfg)
    cloud["kind"] = np.zeros_like(cloud["kind"])
    g, _ = gpu(cfg, cloud)
    g.step(5)
    g.sync()
    ref = oracle.run_steps(cfg, 5, cloud)
    f = g.get_f().reshape(g.N, -1)
    assert rel(f, ref.f) <= TOL
    assert np.abs(g.positions() - ref.x).max() <= 1e-12 * cfg.dx
    rho, U, T = g.moments()
    r0, u0, t0 = ref.moments()
    assert np.abs(rho / r0 - 1).max() <= TOL and np.abs(T / t0 - 1).max() <= TOL


def test_fixed_cloud_3d_ten_steps(torch_cuda):
    """Fixed-cloud (Eulerian, W = 0) mode in 3D: geometry built once and cached (Z21)."""
    cfg = bi.C4.replace(ale=0)
    g, _ = gpu(cfg)
    g.step(10)
    g.sync()
    check_state(g, oracle_run(cfg, 10), cfg)


def test_fixed_cloud_jittered_no_tiles(torch_cuda):
    """Tiles and lattice rows need the regular lattice: a jittered fixed cloud runs the general
    kernel only (transport_info reports neither) and still meets the oracle bar."""
    cfg = bi.CavityConfig("fixjit", 3, 16, 8, ale=0, jitter=0.2, dt=5e-12)
    g, _ = gpu(cfg)
    g.step(5)
    g.sync()
    info = g.transport_info()
    assert info[2] == 0 and info[4] == 0, info
    check_state(g, oracle_run(cfg, 5), cfg)


def test_staged_input_matches_set_f(torch_cuda):
    """bgk_stage_f on a copy stream + bgk_use_staged_f is the same state as bgk_set_f: a
    fixed-cloud run restarted from a staged f^0 reproduces the fresh run bitwise."""
    import torch
    cfg = bi.C1.replace(ale=0, staging=1)
    a, cloud = gpu(cfg)
    b, _ = gpu(cfg, cloud)
    f0 = torch.from_numpy(a.get_f()).pin_memory()
    a.step(3)
    cs = torch.cuda.Stream()
    a.stage_f(f0, cs)
    a.use_staged_f()
    a.step(2)
    b.step(2)
    assert np.array_equal(a.get_f(), b.get_f())


# ------------------------------------ fixed-cloud lattice rows (SURVEY §8(d) lever)
@pytest.mark.parametrize("cfg", [bi.C4.replace(ale=0), bi.CavityConfig("C4r", 3, 24, 8, ale=0)])
def test_lattice_rows_fixed_cloud(torch_cuda, cfg, monkeypatch):
    """Fixed cloud on the lattice: 8 x 8 x 8 tiles of the deep interior run the tabulated 122-point
    stencil (k_transport_tile), groups of 8 line-consecutive particles with identical stencils share
    coefficients and boxes (k_transport_rows), the rest runs the general kernel.  Same oracle bar,
    and the same state as the general kernel alone (BGK_TRANSPORT_ROWS=0) to 1e-13."""
    g, cloud = gpu(cfg)
    g.step(10)
    g.sync()
    info = g.transport_info()
    assert info[2] > 0 and info[4] > 0, info
    assert info[2] * 8 + info[3] + info[4] * 512 == int((cloud["kind"] == 0).sum()), info
    check_state(g, oracle_run(cfg, 10), cfg)
    monkeypatch.setenv("BGK_TRANSPORT_ROWS", "0")
    h, _ = gpu(cfg, cloud)
    h.step(10)
    assert rel(g.get_f(), h.get_f()) <= 1e-13


def test_lattice_rows_c5_sampled(torch_cuda):
    """The bench's secondary workload (C5 fixed cloud) through the lattice-row kernel: one step,
    sampled particles against the oracle evaluated one particle at a time."""
    import torch
    cfg = bi.C5.replace(ale=0)
    g, cloud = gpu(cfg)
    g.step(1)
    g.sync()
    assert g.transport_info()[2] > 0
    kind = cloud["kind"]
    inter = np.nonzero(kind == 0)[0]
    rng = np.random.default_rng(9)
    sample = [int(v) for v in rng.choice(inter, 6, replace=False)] + [int(inter[len(inter) // 2])]
    ref = oracle.sampled_first_step(cfg, cloud, sample)
    fbuf = g.f_internal()
    rows = fbuf[torch.tensor(sample, device=fbuf.device)].reshape(len(sample), -1).cpu().numpy()
    for q, i in enumerate(sample):
        assert rel(rows[q], ref[i]["f"]) <= TOL, (i, rel(rows[q], ref[i]["f"]))


def test_library_lattice_and_default_vmax(torch_cuda):
    """bgk_init_cloud with x = kind = NULL builds the regular cavity lattice itself (same points,
    order and wall ids as bgk_inputs.lattice), and vmax <= 0 defaults to |U_lid| + 4 sqrt(R T0)."""
    from paper_2408_02350_b200 import Bgk
    cfg = bi.C1
    cloud = bi.make_cloud(cfg)
    lib_cloud = {"rho": cloud["rho"], "U": cloud["U"], "T": cloud["T"]}
    g = Bgk(cfg.replace(vmax=-1.0), lib_cloud, device="cuda:0")
    assert np.array_equal(g.positions(), cloud["x"])
    assert np.array_equal(g.kinds(), cloud["kind"])
    g.step(2)
    h, _ = gpu(cfg, cloud)
    h.step(2)
    assert np.array_equal(g.get_f(), h.get_f())


def test_fused_2d_relaxation_matches_unfused(torch_cuda, monkeypatch):
    """2D, N_v = 32, one rank: bgk_step runs transport + moments + relaxation in one kernel (a block
    holds all nodes of a particle).  Ten ALE steps on the jittered cloud agree with the unfused
    kernels (BGK_FUSE=0: transport, moment sums, relaxation) to 1e-13 and with the oracle at the
    parity bar."""
    cfg = bi.CavityConfig("fuse2d", 2, 31, 32, jitter=0.3, dt=3.5e-12)
    g, cloud = gpu(cfg)
    g.step(10)
    g.sync()
    check_state(g, oracle_run(cfg, 10), cfg)
    monkeypatch.setenv("BGK_FUSE", "0")
    h, _ = gpu(cfg, cloud)
    h.step(10)
    h.sync()
    assert rel(g.get_f(), h.get_f()) <= 1e-13
    assert np.abs(g.positions() - h.positions()).max() <= 1e-13 * cfg.dx
