"""Oracle pins: velocity grid (O1), neighbours (O2), WLS (O3), frames (O4),
boundary interpolation weights (O10).  CPU only.

Every check compares the oracle with something other than itself: values the
paper/SPEC print (tests/golden), closed forms, brute force on tiny inputs, an
independent numpy computation, or invariants that a dropped term / wrong sign
/ transposed operand would break.
"""
import math
import os

import numpy as np
import pytest

import bgk_inputs as bi

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    out = {}
    for line in open(os.path.join(GOLD, name)):
        if line.startswith("#") or not line.strip():
            continue
        parts = [p.strip() for p in line.split("|")]
        out[parts[0]] = parts[1:]
    return out


def cfg_of(dims, Nv, vmax, n=5):
    return bi.CavityConfig("t", dims, n, Nv, vmax=vmax)


# ----------------------------------------------------------------- O1 grid
def test_grid_spec_example(oracle_lib):
    g = _golden("spec_examples.txt")["grid_3d_Nv20_vmax1000"][0]
    kv = dict(t.split("=") for t in g.split())
    c = oracle_lib.make_cfg(cfg_of(3, 20, 1000.0))
    nodes = oracle_lib.axis_nodes(c)
    assert len(nodes) == int(kv["nodes"])
    assert oracle_lib.dv(c) == float(kv["dv"])
    assert nodes[0] == float(kv["first"]) and nodes[-1] == float(kv["last"])
    assert oracle_lib.num_nodes(c) == 21 ** 3


def test_grid_small_and_symmetric(oracle_lib):
    c = oracle_lib.make_cfg(cfg_of(2, 2, 1.0))
    assert list(oracle_lib.axis_nodes(c)) == [-1.0, 0.0, 1.0]
    for Nv in (12, 15, 16, 23, 24, 32):
        c = oracle_lib.make_cfg(cfg_of(3, Nv, bi.VMAX_DEFAULT))
        v = oracle_lib.axis_nodes(c)
        np.testing.assert_allclose(v, -v[::-1], rtol=0, atol=1e-12)
        assert abs(v.sum()) < 1e-9


def test_node_flattening_last_axis_fastest(oracle_lib):
    c = oracle_lib.make_cfg(cfg_of(3, 4, 2.0))
    V = oracle_lib.node_velocities(c)
    ax = oracle_lib.axis_nodes(c)
    n = 5
    for k in (0, 1, 7, 31, 124):
        j1, j2, j3 = k // (n * n), (k // n) % n, k % n
        assert tuple(V[k]) == (ax[j1], ax[j2], ax[j3])


# ------------------------------------------------------------ O2 neighbours
def _brute_numpy(x, h2):
    """Independent brute force with the same rounded operations (Z22)."""
    N, d = x.shape
    nbrs = []
    for i in range(N):
        s = np.zeros(N)
        for a in range(d):
            t = x[:, a] - x[i, a]
            s = s + t * t
        m = np.nonzero(s <= h2)[0]
        nbrs.append(m[m != i])
    return nbrs


def _lattice_ball_count(d, r):
    R = int(math.floor(r))
    cnt = 0
    rng = range(-R, R + 1)
    if d == 2:
        cnt = sum(1 for a in rng for b in rng if 0 < a * a + b * b <= r * r)
    else:
        cnt = sum(1 for a in rng for b in rng for c in rng if 0 < a * a + b * b + c * c <= r * r)
    return cnt


@pytest.mark.parametrize("dims,n,expect_int,expect_min", [(2, 21, 28, 17), (3, 12, 122, 65)])
def test_lattice_neighbour_counts(oracle_lib, dims, n, expect_int, expect_min):
    cfg = bi.CavityConfig("t", dims, n, 4)
    x, kind = bi.lattice(cfg)
    off, idx = oracle_lib.neighbors(x, cfg.h2)
    cnt = np.diff(off)
    assert _lattice_ball_count(dims, 3.1) == expect_int
    # deep interior (>= 3 lattice steps from every wall) sees the full ball
    ii = np.rint(x / cfg.dx).astype(int)
    deep = np.all((ii >= 3) & (ii <= n - 4), axis=1)
    assert np.all(cnt[deep] == expect_int)
    assert cnt[kind == 0].min() == expect_min


@pytest.mark.parametrize("dims,N,seed", [(2, 400, 1), (3, 500, 2), (2, 300, 3)])
def test_neighbours_match_independent_bruteforce(oracle_lib, dims, N, seed):
    x = bi.random_cloud(N, dims, seed)
    h2 = 0.12 * 0.12
    off, idx = oracle_lib.neighbors(x, h2)
    ref = _brute_numpy(x, h2)
    for i in range(N):
        got = idx[off[i]:off[i + 1]]
        assert np.array_equal(got, ref[i])
        assert np.all(np.diff(got) > 0)


def test_neighbours_symmetric_and_ties(oracle_lib):
    x = bi.random_cloud(300, 3, 7)
    off, idx = oracle_lib.neighbors(x, 0.2 ** 2)
    pairs = {(i, int(j)) for i in range(300) for j in idx[off[i]:off[i + 1]]}
    assert all((j, i) in pairs for (i, j) in pairs)
    # closed ball: exactly h apart is a neighbour, h(1+1e-9) is not
    h = 0.5
    x2 = np.array([[0.0, 0.0], [0.5, 0.0], [0.0, 0.5 * (1 + 1e-9)]])
    off, idx = oracle_lib.neighbors(x2, h * h)
    assert list(idx[off[0]:off[1]]) == [1]
    assert list(idx[off[1]:off[2]]) == [0]


# ------------------------------------------------------------------ O3 WLS
def test_weight_values(oracle_lib):
    g = _golden("spec_examples.txt")
    pv = _golden("paper_values.txt")
    alpha = float(pv["alpha_w"][0])
    h2 = 0.3 ** 2
    assert oracle_lib.weight(0.0, h2, alpha) == 1.0
    assert abs(oracle_lib.weight(h2, h2, alpha) - float(g["weight_at_h"][0])) < 1e-15
    assert oracle_lib.weight(h2 * 1.0001 ** 2, h2, alpha) == 0.0


def _clouds():
    out = []
    for cfg in (bi.C1, bi.C1.replace(jitter=0.3), bi.CavityConfig("t3", 3, 9, 4),
                bi.CavityConfig("t3j", 3, 9, 4, jitter=0.3)):
        x, kind = bi.lattice(cfg)
        out.append((cfg, x, kind))
    return out


@pytest.mark.parametrize("k", range(4))
def test_wls_inverse_and_linear_exactness(oracle_lib, k):
    cfg, x, kind = _clouds()[k]
    d = cfg.dims
    off, idx = oracle_lib.neighbors(x, cfg.h2)
    S, a, fr, rot = oracle_lib.wls_all(x, kind, off, idx, cfg.h2)
    rng = np.random.default_rng(k)
    g = rng.normal(size=d) / cfg.dx
    f = 0.7 + x @ g
    for i in np.nonzero(kind == 0)[0]:
        nb = idx[off[i]:off[i + 1]]
        D = x[nb] - x[i]
        w = np.exp(-6.0 * (D * D).sum(1) / cfg.h2)
        A = (D * w[:, None]).T @ D              # independent M^T W M
        np.testing.assert_allclose(S[i] @ A, np.eye(d), atol=1e-12)
        grad = (a[off[i]:off[i + 1]] * (f[nb] - f[i])[:, None]).sum(0)
        np.testing.assert_allclose(grad, g, rtol=1e-12, atol=1e-12 * np.abs(g).max())


def test_wls_quadratic_exact_on_symmetric_stencils_only(oracle_lib):
    cfg = bi.CavityConfig("t", 2, 15, 4)
    x, kind = bi.lattice(cfg)
    off, idx = oracle_lib.neighbors(x, cfg.h2)
    S, a, fr, rot = oracle_lib.wls_all(x, kind, off, idx, cfg.h2)
    xs = x / cfg.dx
    f = 0.3 * xs[:, 0] ** 2 - 0.2 * xs[:, 0] * xs[:, 1] + 0.5 * xs[:, 1] ** 2
    ii = np.rint(xs).astype(int)
    errs_sym, errs_wall = [], []
    for i in np.nonzero(kind == 0)[0]:
        nb = idx[off[i]:off[i + 1]]
        grad = (a[off[i]:off[i + 1]] * (f[nb] - f[i])[:, None]).sum(0) * cfg.dx
        exact = np.array([0.6 * xs[i, 0] - 0.2 * xs[i, 1], -0.2 * xs[i, 0] + 1.0 * xs[i, 1]])
        e = np.abs(grad - exact).max() / np.abs(exact).max()
        (errs_sym if np.all((ii[i] >= 3) & (ii[i] <= 11)) else errs_wall).append(e)
    assert max(errs_sym) < 1e-12
    assert max(errs_wall) > 1e-3    # one-sided stencils are not quadratic-exact (SURVEY §0 finding 6)


def test_wls_deficient_collinear(oracle_lib):
    x = np.array([[0.0, 0.0], [0.1, 0.0], [0.2, 0.0], [-0.1, 0.0], [-0.2, 0.0]])
    with pytest.raises(oracle_lib.OracleError):
        oracle_lib.wls_one(x, 0, np.array([1, 2, 3, 4]), 0.25 ** 2)
    with pytest.raises(oracle_lib.OracleError):   # m < d+2
        oracle_lib.wls_one(np.array([[0.0, 0.0], [0.1, 0.0], [0.0, 0.1]]), 0, np.array([1, 2]), 1.0)


# ---------------------------------------------------------------- O4 frames
def test_frames_orthonormal_right_handed(oracle_lib):
    rng = np.random.default_rng(3)
    for _ in range(200):
        for d in (2, 3):
            dj = rng.normal(size=d)
            F = oracle_lib.frame(dj)
            np.testing.assert_allclose(F @ F.T, np.eye(d), atol=1e-14)
            assert abs(np.linalg.det(F) - 1.0) < 1e-14
            np.testing.assert_allclose(F[0], dj / np.linalg.norm(dj), atol=1e-15)
    # neighbour due east: n = (1,0), t = (0,1)
    F = oracle_lib.frame([0.3, 0.0])
    assert np.array_equal(F, np.array([[1.0, 0.0], [-0.0, 1.0]]))
    # Z10: dx = dy = 0 -> phi = 0 -> b = (0, 1, 0), t = (+-1, 0, 0)
    F = oracle_lib.frame([0.0, 0.0, 2.0])
    np.testing.assert_allclose(F[2], [0, 1, 0], atol=0)
    np.testing.assert_allclose(F[1], [1, 0, 0], atol=1e-16)
    np.testing.assert_allclose(F[0], [0, 0, 1], atol=1e-16)
    # Z26: vertical to rounding (|dxy| <= 1e-8 r) is treated as vertical, whatever the sign of the
    # tiny offset; just above the threshold the true azimuth is used
    for e in ((1e-9, 0.0), (-1e-9, 3e-10), (0.0, -5e-9)):
        F = oracle_lib.frame([e[0], e[1], 1.0])
        np.testing.assert_allclose(F[2], [0, 1, 0], atol=0)
        assert F[0][1] == 0.0 and abs(F[0][2] - 1.0) < 1e-15
        assert 0.0 <= F[0][0] <= 1e-8   # sin(theta) >= 0 at phi = 0 (acos rounds it to 0 here)
    F = oracle_lib.frame([-2e-8, 0.0, 1.0])
    np.testing.assert_allclose(F[2], [0, -1, 0], atol=1e-15)


def test_frames_generic_angle_are_spherical_unit_vectors(oracle_lib):
    """All three 3D frame rows at generic angles, pinned by their geometric meaning rather
    than the trigonometric formula: n = e_r is the pair direction, b = e_phi is the horizontal unit
    vector z x n / |z x n| (this fixes the rotation of (t, b) about n that orthonormality and
    right-handedness leave free), and t = e_theta = b x n (so t_z = -sin(theta) <= 0, t lies in the
    vertical plane through n and z)."""
    rng = np.random.default_rng(17)
    z = np.array([0.0, 0.0, 1.0])
    for _ in range(500):
        dj = rng.normal(size=3) * rng.uniform(0.1, 3.0)
        F = oracle_lib.frame(dj)
        n = dj / np.linalg.norm(dj)
        b = np.cross(z, n)
        b /= np.linalg.norm(b)
        t = np.cross(b, n)
        np.testing.assert_allclose(F[0], n, atol=2e-15)
        np.testing.assert_allclose(F[2], b, atol=2e-15)
        np.testing.assert_allclose(F[1], t, atol=2e-15)
        assert F[2][2] == 0.0 and F[1][2] <= 0.0
        # t is coplanar with z and n (zero triple product), and points away from the north pole
        assert abs(np.dot(np.cross(z, n), F[1])) <= 2e-15
        assert np.dot(F[1], z - n[2] * n) <= 1e-15
    # azimuth quadrants: b follows phi = atan2(dy, dx) through all four quadrants
    for dx_, dy_, bx, by in ((1, 1, -1, 1), (-1, 1, -1, -1), (-1, -1, 1, -1), (1, -1, 1, 1)):
        F = oracle_lib.frame([dx_, dy_, 0.5])
        np.testing.assert_allclose(F[2][:2], np.array([bx, by]) / np.sqrt(2), atol=1e-15)


@pytest.mark.parametrize("k", range(4))
def test_rotation_positive_abar_and_completeness(oracle_lib, k):
    cfg, x, kind = _clouds()[k]
    off, idx = oracle_lib.neighbors(x, cfg.h2)
    S, a, fr, rot = oracle_lib.wls_all(x, kind, off, idx, cfg.h2)
    inter = np.repeat(kind == 0, np.diff(off))
    rot, fr, a = rot[inter], fr[inter], a[inter]
    assert np.all(rot[:, 0] > 0)   # abar = w d^T S d / r > 0 for SPD S
    back = np.einsum("pe,pea->pa", rot, fr)   # sum_e rot_e * frame_e = a
    np.testing.assert_allclose(back, a, rtol=0, atol=1e-13 * np.abs(a).max())


# ------------------------------------------------------ boundary weights (O10)
@pytest.mark.parametrize("dims,n", [(2, 21), (3, 10)])
def test_boundary_weights_reproduce_linear(oracle_lib, dims, n):
    cfg = bi.CavityConfig("t", dims, n, 4)
    x, kind = bi.lattice(cfg)
    off, idx = oracle_lib.neighbors(x, cfg.h2)
    cw = oracle_lib.boundary_weights(x, kind, off, idx, cfg.h2)
    rng = np.random.default_rng(dims)
    g = rng.normal(size=dims) / cfg.dx
    f = 1.3 + x @ g
    for b in np.nonzero(kind != 0)[0]:
        s, e = off[b], off[b + 1]
        c = cw[s:e]
        nb = idx[s:e]
        assert np.all(c[kind[nb] != 0] == 0.0)
        assert abs(c.sum() - 1.0) < 1e-13
        assert abs(c @ f[nb] - f[b]) < 1e-12 * abs(f).max()
    # corner weights can be negative (SURVEY §7 hard parts)
    assert cw.min() < 0


# ------------------------------------------------ second-order WLS (NEXT(3))
@pytest.mark.parametrize("k", range(4))
def test_wls_order2_reproduces_quadratics_on_any_stencil(oracle_lib, k):
    """Second-order Taylor WLS: the gradient of any quadratic is exact on every non-deficient
    stencil -- walls, jittered clouds included -- not only on symmetric ones."""
    cfg, x, kind = _clouds()[k]
    d = cfg.dims
    off, idx = oracle_lib.neighbors(x, cfg.h2)
    S, a, fr, rot = oracle_lib.wls_all(x, kind, off, idx, cfg.h2, order=2)
    rng = np.random.default_rng(10 + k)
    xs = x / cfg.dx
    g = rng.normal(size=d)
    H = rng.normal(size=(d, d))
    H = H + H.T
    f = 0.5 + xs @ g + 0.5 * np.einsum("ni,ij,nj->n", xs, H, xs)
    worst = 0.0
    for i in np.nonzero(kind == 0)[0]:
        nb = idx[off[i]:off[i + 1]]
        grad = (a[off[i]:off[i + 1]] * (f[nb] - f[i])[:, None]).sum(0) * cfg.dx
        exact = g + H @ xs[i]
        worst = max(worst, np.abs(grad - exact).max() / np.abs(exact).max())
    assert worst < 1e-11
    # first order is NOT quadratic-exact on the same clouds' wall stencils (sanity of the pin)
    if k in (0, 2):
        S1, a1, _, _ = oracle_lib.wls_all(x, kind, off, idx, cfg.h2, order=1)
        errs = []
        for i in np.nonzero(kind == 0)[0]:
            nb = idx[off[i]:off[i + 1]]
            grad = (a1[off[i]:off[i + 1]] * (f[nb] - f[i])[:, None]).sum(0) * cfg.dx
            exact = g + H @ xs[i]
            errs.append(np.abs(grad - exact).max() / np.abs(exact).max())
        assert max(errs) > 1e-3


def test_wls_order2_linear_exact_and_deficiency(oracle_lib):
    cfg, x, kind = _clouds()[3]
    off, idx = oracle_lib.neighbors(x, cfg.h2)
    S, a, fr, rot = oracle_lib.wls_all(x, kind, off, idx, cfg.h2, order=2)
    g = np.array([1.0, -2.0, 0.5]) / cfg.dx
    f = 3.0 + x @ g
    for i in np.nonzero(kind == 0)[0][::5]:
        nb = idx[off[i]:off[i + 1]]
        grad = (a[off[i]:off[i + 1]] * (f[nb] - f[i])[:, None]).sum(0)
        np.testing.assert_allclose(grad, g, rtol=1e-11)
    # a 6-neighbour cross stencil cannot determine 9 second-order unknowns
    hx = 0.1
    pts = [np.zeros(3)] + [s * hx * np.eye(3)[a] for a in range(3) for s in (1, -1)]
    with pytest.raises(oracle_lib.OracleError):
        oracle_lib.wls_one(np.array(pts), 0, np.arange(1, 7, dtype=np.int32), (1.01 * hx) ** 2, order=2)
