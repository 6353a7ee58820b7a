"""The shared input generators (bgk_inputs): lattice counts, wall tagging, seeding, shards."""
import numpy as np
import pytest

import bgk_inputs as bi


def test_lattice_counts_spec_examples():
    x, kind = bi.lattice(bi.CavityConfig("a", 2, 200, 4))
    assert len(x) == 40000 and (kind != 0).sum() == 4 * 199
    x, kind = bi.lattice(bi.CavityConfig("b", 2, 3, 4, L=1.0))
    assert len(x) == 9 and (kind != 0).sum() == 8 and (kind == 0).sum() == 1
    x, kind = bi.lattice(bi.CavityConfig("c", 3, 20, 4))
    assert len(x) == 8000                                               # SPEC.md:68 / PAPER.md:505
    for n, N in ((20, 8000), (30, 27000), (40, 64000)):
        assert bi.CavityConfig("d", 3, n, 4).n_particles == N


def test_wall_ids_and_ties():
    cfg = bi.CavityConfig("t", 3, 5, 4)
    x, kind = bi.lattice(cfg)
    L = cfg.L
    # every particle with a coordinate equal to 0 or L is boundary
    on_face = np.any((x == 0.0) | (x == L), axis=1)
    assert np.array_equal(on_face, kind != 0)
    # the lid id (6) only where z = L and no other wall applies
    lid = kind == 6
    assert np.all(x[lid, 2] == L)
    assert np.all((x[lid, 0] > 0) & (x[lid, 0] < L) & (x[lid, 1] > 0) & (x[lid, 1] < L))
    # corner (0,0,L) takes wall 1 (stationary)
    corner = np.nonzero((x[:, 0] == 0) & (x[:, 1] == 0) & (x[:, 2] == L))[0][0]
    assert kind[corner] == 1
    # index order: x fastest
    assert x[1, 0] > x[0, 0] and x[1, 1] == x[0, 1]


def test_jitter_seeded_and_interior_only():
    a, ka = bi.lattice(bi.C3)
    b, kb = bi.lattice(bi.C3)
    assert np.array_equal(a, b)
    r, _ = bi.lattice(bi.C3.replace(jitter=0.0))
    moved = np.any(a != r, axis=1)
    assert np.array_equal(moved, ka == 0)
    assert np.abs(a - r).max() <= 0.3 * bi.C3.dx


def test_stress_fields_shape():
    cloud = bi.make_cloud(bi.C4)
    assert cloud["U"].shape == (8000, 3) and np.abs(cloud["U"]).max() <= 10.0
    assert cloud["rho"].min() > 0.9 * bi.C4.rho0 and cloud["T"].min() > 0.9 * bi.T0


@pytest.mark.parametrize("n,w", [(625, 8), (625, 1), (33, 4), (289, 2)])
def test_column_shards_cover(n, w):
    sh = bi.column_shards(n, w)
    assert sh[0][0] == 0 and sh[-1][1] == n
    assert all(sh[i][1] == sh[i + 1][0] for i in range(w - 1))
    sizes = [b - a for a, b in sh]
    assert max(sizes) - min(sizes) <= 1
