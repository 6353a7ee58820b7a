"""Parity of the bench's exact transport instantiation (C5 velocity grid) over ten steps.

bench.py times C5 (40^3 particles x 25^3 nodes, N_v = 24, ALE, particle management on).  Its
transport is k_transport<3, R = 25, ...> in blocks of 2 warps over 640-column (128-B) padded
rows, 20 column groups of 32 columns, one v_1 chunk -- an instantiation used only when
N_v = 24.  Two checks hold it to the north-star bar (1e-10 relative max-norm on f, rho, U, T
after 10 steps; BASELINE.json):

  * small stress clouds on C5's velocity grid (same N_v, v_max, dt, management) replayed by the
    oracle in full, element by element;
  * the full C5 workload against tests/golden/c5_10steps_oracle.npz, written once by
    tools/make_c5_golden.py from oracle/ alone: every particle's (rho, U, T) and position, and
    the full f rows of a fixed sample.

Citations: PAPER.md:163-171 and 384-481 (transport), 185-199 (moments, relaxation), 177-180
(ALE), 489-492 (management); SURVEY.md §8(d) C5.
"""
import json
import math
import os

import numpy as np
import pytest

import bgk_inputs as bi
import oracle

pytestmark = pytest.mark.gpu

TOL = 1e-10
SIG = math.sqrt(bi.R_GAS * bi.T0)
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "c5_10steps_oracle.npz")


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def rel(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


def bench_like(cfg):
    """The configuration bench.py runs: management on, host-input staging buffer carved."""
    return cfg.replace(manage=1, staging=1)


def assert_headline_kernel(g):
    np_, R = g.transport_info()[:2]
    assert (np_, R) == (1, 25), "not the C5 transport instantiation (one particle per warp, R = 25)"
    assert g.Kloc == 625 * 25


@pytest.mark.parametrize("cfg", [
    bi.CavityConfig("C5grid_14c", 3, 14, 24),                          # lattice, stress start
    bi.CavityConfig("C5grid_12j", 3, 12, 24, jitter=0.25, dt=5e-12),   # jittered: ragged lists
])
def test_c5_velocity_grid_ten_steps(torch_cuda, cfg):
    from paper_2408_02350_b200 import Bgk
    cfg = bench_like(cfg)
    cloud = bi.make_cloud(cfg)
    g = Bgk(cfg, cloud, device="cuda:0")
    assert_headline_kernel(g)
    g.step(10)
    g.sync()
    ref = oracle.run_steps(cfg, 10, cloud)
    assert g.N == ref.x.shape[0]
    f = g.get_f().reshape(g.N, -1)
    assert rel(f, ref.f) <= TOL, rel(f, ref.f)
    rho, U, T = g.moments()
    r0, u0, t0 = ref.moments()
    assert np.abs(rho / r0 - 1).max() <= TOL
    assert np.abs(U - u0).max() / SIG <= TOL
    assert np.abs(T / t0 - 1).max() <= TOL
    inter = ref.kind == 0
    m = g.macro()
    assert np.abs(m[inter, 0] / ref.macro[inter, 0] - 1).max() <= TOL
    assert np.abs(m[inter, 1:4] - ref.macro[inter, 1:4]).max() / SIG <= TOL
    assert np.abs(m[inter, 4] / ref.macro[inter, 4] - 1).max() <= TOL
    assert np.abs(g.positions() - ref.x).max() <= 1e-12 * cfg.dx


def test_c5_full_ten_steps_against_oracle_golden(torch_cuda):
    """Full C5 (64 000 particles x 15 625 nodes), ten ALE steps with management, in bench.py's
    launch configuration, against the oracle-written golden."""
    import torch
    from paper_2408_02350_b200 import Bgk
    gold = np.load(GOLDEN)
    meta = json.loads(str(gold["meta"]))
    assert meta["config"] == bi.C5.name and meta["steps"] == 10 and meta["manage"] == 1
    cfg = bench_like(bi.C5)
    cloud = bi.make_cloud(cfg)
    g = Bgk(cfg, cloud, device="cuda:0")
    assert_headline_kernel(g)
    g.step(10)
    g.sync()
    assert g.N == len(gold["x"])
    assert np.abs(g.positions() - gold["x"]).max() <= 1e-12 * cfg.dx
    rho, U, T = g.moments()
    assert np.abs(rho / gold["rho"] - 1).max() <= TOL
    assert np.abs(U - gold["U"]).max() / SIG <= TOL
    assert np.abs(T / gold["T"] - 1).max() <= TOL
    inter = cloud["kind"] == 0
    m = g.macro()
    gm = gold["macro"]
    assert np.abs(m[inter, 0] / gm[inter, 0] - 1).max() <= TOL
    assert np.abs(m[inter, 1:4] - gm[inter, 1:4]).max() / SIG <= TOL
    assert np.abs(m[inter, 4] / gm[inter, 4] - 1).max() <= TOL
    sample = [int(i) for i in gold["sample"]]
    fbuf = g.f_internal()
    rows = fbuf[torch.tensor(sample, device=fbuf.device)].reshape(len(sample), -1).cpu().numpy()
    fr = gold["f_rows"]
    assert rel(rows, fr) <= TOL, rel(rows, fr)
    for q in range(len(sample)):                     # every sampled row on its own scale too
        assert rel(rows[q], fr[q]) <= TOL, (sample[q], rel(rows[q], fr[q]))
