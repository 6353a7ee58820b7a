"""Whole-step CUDA graphs (paper_2408_02350_b200/csrc/graph.cu) against the eager phases and the oracle.

bgk_step replays each step as one graph from the second step on; with particle management the graph
carries two conditional nodes (the device decides whether the pass changed the cloud).  Checked:
  * graph steps are bitwise equal to the same steps run phase by phase (bgk_run_phase, eager);
  * managed runs through graphs match the CPU oracle at the north-star bar (1e-10), including a
    run where a pass changes the cloud after graphs are in use (the skip / reconcile / eager re-run
    path; BGK_TEST_GRAPH_SKIP_AT forces one graph step to count as changed);
  * graph_info shows that graphs actually ran.
Citations: PAPER.md:489-492 (particle management), SURVEY.md §8(b) (asynchronous bgk_step).
"""
import math
import os
import subprocess
import sys

import numpy as np
import pytest

import bgk_inputs as bi
import oracle

pytestmark = pytest.mark.gpu
TOL = 1e-10
SIG = math.sqrt(bi.R_GAS * bi.T0)
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def rel(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


@pytest.mark.parametrize("cfg", [bi.C1, bi.CavityConfig("g3", 3, 9, 8), bi.C1.replace(ale=0),
                                 bi.CavityConfig("g3m", 3, 9, 8, manage=1)])
def test_graph_steps_bitwise_equal_eager_phases(torch_cuda, cfg):
    from paper_2408_02350_b200 import Bgk
    cloud = bi.make_cloud(cfg)
    g = Bgk(cfg, cloud, device="cuda:0")
    e = Bgk(cfg, cloud, device="cuda:0")
    g.step(6)
    for _ in range(6):
        for q in range(6):
            e.run_phase(q)
    g.sync()
    e.sync()
    info = g.graph_info()
    assert info[0] == 1 and info[1] >= 4, info          # graphs usable and used
    assert np.array_equal(g.get_f(), e.get_f())
    assert np.array_equal(g.positions(), e.positions())
    assert np.array_equal(g.macro(), e.macro())
    g.close()
    e.close()


def test_graph_managed_run_matches_oracle(torch_cuda):
    from paper_2408_02350_b200 import Bgk
    cfg = bi.CavityConfig("gM2", 2, 21, 12, manage=1, defects=2, m_min=21, jitter=0.05, dt=5e-12)
    cloud = bi.make_cloud(cfg)
    g = Bgk(cfg, cloud, device="cuda:0")
    g.step(8)
    g.sync()
    ref = oracle.run_steps(cfg, 8, cloud)
    assert g.N == ref.x.shape[0]
    assert rel(g.get_f().reshape(g.N, -1), ref.f) <= TOL
    assert np.abs(g.positions() - ref.x).max() <= 1e-12 * cfg.dx
    assert g.graph_info()[1] >= 5
    g.close()


_SKIP_SCRIPT = r"""
import math, os, sys
sys.path.insert(0, sys.argv[1])
import numpy as np
import bgk_inputs as bi
import oracle
from paper_2408_02350_b200 import Bgk
cfg = bi.CavityConfig("gM3", 3, 10, 6, manage=1, defects=1, jitter=0.05, dt=5e-12)
cloud = bi.make_cloud(cfg)
g = Bgk(cfg, cloud, device="cuda:0")
g.step(8)
rho, U, T = g.moments()
info = g.graph_info()
ref = oracle.run_steps(cfg, 8, cloud)
r0, u0, t0 = ref.moments()
f = g.get_f().reshape(g.N, -1)
err = float(np.abs(f - ref.f).max() / np.abs(ref.f).max())
print("RESULT", info[1], info[3], err, float(np.abs(rho / r0 - 1).max()), g.N == ref.x.shape[0])
"""


def test_graph_skip_reconcile_rerun(torch_cuda):
    """A graph step that counts as a cloud change (forced by the test hook at the second graph step)
    skips itself and the steps queued after it; moments() reconciles and re-runs them (the first
    eagerly): the result is the oracle's 8 managed steps (the first pass merges the defect pair and
    fills the hole; later passes change nothing)."""
    env = dict(os.environ, BGK_TEST_GRAPH_SKIP_AT="1")
    out = subprocess.run([sys.executable, "-c", _SKIP_SCRIPT, ROOT], env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("RESULT")][-1].split()
    launched, rerun, err, rerr, same_n = int(line[1]), int(line[2]), float(line[3]), float(line[4]), line[5]
    assert rerun >= 1, line                   # the skip happened and was re-run
    assert launched >= 2, line
    assert same_n == "True"
    assert err <= TOL and rerr <= TOL, line
