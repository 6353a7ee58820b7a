"""Small runs for compute-sanitizer (memcheck / racecheck / synccheck / initcheck) -- every kernel of
the step on configurations that finish in seconds even under instrumentation (single
writer per output, no races).

    compute-sanitizer --tool memcheck  python tools/sanitize_run.py [case ...]
    compute-sanitizer --tool racecheck python tools/sanitize_run.py [case ...]

Cases: c1 (2D Chu, 21^2 x 13^2, ALE, 33-column tail not used), c2s (2D, N_v = 32: TMA groups + tail
columns), c3d (3D 8^3 x 9^3), c5g (3D on C5's velocity grid, the bench's R = 25 instantiation, 9^3
particles), m2 / m3 (particle management with merges and fills), fixed (3D fixed cloud: lattice-row
kernel), shard (column-sharded contexts exchanging the two sums), wls2 (second-order WLS).
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bgk_inputs as bi  # noqa: E402
from paper_2408_02350_b200 import Bgk  # noqa: E402

CASES = {
    "c1": bi.C1,
    "c2s": bi.CavityConfig("c2s", 2, 15, 32, dt=4e-12),
    "c3d": bi.CavityConfig("c3d", 3, 8, 8),
    "c5g": bi.CavityConfig("c5g", 3, 9, 24, manage=1),
    "m2": bi.CavityConfig("M2", 2, 21, 12, manage=1, defects=2, m_min=21, jitter=0.05, dt=5e-12),
    "m3": bi.CavityConfig("M3", 3, 12, 6, manage=1, defects=2, m_min=84, jitter=0.05, dt=5e-12),
    "fixed": bi.CavityConfig("fixed", 3, 12, 6, ale=0),
    "wls2": bi.CavityConfig("wls2", 3, 8, 6, wls_order=2, jitter=0.1, dt=5e-12),
}


def run(name, steps=2):
    cfg = CASES[name]
    cloud = bi.make_cloud(cfg)
    g = Bgk(cfg, cloud, device="cuda:0")
    g.step(steps)
    g.sync()
    g.stable_dt()
    rho, U, T = g.moments()
    f = g.get_f()
    assert np.all(np.isfinite(f)) and np.all(rho > 0)
    g.set_f(f)
    g.step(1)
    g.sync()
    print(f"{name}: ok ({steps + 1} steps, N = {g.N})", flush=True)
    g.close()


def run_shard():
    cfg = bi.CavityConfig("shard", 3, 8, 8)
    cloud = bi.make_cloud(cfg)
    shards = bi.column_shards((cfg.Nv + 1) ** 2, 2)
    ranks = [Bgk(cfg, cloud, col_range=s, device="cuda:0") for s in shards]
    for _ in range(2):
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
    for r in ranks:
        r.sync()
    print("shard: ok", flush=True)


if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES) + ["shard"]
    for n in names:
        if n == "shard":
            run_shard()
        else:
            run(n)
