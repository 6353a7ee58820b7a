"""Scaling sweeps of the paper's Figs. 6-7 on one B200.

Fig. 6: 3D driven cavity, fixed velocity grid N_v = 15 (16 nodes per axis, no zero node), initial
spatial grids n^3; Fig. 7: N = 40^3 particles, velocity grids N_v.  Both run to t_final = 400 dt
through the public API (bgk_step, ALE mode, the paper's equilibrium start), timed on the device
with CUDA events around the 400 steps.  The paper's curves are images (not recoverable), so
this is a characterisation of the B200 path, not a comparison.  One JSON line per run.

usage: python tools/sweeps.py [--steps 400] [--which n|nv|both] [--quick]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bgk_inputs as bi  # noqa: E402
from paper_2408_02350_b200 import Bgk  # noqa: E402


def run(cfg, steps):
    cloud = bi.make_cloud(cfg)
    g = Bgk(cfg, cloud, device="cuda:0")
    g.step(3)                       # warm-up (geometry, first launches)
    g.sync()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    e0.record(st)
    g.step(steps)
    e1.record(st)
    g.sync()
    torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    ms = e0.elapsed_time(e1)
    rho, U, T = g.moments()
    n_nodes = (cfg.Nv + 1) ** cfg.dims
    out = {"config": cfg.name, "n_per_axis": cfg.n_per_axis, "particles": len(cloud["kind"]),
           "Nv": cfg.Nv, "velocity_nodes": n_nodes, "steps": steps, "device_s": ms / 1e3, "wall_s": wall,
           "ms_per_step": ms / steps, "updates_per_s": len(cloud["kind"]) * n_nodes * steps / (ms / 1e3),
           "rho_minmax": [float(rho.min()), float(rho.max())], "T_minmax": [float(T.min()), float(T.max())]}
    g.close()
    del g
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--which", default="both", choices=["n", "nv", "both"])
    ap.add_argument("--quick", action="store_true", help="small sizes only (smoke)")
    a = ap.parse_args()
    base = dict(dims=3, Kn=1.0, dt=1.0e-11, ale=1, init="equilibrium")
    runs = []
    if a.which in ("n", "both"):
        for n in ((10, 14) if a.quick else (20, 30, 40, 50, 60)):
            runs.append(bi.CavityConfig(f"fig6_n{n}_Nv15", n_per_axis=n, Nv=15, **base))
    if a.which in ("nv", "both"):
        for nv in ((4, 6) if a.quick else (8, 12, 15, 16, 20, 24, 28)):
            runs.append(bi.CavityConfig(f"fig7_n40_Nv{nv}", n_per_axis=10 if a.quick else 40, Nv=nv, **base))
    for cfg in runs:
        print(json.dumps(run(cfg, a.steps)), flush=True)


if __name__ == "__main__":
    main()
