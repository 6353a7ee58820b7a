"""Per-shard step times on ONE GPU -> predicted multi-GPU efficiency.

A velocity-sharded rank (bgk_inputs.column_shards) runs the split-phase step on its column range:
  step_transport  (replicated geometry + transport of its columns + rank-local moment sums)
  -- all_reduce(SUM) of [N, 5] fp64 --
  step_relax      (relaxation of its columns, ALE move, boundary interpolation + local wall flux)
  -- all_reduce(SUM) of [N] fp64 --
  step_boundary   (outgoing half of the boundary rows)
This tool times one rank's phases (CUDA events) for every shard of P = 1, 2, 4, 8 on one GPU.  The
two all-reduces are emulated by copying in the full-grid moment sums and wall fluxes of the
unsharded run at the same step (recorded once), so every shard's state evolves as in a real run
(its own slab sums alone would give the slab's mean velocity, hundreds of m/s, and scramble the ALE
cloud within a few steps).  The predicted step at P ranks is
    T_P = max_r (T_transport_r + T_relax_r + T_boundary_r) + T_allreduce,
T_allreduce a stated estimate for the two small NCCL all-reduces over NVLink 5 (latency-bound:
2.56 MB + 0.5 MB at C5), and the predicted efficiency E_P = T_1 / (P T_P).  Prints one JSON line.

    python tools/shard_times.py [--config C5_3d_40cube_Nv24] [--steps 5] [--allreduce-us 60]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bgk_inputs as bi  # noqa: E402
from paper_2408_02350_b200 import Bgk  # noqa: E402


def time_rank(cfg, cloud, col_range, steps, warmup, ref=None):
    """ref: None (record the full-grid sums of every step into a list) or that list (feed them)."""
    g = Bgk(cfg, cloud, col_range=col_range, device="cuda:0")
    st = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    acc = np.zeros(3)
    rec = [] if ref is None else None
    for n in range(warmup + steps):
        ev[0].record(st)
        g.step_transport()
        if ref is not None:
            g.buffer(0).copy_(ref[n][0])            # the all-reduced moment sums (emulated)
        ev[1].record(st)
        g.step_relax()
        if ref is not None:
            g.buffer(1).copy_(ref[n][1])            # the all-reduced wall flux (emulated)
        ev[2].record(st)
        g.step_boundary()
        ev[3].record(st)
        torch.cuda.synchronize()
        if rec is not None:
            rec.append((g.buffer(0).clone(), g.buffer(1).clone()))
        if n >= warmup:
            acc += [ev[q].elapsed_time(ev[q + 1]) for q in range(3)]
    try:
        g.sync()
    except Exception:          # a slab's state may drift without the all-reduce; timing is unaffected
        pass
    info = g.transport_info()
    g.close()
    del g
    torch.cuda.empty_cache()
    t = acc / steps
    out = {"col_range": list(col_range), "ncol": col_range[1] - col_range[0], "transport_ms": t[0],
           "relax_ms": t[1], "boundary_ms": t[2], "step_ms": float(t.sum()), "R": info[1]}
    return out, rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5_3d_40cube_Nv24")
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--allreduce-us", type=float, default=60.0,
                    help="estimate for the two all-reduces per step (NVLink 5, latency-bound sizes)")
    ap.add_argument("--ranks", default="1,2,4,8")
    a = ap.parse_args()
    cfg = bi.CONFIGS[a.config].replace(manage=1)
    cloud = bi.make_cloud(cfg)
    ncol = (cfg.Nv + 1) ** (cfg.dims - 1)
    out = {"config": cfg.name, "allreduce_ms_estimate": a.allreduce_us / 1e3, "ranks": {}}
    t1 = None
    r1, ref = time_rank(cfg, cloud, (0, ncol), a.steps, a.warmup)   # the full grid; its sums per step
    for P in [int(x) for x in a.ranks.split(",")]:
        shards = bi.column_shards(ncol, P)
        # ranks with the same column count run the same kernels: time one per distinct width
        seen, rows = {}, []
        for s in shards:
            w = s[1] - s[0]
            if w not in seen:
                seen[w] = r1 if P == 1 else time_rank(cfg, cloud, s, a.steps, a.warmup, ref)[0]
            rows.append(seen[w])
        tmax = max(r["step_ms"] for r in rows)
        tp = tmax + (a.allreduce_us / 1e3 if P > 1 else 0.0)
        if P == 1:
            t1 = tp
        out["ranks"][P] = {"shards": [list(s) for s in shards], "per_width": list(seen.values()),
                           "max_rank_step_ms": tmax, "predicted_step_ms": tp,
                           "predicted_efficiency": (t1 / (P * tp)) if t1 else None}
        print(f"P={P}: max rank step {tmax:.3f} ms, predicted {tp:.3f} ms, "
              f"efficiency {(t1 / (P * tp)) if t1 else float('nan'):.3f}", file=sys.stderr, flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
