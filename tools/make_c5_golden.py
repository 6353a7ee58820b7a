"""Write the C5 ten-step golden (tests/golden/c5_10steps_oracle.npz) from the CPU oracle ONLY.

The bench workload (BASELINE.json configs[4]: 3D driven cavity, 40^3 particles
x 25^3 velocity nodes, Kn = 1, dt = 1e-11, ALE, parity-stress start, particle management on as in
bench.py) is stepped ten times by ``oracle.run_steps`` -- the plain fp64 C oracle, OpenMP over
particles -- and the following are stored:

  * rho, U, T of every particle after step 10 (``State.moments``: SPEC moments_3d);
  * macro: the recovered (rho, U, T) at interior particles after step 10;
  * x: every position after step 10 (ALE motion);
  * f rows of a fixed sample of particles (random interior, the first / last interior, near-lid
    interior, lid, side-wall and corner boundary particles), all 15 625 nodes each;
  * the per-step management reports (merges / fills; none are expected on the lattice).

Nothing here imports the CUDA package: the expected values come from ``oracle/`` alone
(task rule ③).  About 20-40 min on 8 host cores; run once:

    python tools/make_c5_golden.py [--steps 10] [--out tests/golden/c5_10steps_oracle.npz]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bgk_inputs as bi  # noqa: E402
import oracle  # noqa: E402


def sample_particles(cloud, n_random=8, seed=24080235):
    """The sampled rows: deterministic from the seeded cloud (no method arithmetic)."""
    kind = cloud["kind"]
    x = cloud["x"]
    inter = np.nonzero(kind == 0)[0]
    rng = np.random.default_rng(seed)
    s = [int(v) for v in rng.choice(inter, n_random, replace=False)]
    s += [int(inter[0]), int(inter[-1])]
    top = inter[np.argsort(-x[inter, 2], kind="stable")]     # the interior layer under the lid
    s += [int(top[0]), int(top[len(top) // 7])]
    for wid in (6, 2, 1):                                    # lid, x = L wall, corner / x = 0 wall
        b = np.nonzero(kind == wid)[0]
        s += [int(b[len(b) // 3])]
    s.append(int(np.nonzero(kind == 1)[0][0]))               # the (0, 0, 0) corner
    return sorted(set(s))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "c5_10steps_oracle.npz"))
    ap.add_argument("--config", default="C5_3d_40cube_Nv24")
    args = ap.parse_args()
    cfg = bi.CONFIGS[args.config].replace(manage=1)          # bench.py's step: management on
    cloud = bi.make_cloud(cfg)
    sample = sample_particles(cloud)
    oracle.build()
    t0 = time.time()
    st = oracle.State(oracle.make_cfg(cfg), cloud, manage=oracle.manage_params(cfg))
    for n in range(args.steps):
        st.step(1)
        print(f"step {n + 1}/{args.steps}: {time.time() - t0:.0f} s, report {st.reports[-1]}", flush=True)
    N = st.x.shape[0]
    assert N == len(cloud["x"]), "management changed the cloud (not expected on the C5 lattice)"
    rho, U, T = st.moments()
    meta = {"config": cfg.name, "steps": args.steps, "manage": 1, "init": cfg.init, "dt": cfg.dt,
            "threads": oracle.omp_threads(), "seconds": round(time.time() - t0, 1),
            "source": "oracle.run_steps (oracle/bgk_oracle.c or_manage + or_step), tools/make_c5_golden.py",
            "cites": "PAPER.md:163-199 (transport, moments, relaxation), 177-180 (ALE), 489-492 (management); "
                     "SURVEY.md §8(c) O1-O11, §8(d) C5"}
    np.savez_compressed(args.out, rho=rho, U=U, T=T, macro=st.macro, x=st.x,
                        sample=np.array(sample, dtype=np.int64), f_rows=st.f[sample],
                        reports=np.array(st.reports, dtype=np.int64), meta=json.dumps(meta))
    print(json.dumps(meta), flush=True)


if __name__ == "__main__":
    main()
