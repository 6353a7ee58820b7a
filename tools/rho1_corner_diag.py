"""Diagnostic for DESIGN.md Z30: run the rho0 = 1 ALE cavity with management until the lid corner's
interpolation system fails, then report the corner's interior stencil and the fill candidate."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bgk_inputs as bi  # noqa: E402
from paper_2408_02350_b200 import Bgk  # noqa: E402

cfg = bi.C2.replace(rho_init=1.0, init="equilibrium", manage=1)
g = Bgk(cfg, bi.make_cloud(cfg), device="cuda:0")
last_x = last_k = None
steps = 0
err = None
try:
    for it in range(100):
        g.step(100)
        g.sync()
        steps += 100
        last_x, last_k = g.positions(), g.kinds()
except Exception as e:
    err = str(e)
x, k = last_x, last_k
corner = np.array([0.0, cfg.L])
d = np.sqrt(((x - corner) ** 2).sum(1))
near = np.nonzero((k == 0) & (d <= cfg.h))[0]
cand = corner + 0.5 * cfg.h * np.array([1.0, -1.0])
dc = np.sqrt(((x - cand) ** 2).sum(1))
out = {"steps_ok": steps, "error": err, "dx": cfg.dx, "h": cfg.h,
       "corner_interior_stencil": [[float(v) / cfg.dx for v in (x[i] - corner)] for i in near],
       "candidate_nearest_dx": float(np.sort(dc)[0] / cfg.dx),
       "nearest_to_candidate": [[float(v) / cfg.dx for v in (x[i] - corner)] for i in np.argsort(dc)[:4]]}
print(json.dumps(out))
