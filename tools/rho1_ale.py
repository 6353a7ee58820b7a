"""Diagnostic: the rho0 = 1 cavity (Kn = 0.110) on the moving cloud with particle management, to
steady state -- how far the ALE run gets (DESIGN.md NEXT(2), Z30).  Prints one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bgk_inputs as bi  # noqa: E402
from paper_2408_02350_b200 import Bgk  # noqa: E402

cfg = bi.C2.replace(rho_init=1.0, init="equilibrium", manage=1)
g = Bgk(cfg, bi.make_cloud(cfg), device="cuda:0")
out = {"config": "C2 rho0=1 ALE + management", "steps": 0, "steady": False, "error": None}
prev = None
t0 = time.time()
try:
    for it in range(200):
        g.step(200)
        g.sync()
        out["steps"] += 200
        kind = g.kinds()
        inter = kind == 0
        U = g.macro()[:, 1:3]
        if prev is not None and len(prev) == len(U):
            num = np.linalg.norm(U[inter] - prev[inter])
            den = np.linalg.norm(U[inter])
            out["rel_change"] = float(num / den)
            if den > 0 and num / den < 1e-3:
                out["steady"] = True
                break
        prev = U.copy()
except Exception as e:
    out["error"] = str(e)
out["N"] = g.N
out["manage_report"] = g.manage_report()
out["graph_info"] = g.graph_info()
out["seconds"] = time.time() - t0
print(json.dumps(out))
