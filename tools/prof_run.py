"""Minimal driver for ncu: a few whole steps of a workload through the C ABI (no timing)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bgk_inputs as bi  # noqa: E402
from paper_2408_02350_b200 import Bgk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5_3d_40cube_Nv24")
ap.add_argument("--steps", type=int, default=3)
a = ap.parse_args()
cfg = bi.CONFIGS[a.config]
g = Bgk(cfg, bi.make_cloud(cfg), device="cuda:0")
g.step(a.steps)
g.sync()
torch.cuda.synchronize()
print("done", cfg.name, a.steps)
