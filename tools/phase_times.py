"""Per-phase CUDA-event times of a workload (used for tuning runs; prints one JSON line)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bgk_inputs as bi  # noqa: E402
from paper_2408_02350_b200 import Bgk, _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5_3d_40cube_Nv24")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--fixed", action="store_true", help="fixed cloud (W = 0, geometry cached), no management")
a = ap.parse_args()
cfg = bi.CONFIGS[a.config]
if a.fixed:
    cfg = cfg.replace(ale=0, manage=0)
g = Bgk(cfg, bi.make_cloud(cfg), device="cuda:0")
g.step(a.warmup)
try:
    g.sync()
except Exception as ex:  # experiment builds may produce garbage states
    print('warning:', ex, file=sys.stderr)
st = torch.cuda.current_stream()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
acc = [0.0] * 6
for _ in range(a.steps):
    ev[0].record(st)
    for q in range(6):
        g.run_phase(q)
        ev[q + 1].record(st)
    torch.cuda.synchronize()
    for q in range(6):
        acc[q] += ev[q].elapsed_time(ev[q + 1])
try:
    g.sync()
except Exception as ex:
    print('warning:', ex, file=sys.stderr)
out = {p: acc[i] / a.steps for i, p in enumerate(_lib.PHASES)}
out["total"] = sum(out.values())
out["knobs"] = {k: v for k, v in os.environ.items() if k.startswith("BGK_")}
out["config"] = cfg.name
print(json.dumps(out))
