"""Parity drift diagnostics for the second-order WLS path: rel max-norm of f vs the oracle per step."""
import sys
import numpy as np
import bgk_inputs as bi
import oracle
from paper_2408_02350_b200 import Bgk

oracle.build()


def rel(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


cases = [bi.C4, bi.C4.replace(wls_order=2), bi.C4.replace(wls_order=2, ale=0),
         bi.C4.replace(wls_order=2, Nv=8), bi.C1.replace(wls_order=2)]
for cfg in cases:
    cloud = bi.make_cloud(cfg)
    g = Bgk(cfg, cloud, device="cuda:0")
    out = []
    for n in (1, 2, 5, 10):
        g2 = Bgk(cfg, cloud, device="cuda:0")
        g2.step(n)
        g2.sync()
        ref = oracle.run_steps(cfg, n)
        out.append("%d:%.2e" % (n, rel(g2.get_f().reshape(g2.N, -1), ref.f)))
    print(cfg.name, cfg.wls_order, cfg.ale, cfg.Nv, " ".join(out), flush=True)
