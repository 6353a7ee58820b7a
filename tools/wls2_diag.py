"""Which step/particle makes order-2 ALE parity jump: neighbour lists, positions, f error map."""
import numpy as np
import bgk_inputs as bi
import oracle
from paper_2408_02350_b200 import Bgk

oracle.build()
cfg = bi.C4.replace(wls_order=2)
cloud = bi.make_cloud(cfg)
g = Bgk(cfg, cloud, device="cuda:0")
for n in range(1, 6):
    g.step(1)
    g.sync()
    ref = oracle.run_steps(cfg, n)
    xg = g.positions()
    f = g.get_f().reshape(g.N, -1)
    err = np.abs(f - ref.f).max(1) / np.abs(ref.f).max()
    worst = np.argsort(err)[-5:][::-1]
    offg, idxg = oracle.neighbors(xg, cfg.h2)
    offr, idxr = oracle.neighbors(ref.x, cfg.h2)
    same = np.array_equal(offg, offr) and np.array_equal(idxg, idxr)
    print("step", n, "pos diff/dx %.2e" % (np.abs(xg - ref.x).max() / cfg.dx), "nb same", same,
          "worst", [(int(i), "%.2e" % err[i], int(cloud["kind"][i])) for i in worst], flush=True)
    # pre-step geometry of this step was built on x^{n-1}: report ill-conditioning of worst particle
    if err.max() > 1e-12:
        xs = ref.x
        i = int(worst[0])
        nb = idxr[offr[i]:offr[i + 1]]
        d2 = ((xs[nb] - xs[i]) ** 2).sum(1)
        print("   worst particle", i, "x/dx", xs[i] / cfg.dx, "m", len(nb), "min |d2-h2|/h2 %.2e" % (np.abs(d2 - cfg.h2).min() / cfg.h2))
        U = ref.macro[i]
        print("   macro", U)
