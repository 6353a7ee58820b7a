"""The velocity-sharded step through torch.distributed (Bgk.step_sharded) on one GPU.

Two processes share cuda:0 and a gloo process group (NCCL refuses two ranks on one
device); each owns half of the velocity columns and the only exchange is the two
all-reduces of Bgk.step_sharded.  The gathered distribution must match the oracle to the
parity tolerance.  On a multi-GPU box bench.py runs the same code with NCCL.
"""
import os
import socket

import numpy as np
import pytest

import bgk_inputs as bi

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, cfg, steps, q):
    import torch
    import torch.distributed as dist
    from paper_2408_02350_b200 import Bgk
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cloud = bi.make_cloud(cfg)
    ncol = (cfg.Nv + 1) ** (cfg.dims - 1)
    shard = bi.column_shards(ncol, world)[rank]
    g = Bgk(cfg, cloud, col_range=shard, device="cuda:0")
    for _ in range(steps):
        g.step_sharded()
    torch.cuda.synchronize()
    f = g.get_f()
    rho, U, T = g.moments_sharded()
    q.put((rank, shard, f, rho))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [bi.C1, bi.CavityConfig("c4s", 3, 10, 8)])
def test_two_rank_sharded_step_matches_oracle(cfg):
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import oracle
    steps = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, cfg, steps, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ref = oracle.run_steps(cfg, steps)
    N = len(ref.x)
    n1 = cfg.Nv + 1
    ncol = n1 ** (cfg.dims - 1)
    nv = 2 if cfg.dims == 2 else 1
    full = np.zeros((N, nv, n1, ncol))
    for _, (c0, c1), f, _ in res:
        full[:, :, :, c0:c1] = f.reshape(N, nv, n1, c1 - c0)
    err = np.abs(full.reshape(N, -1) - ref.f).max() / np.abs(ref.f).max()
    assert err <= 1e-10
    r0, _, _ = ref.moments()
    for _, _, _, rho in res:
        assert np.abs(rho / r0 - 1).max() <= 1e-10
