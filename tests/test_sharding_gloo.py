"""World-size-2 gloo test (CPU) of the velocity-sharding decomposition the multi-GPU path uses.

Each rank owns a contiguous column range (bgk_inputs.column_shards) of the velocity grid,
forms the rank-local moment sums (sum f, sum v f, sum |v|^2 f [+ g2]) and the rank-local
incoming wall flux over its columns only, and the two buffers are all-reduced -- exactly
the two exchanges of Bgk.step_sharded.  The reduced sums must give the oracle's
(rho, U, T) of the full row and the oracle's full incoming flux.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bgk_inputs as bi


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, dims, Nv, out_q):
    import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = bi.CavityConfig("g", dims, 5, Nv)
    c = oracle.make_cfg(cfg)
    K = oracle.num_nodes(c)
    n1 = Nv + 1
    ncol = n1 ** (dims - 1)
    V = oracle.node_velocities(c).reshape(n1, ncol, dims)
    rng = np.random.default_rng(0)                  # same row on every rank
    rows = [oracle.maxwellian_row(c, 0.3, rng.uniform(-20, 20, dims), 280.0) * rng.uniform(0.9, 1.1)
            for _ in range(3)]
    c0, c1 = bi.column_shards(ncol, world)[rank]
    sums = torch.zeros(len(rows), 5, dtype=torch.float64)
    flux = torch.zeros(len(rows), dtype=torch.float64)
    n = oracle.wall_normal(dims, 1)
    for r, f in enumerate(rows):
        g1 = f[:K].reshape(n1, ncol)[:, c0:c1]
        v = V[:, c0:c1]
        sums[r, 0] = g1.sum()
        for a in range(dims):
            sums[r, 1 + a] = (v[..., a] * g1).sum()
        e = ((v ** 2).sum(-1) * g1).sum()
        if dims == 2:
            e += f[K:].reshape(n1, ncol)[:, c0:c1].sum()
        sums[r, 1 + dims] = e
        vn = v @ n
        flux[r] = (np.where(vn < 0, vn, 0.0) * g1).sum()
    dist.all_reduce(sums)
    dist.all_reduce(flux)
    if rank == 0:
        dv = oracle.dv(c)
        errs = []
        for r, f in enumerate(rows):
            s = sums[r].numpy()
            w = dv ** dims
            rho = s[0] * w
            U = s[1:1 + dims] / s[0]
            T = (s[1 + dims] * w - rho * (U @ U)) / (3 * rho * bi.R_GAS)
            r0, u0, t0 = oracle.moments_row(c, f)
            Vf = oracle.node_velocities(c)
            vn = Vf @ n
            fl0 = (np.where(vn < 0, vn, 0.0) * f[:K]).sum()
            errs.append(max(abs(rho / r0 - 1), np.abs(U - u0).max() / 237.0, abs(T / t0 - 1),
                            abs(flux[r].item() / fl0 - 1)))
        out_q.put(max(errs))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("dims,Nv", [(2, 12), (3, 8)])
def test_two_rank_gloo_decomposition(dims, Nv):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, dims, Nv, q)) for r in range(2)]
    for p in procs:
        p.start()
    err = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert err < 1e-12
