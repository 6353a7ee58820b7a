"""Benchmark: particle x velocity updates/s of the fp64 BGK step (and achieved HBM GB/s).

Workload (BASELINE.json north_star target): 3D driven cavity C5, 40^3 particles x 25^3
velocity nodes (Nv = 24), Kn = 1, dt = 1e-11, ALE mode (neighbours + WLS rebuilt every
step), synthetic seeded "stress" initial state (bgk_inputs).  One "step" is the whole hot
path: neighbour search, particle management (merge / fill pass; --manage 0 turns it off), WLS,
transport, moments, Maxwellian + relaxation, ALE move, diffuse-reflection walls.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl ours|reference]

N > 1 is launched with torch.distributed.run (one rank per GPU); the velocity grid is
sharded by columns and the only data exchange is two NCCL all-reduces per step (moment
sums [N,5] and wall flux [N]).  --impl reference times the CPU oracle (the paper-defined
reference of this tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bgk_inputs as bi  # noqa: E402

METRIC = "particle x velocity updates/s per BGK step (fp64) and achieved HBM GB/s"
UNIT = "updates/s"
FP64_LANES_PER_SM = 64           # B200: 64 FP64 FMA lanes per SM (B200_PROFILING / datasheet 37 TF)
N_SM = 148


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = "clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- CPU oracle baseline
class _AllRows:
    """f^0 rows of a whole cloud (built once by the oracle's or_init_f) as the row cache the sampled
    driver reads: the input state exists before the timed region, as on the GPU."""

    def __init__(self, F0):
        self.F0 = F0

    def __contains__(self, j):
        return True

    def __getitem__(self, j):
        return self.F0[j]


def cpu_info():
    model = ""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count() or 1, "cpu_model": model}


def oracle_sample_rate(cfg, cloud, seconds: float = 10.0, threads: int = 0, max_particles: int = 65536,
                       rows=None):
    """Time the oracle (as it stands) on interior particles of the workload: each task is the
    oracle's whole first step at one particle -- brute-force neighbour list, WLS + frames, transport
    over all K nodes, moments, tau, Maxwellian, relaxation, ALE move (oracle.sampled_first_step).
    The input state f^0 is built before the timed region (``rows``).  Returns (updates/s, threads,
    sample description)."""
    import concurrent.futures as cf

    import oracle
    oracle.build()
    kind = cloud["kind"]
    inter = np.nonzero(kind == 0)[0]
    rng = np.random.default_rng(2408)
    order = rng.permutation(inter)[:max_particles]
    threads = threads or (os.cpu_count() or 1)
    if rows is None:
        c = oracle.make_cfg(cfg)
        rows = _AllRows(oracle.init_f(c, cloud["rho"], cloud["U"], cloud["T"]))
    K = cfg.n_nodes
    done = 0
    t0 = time.perf_counter()
    if threads == 1:
        for i in order:
            oracle.sampled_first_step(cfg, cloud, [int(i)], f0=rows)
            done += 1
            if time.perf_counter() - t0 > seconds:
                break
    else:
        with cf.ThreadPoolExecutor(threads) as ex:   # ctypes releases the GIL inside the C oracle
            it = iter(order)
            futs = set()
            while True:
                while len(futs) < 2 * threads:
                    try:
                        i = int(next(it))
                    except StopIteration:
                        break
                    futs.add(ex.submit(oracle.sampled_first_step, cfg, cloud, [i], None, rows))
                if not futs:
                    break
                fin, futs = cf.wait(futs, return_when=cf.FIRST_COMPLETED)
                done += len(fin)
                if time.perf_counter() - t0 > seconds:
                    cf.wait(futs)                    # in-flight particles finish inside the timed region
                    done += len(futs)
                    break
    dt = time.perf_counter() - t0
    rate = done * K / dt
    desc = (f"oracle whole first step (neighbours, WLS, transport, moments, relaxation, move) at {done} random "
            f"interior particles of {cfg.name} (all {K} nodes each; f^0 built before timing), {threads} "
            f"thread(s), {dt:.1f} s")
    return rate, threads, desc


def oracle_whole_steps(cfg, steps: int, threads: int):
    """Seconds per whole-cloud oracle step (or_step: geometry, transport, moments, relaxation, move,
    boundary) at `threads` OpenMP threads; the initial state is built before timing."""
    import oracle
    oracle.build()
    prev = oracle.omp_threads()
    oracle.set_threads(threads)
    try:
        st = oracle.State(oracle.make_cfg(cfg), bi.make_cloud(cfg))
        t0 = time.perf_counter()
        st.step(steps)
        dt = (time.perf_counter() - t0) / steps
    finally:
        oracle.set_threads(prev)
    return dt


def cpu_baseline(cfg, cloud, seconds: float, full: bool = False):
    """The paper's CPU (1 thread) and OMP (all cores) columns (Tables 1-2) for this
    host: the bench workload sampled per particle at 1 thread and at all cores, and whole oracle steps
    of the two small configs (C1 2D, C4 3D) at 1 thread and all cores (C4 at 1 thread takes ~2 min:
    only with ``full``)."""
    import oracle
    info = cpu_info()
    ncores = info["nproc"]
    c = oracle.make_cfg(cfg)
    rows = _AllRows(oracle.init_f(c, cloud["rho"], cloud["U"], cloud["T"]))
    par, par_threads, par_desc = oracle_sample_rate(cfg, cloud, seconds, ncores, rows=rows)
    seq, _, seq_desc = oracle_sample_rate(cfg, cloud, seconds, 1, rows=rows)
    del rows
    whole = {}
    for wc, steps in ((bi.C1, 3), (bi.C4, 1)):
        upd = wc.n_particles * wc.n_nodes
        tp = oracle_whole_steps(wc, steps, ncores)
        whole[wc.name] = {"par_s_per_step": tp, "par_updates_per_s": upd / tp, "par_threads": ncores}
        if full or wc.dims == 2:
            t1 = oracle_whole_steps(wc, steps, 1)
            whole[wc.name].update({"seq_s_per_step": t1, "seq_updates_per_s": upd / t1})
    return {"value": par, "unit": UNIT, "cores": par_threads, "kind": "oracle", "sample": par_desc,
            "sequential": {"value": seq, "unit": UNIT, "cores": 1, "sample": seq_desc},
            "whole_steps": whole, **info}


def lean_count(dims: int) -> float:
    """fp64 instructions per (particle, neighbour, node) triple -- 10 in 3D, 8 in
    2D-Chu (two projections, two neg-parts, C, two accumulates shared by g1 and g2, sum C)."""
    return 10.0 if dims == 3 else 8.0


def measure_2d(cfg, dev, steps: int, warmup: int, peaks: dict):
    """A 2D workload as a secondary bench line (the configs where the HBM
    roofline is the binding one): whole ALE steps with particle management (CUDA events, the graph
    path of bgk_step), per-phase times, achieved HBM GB/s at 32 B per value and two values (g1, g2)
    per node, and the transport's fp64 roofline at the 2D lean count."""
    import torch

    from paper_2408_02350_b200 import Bgk
    from paper_2408_02350_b200 import _lib
    cfg = cfg.replace(manage=1)
    cloud = bi.make_cloud(cfg)
    g = Bgk(cfg, cloud, device=dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(warmup):
        g.step(1)
    g.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    e0.record(stream)
    for _ in range(steps):
        g.step(1)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / steps
    g.sync()
    phases = _lib.PHASES
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(phases) + 1)]
    acc = np.zeros(len(phases))
    nph = 10
    for _ in range(nph):
        ev[0].record(stream)
        for q in range(len(phases)):
            g.run_phase(q)
            ev[q + 1].record(stream)
        torch.cuda.synchronize(dev)
        acc += [ev[q].elapsed_time(ev[q + 1]) for q in range(len(phases))]
    ph = {p: float(v / nph) for p, v in zip(phases, acc)}
    g.sync()
    N, K = g.N, cfg.n_nodes
    off, _ = g.neighbors()
    sum_m = int(np.diff(off)[cloud["kind"] == 0].sum())
    hbm_gbs = 32.0 * 2 * N * K / (ms / 1e3) / 1e9
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    peak_instr = N_SM * FP64_LANES_PER_SM * sm_max * 1e6
    algo = lean_count(2) * sum_m * K
    info = g.transport_info()
    g.close()
    return {"workload": cfg.name, "ms_per_step": ms, "value": N * K / (ms / 1e3), "unit": UNIT, "steps": steps,
            "particles": N, "velocity_nodes": K, "interior_pairs": sum_m, "particle_management": True,
            "hbm_gbs": hbm_gbs, "hbm_frac": hbm_gbs / float(peaks.get("hbm_gbs", 6650.0)),
            "hbm_bytes_per_step": 32.0 * 2 * N * K, "phases_ms": ph,
            "transport_roofline": {"bound": "alu", "achieved": algo / (ph["transport"] / 1e3) / 1e12,
                                   "peak": peak_instr / 1e12, "unit": "T fp64-instr/s",
                                   "frac": algo / (ph["transport"] / 1e3) / peak_instr,
                                   "per_unit": f"{lean_count(2):g} fp64 instr per triple x {sum_m} pairs x {K} nodes"},
            "transport_mapping": {"particles_per_warp": info[0], "nodes_per_lane": info[1]}}


# ---------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2408_02350_b200 import Bgk
    from paper_2408_02350_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # validation knobs for the multi-rank path on a one-GPU box: every rank on device
    # BGK_BENCH_DEVICE, collectives over BGK_DIST_BACKEND (gloo); production uses NCCL, one GPU per rank
    local = int(os.environ.get("BGK_BENCH_DEVICE", local))
    backend = os.environ.get("BGK_DIST_BACKEND", "nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    cfg = bi.CONFIGS[args.config] if args.config in bi.CONFIGS else getattr(bi, args.config)
    if args.manage and cfg.ale:
        cfg = cfg.replace(manage=1)      # the paper's step includes "Particle Organization" (Table 3)
    if not args.no_e2e:
        cfg = cfg.replace(staging=1)     # e2e: host inputs staged on a copy stream, overlapped with steps
    cloud = bi.make_cloud(cfg)
    ncol = (cfg.Nv + 1) ** (cfg.dims - 1)
    shard = bi.column_shards(ncol, world)[rank]
    g = Bgk(cfg, cloud, col_range=shard if world > 1 else None, device=dev)
    N, K = g.N, cfg.n_nodes
    n_int = int((cloud["kind"] == 0).sum())
    stream = torch.cuda.current_stream(dev)

    def step():
        if world > 1:
            g.step_sharded()
        else:
            g.step(1)

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        step()
    g.sync()
    barrier()
    # ---- timed region: K whole steps (inputs are HBM-resident; f = N*K*8 B >> L2)
    peaks, peak_src = load_peaks()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        barrier()
    ms = e0.elapsed_time(e1)
    g.sync()
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    ms_step = ms / args.steps
    updates = N * K * args.steps
    value = updates / (ms / 1e3)

    # ---- per-phase breakdown (paper Table 3), CUDA events on the launching stream
    phases = _lib.PHASES
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(phases) + 1)]
    acc = np.zeros(len(phases))
    nph = max(2, min(args.steps, 5))
    barrier()
    for _ in range(nph):
        ev[0].record(stream)
        for q in range(len(phases)):
            g.run_phase(q)
            if world > 1 and q == 2:
                dist.all_reduce(g.buffer(_lib.BUF_MOMENT_SUMS))
            if world > 1 and q == 4:
                dist.all_reduce(g.buffer(_lib.BUF_WALL_FLUX))
            ev[q + 1].record(stream)
        torch.cuda.synchronize(dev)
        acc += [ev[q].elapsed_time(ev[q + 1]) for q in range(len(phases))]
    phase_ms = {p: float(v / nph) for p, v in zip(phases, acc)}
    g.sync()

    # ---- roofline of the dominant kernel (transport): fp64-issue bound
    off, idx = g.neighbors()
    inter = cloud["kind"] == 0
    sum_m = int(np.diff(off)[inter].sum())
    k_loc = g.Kloc
    t_tr = phase_ms["transport"] / 1e3
    # SURVEY.md §8(d) lean count: 3D 10 (3 projections + 5 add/abs + 2 accumulates), 2D-Chu 8
    instr_per_triple = lean_count(cfg.dims)
    algo_instr = instr_per_triple * sum_m * k_loc
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    peak_instr = N_SM * FP64_LANES_PER_SM * sm_max * 1e6
    traffic, traffic_src = None, None
    tp = os.path.join(ROOT, "profiles", "transport_traffic.json")
    if os.path.exists(tp):
        try:
            tj = json.load(open(tp))
            traffic = tj.get(cfg.name)
            traffic_src = tj.get("_note")
        except Exception:
            traffic = None
    roofline = {"bound": "alu", "kernel": "k_transport (fp64 pipe)",
                "achieved": algo_instr / t_tr / 1e12, "peak": peak_instr / 1e12,
                "unit": "T fp64-instr/s", "frac": algo_instr / t_tr / peak_instr, "traffic": traffic,
                "traffic_src": traffic_src,
                "per_unit": f"{instr_per_triple:g} fp64 instr per (particle, neighbour, node) triple; "
                            f"{sum_m} interior pairs x {k_loc} local nodes",
                "peak_src": f"{N_SM} SM x {FP64_LANES_PER_SM} FP64 lanes x {sm_max:.0f} MHz (sm_max of "
                            f"{peak_src} peaks)"}
    # achieved HBM (algorithmic): 32 B per particle-velocity value per step
    # (read f^n, write ftilde, read ftilde, write f^{n+1})
    nval = 2 if cfg.dims == 2 else 1
    bytes_step = 32.0 * N * K * nval
    hbm_gbs = bytes_step / (ms_step / 1e3) / 1e9

    # ---- e2e through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        Kl = g.Kloc
        N_e = g.N                        # the cloud as it is now (management may have changed it)
        host_f = torch.empty((N_e, nval, Kl), dtype=torch.float64, pin_memory=True)
        g.get_f(host_f)
        rho = torch.empty(N, dtype=torch.float64, pin_memory=True)
        U = torch.empty((N, cfg.dims), dtype=torch.float64, pin_memory=True)
        T = torch.empty(N, dtype=torch.float64, pin_memory=True)
        n_e2e = max(1, min(args.steps, args.e2e_steps))
        copy_stream = torch.cuda.Stream(dev)
        barrier()
        t0 = time.perf_counter()
        # every step: H2D of that step's input state from pinned host memory (on a copy stream,
        # issued one step ahead so it overlaps the previous step's compute), the step, and a
        # D2H read of its result (rho, U, T)
        g.stage_f(host_f, copy_stream)
        for n in range(n_e2e):
            g.use_staged_f()
            if n + 1 < n_e2e:
                g.stage_f(host_f, copy_stream)
            if world > 1:
                g.step_sharded()
                rr, uu, tt = g.moments_sharded()
            else:
                g.step(1)
                rr, uu, tt = g.moments()
            if g.N != N_e and n + 1 < n_e2e:
                # particle management changed the cloud: the staged rows are stale (bgk_use_staged_f
                # would refuse them) -- size the host buffer for the new N and stage again
                copy_stream.synchronize()
                N_e = g.N
                host_f = torch.empty((N_e, nval, Kl), dtype=torch.float64, pin_memory=True)
                g.get_f(host_f)
                g.stage_f(host_f, copy_stream)
        copy_stream.synchronize()
        barrier()
        dt_e2e = time.perf_counter() - t0
        tt_ = torch.tensor([dt_e2e], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tt_, op=dist.ReduceOp.MAX)
        dt_e2e = float(tt_.item())
        e2e = {"value": N * K * n_e2e / dt_e2e, "unit": UNIT,
               "h2d_bytes_per_step": int(host_f.numel() * 8 * world),
               "d2h_bytes_per_step": int(N_e * (cfg.dims + 2) * 8),
               "steps": n_e2e,
               "path": "bgk_stage_f(pinned host, copy stream, one step ahead) + bgk_use_staged_f + bgk_step "
                       "+ bgk_moments(host)"}

    launches = g.launches_per_step() * args.steps
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name, "particles": N, "interior": n_int, "velocity_nodes": K,
                   "interior_pairs": sum_m, "ale": bool(cfg.ale), "init": cfg.init, "dt": cfg.dt,
                   "particle_management": bool(cfg.manage),
                   "parallelism": f"velocity-sharded x{world}" if world > 1 else "single GPU",
                   "l2": f"inputs larger than L2 (f = {N * K * nval * 8 / 1e9:.1f} GB per buffer)"},
        "hbm_gbs": hbm_gbs, "hbm_frac": hbm_gbs / float(peaks.get("hbm_gbs", 6650.0)),
        "phases_ms": phase_ms,
        "roofline": roofline,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if world == 1 and cfg.ale and not args.no_secondary:
        # the fixed-cloud (Eulerian, W = 0, geometry cached) C5 run as the secondary
        # number -- the same kernels, without the per-step neighbour search / WLS / management
        g.close()
        del g
        torch.cuda.empty_cache()
        cfg2 = cfg.replace(ale=0, manage=0)
        g2 = Bgk(cfg2, cloud, device=dev)
        for _ in range(max(2, args.warmup)):
            g2.step(1)
        g2.sync()
        barrier()
        n2 = max(3, min(args.steps, 5))
        e0.record(stream)
        for _ in range(n2):
            g2.step(1)
        e1.record(stream)
        barrier()
        ms2 = e0.elapsed_time(e1) / n2
        g2.sync()
        info = g2.transport_info()
        out["secondary"] = {"workload": cfg2.name + " fixed cloud (W = 0, geometry cached)", "ms_per_step": ms2,
                            "value": N * K / (ms2 / 1e3), "unit": UNIT, "steps": n2,
                            "lattice_row_groups": info[2], "general_kernel_particles": info[3],
                            "deep_tiles": info[4], "deep_tile_particles": info[4] * 512,
                            "hbm_gbs": 32.0 * N * K / (ms2 / 1e3) / 1e9,
                            "hbm_frac": 32.0 * N * K / (ms2 / 1e3) / 1e9 / float(peaks.get("hbm_gbs", 6650.0))}
        g2.close()
    if world == 1 and cfg.dims == 3 and not args.no_secondary:
        out["secondary_2d"] = [measure_2d(c2, dev, 50, 5, peaks) for c2 in (bi.C2, bi.C3)]
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(cfg, cloud, args.cpu_seconds, args.cpu_full)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------------- reference arm (oracle)
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = bi.CONFIGS[args.config] if args.config in bi.CONFIGS else getattr(bi, args.config)
    cloud = bi.make_cloud(cfg)
    import oracle
    per = max(5.0, min(30.0, 150.0 / max(1, args.steps + args.warmup)))
    rows = _AllRows(oracle.init_f(oracle.make_cfg(cfg), cloud["rho"], cloud["U"], cloud["T"]))
    for _ in range(args.warmup):
        oracle_sample_rate(cfg, cloud, seconds=per / 3, rows=rows)
    rates, cores, desc = [], 1, ""
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r, cores, desc = oracle_sample_rate(cfg, cloud, seconds=per, rows=rows)
        rates.append(r)
    wall = time.perf_counter() - t0
    value = float(np.mean(rates))
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall / args.steps * 1e3,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic",
           "config": {"workload": cfg.name, "particles": cfg.n_particles, "velocity_nodes": cfg.n_nodes},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5_3d_40cube_Nv24")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--e2e-steps", type=int, default=6)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the fixed-cloud secondary number")
    ap.add_argument("--manage", type=int, default=1, choices=[0, 1],
                    help="particle management pass in every ALE step (the paper's Particle Organization)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-full", action="store_true", help="also time a whole C4 oracle step at 1 thread (~2 min)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
