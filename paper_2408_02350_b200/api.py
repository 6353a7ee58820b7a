"""Thin Python binding of the C ABI (include/bgk.h) -- argument marshalling only.

PyTorch supplies the device workspace (one uint8 tensor), the stream
(``torch.cuda.current_stream().cuda_stream``) and, for velocity-sharded runs,
the process group that all-reduces the two small buffers between the split
phases.  Every step of the method runs in the library's CUDA kernels.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Tuple

import numpy as np
import torch

from . import _lib
from ._lib import BgkConfig, BgkError

ALPHA_W = 6.0


def make_config(cfg, col_range: Optional[Tuple[int, int]] = None, max_neighbors: int = 0,
                dt: Optional[float] = None) -> BgkConfig:
    """bgk_config from a bgk_inputs.CavityConfig (workload recipe)."""
    import bgk_inputs as bi
    c = BgkConfig()
    c.dims, c.Nv, c.vmax, c.L = cfg.dims, cfg.Nv, cfg.vmax, cfg.L
    c.h, c.h2, c.alpha_w = cfg.h, cfg.h2, bi.ALPHA_W
    c.dt = cfg.dt if dt is None else dt
    c.R, c.kb, c.dmol, c.T_wall = bi.R_GAS, bi.K_B, bi.D_MOL, bi.T0
    for a in range(3):
        c.U_lid[a] = cfg.U_lid[a]
    c.dx, c.ale = cfg.dx, cfg.ale
    if col_range is None:
        c.col_begin = c.col_end = 0
    else:
        c.col_begin, c.col_end = col_range
    c.max_neighbors = max_neighbors
    c.wls_order = getattr(cfg, "wls_order", 1)
    c.manage = getattr(cfg, "manage", 0)
    c.m_min = getattr(cfg, "m_min", 0)
    c.r_merge = getattr(cfg, "r_merge", 0.0)
    c.max_particles = cfg.capacity if getattr(cfg, "manage", 0) else 0
    c.staging = getattr(cfg, "staging", 0)
    return c


def _ptr(a) -> Optional[int]:
    if a is None:
        return None
    if isinstance(a, torch.Tensor):
        assert a.is_contiguous()
        return a.data_ptr()
    assert isinstance(a, np.ndarray) and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


class Bgk:
    """One rank's BGK solver state behind the C ABI."""

    def __init__(self, cfg, cloud: dict, col_range=None, max_neighbors: int = 0, device=None,
                 dt: Optional[float] = None):
        self.L = _lib.load()
        self.cfg = cfg
        self.dims = cfg.dims
        self.nval = 2 if cfg.dims == 2 else 1
        self.device = torch.device(device if device is not None else "cuda")
        self.c = make_config(cfg, col_range, max_neighbors, dt)
        N = int(len(cloud["x"])) if cloud.get("x") is not None else cfg.n_particles
        self._N = N
        n1 = cfg.Nv + 1
        ncol_g = n1 ** (cfg.dims - 1)
        self.col_range = (0, ncol_g) if col_range is None else tuple(col_range)
        self.ncol = self.col_range[1] - self.col_range[0]
        self.n1 = n1
        self.Kloc = n1 * self.ncol
        nbytes = C.c_size_t(0)
        self._check(self.L.bgk_workspace_size(C.byref(self.c), N, C.byref(nbytes)), ctx=False)
        self.ws = torch.empty(int(nbytes.value), dtype=torch.uint8, device=self.device)
        lattice = cloud.get("x") is None                     # the library builds the regular lattice
        x = None if lattice else np.ascontiguousarray(cloud["x"], dtype=np.float64)
        kind = None if lattice else np.ascontiguousarray(cloud["kind"], dtype=np.int8)
        macro0 = None
        if "rho" in cloud:
            macro0 = np.ascontiguousarray(np.column_stack([cloud["rho"], cloud["U"], cloud["T"]]), dtype=np.float64)
        self.ctx = C.c_void_p()
        with torch.cuda.device(self.device):
            st = self.L.bgk_init_cloud(C.byref(self.c), _ptr(x), _ptr(kind), _ptr(macro0), N,
                                       self.ws.data_ptr(), int(nbytes.value), self.stream, C.byref(self.ctx))
        self._check(st, ctx=False)
        self.kind = kind

    # ------------------------------------------------------------ helpers
    @property
    def N(self) -> int:
        """Current particle count (particle management may change it)."""
        if getattr(self, "ctx", None) and self.c.manage:
            n = C.c_int64(0)
            self._check(self.L.bgk_count(self.ctx, C.byref(n), None, None, None))
            self._N = int(n.value)
        return self._N

    def counts(self):
        """(N, interior, boundary, capacity)."""
        v = [C.c_int64(0) for _ in range(4)]
        self._check(self.L.bgk_count(self.ctx, *[C.byref(q) for q in v]))
        return tuple(int(q.value) for q in v)

    def manage(self):
        """One particle-management pass (bgk_manage); returns its report tuple
        (merges, merges kept, inserts, inserts deficient, inserts over capacity, N)."""
        rep = np.zeros(6, dtype=np.int64)
        self._check(self.L.bgk_manage(self.ctx, _ptr(rep), self.stream))
        return tuple(int(v) for v in rep)

    def stage_f(self, f, copy_stream=None):
        """Enqueue the host -> device copy of the next input state (canonical layout) on
        `copy_stream` (a torch.cuda.Stream); returns at once (bgk_stage_f)."""
        cs = copy_stream.cuda_stream if copy_stream is not None else self.stream
        self._check(self.L.bgk_stage_f(self.ctx, _ptr(f), cs))

    def use_staged_f(self):
        """The next step starts from the staged state (bgk_use_staged_f; stream-ordered)."""
        self._check(self.L.bgk_use_staged_f(self.ctx, self.stream))

    def transport_info(self):
        """(particles per warp, rows per lane, lattice-row groups, particles left to the general kernel,
        deep-interior tiles of 512 particles)."""
        v = np.zeros(5, dtype=np.int64)
        self._check(self.L.bgk_transport_info(self.ctx, _ptr(v)))
        return tuple(int(q) for q in v)

    def graph_info(self):
        """(graphs usable, steps launched as graphs, captures, steps re-run after a skip)."""
        v = np.zeros(4, dtype=np.int64)
        self._check(self.L.bgk_graph_info(self.ctx, _ptr(v)))
        return tuple(int(q) for q in v)

    def kinds(self):
        k = np.zeros(self.N, dtype=np.int8)
        self._check(self.L.bgk_get_kind(self.ctx, _ptr(k), self.stream))
        return k

    def manage_report(self):
        rep = np.zeros(6, dtype=np.int64)
        self._check(self.L.bgk_manage_report(self.ctx, _ptr(rep)))
        return tuple(int(v) for v in rep)

    @property
    def stream(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    def _check(self, st: int, ctx: bool = True):
        if st != _lib.BGK_OK:
            msg, part = "", -1
            if ctx and getattr(self, "ctx", None):
                p = C.c_int64(-1)
                m = self.L.bgk_last_error(self.ctx, C.byref(p))
                msg, part = (m.decode() if m else ""), p.value
            raise BgkError(st, msg, part)

    def close(self):
        if getattr(self, "ctx", None):
            self.L.bgk_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ the step
    def step(self, n: int = 1):
        self._check(self.L.bgk_step(self.ctx, int(n), self.stream))

    def step_transport(self):
        self._check(self.L.bgk_step_transport(self.ctx, self.stream))

    def step_relax(self):
        self._check(self.L.bgk_step_relax(self.ctx, self.stream))

    def step_boundary(self):
        self._check(self.L.bgk_step_boundary(self.ctx, self.stream))

    def run_phase(self, phase: int):
        self._check(self.L.bgk_run_phase(self.ctx, int(phase), self.stream))

    def step_sharded(self, group=None):
        """One step of a velocity-sharded run: the only data exchange is two
        all-reduces (moment sums [N,5], wall flux [N]) over the process group."""
        import torch.distributed as dist
        self.step_transport()
        dist.all_reduce(self.buffer(_lib.BUF_MOMENT_SUMS), group=group)
        self.step_relax()
        dist.all_reduce(self.buffer(_lib.BUF_WALL_FLUX), group=group)
        self.step_boundary()

    def buffer(self, which: int) -> torch.Tensor:
        """float64 view of an internal buffer (inside the workspace tensor)."""
        ptr, nb = C.c_void_p(), C.c_size_t(0)
        self._check(self.L.bgk_buffer(self.ctx, int(which), C.byref(ptr), C.byref(nb)))
        off = ptr.value - self.ws.data_ptr()
        return self.ws[off:off + nb.value].view(torch.float64)

    @property
    def ncs(self) -> int:
        """Stored column stride of the internal layout f[N][n1][ncs][nval] (include/bgk.h BGK_BUF_F):
        the local column count padded in 3D (128-byte rows), read off the buffer's size."""
        return self.buffer(_lib.BUF_F).numel() // (self.N * self.n1 * self.nval)

    def f_internal(self) -> torch.Tensor:
        """The current distribution buffer as a [N, n1, ncol, nval] view (padding stripped)."""
        f = self.buffer(_lib.BUF_F).view(self.N, self.n1, self.ncs, self.nval)
        return f[:, :, : self.ncol, :]

    def sync(self):
        self._check(self.L.bgk_sync(self.ctx, self.stream))

    # ------------------------------------------------------------ geometry
    def build_neighbors(self):
        need = C.c_int64(0)
        self._check(self.L.bgk_build_neighbors(self.ctx, None, None, 0, C.byref(need), self.stream))
        return int(need.value)

    def wls_coeffs(self):
        self._check(self.L.bgk_wls_coeffs(self.ctx, self.stream))

    def neighbors(self):
        nnz = C.c_int64(0)
        off = np.zeros(self.N + 1, dtype=np.int64)
        self._check(self.L.bgk_get_neighbors(self.ctx, _ptr(off), None, C.byref(nnz), self.stream))
        idx = np.zeros(max(int(nnz.value), 1), dtype=np.int32)
        self._check(self.L.bgk_get_neighbors(self.ctx, _ptr(off), _ptr(idx), C.byref(nnz), self.stream))
        return off, idx[: int(nnz.value)]

    def wls(self):
        off, idx = self.neighbors()
        d, nnz = self.dims, len(idx)
        S = np.zeros((self.N, d, d))
        rot = np.zeros((max(nnz, 1), d))
        fr = np.zeros((max(nnz, 1), d, d))
        cw = np.zeros(max(nnz, 1))
        self._check(self.L.bgk_get_wls(self.ctx, _ptr(S), _ptr(rot), _ptr(fr), _ptr(cw), self.stream))
        return S, rot[:nnz], fr[:nnz], cw[:nnz]

    def stable_dt(self) -> float:
        v = C.c_double(0.0)
        self._check(self.L.bgk_stable_dt(self.ctx, C.byref(v), self.stream))
        return float(v.value)

    def launches_per_step(self) -> int:
        v = C.c_int64(0)
        self._check(self.L.bgk_launches_per_step(self.ctx, C.byref(v)))
        return int(v.value)

    # ------------------------------------------------------------ state I/O
    def get_f(self, out=None):
        """Canonical layout [N, nval, n1*ncol_local] (host numpy by default, or a given tensor/array)."""
        if out is None:
            out = np.zeros((self.N, self.nval, self.Kloc))
        self._check(self.L.bgk_get_f(self.ctx, _ptr(out), self.stream))
        return out

    def set_f(self, f):
        if isinstance(f, np.ndarray):
            f = np.ascontiguousarray(f, dtype=np.float64)
        self._check(self.L.bgk_set_f(self.ctx, _ptr(f), self.stream))

    def positions(self):
        x = np.zeros((self.N, self.dims))
        self._check(self.L.bgk_get_positions(self.ctx, _ptr(x), self.stream))
        return x

    def macro(self):
        m = np.zeros((self.N, self.dims + 2))
        self._check(self.L.bgk_get_macro(self.ctx, _ptr(m), self.stream))
        return m

    def moments(self, out=None):
        """(rho[N], U[N,d], T[N]) of the current distribution (single rank)."""
        rho = np.zeros(self.N)
        U = np.zeros((self.N, self.dims))
        T = np.zeros(self.N)
        self._check(self.L.bgk_moments(self.ctx, _ptr(rho), _ptr(U), _ptr(T), self.stream))
        return rho, U, T

    def moments_sharded(self, group=None):
        import torch.distributed as dist
        self._check(self.L.bgk_moments_partial(self.ctx, self.stream))
        dist.all_reduce(self.buffer(_lib.BUF_MOMENT_SUMS), group=group)
        rho = np.zeros(self.N)
        U = np.zeros((self.N, self.dims))
        T = np.zeros(self.N)
        self._check(self.L.bgk_moments_finalize(self.ctx, _ptr(rho), _ptr(U), _ptr(T), self.stream))
        return rho, U, T
