"""Seeded synthetic inputs shared by the CUDA path and the CPU oracle.

This module is the ONLY code both sides share.  It holds the workload
recipe -- particle positions, particle kinds, initial macroscopic fields and
the scalar configuration -- and none of the method's arithmetic (no
Maxwellian, no moments, no weights, no neighbour tests, no flux).  Each side
computes f^0 = M(rho^0, U^0, T^0) itself from the fields generated here.

Recipe:
  * cavity [0, L]^d, L = 1e-6 m, Argon constants of PAPER.md:535
    (d = 0.368e-9 m, k_B = 1.3806e-23, R = 208, T0 = T_wall = 270 K),
    lid velocity (1, 0[, 0]) on y = L (2D) or z = L (3D);
  * regular lattice with n points per axis, dx = L/(n-1), lattice
    points on the faces are boundary particles; an edge/corner point takes the
    lowest wall id, and the lid has the highest id, so ties go to a stationary
    wall;
  * optional jitter of interior points by U(-j, j)*dx per coordinate
    (numpy PCG64, seed given in the config);
  * h = 3.1 dx, h2 = h*h computed once here and handed to both
    sides;
  * v_max = |U_wall| + 4 sqrt(R T0);
  * rho0 from Kn: rho0 = k_B / (sqrt(2) pi R d^2 Kn L), stored
    as literal numbers below and pinned by a test against the oracle's
    mean-free-path formula;
  * initial fields: "equilibrium" = uniform (rho0, 0, T0), or
    "stress" = rho0 (1 + 0.1 prod_a sin(pi x_a/L)),
    U = 10 m/s (sin 2 pi y/L, -sin 2 pi x/L[, 0]), T = T0 (1 + 0.05 cos pi x/L)
    (so every (particle, velocity) has O(1) transport).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

# Argon driven cavity constants.
L_CAVITY = 1.0e-6
D_MOL = 0.368e-9
K_B = 1.3806e-23
R_GAS = 208.0
T0 = 270.0
H_FACTOR = 3.1
ALPHA_W = 6.0

# rho0 for Kn = 0.1 / 1 / 10 (Z13): k_B/(sqrt(2) pi R d^2 Kn L), evaluated in fp64.
RHO0_BY_KN = {0.1: 1.1031740216824177, 1.0: 0.11031740216824179, 10.0: 0.011031740216824178}

# v_max = |U_wall| + 4 sqrt(R T0) = 1 + 4 sqrt(56160)  (Z4)
VMAX_DEFAULT = 948.924047590312


@dataclasses.dataclass(frozen=True)
class CavityConfig:
    name: str
    dims: int                 # 2 = Chu-reduced 2D, 3 = full 3D
    n_per_axis: int
    Nv: int                   # velocity cells per axis -> Nv+1 nodes per axis (Z3)
    Kn: float = 1.0
    dt: float = 1.0e-11
    ale: int = 1              # 1 = ALE (W = U^n, particles move, geometry rebuilt); 0 = fixed cloud
    jitter: float = 0.0       # interior jitter amplitude in units of dx
    seed: int = 2408023500
    init: str = "stress"      # "stress" | "equilibrium"
    vmax: float = VMAX_DEFAULT
    lid: float = 1.0          # lid speed; 0 gives an all-stationary box
    wls_order: int = 1        # Taylor order of the WLS derivative (1: the paper's scheme; 2: P:368-369)
    L: float = L_CAVITY
    # particle management (Z28): merge/fill pass at the
    # start of every ALE step when manage = 1; r_merge <= 0 -> 0.2 dx, m_min <= 0 -> dims + 3
    # (S:351-352); max_particles <= 0 -> N + N // 8 + 64 (capacity for inserted particles)
    manage: int = 0
    r_merge: float = 0.0
    m_min: int = 0
    max_particles: int = 0
    defects: int = 0          # management workloads: `defects` close pairs + `defects` holes (lattice())
    staging: int = 0          # 1: input staging buffer for overlapped host -> device copies (e2e)
    rho_init: float = 0.0     # > 0: initial density given directly (the paper's rho0 = 1 case),
                              # overriding the Kn table; Kn is then k_B/(sqrt(2) pi R d^2 rho L)

    @property
    def rho0(self) -> float:
        return self.rho_init if self.rho_init > 0 else RHO0_BY_KN[self.Kn]

    @property
    def dx(self) -> float:
        return self.L / (self.n_per_axis - 1)

    @property
    def h(self) -> float:
        return H_FACTOR * self.dx

    @property
    def h2(self) -> float:
        h = self.h
        return h * h

    @property
    def n_nodes(self) -> int:
        return (self.Nv + 1) ** self.dims

    @property
    def n_particles(self) -> int:
        return self.n_per_axis ** self.dims

    @property
    def merge_radius(self) -> float:
        return self.r_merge if self.r_merge > 0 else 0.2 * self.dx

    @property
    def min_neighbors(self) -> int:
        return self.m_min if self.m_min > 0 else self.dims + 3

    @property
    def capacity(self) -> int:
        n = self.n_particles
        return self.max_particles if self.max_particles > 0 else n + n // 8 + 64

    @property
    def U_lid(self) -> tuple:
        return (self.lid, 0.0, 0.0)

    def replace(self, **kw) -> "CavityConfig":
        return dataclasses.replace(self, **kw)


# The five workloads of BASELINE.json "configs".
C1 = CavityConfig("C1_2d_21x21_Nv12", 2, 21, 12, Kn=1.0, dt=1.0e-11)
C2 = CavityConfig("C2_2d_101x101_Nv32", 2, 101, 32, Kn=1.0, dt=6.0e-12)
C3 = CavityConfig("C3_2d_141x141_jitter_Nv32", 2, 141, 32, Kn=1.0, dt=3.5e-12, jitter=0.3)
C4 = CavityConfig("C4_3d_20cube_Nv16", 3, 20, 16, Kn=1.0, dt=1.0e-11)
C5 = CavityConfig("C5_3d_40cube_Nv24", 3, 40, 24, Kn=1.0, dt=1.0e-11)
CONFIGS = {c.name: c for c in (C1, C2, C3, C4, C5)}


def lattice(cfg: CavityConfig):
    """Positions (N, d) float64 and kinds (N,) int8 of the seeded cavity cloud.

    Particle index = ix + n*iy (+ n^2*iz): x fastest.  kind 0 = interior,
    1..2d = wall id: 1: x=0, 2: x=L, 3: y=0, 4: y=L, (5: z=0, 6: z=L); the lid
    is wall 2d.  Edge and corner points take the lowest wall id they lie on.
    """
    n, d, L = cfg.n_per_axis, cfg.dims, cfg.L
    if n < 3:
        raise ValueError("n_per_axis must be >= 3 (SPEC.md:62)")
    dx = L / (n - 1)
    axis = np.arange(n, dtype=np.float64) * dx
    axis[-1] = L
    grids = np.meshgrid(*([np.arange(n)] * d), indexing="ij")
    # meshgrid 'ij' gives index (i0, i1, i2) with i_last fastest; we want x fastest.
    idx = [g.reshape(-1) for g in grids][::-1]  # idx[0] = ix (fastest), ...
    N = n ** d
    x = np.empty((N, d), dtype=np.float64)
    kind = np.zeros(N, dtype=np.int8)
    for a in range(d):
        x[:, a] = axis[idx[a]]
    # wall id: assign from the highest id down so the LOWEST id a point lies on wins.
    for wid in range(2 * d, 0, -1):
        a, side = (wid - 1) // 2, (wid - 1) % 2
        on = (idx[a] == 0) if side == 0 else (idx[a] == n - 1)
        kind[on] = wid
    if cfg.jitter > 0.0:
        rng = np.random.Generator(np.random.PCG64(cfg.seed))
        J = rng.uniform(-cfg.jitter, cfg.jitter, size=(N, d)) * dx
        interior = kind == 0
        x[interior] += J[interior]
    if cfg.defects > 0:
        x, kind = _apply_defects(cfg, x, kind, idx)
    return x, kind


def _apply_defects(cfg: CavityConfig, x, kind, idx):
    """Management workload (seeded, PCG64(seed + 1)): `defects` interior particles are moved by
    0.95 dx along +x towards their interior +x neighbour (a pair 0.05 dx apart, below the
    default merge radius 0.2 dx), and `defects` holes are cut by removing a 2^d block of
    interior particles (lattice positions only; the rest of the cloud is untouched)."""
    n, d, dx = cfg.n_per_axis, cfg.dims, cfg.dx
    rng = np.random.Generator(np.random.PCG64(cfg.seed + 1))
    ijk = np.stack(idx, axis=1)                       # (N, d) lattice indices, x first
    deep = np.all((ijk >= 2) & (ijk <= n - 4), axis=1)
    cand = np.nonzero(deep)[0]
    pick = rng.permutation(cand)
    used = np.zeros(len(x), dtype=bool)
    moved, holes = 0, []
    stride = np.array([n ** a for a in range(d)])
    for i in pick:
        if moved < cfg.defects:
            j = i + 1                                  # +x neighbour (x fastest)
            block = [i, j]
            if used[block].any():
                continue
            x[i, 0] += 0.95 * dx
            used[np.clip(np.arange(i - 2 * n ** (d - 1), i + 2 * n ** (d - 1) + 1), 0, len(x) - 1)] = True
            moved += 1
        elif len(holes) < cfg.defects:
            corner = ijk[i]
            offs = np.array(np.meshgrid(*([[0, 1]] * d), indexing="ij")).reshape(d, -1).T
            block = (corner[None, :] + offs) @ stride
            if used[block].any():
                continue
            holes.extend(block.tolist())
            used[np.clip(np.arange(i - 3 * n ** (d - 1), i + 3 * n ** (d - 1) + 1), 0, len(x) - 1)] = True
        else:
            break
    keep = np.ones(len(x), dtype=bool)
    keep[holes] = False
    return x[keep], kind[keep]


def initial_fields(cfg: CavityConfig, x: np.ndarray):
    """Initial (rho, U, T) per particle: arrays (N,), (N, d), (N,)."""
    N, d = x.shape
    L = cfg.L
    rho = np.full(N, cfg.rho0)
    U = np.zeros((N, d))
    T = np.full(N, T0)
    if cfg.init == "equilibrium":
        return rho, U, T
    if cfg.init != "stress":
        raise ValueError(cfg.init)
    prod = np.ones(N)
    for a in range(d):
        prod *= np.sin(math.pi * x[:, a] / L)
    rho = cfg.rho0 * (1.0 + 0.1 * prod)
    U[:, 0] = 10.0 * np.sin(2.0 * math.pi * x[:, 1] / L)
    U[:, 1] = -10.0 * np.sin(2.0 * math.pi * x[:, 0] / L)
    T = T0 * (1.0 + 0.05 * np.cos(math.pi * x[:, 0] / L))
    return rho, U, T


def make_cloud(cfg: CavityConfig):
    """Everything a run needs as plain numpy arrays (host)."""
    x, kind = lattice(cfg)
    rho, U, T = initial_fields(cfg, x)
    return {"x": x, "kind": kind, "rho": rho, "U": U, "T": T}


def random_cloud(n: int, dims: int, seed: int, L: float = 1.0):
    """Uniform random points in [0, L]^d (neighbour-search stress input)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.uniform(0.0, L, size=(n, dims))


def column_shards(n_cols: int, world: int):
    """Contiguous column ranges [c0, c1) of the velocity plane for each rank.

    The velocity grid is sharded by "columns" (all nodes that share the
    fastest d-1 indices, i.e. a line along the slowest axis v_1); rank r owns
    columns [c0_r, c1_r).  Sizes differ by at most one.
    """
    if world < 1 or world > n_cols:
        raise ValueError("world size must be in [1, n_cols]")
    base, rem = divmod(n_cols, world)
    out, c = [], 0
    for r in range(world):
        sz = base + (1 if r < rem else 0)
        out.append((c, c + sz))
        c += sz
    return out
