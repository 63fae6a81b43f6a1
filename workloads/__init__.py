"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This module holds none of the method's arithmetic: it only draws particle positions and
velocities (DESIGN.md §4 input recipe) and names the BASELINE.json configurations.
Positions are i.i.d. uniform in the periodic box; velocities are i.i.d.
N(0, kT) per component with the mean subtracted.  numpy PCG64, init_seed=1;
DPD seed=42.
"""
from __future__ import annotations

from dataclasses import dataclass, field, asdict

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    box: tuple
    rho: float
    a: float
    gamma: float
    kT: float
    power: float
    dt: float
    rc: float = 1.0
    seed: int = 42
    body_f: float = 0.0
    steps: int = 100
    grid: tuple = (1, 1, 1)  # rank grid for multi-GPU configs (S1)

    @property
    def n(self) -> int:
        return int(round(self.rho * self.box[0] * self.box[1] * self.box[2]))

    def as_dict(self):
        return asdict(self)


# BASELINE.json "configs":
CONFIGS = {
    # 1: parity -- 8^3, rho=3, a=25, gamma=45, kT=1, k=0.5, dt=0.01, 100 steps vs oracle
    "parity": Config("parity", (8.0, 8.0, 8.0), 3.0, 25.0, 45.0, 1.0, 0.5, 0.01, steps=100),
    # 2: equilibrium 64^3 rho=8; paper PP benchmark params a=50, kT=1, gamma=20, dt=0.002
    "eq64": Config("eq64", (64.0, 64.0, 64.0), 8.0, 50.0, 20.0, 1.0, 0.5, 0.002, steps=1000),
    # 3: periodic Poiseuille 96^3, Fig.-3 params, f = 0.005 (C-16)
    "pois96": Config("pois96", (96.0, 96.0, 96.0), 8.0, 10.0, 20.0, 1.0, 0.5, 0.005, body_f=0.005,
                     steps=120000),
    # 4: weak scaling, 128^3 per GPU, config-2 params
    "weak128": Config("weak128", (128.0, 128.0, 128.0), 8.0, 50.0, 20.0, 1.0, 0.5, 0.002, steps=100),
    # 5: strong scaling 256^3 total
    "strong256": Config("strong256", (256.0, 256.0, 256.0), 8.0, 50.0, 20.0, 1.0, 0.5, 0.002, steps=100),
}


def with_box(cfg: Config, box) -> Config:
    d = cfg.as_dict()
    d["box"] = tuple(float(b) for b in box)
    return Config(**d)


def make_particles(box, rho: float, kT: float, init_seed: int = 1, n: int | None = None):
    """Uniform positions in [0, L) and Maxwell-Boltzmann velocities, mean removed.
    Returns float32 arrays pos[n,3], vel[n,3]."""
    rng = np.random.Generator(np.random.PCG64(init_seed))
    L = np.asarray(box, dtype=np.float64)
    if n is None:
        n = int(round(rho * L[0] * L[1] * L[2]))
    pos = rng.random((n, 3)) * L
    pos = pos.astype(np.float32)
    # float32 rounding can land exactly on L; keep the open interval [0, L)
    for k in range(3):
        bad = pos[:, k] >= np.float32(L[k])
        pos[bad, k] = 0.0
    vel = rng.normal(0.0, np.sqrt(kT), size=(n, 3)) if kT > 0 else np.zeros((n, 3))
    if n > 0:
        vel -= vel.mean(axis=0, keepdims=True)
    return pos, vel.astype(np.float32)


def make_config(cfg: Config, init_seed: int = 1):
    return make_particles(cfg.box, cfg.rho, cfg.kT, init_seed)
