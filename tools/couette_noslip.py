"""Plane Couette flow between SDF walls (NEXT-3): measured shear rate
against 2U/H and the fluid velocity at the walls.  Walls at z = 2 and z = L_z - 2 moving at
-U / +U along x; frozen layer carved either from the uniform start or from an equilibrated
periodic fluid ("the same radial distribution function as the fluid").
usage: python tools/couette_noslip.py set equil  (set: gw | paper; equil: 0 | 1)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import workloads  # noqa: E402
from paper_1911_04712_b200 import capi  # noqa: E402

SETS = {  # (rho, a, gamma, kT, k, dt)
    "gw": (3.0, 25.0, 4.5, 1.0, 0.5, 0.01),        # Groot-Warren water (round-1 test)
    "paper": (10.0, 10.0, 10.0, 0.5, 0.125, 0.001),  # the paper's wall validation (Taylor-Couette)
    "jeffery": (8.0, 25.0, 50.0, 0.5, 0.5, 0.005),  # the paper's moving-plate setup
}


def run(name, equil, U=1.0, box=(10.0, 10.0, 20.0), t_relax=20.0, t_sample=20.0, seed=2):
    rho, a, gamma, kT, k, dt = SETS[name]
    H = box[2] - 4.0
    d = capi.DPD(box, 1.0, a, gamma, kT, k, dt, 42)
    pos, vel = workloads.make_particles(box, rho, kT, init_seed=seed)
    d.set_particles(pos, vel)
    if equil:  # periodic fluid relaxes its structure first; the carve then freezes an equilibrium layer
        d.step(int(round(10.0 / dt)))
        pos, vel = d.get_particles()
    vel = vel.copy()
    vel[:, 0] += U * (np.clip(pos[:, 2], 2.0, box[2] - 2.0) - 0.5 * box[2]) / (0.5 * H)  # start on the profile
    lo = (1, (0.0, 0.0, -1.0, -2.0), (-U, 0.0, 0.0))
    hi = (1, (0.0, 0.0, 1.0, box[2] - 2.0), (U, 0.0, 0.0))
    d.set_walls([lo, hi])
    d.set_particles(pos, vel)
    d.wall_carve(1)
    fluid = d.get_species() == 0
    d.step(int(round(t_relax / dt)))
    nb = 16
    edges = np.linspace(2.0, box[2] - 2.0, nb + 1)
    acc, cnt = np.zeros(nb), np.zeros(nb)
    every = max(1, int(round(0.1 / dt)))
    for _ in range(int(round(t_sample / (every * dt)))):
        d.step(every)
        x, v = d.get_particles()
        kk = np.clip(np.digitize(x[fluid, 2], edges) - 1, 0, nb - 1)
        acc += np.bincount(kk, weights=v[fluid, 0], minlength=nb)
        cnt += np.bincount(kk, minlength=nb)
    zc = 0.5 * (edges[1:] + edges[:-1])
    prof = acc / np.maximum(cnt, 1)
    dens = cnt / cnt.mean()
    slope, icpt = np.polyfit(zc[2:-2], prof[2:-2], 1)  # bulk fit, away from the wall layers
    return {"set": name, "equilibrated_carve": bool(equil), "params": dict(zip(["rho", "a", "gamma", "kT", "k", "dt"],
                                                                              SETS[name])),
            "slope_over_2U_H": slope / (2 * U / H), "v_wall_lo": slope * 2.0 + icpt + U,
            "v_wall_hi": slope * (box[2] - 2.0) + icpt - U, "profile": prof.round(4).tolist(),
            "density_profile": dens.round(3).tolist()}


if __name__ == "__main__":
    print(json.dumps(run(sys.argv[1], int(sys.argv[2]))))
