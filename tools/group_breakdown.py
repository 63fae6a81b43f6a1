"""Per-kernel-class time of one member of an in-process group (CUDA events around each
launch on the shared stream), against the same box as one domain.
With mode loopback: the one-rank NCCL context of the whole box whose split dimensions are
their own neighbour (dpd_create_loopback); "nccl" is the time of the send/recv groups.
usage: python tools/group_breakdown.py [L=128] [grid=2,2,2] [steps=20] [mode=group|loopback]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import workloads  # noqa: E402
from paper_1911_04712_b200 import capi  # noqa: E402

L = float(sys.argv[1]) if len(sys.argv) > 1 else 128.0
grid = tuple(int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "2,2,2").split(","))
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
cfg = workloads.with_box(workloads.CONFIGS["eq64"], (L, L, L))
pos, vel = workloads.make_config(cfg)
if len(sys.argv) > 4 and sys.argv[4] == "loopback":
    c = capi.dpd_create_loopback(cfg.box, cfg.rc, cfg.a, cfg.gamma, cfg.kT, cfg.power, cfg.dt, cfg.seed, grid)
    capi.dpd_set_particles_ex(c, pos, vel, np.arange(pos.shape[0], dtype=np.int32), 0)
    capi.dpd_step(c, 10)
    capi.dpd_set_timing(c, True)
    capi.dpd_step(c, steps)
    t = {k: round(1e3 * ms / steps, 1) for k, (ms, nl) in capi.dpd_get_timing(c).items() if nl}
    print(json.dumps({"box": L, "split": grid, "mode": "loopback", "us_per_step": t}))
    capi.dpd_destroy(c)
    sys.exit(0)
ctxs = capi.dpd_create_group(cfg.box, cfg.rc, cfg.a, cfg.gamma, cfg.kT, cfg.power, cfg.dt, cfg.seed, grid)
ids = np.arange(pos.shape[0], dtype=np.int32)
for c in ctxs:
    capi.dpd_set_particles_ex(c, pos, vel, ids, 0)
capi.dpd_group_step(ctxs, 10)
for c in ctxs:
    capi.dpd_set_timing(c, True)
capi.dpd_group_step(ctxs, steps)
tot = {}
for c in ctxs:
    for k, (ms, nl) in capi.dpd_get_timing(c).items():
        if nl:
            tot[k] = tot.get(k, 0.0) + ms
per_member_step_us = {k: round(1e3 * v / (steps * len(ctxs)), 1) for k, v in sorted(tot.items(), key=lambda x: -x[1])}
print(json.dumps({"box": L, "grid": grid, "us_per_member_step": per_member_step_us,
                  "sum_us": round(sum(per_member_step_us.values()), 1)}))
for c in ctxs:
    capi.dpd_destroy(c)
