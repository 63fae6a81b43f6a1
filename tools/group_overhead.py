"""Decomposition overhead on one GPU: the same global box stepped as one domain and as an
in-process group of subdomains (dpd_create_group: the NCCL path's kernels -- migration,
ghost pack, halo binning, one-sided halo forces -- with device copies as the transport).
Times dpd_step / dpd_group_step with CUDA events after warm-up; prints one JSON line.
mode serial: every phase of every member on one stream (device copies of the packed
counts); mode graph: the production task graph per member (ghost pack / exchange / sort on
the communication streams, concurrent with the interior forces) with the capacity-padded
messages the NCCL path sends (option group_task_graph); mode loopback: ONE subdomain of
the whole box whose dimensions with grid[k] = 1 in "split" are their own neighbour
(dpd_create_loopback): the production task graph with the real NCCL send/recv (to the rank
itself) -- at L = 128 and split 1,1,1 this is the per-GPU step of the weak-scaling series
(128^3 per GPU, six exchanged faces) with the transfer through NCCL's self path.
usage: python tools/group_overhead.py [L=128] [grid=2,2,2] [steps=50] [mode=graph|serial|loopback]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_1911_04712_b200 import capi  # noqa: E402

L = float(sys.argv[1]) if len(sys.argv) > 1 else 128.0
grid = tuple(int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "2,2,2").split(","))
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 50
mode = sys.argv[4] if len(sys.argv) > 4 else "graph"
cfg = workloads.with_box(workloads.CONFIGS["eq64"], (L, L, L))
pos, vel = workloads.make_config(cfg)
n = pos.shape[0]


def timed(run, k):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    run(k)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / k


d = capi.DPD(cfg.box, cfg.rc, cfg.a, cfg.gamma, cfg.kT, cfg.power, cfg.dt, cfg.seed)
d.set_particles(pos, vel)
d.step(10)
t_single = timed(d.step, steps)
del d
if mode == "loopback":
    c = capi.dpd_create_loopback(cfg.box, cfg.rc, cfg.a, cfg.gamma, cfg.kT, cfg.power, cfg.dt, cfg.seed, grid)
    capi.dpd_set_particles_ex(c, pos, vel, np.arange(n, dtype=np.int32), 0)
    capi.dpd_step(c, 10)
    t_loop = timed(lambda k: capi.dpd_step(c, k), steps)
    cnt = capi.dpd_get_count(c)
    sched = [f"{slot}:{name}" for slot, name, _ in capi.dpd_step_schedule(c)]
    capi.dpd_destroy(c)
    print(json.dumps({"box": L, "n": n, "split": grid, "steps": steps, "mode": mode, "ms_per_step_single": t_single,
                      "ms_per_step_loopback": t_loop, "overhead": t_loop / t_single - 1.0,
                      "particles_conserved": int(cnt) == n, "schedule": sched}))
    sys.exit(0)
ctxs = capi.dpd_create_group(cfg.box, cfg.rc, cfg.a, cfg.gamma, cfg.kT, cfg.power, cfg.dt, cfg.seed, grid)
capi.dpd_set_option(ctxs[0], "group_task_graph", 1 if mode == "graph" else 0)
ids = np.arange(n, dtype=np.int32)
for c in ctxs:
    capi.dpd_set_particles_ex(c, pos, vel, ids, 0)
capi.dpd_group_step(ctxs, 10)
t_group = timed(lambda k: capi.dpd_group_step(ctxs, k), steps)
counts = [capi.dpd_get_count(c) for c in ctxs]
for c in ctxs:
    capi.dpd_destroy(c)
print(json.dumps({"box": L, "n": n, "grid": grid, "steps": steps, "mode": mode, "ms_per_step_single": t_single,
                  "ms_per_step_group": t_group, "overhead": t_group / t_single - 1.0,
                  "particles_conserved": int(sum(counts)) == n}))
