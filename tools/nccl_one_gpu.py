"""Probe: the NCCL multi-GPU path (dpd_create_dist, task-graph step with ghost exchange on the
comm stream) with 2 ranks sharing cuda:0.  Launch:
  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 tools/nccl_one_gpu.py
NCCL may refuse two ranks on one device ("Duplicate GPU"); the script reports what happened."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads  # noqa: E402
from paper_1911_04712_b200 import capi  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("gloo")
cfg = workloads.with_box(workloads.CONFIGS["parity"], (12.0, 12.0, 12.0))
grid = (world, 1, 1)
sub = (cfg.box[0] / world, cfg.box[1], cfg.box[2])
uid = torch.zeros(128, dtype=torch.uint8)
if rank == 0:
    uid = torch.from_numpy(capi.dpd_nccl_unique_id())
dist.broadcast(uid, 0)
try:
    ctx = capi.dpd_create_dist(cfg.box, cfg.rc, cfg.a, cfg.gamma, cfg.kT, cfg.power, cfg.dt, cfg.seed, rank, world,
                               grid, uid.numpy())
except Exception as e:  # noqa: BLE001
    print(f"rank {rank}: dpd_create_dist failed: {e}", flush=True)
    sys.exit(0)
pos, vel = workloads.make_config(cfg)
ids = np.arange(len(pos), dtype=np.int32)
mine = (pos[:, 0] >= rank * sub[0]) & (pos[:, 0] < (rank + 1) * sub[0])
capi.dpd_set_particles_ex(ctx, np.ascontiguousarray(pos[mine]), np.ascontiguousarray(vel[mine]),
                          np.ascontiguousarray(ids[mine]), 0)
f_loc, id_loc = capi.dpd_get_forces_ex(ctx)
print(f"rank {rank}: schedule {[t[1] for t in capi.dpd_step_schedule(ctx)]}", flush=True)
capi.dpd_step(ctx, 50)
x, v, i2 = capi.dpd_get_particles_ex(ctx)
n = torch.tensor([len(i2)])
dist.all_reduce(n)
# reference: single-domain run of the same state
if rank == 0:
    d = capi.DPD(cfg.box, cfg.rc, cfg.a, cfg.gamma, cfg.kT, cfg.power, cfg.dt, cfg.seed)
    d.set_particles(pos, vel)
    f_ref = d.get_forces()
    d.step(50)
    xr, vr = d.get_particles()
parts = [None] * world
dist.all_gather_object(parts, (f_loc, id_loc, x, v, i2))
if rank == 0:
    F = np.zeros_like(f_ref)
    X = np.zeros_like(xr)
    for f, idl, xx, vv, ii in parts:
        F[idl] = f
        X[ii] = xx
    err = np.abs(F - f_ref).max() / np.abs(f_ref).max()
    dx = np.abs(X - xr)
    dx = np.minimum(dx, 12.0 - dx).max()
    print(f"NCCL 2-rank on one GPU: total n {int(n)} (expect {len(pos)}), prime force rel err {err:.2e}, "
          f"max |x - x_single| after 50 steps {dx:.2e}", flush=True)
capi.dpd_destroy(ctx)
dist.destroy_process_group()
