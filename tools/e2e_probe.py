import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import workloads
from paper_1911_04712_b200 import capi
cfg = workloads.CONFIGS["eq64"]
torch.cuda.set_device(0)
stream = torch.cuda.Stream()
ctx = capi.dpd_create(cfg.box, cfg.rc, cfg.a, cfg.gamma, cfg.kT, cfg.power, cfg.dt, cfg.seed)
capi.dpd_set_stream(ctx, stream.cuda_stream)
pos, vel = workloads.make_particles(cfg.box, cfg.rho, cfg.kT, init_seed=1)
n = pos.shape[0]
pos_h = torch.from_numpy(pos).pin_memory(); vel_h = torch.from_numpy(vel).pin_memory()
out_pos = torch.empty((n, 3), dtype=torch.float32).pin_memory(); out_vel = torch.empty((n, 3), dtype=torch.float32).pin_memory()
capi.dpd_set_particles_ex(ctx, pos_h, vel_h, None, 0); capi.dpd_step(ctx, 20)
for rep in range(3):
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    t0 = time.perf_counter()
    ev[0].record(stream)
    capi.dpd_set_particles_ex(ctx, pos_h, vel_h, None, 0)
    t1 = time.perf_counter()
    ev[1].record(stream)
    capi.dpd_step_async(ctx, int(os.environ.get("K", "200")))
    ev[2].record(stream)
    capi.dpd_get_particles(ctx, out_pos, out_vel)
    ev[3].record(stream)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print("set %.2f ms (host %.2f)  steps %.2f ms  get %.2f ms  total %.2f (wall %.2f)" % (
        ev[0].elapsed_time(ev[1]), 1e3*(t1-t0), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3]), ev[0].elapsed_time(ev[3]), 1e3*(t3-t0)))
capi.dpd_set_timing(ctx, True)
capi.dpd_set_particles_ex(ctx, pos_h, vel_h, None, 0)
capi.dpd_get_particles(ctx, out_pos, out_vel)
print({k: v for k, v in capi.dpd_get_timing(ctx).items() if v[1]})
