import sys, time, json
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import workloads
from paper_1911_04712_b200 import capi
cfg = workloads.CONFIGS["eq64"]
pos, vel = workloads.make_config(cfg)
ctx = capi.dpd_create(cfg.box, cfg.rc, cfg.a, cfg.gamma, cfg.kT, cfg.power, cfg.dt, cfg.seed)
s = torch.cuda.Stream()
capi.dpd_set_stream(ctx, s.cuda_stream)
capi.dpd_set_particles_ex(ctx, pos, vel, None, 0)
capi.dpd_step(ctx, 220)
res = []
for rep in range(12):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s); capi.dpd_step_async(ctx, 200); e1.record(s); capi.dpd_sync(ctx)
    res.append(round(e0.elapsed_time(e1) / 200, 4))
print(res)
# per-step times within one 200-step region
ev = [torch.cuda.Event(enable_timing=True) for _ in range(201)]
torch.cuda.synchronize()
ev[0].record(s)
for i in range(200):
    capi.dpd_step_async(ctx, 1); ev[i + 1].record(s)
capi.dpd_sync(ctx)
st = [ev[i].elapsed_time(ev[i + 1]) for i in range(200)]
print("per-step min %.4f median %.4f max %.4f" % (min(st), sorted(st)[100], max(st)), sorted(st)[-5:])
