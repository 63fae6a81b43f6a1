import sys; sys.path.insert(0, '.')
import numpy as np, workloads
from paper_1911_04712_b200 import capi
cfg = workloads.CONFIGS["eq64"]
pos, vel = workloads.make_config(cfg)
d = capi.DPD(cfg.box, cfg.rc, cfg.a, cfg.gamma, cfg.kT, cfg.power, cfg.dt, cfg.seed)
d.set_particles(pos, vel)
print("after set", [d.get_stat(k) for k in ["fallback_staged", "fallback_home", "full_list_particles"]])
d.step(10)
print("after 10", [d.get_stat(k) for k in ["fallback_staged", "fallback_home", "full_list_particles"]])
x, u, f, ids = d.get_state()
# max half-stencil hits estimate: count neighbours within rc for a sample via cell grid
cfg1 = workloads.CONFIGS["parity"]
