"""One 2x2x2 in-process group step of BASELINE config 4 (128^3 rho = 8 per subdomain) for an
ncu capture of the halo kernels (k_ghost_pack_cells, k_ghost_bin / scatter,
k_force_halo_cells).  usage: ncu ... python tools/halo_capture.py [L=256]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import workloads  # noqa: E402
from paper_1911_04712_b200 import capi  # noqa: E402

L = float(sys.argv[1]) if len(sys.argv) > 1 else 256.0
cfg = workloads.with_box(workloads.CONFIGS["eq64"], (L, L, L))
pos, vel = workloads.make_config(cfg)
ctxs = capi.dpd_create_group(cfg.box, cfg.rc, cfg.a, cfg.gamma, cfg.kT, cfg.power, cfg.dt, cfg.seed, (2, 2, 2))
capi.dpd_set_option(ctxs[0], "group_task_graph", 1)
ids = np.arange(pos.shape[0], dtype=np.int32)
for c in ctxs:
    capi.dpd_set_particles_ex(c, pos, vel, ids, 0)
capi.dpd_group_step(ctxs, 2)
for c in ctxs:
    capi.dpd_destroy(c)
print("ok")
