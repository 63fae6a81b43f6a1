"""Small end-to-end run for compute-sanitizer (memcheck / racecheck / synccheck):
config-1 box on one domain (the tiled and the reference force kernel), the species matrix,
asynchronous dumps (snapshot kernel + copy stream + writer thread) and a 2x2x2 in-process
group, serialised and as the production task graph (comm streams, CUDA events); with
SANITIZE_LOOPBACK=1 also the one-rank NCCL loopback context (split x, y, z)."""
import tempfile
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import workloads  # noqa: E402
from paper_1911_04712_b200 import capi  # noqa: E402

cfg = workloads.CONFIGS["parity"]
pos, vel = workloads.make_config(cfg)
# a ragged box at rho = 8: partial edge tiles (1-3 home cells wide), sweep blocks running into
# the sentinel gaps after every staged row
rg = workloads.Config("ragged", (11.3, 9.7, 7.2), 8.0, 25.0, 4.5, 1.0, 0.5, 0.005)
rp, rv = workloads.make_config(rg)
d = capi.DPD(rg.box, rg.rc, rg.a, rg.gamma, rg.kT, rg.power, rg.dt, rg.seed)
d.set_particles(rp, rv)
d.step(3)
d.get_forces()
for k in (0, 1):
    d = capi.DPD(cfg.box, cfg.rc, cfg.a, cfg.gamma, cfg.kT, cfg.power, cfg.dt, cfg.seed)
    d.set_option("force_kernel", k)
    d.set_particles(pos, vel)
    d.step(3)
    d.get_forces()
d = capi.DPD(cfg.box, cfg.rc, cfg.a, cfg.gamma, cfg.kT, cfg.power, cfg.dt, cfg.seed)
d.set_species(np.array([[25.0, 40.0], [40.0, 25.0]]), np.array([[45.0, 10.0], [10.0, 45.0]]))
d.set_particles_typed(pos, vel, None, (np.arange(len(pos)) % 2).astype(np.int32))
d.step(3)
with tempfile.TemporaryDirectory() as tmp:
    d.dump_open(os.path.join(tmp, "s"), 2)
    d.dump_every(2)
    d.step(5)
    d.dump_now()
    assert d.dump_close() == 4  # steps 4, 6, 8 and dump_now at 8
big = workloads.with_box(cfg, (12.0, 12.0, 12.0))
p2, v2 = workloads.make_config(big)
for graph in (0, 1):
    ctxs = capi.dpd_create_group(big.box, big.rc, big.a, big.gamma, big.kT, big.power, big.dt, big.seed, (2, 2, 2))
    capi.dpd_set_option(ctxs[0], "group_task_graph", graph)
    ids = np.arange(p2.shape[0], dtype=np.int32)
    for c in ctxs:
        capi.dpd_set_particles_ex(c, p2, v2, ids, 0)
    capi.dpd_group_step(ctxs, 3)
    for c in ctxs:
        capi.dpd_destroy(c)
if os.environ.get("SANITIZE_LOOPBACK") == "1":
    c = capi.dpd_create_loopback(big.box, big.rc, big.a, big.gamma, big.kT, big.power, big.dt, big.seed, (1, 1, 1))
    capi.dpd_set_particles_ex(c, p2, v2, np.arange(p2.shape[0], dtype=np.int32), 0)
    capi.dpd_step(c, 3)
    capi.dpd_get_state(c)
    capi.dpd_destroy(c)
print("sanitize run ok")
