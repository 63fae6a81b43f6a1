"""The NCCL data plane on one GPU: a
one-rank context whose split dimensions are their own neighbour (dpd_create_loopback).
Ghosts and migrants are packed into the capacity-padded 26-direction messages and sent with
ncclSend / ncclRecv to the rank itself, inside the production task graph (ghost pack /
exchange / sort on the communication stream, concurrent with the interior forces,
CUDA-event edges), and the set-time density is an ncclAllReduce.  The pool has one B200 per
box and NCCL rejects two ranks on one device (profiles/r02_nccl_one_gpu.log), so this is
where exchange_nccl runs on hardware.  Checked against the oracle's all-pairs sums (C-1)
with the per-step protocol of C-13, and against the periodic single-domain context."""
import numpy as np
import pytest

import oracle
import workloads
from test_gpu_parity import FORCE_TOL, boundary_eps, by_id, check_forces

pytestmark = pytest.mark.gpu

SPLITS = [(1, 0, 0), (0, 1, 1), (1, 1, 1)]


def _loopback(cfg, split):
    from paper_1911_04712_b200 import capi
    return capi, capi.dpd_create_loopback(cfg.box, cfg.rc, cfg.a, cfg.gamma, cfg.kT, cfg.power, cfg.dt, cfg.seed,
                                          split)


def _params(cfg):
    return oracle.DPDParams(box=cfg.box, rc=cfg.rc, a=cfg.a, gamma=cfg.gamma, kT=cfg.kT, power=cfg.power,
                            dt=cfg.dt, seed=cfg.seed, body_f=cfg.body_f)


def test_loopback_rejects_no_split():
    from paper_1911_04712_b200 import capi
    cfg = workloads.CONFIGS["parity"]
    with pytest.raises(capi.DPDError):
        capi.dpd_create_loopback(cfg.box, cfg.rc, cfg.a, cfg.gamma, cfg.kT, cfg.power, cfg.dt, cfg.seed, (0, 0, 0))


@pytest.mark.parametrize("split", SPLITS)
def test_loopback_prime_and_per_step_parity(split):
    """Prime forces (ghost exchange through NCCL, then local + halo forces), then 30 steps at
    dt = 0.01: every step the oracle recomputes F(x_s, u_s, s) from the GPU state (C-13);
    particles leave through a split face, travel as migration messages and come back."""
    cfg = workloads.with_box(workloads.CONFIGS["parity"], (9.0, 8.0, 10.0))
    p = _params(cfg)
    pos0, vel0 = workloads.make_config(cfg)
    n = pos0.shape[0]
    capi, c = _loopback(cfg, split)
    try:
        ids0 = np.arange(n, dtype=np.int32)
        capi.dpd_set_particles_ex(c, pos0, vel0, ids0, 0)
        assert capi.dpd_get_count(c) == n
        pos, u, f, ids = capi.dpd_get_state(c)
        x_id, u_id, f_id = by_id(ids, pos, u, f)
        np.testing.assert_allclose(x_id, pos0, atol=1e-5)
        F_ref, allow, _ = oracle.forces(p, x_id, u_id, 0, eps=boundary_eps(cfg.box))
        check_forces(f_id, F_ref, allow)
        sched = {name: slot for slot, name, _ in capi.dpd_step_schedule(c)}
        assert sched["migrate_exchange"] == 0 and sched["ghost_exchange"] == 1 and sched["force_local"] == 0
        assert sched["halo_force"] == 1 and sched["join"] == 0  # halo forces beside the interior ones
        for s in range(1, 31):
            capi.dpd_step(c, 1)
            pos, u, f, ids = capi.dpd_get_state(c)
            assert len(ids) == n and np.array_equal(np.sort(ids), ids0), "particles lost or duplicated"
            assert capi.dpd_get_step(c) == s
            x_id, u_id, f_id = by_id(ids, pos, u, f)
            assert np.all(x_id >= 0) and np.all(x_id < np.asarray(cfg.box, np.float32))
            F_ref, allow, _ = oracle.forces(p, x_id, u_id, s, eps=boundary_eps(cfg.box))
            check_forces(f_id, F_ref, allow)
    finally:
        capi.dpd_destroy(c)


@pytest.mark.parametrize("split", [(1, 1, 1)])
def test_loopback_matches_single_domain(split):
    """Same initial state on the periodic single domain and on the loopback context: the
    per-particle state after 0, 1 and 5 steps agrees to fp32 accuracy (the global ids key the pair
    RNG, C-7/C-19, so both draw the same xi; only the summation order differs)."""
    from paper_1911_04712_b200 import capi
    cfg = workloads.with_box(workloads.CONFIGS["eq64"], (16.0, 16.0, 16.0))
    pos0, vel0 = workloads.make_config(cfg)
    single = capi.DPD(cfg.box, cfg.rc, cfg.a, cfg.gamma, cfg.kT, cfg.power, cfg.dt, cfg.seed)
    single.set_particles(pos0, vel0)
    _, c = _loopback(cfg, split)
    try:
        capi.dpd_set_particles_ex(c, pos0, vel0, np.arange(pos0.shape[0], dtype=np.int32), 0)
        for nsteps in (0, 1, 4):
            if nsteps:
                capi.dpd_step(c, nsteps)
                single.step(nsteps)
            pos, u, f, ids = capi.dpd_get_state(c)
            x1, u1, f1, ids1 = single.get_state()
            a = by_id(ids, pos, u, f)
            b = by_id(ids1, x1, u1, f1)
            d = np.abs(a[0] - b[0])
            d = np.minimum(d, np.asarray(cfg.box, np.float32) - d)  # a wrap on one side only
            assert d.max() < 1e-4
            np.testing.assert_allclose(a[1], b[1], atol=2e-3)
            assert np.abs(a[2] - b[2]).max() < 10 * FORCE_TOL * np.abs(b[2]).max()
    finally:
        capi.dpd_destroy(c)


def test_loopback_rejects_too_many_cells_per_dimension():
    """The boundary-cell list packs 10-bit cell coordinates: a decomposed subdomain must stay
    below 1024 cells per dimension, refused at create (DPD_ERR_CONFIG), not overflowed."""
    from paper_1911_04712_b200 import capi
    cfg = workloads.CONFIGS["parity"]
    with pytest.raises(capi.DPDError):
        capi.dpd_create_loopback((1100.0, 4.0, 4.0), cfg.rc, cfg.a, cfg.gamma, cfg.kT, cfg.power, cfg.dt, cfg.seed,
                                 (0, 1, 0))
    c = capi.dpd_create_loopback((1000.0, 4.0, 4.0), cfg.rc, cfg.a, cfg.gamma, cfg.kT, cfg.power, cfg.dt, cfg.seed,
                                 (0, 1, 0))
    capi.dpd_destroy(c)
