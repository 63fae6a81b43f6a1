"""3D domain decomposition on one GPU: an
in-process group of subdomain contexts exchanging ghosts and migrants by device copies runs
the same kernels as the NCCL path.  Checked against the oracle's all-pairs sums (the plain
definition, C-1) with the per-step protocol of C-13, plus particle/id conservation."""
import numpy as np
import pytest

import oracle
import workloads
from test_gpu_parity import FORCE_TOL, boundary_eps, by_id, check_forces

pytestmark = pytest.mark.gpu


def make_group(cfg, grid):
    from paper_1911_04712_b200 import capi
    ctxs = capi.dpd_create_group(cfg.box, cfg.rc, cfg.a, cfg.gamma, cfg.kT, cfg.power, cfg.dt, cfg.seed, grid)
    return capi, ctxs


def gather_state(capi, ctxs):
    parts = [capi.dpd_get_state(c) for c in ctxs]
    pos = np.concatenate([p[0] for p in parts])
    u = np.concatenate([p[1] for p in parts])
    f = np.concatenate([p[2] for p in parts])
    ids = np.concatenate([p[3] for p in parts])
    return pos, u, f, ids


def destroy(capi, ctxs):
    for c in ctxs:
        capi.dpd_destroy(c)


@pytest.mark.parametrize("grid", [(2, 1, 1), (2, 2, 1), (2, 2, 2), (3, 1, 2)])
def test_group_prime_forces_match_oracle(grid):
    cfg = workloads.with_box(workloads.CONFIGS["parity"], (12.0, 12.0, 12.0))
    p = oracle.DPDParams(box=cfg.box, rc=cfg.rc, a=cfg.a, gamma=cfg.gamma, kT=cfg.kT, power=cfg.power, dt=cfg.dt,
                         seed=cfg.seed)
    pos0, vel0 = workloads.make_config(cfg)
    capi, ctxs = make_group(cfg, grid)
    try:
        ids0 = np.arange(pos0.shape[0], dtype=np.int32)
        for c in ctxs:  # every member receives the global set and keeps its own share
            capi.dpd_set_particles_ex(c, pos0, vel0, ids0, 0)
        capi.dpd_group_step(ctxs, 0)  # prime: ghost exchange + forces
        counts = [capi.dpd_get_count(c) for c in ctxs]
        assert sum(counts) == pos0.shape[0] and min(counts) > 0
        pos, u, f, ids = gather_state(capi, ctxs)
        assert np.array_equal(np.sort(ids), ids0)
        x_id, u_id, f_id = by_id(ids, pos, u, f)
        np.testing.assert_allclose(x_id, pos0, atol=1e-5)  # local frames map back exactly
        F_ref, allow, _ = oracle.forces(p, x_id, u_id, 0, eps=boundary_eps(cfg.box))
        check_forces(f_id, F_ref, allow)
    finally:
        destroy(capi, ctxs)


@pytest.mark.parametrize("graph", [0, 1])
@pytest.mark.parametrize("grid", [(2, 1, 1), (2, 2, 2)])
def test_group_per_step_parity_with_migration(grid, graph):
    """30 steps at dt = 0.01 (config-1 parameters): particles migrate between subdomains; each
    step the oracle recomputes F(x_s, u_s, s) from the gathered GPU state (C-13).  graph = 1
    runs the production step: the task graph of build_step_graph for every member (ghost
    pack / exchange / sort on the communication streams, concurrent with the interior forces,
    CUDA-event edges) with the NCCL send/recv swapped for a device copy of the same
    capacity-padded messages."""
    cfg = workloads.with_box(workloads.CONFIGS["parity"], (12.0, 12.0, 12.0))
    p = oracle.DPDParams(box=cfg.box, rc=cfg.rc, a=cfg.a, gamma=cfg.gamma, kT=cfg.kT, power=cfg.power, dt=cfg.dt,
                         seed=cfg.seed)
    pos0, vel0 = workloads.make_config(cfg)
    n = pos0.shape[0]
    capi, ctxs = make_group(cfg, grid)
    try:
        capi.dpd_set_option(ctxs[0], "group_task_graph", graph)
        ids0 = np.arange(n, dtype=np.int32)
        for c in ctxs:
            capi.dpd_set_particles_ex(c, pos0, vel0, ids0, 0)
        capi.dpd_group_step(ctxs, 0)
        start_counts = [capi.dpd_get_count(c) for c in ctxs]
        for s in range(1, 31):
            capi.dpd_group_step(ctxs, 1)
            pos, u, f, ids = gather_state(capi, ctxs)
            assert len(ids) == n and np.array_equal(np.sort(ids), ids0), "particles lost or duplicated"
            assert all(capi.dpd_get_step(c) == s for c in ctxs)
            x_id, u_id, f_id = by_id(ids, pos, u, f)
            F_ref, allow, _ = oracle.forces(p, x_id, u_id, s, eps=boundary_eps(cfg.box))
            check_forces(f_id, F_ref, allow)
        moved = sum(abs(capi.dpd_get_count(c) - k) for c, k in zip(ctxs, start_counts))
        assert moved > 0  # migration actually happened
    finally:
        destroy(capi, ctxs)


@pytest.mark.parametrize("graph", [0, 1])
def test_group_matches_single_domain(graph):
    """Same initial state on one domain and on a 2x2x2 group: forces after 5 steps agree to
    fp32 accuracy (identical RNG words: global ids key the pair RNG, C-7/C-19)."""
    from paper_1911_04712_b200 import capi
    cfg = workloads.with_box(workloads.CONFIGS["eq64"], (16.0, 16.0, 16.0))
    pos0, vel0 = workloads.make_config(cfg)
    single = capi.DPD(cfg.box, cfg.rc, cfg.a, cfg.gamma, cfg.kT, cfg.power, cfg.dt, cfg.seed)
    single.set_particles(pos0, vel0)
    _, ctxs = make_group(cfg, (2, 2, 2))
    try:
        capi.dpd_set_option(ctxs[0], "group_task_graph", graph)
        ids0 = np.arange(pos0.shape[0], dtype=np.int32)
        for c in ctxs:
            capi.dpd_set_particles_ex(c, pos0, vel0, ids0, 0)
        capi.dpd_group_step(ctxs, 0)
        pos, u, f, ids = gather_state(capi, ctxs)
        x1, u1, f1, ids1 = single.get_state()
        a = by_id(ids, pos, f)
        b = by_id(ids1, x1, f1)
        np.testing.assert_allclose(a[0], b[0], atol=1e-5)
        scale = np.abs(b[1]).max()
        assert np.abs(a[1] - b[1]).max() < FORCE_TOL * scale
    finally:
        destroy(capi, ctxs)


def test_group_temperature_and_momentum():
    """Equilibrium on a 2x2x1 group (rho = 8, Table-2 parameters): T = kT within 1%
    and total momentum conserved through migration and halo forces."""
    cfg = workloads.with_box(workloads.CONFIGS["eq64"], (16.0, 16.0, 16.0))
    pos0, vel0 = workloads.make_config(cfg)
    capi, ctxs = make_group(cfg, (2, 2, 1))
    try:
        ids0 = np.arange(pos0.shape[0], dtype=np.int32)
        for c in ctxs:
            capi.dpd_set_particles_ex(c, pos0, vel0, ids0, 0)
        capi.dpd_group_step(ctxs, 200)
        Ts, Ps = [], []
        for _ in range(60):
            capi.dpd_group_step(ctxs, 10)
            vs = np.concatenate([capi.dpd_get_particles_ex(c)[1] for c in ctxs]).astype(np.float64)
            assert vs.shape[0] == pos0.shape[0]
            Ts.append(oracle.temperature(vs))
            Ps.append(vs.sum(axis=0))
        assert abs(np.mean(Ts) - 1.0) < 0.01, np.mean(Ts)
        assert np.abs(np.array(Ps)).max() < 1e-2 * np.sqrt(pos0.shape[0])
    finally:
        destroy(capi, ctxs)


@pytest.mark.parametrize("name", ["weak128", "strong256"])
def test_group_full_size_sampled_parity(name):
    """2x2x2 group over BASELINE config 4's 128^3 box (16.8 M particles, 64^3 per subdomain)
    and config 5's 256^3 box (134 M particles, 128^3 per subdomain: the weak-scaling subdomain
    of the multi-GPU bench) at rho = 8: after the prime and 3 steps with migration, sampled
    all-j force sums (local + halo pairs) against the oracle's plain definition (C-1), every id
    present exactly once, sum F = 0."""
    cfg = workloads.CONFIGS[name]
    p = oracle.DPDParams(box=cfg.box, rc=cfg.rc, a=cfg.a, gamma=cfg.gamma, kT=cfg.kT, power=cfg.power, dt=cfg.dt,
                         seed=cfg.seed)
    pos0, vel0 = workloads.make_config(cfg)
    n = pos0.shape[0]
    capi, ctxs = make_group(cfg, (2, 2, 2))
    try:
        ids0 = np.arange(n, dtype=np.int32)
        for c in ctxs:
            capi.dpd_set_particles_ex(c, pos0, vel0, ids0, 0)
        capi.dpd_group_step(ctxs, 0)
        capi.dpd_group_step(ctxs, 3)
        steps = {capi.dpd_get_step(c) for c in ctxs}
        assert len(steps) == 1
        pos, u, f, ids = gather_state(capi, ctxs)
        assert pos.shape[0] == n and np.array_equal(np.sort(ids), ids0)
        # boundary particles sit in the halo of up to 7 other subdomains: sample those too
        rng = np.random.default_rng(7)
        half = cfg.box[0] / 2.0  # subdomain edge
        near = np.where(np.any(np.abs(np.mod(pos, half) - half / 2.0) > half / 2.0 - 1.0, axis=1))[0]
        sel = np.concatenate([rng.choice(n, 16, replace=False), rng.choice(near, 16, replace=False)])
        F_ref, allow = oracle.forces_subset(p, pos, u, steps.pop(), sel, ids=ids.astype(np.uint32),
                                            eps=boundary_eps(cfg.box))
        scale = np.abs(f).max()
        err = np.abs(f[sel].astype(np.float64) - F_ref).max(axis=1)
        assert np.all(err <= FORCE_TOL * scale + allow), (err.max(), scale)
        assert np.abs(f.astype(np.float64).sum(0)).max() < 1e-5 * np.abs(f).sum()
    finally:
        destroy(capi, ctxs)


def test_ghost_capacity_overflow_is_reported():
    """Message slots sized far below the boundary-layer occupancy (message_capacity_percent =
    10): the ghost pack counts the overflow, writes only what fits and the step reports
    DPD_ERR_CAPACITY instead of corrupting memory."""
    from paper_1911_04712_b200 import capi
    cfg = workloads.with_box(workloads.CONFIGS["parity"], (12.0, 12.0, 12.0))
    pos0, vel0 = workloads.make_config(cfg)
    _, ctxs = make_group(cfg, (2, 1, 1))
    try:
        ids0 = np.arange(pos0.shape[0], dtype=np.int32)
        for c in ctxs:
            capi.dpd_set_option(c, "message_capacity_percent", 10)
            capi.dpd_set_particles_ex(c, pos0, vel0, ids0, 0)
        with pytest.raises(capi.DPDError) as e:
            capi.dpd_group_step(ctxs, 1)
        assert e.value.code == capi.DPD_ERR_CAPACITY
    finally:
        destroy(capi, ctxs)


def test_group_empty_and_one_sided_sets():
    """Edge cases of the decomposition: an empty set (n = 0) steps without work on every
    member, and a set living entirely inside one subdomain leaves the others empty but still
    exchanging (zero-count messages) while it expands into them."""
    from paper_1911_04712_b200 import capi
    cfg = workloads.with_box(workloads.CONFIGS["parity"], (12.0, 12.0, 12.0))
    _, ctxs = make_group(cfg, (2, 2, 1))
    try:
        e = np.zeros((0, 3), np.float32)
        for c in ctxs:
            capi.dpd_set_particles_ex(c, e, e, np.zeros(0, np.int32), 0)
        capi.dpd_group_step(ctxs, 5)
        assert [capi.dpd_get_count(c) for c in ctxs] == [0, 0, 0, 0]
        pos0, vel0 = workloads.make_config(cfg)
        inside = np.all(pos0 < 5.5, axis=1)  # all in member 0's subdomain [0, 6)^2 x [0, 12)
        pos1, vel1 = pos0[inside], vel0[inside]  # the block expands into the empty members
        ids1 = np.arange(pos1.shape[0], dtype=np.int32)
        for c in ctxs:
            # message slots are sized from the global density (here ~1/5 of member 0's):
            # a non-uniform set needs the documented head-room option
            capi.dpd_set_option(c, "message_capacity_percent", 800)
            capi.dpd_set_particles_ex(c, pos1, vel1, ids1, 0)
        assert [capi.dpd_get_count(c) for c in ctxs][1:] == [0, 0, 0]
        capi.dpd_group_step(ctxs, 100)
        counts = [capi.dpd_get_count(c) for c in ctxs]
        assert sum(counts) == pos1.shape[0] and min(counts[1:]) > 0
        ids = np.concatenate([gather_state(capi, [c])[3] for c in ctxs])
        assert np.array_equal(np.sort(ids), ids1)
    finally:
        destroy(capi, ctxs)


@pytest.mark.parametrize("graph", [0, 1])
def test_member_array_capacity_overflow_is_reported(graph):
    """A dense block drifting into an empty member fills that member's particle arrays (sized
    at set time from its own share: 1.1 n + 12 sqrt(n) + 4096) past their capacity: the step
    reports DPD_ERR_CAPACITY (the scatter refuses slots beyond the arrays) instead of writing
    past them."""
    from paper_1911_04712_b200 import capi
    # force-free particles (a = gamma = kT = 0): the slab drifts intact at u = 3 along x
    cfg = workloads.Config("capacity", (12.0, 12.0, 12.0), 3.0, 0.0, 0.0, 0.0, 0.5, 0.01)
    rng = np.random.default_rng(3)
    n = 9000
    pos = np.empty((n, 3), np.float32)
    pos[:, 0] = 4.9 + rng.random(n) * 1.0  # a slab against member 1's face at x = 6
    pos[:, 1:] = rng.random((n, 2)) * 12.0
    vel = np.zeros((n, 3), np.float32)
    vel[:, 0] = 3.0
    _, ctxs = make_group(cfg, (2, 1, 1))
    try:
        capi.dpd_set_option(ctxs[0], "group_task_graph", graph)
        ids = np.arange(n, dtype=np.int32)
        for c in ctxs:
            capi.dpd_set_option(c, "message_capacity_percent", 100000)  # the messages are not the limit
            capi.dpd_set_particles_ex(c, pos, vel, ids, 0)
        assert capi.dpd_get_count(ctxs[1]) == 0
        with pytest.raises(capi.DPDError) as e:
            capi.dpd_group_step(ctxs, 60)
        assert e.value.code == capi.DPD_ERR_CAPACITY
    finally:
        destroy(capi, ctxs)
