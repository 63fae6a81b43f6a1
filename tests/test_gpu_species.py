"""Species interaction matrix on the CUDA path against the
oracle.  Same bars as tests/test_gpu_parity.py: forces within 1e-4 max|F| + the C-12
boundary allowance; species bit-exact through steps, migration and ghost exchange."""
import numpy as np
import pytest

import oracle
import workloads
from test_gpu_parity import boundary_eps, by_id, check_forces, window_kw, windows

pytestmark = pytest.mark.gpu

A3 = np.array([[25.0, 10.0, 25.0], [10.0, 40.0, 0.0], [25.0, 0.0, 25.0]])
G3 = np.array([[4.5, 9.0, 0.0], [9.0, 20.0, 4.5], [0.0, 4.5, 45.0]])


def _species(n, seed=8, ns=3):
    return np.random.default_rng(seed).integers(0, ns, n).astype(np.int32)


def _params(cfg, sp):
    return oracle.DPDParams(box=cfg.box, rc=cfg.rc, a=cfg.a, gamma=cfg.gamma, kT=cfg.kT, power=cfg.power,
                            dt=cfg.dt, seed=cfg.seed, amat=A3, gmat=G3, species=sp)


@pytest.mark.parametrize("kernel", [0, 1])
@pytest.mark.parametrize("power", [0.5, 1.0])
def test_prime_forces_match_oracle(kernel, power):
    from paper_1911_04712_b200 import capi
    cfg = workloads.CONFIGS["parity"]
    pos, vel = workloads.make_config(cfg)
    sp = _species(len(pos))
    d = capi.DPD(cfg.box, cfg.rc, cfg.a, cfg.gamma, cfg.kT, power, cfg.dt, cfg.seed)
    d.set_option("force_kernel", kernel)
    d.set_species(A3, G3)
    d.set_particles_typed(pos, vel, None, sp, 0)
    p = _params(cfg, sp)
    p.power = power
    F_ref, allow, _ = oracle.forces(p, pos, vel, 0, **window_kw(cfg.box))
    check_forces(d.get_forces(), F_ref, allow)
    assert np.array_equal(d.get_species(), sp)


def test_per_step_parity_with_species():
    """30 steps, C-13 protocol: each step the oracle is fed the GPU state (ids, species)."""
    from paper_1911_04712_b200 import capi
    cfg = workloads.CONFIGS["parity"]
    pos0, vel0 = workloads.make_config(cfg)
    n = len(pos0)
    sp0 = _species(n, seed=12)
    d = capi.DPD(cfg.box, cfg.rc, cfg.a, cfg.gamma, cfg.kT, cfg.power, cfg.dt, cfg.seed)
    d.set_species(A3, G3)
    d.set_particles_typed(pos0, vel0, None, sp0, 0)
    eps, eps_img = windows(cfg.box)
    for s in range(31):
        pos, u, F, ids = d.get_state()
        x_id, u_id, F_id = by_id(ids, pos, u, F)
        spec, sids = d.get_species_ex()
        assert np.array_equal(spec[np.argsort(sids)], sp0)
        F_ref, allow, _ = oracle.forces(_params(cfg, sp0), x_id, u_id, s, eps=eps, eps_image=eps_img)
        check_forces(F_id, F_ref, allow)
        if s < 30:
            d.step(1)


def test_species_survive_migration_and_ghosts():
    """2x2x1 in-process group at dt = 0.01: species follow their particles across ranks, and
    forces across subdomain faces (ghost pairs) use the right matrix entries."""
    from paper_1911_04712_b200 import capi
    cfg = workloads.CONFIGS["parity"]
    grid = (2, 2, 1)
    gbox = tuple(cfg.box[k] * grid[k] for k in range(3))
    pos, vel = workloads.make_particles(gbox, cfg.rho, cfg.kT, init_seed=3)
    n = len(pos)
    sp = _species(n, seed=5)
    ids = np.arange(n, dtype=np.int32)
    ctxs = capi.dpd_create_group(gbox, cfg.rc, cfg.a, cfg.gamma, cfg.kT, cfg.power, cfg.dt, cfg.seed, grid)
    try:
        for c in ctxs:
            capi.dpd_set_species(c, A3, G3)
            capi.dpd_set_particles_typed(c, pos, vel, ids, sp, 0)
        capi.dpd_group_step(ctxs, 0)  # prime
        p = oracle.DPDParams(box=gbox, rc=cfg.rc, a=cfg.a, gamma=cfg.gamma, kT=cfg.kT, power=cfg.power,
                             dt=cfg.dt, seed=cfg.seed, amat=A3, gmat=G3)
        eps = boundary_eps(gbox)
        for s in range(0, 21, 5):
            if s:
                capi.dpd_group_step(ctxs, 5)
            X, U, F, I, S = [], [], [], [], []
            for c in ctxs:
                x, u, f, i = capi.dpd_get_state(c)
                spec, sids = capi.dpd_get_species_ex(c)
                assert np.array_equal(sids, i)
                X.append(x); U.append(u); F.append(f); I.append(i); S.append(spec)
            X, U, F, I, S = map(np.concatenate, (X, U, F, I, S))
            assert np.array_equal(np.sort(I), np.arange(n))
            x_id, u_id, F_id, s_id = by_id(I, X, U, F, S)
            assert np.array_equal(s_id, sp)
            p.species = sp
            F_ref, allow, _ = oracle.forces(p, x_id, u_id, s, eps=eps)
            check_forces(F_id, F_ref, allow)
    finally:
        for c in ctxs:
            capi.dpd_destroy(c)


def test_mixed_viscosity_temperature():
    """Fluctuation-dissipation holds per pair (sigma_ij^2 = 2 gamma_ij kT): a 50/50
    mixture with gamma 4.5 / 45 and cross 20 equilibrates at T = kT within 1 %."""
    from paper_1911_04712_b200 import capi
    cfg = workloads.with_box(workloads.CONFIGS["parity"], (16.0, 16.0, 16.0))  # rho = 3, dt = 0.01
    pos, vel = workloads.make_config(cfg)
    sp = _species(len(pos), seed=1, ns=2)
    A = np.full((2, 2), 25.0)
    G = np.array([[4.5, 20.0], [20.0, 45.0]])
    d = capi.DPD(cfg.box, cfg.rc, cfg.a, cfg.gamma, cfg.kT, cfg.power, cfg.dt, cfg.seed)
    d.set_species(A, G)
    d.set_particles_typed(pos, vel, None, sp, 0)
    d.step(300)
    Ts = []
    for _ in range(60):
        d.step(10)
        _, v = d.get_particles()
        Ts.append(oracle.temperature(v))
    T = float(np.mean(Ts))
    assert abs(T - cfg.kT) < 0.01 * cfg.kT, T


def test_species_errors():
    from paper_1911_04712_b200 import capi
    cfg = workloads.CONFIGS["parity"]
    pos, vel = workloads.make_config(cfg)
    d = capi.DPD(cfg.box, cfg.rc, cfg.a, cfg.gamma, cfg.kT, cfg.power, cfg.dt, cfg.seed)
    with pytest.raises(capi.DPDError) as e:
        d.set_species(np.array([[1.0, 2.0], [3.0, 1.0]]), np.ones((2, 2)))
    assert e.value.code == capi.DPD_ERR_CONFIG
    with pytest.raises(capi.DPDError):
        d.set_species(np.ones((5, 5)), np.ones((5, 5)))
    d.set_species(A3, G3)
    bad = _species(len(pos))
    bad[7] = 3
    with pytest.raises(capi.DPDError) as e:
        d.set_particles_typed(pos, vel, None, bad, 0)
    assert e.value.code == capi.DPD_ERR_ARG
    # ids >= 2^30 cannot carry a species through the tiled kernel's staged id word
    big = np.arange(len(pos), dtype=np.int32) + (1 << 30)
    with pytest.raises(capi.DPDError) as e:
        d.set_particles_typed(pos, vel, big, _species(len(pos)), 0)
    assert e.value.code == capi.DPD_ERR_ARG
    d.set_particles_typed(pos, vel, None, _species(len(pos)), 0)
    with pytest.raises(capi.DPDError) as e:
        d.set_species(A3, G3)
    assert e.value.code == capi.DPD_ERR_ARG
    # without a species matrix the full 31-bit id range is legal
    d1 = capi.DPD(cfg.box, cfg.rc, cfg.a, cfg.gamma, cfg.kT, cfg.power, cfg.dt, cfg.seed)
    d1.set_particles_typed(pos, vel, big, None, 0)
    _, _, F, ids = d1.get_state()
    assert np.all(np.isfinite(F)) and ids.min() >= (1 << 30)
