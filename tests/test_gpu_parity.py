"""CUDA path (through the C-ABI) against the oracle: parity gate of DESIGN.md §7.

Bars (north_star):
  * cell indices, per-cell counts, starts and RNG words: bit-exact
  * per-step forces: |F_gpu - F_oracle|_inf <= 1e-4 max|F| + boundary allowance (C-12)
  * per-step protocol: the oracle is fed the GPU state of each step (C-13)
"""
import numpy as np
import pytest

import oracle
import workloads

pytestmark = pytest.mark.gpu

FORCE_TOL = 1e-4


KERNELS = [0, 1]  # 0: tiled (production), 1: reference thread-per-particle (cross-check)


def _ctx(cfg, seed=None, kernel=0):
    from paper_1911_04712_b200 import capi
    d = capi.DPD(cfg.box, cfg.rc, cfg.a, cfg.gamma, cfg.kT, cfg.power, cfg.dt, cfg.seed if seed is None else seed)
    d.set_option("force_kernel", kernel)
    return d


def _params(cfg):
    return oracle.DPDParams(box=cfg.box, rc=cfg.rc, a=cfg.a, gamma=cfg.gamma, kT=cfg.kT, power=cfg.power,
                            dt=cfg.dt, seed=cfg.seed, body_f=cfg.body_f)


def boundary_eps(box):
    # fp32 positions near L carry an absolute error of ~ulp(L); widen the C-12 window to it
    # (used where the GPU works in shifted local frames: the decomposed group tests)
    return max(1e-5, 16 * float(np.spacing(np.float32(max(box)))))


def windows(box, rc=1.0):
    """Per-pair C-12 windows (eps, eps_image): a pair inside the box differs from the fp64
    definition only by the fp32 rounding of r^2 (a few ulp of r_c); a pair across a
    periodic edge also carries the rounding of the shifted image x_j +- L (<= ulp(L) / 2
    per coordinate, sqrt(3)/2 ulp(L) in r)."""
    eps = 4.0 * float(np.spacing(np.float32(rc)))
    return eps, max(eps, 2.0 * float(np.spacing(np.float32(max(box)))))


def window_kw(box, rc=1.0):
    eps, eps_img = windows(box, rc)
    return {"eps": eps, "eps_image": eps_img}


def face_sample(pos, box, n_random, n_face, seed):
    """Particle indices: n_random uniform ones plus n_face within r_c of each of the six
    periodic faces (the pairs that cross a periodic edge)."""
    rng = np.random.default_rng(seed)
    n = pos.shape[0]
    sel = [rng.choice(n, n_random, replace=False)]
    for d in range(3):
        for near in (pos[:, d] < 1.0, pos[:, d] >= box[d] - 1.0):
            idx = np.flatnonzero(near)
            sel.append(rng.choice(idx, min(n_face, idx.size), replace=False))
    return np.unique(np.concatenate(sel))


def by_id(ids, *arrays):
    order = np.argsort(ids)
    return [a[order] for a in arrays]


def check_forces(F_gpu, F_ref, allow, tol=FORCE_TOL):
    scale = np.abs(F_ref).max()
    err = np.abs(F_gpu.astype(np.float64) - F_ref).max(axis=1)
    bad = err > tol * scale + allow
    assert not bad.any(), (f"{bad.sum()} particles off; worst {err.max():.3e} vs tol {tol * scale:.3e}; "
                           f"max allow {allow.max():.3e}")
    return err.max() / scale


def test_device_philox_known_answers():
    from paper_1911_04712_b200 import capi
    from conftest import read_golden
    rows = [[int(t, 16) for t in r] for r in read_golden("philox2x32_10_kat.txt")]
    ctr = np.array([r[0:2] for r in rows], np.uint32)
    key = np.array([r[2] for r in rows], np.uint32)
    out = capi.dpd_debug_philox(ctr, key)
    assert np.array_equal(out, np.array([r[3:5] for r in rows], np.uint32))


def test_device_pair_words_and_xi_match_oracle():
    from paper_1911_04712_b200 import capi
    rng = np.random.default_rng(11)
    n = 200000
    q = np.zeros((n, 4), np.uint32)
    q[:, 0] = rng.integers(0, 2**31, n)
    q[:, 1] = rng.integers(0, 2**31, n)
    steps = rng.integers(0, 2**40, n)
    q[:, 2] = steps & 0xFFFFFFFF
    q[:, 3] = steps >> 32
    words, xi = capi.dpd_debug_pair_words(q, 42)
    for k in range(0, n, 1999):
        assert oracle.pair_words(42, int(steps[k]), int(q[k, 0]), int(q[k, 1])) == (int(words[k, 0]), int(words[k, 1]))
    xi_ref = np.array([oracle.xi(int(a), int(b)) for a, b in words[:20000]])
    err = np.abs(xi[:20000] - xi_ref)
    assert err.max() < 2e-3, err.max()          # worst case: u1 -> 1 where sqrt amplifies log error
    assert np.median(err) < 1e-6


def test_hand_placed_pair_worked_values():
    from conftest import read_golden
    # SURVEY App. B / tests/golden/pair_worked_values.txt through set_particles + get_forces
    cfg = workloads.CONFIGS["parity"]
    d = _ctx(cfg)
    pos = np.array([[1.0, 1.0, 1.0], [1.5, 1.0, 1.0]], np.float32)
    vel = np.zeros_like(pos)
    d.set_particles(pos, vel)
    f = d.get_forces()
    ref = {(int(r[0]), int(r[1]), int(r[2])): float(r[6]) for r in read_golden("pair_worked_values.txt")}
    np.testing.assert_allclose(f[0], [ref[(0, 1, 0)], 0, 0], rtol=0, atol=1e-4 * abs(ref[(0, 1, 0)]))
    np.testing.assert_allclose(f[1], -f[0], rtol=0, atol=0)
    # conservative-only and dissipative-only hand examples
    from paper_1911_04712_b200 import capi
    d2 = capi.DPD((8.0, 8.0, 8.0), 1.0, 10.0, 0.0, 0.0, 1.0, 0.01, 42)
    d2.set_particles(np.array([[2.0, 2.0, 2.0], [2.5, 2.0, 2.0]], np.float32), np.zeros((2, 3), np.float32))
    np.testing.assert_allclose(d2.get_forces()[0], [-5.0, 0, 0], atol=1e-5)
    d3 = capi.DPD((8.0, 8.0, 8.0), 1.0, 0.0, 4.0, 0.0, 1.0, 0.01, 42)
    d3.set_particles(np.array([[2.0, 2.0, 2.0], [2.5, 2.0, 2.0]], np.float32),
                     np.array([[-1.0, 0, 0], [1.0, 0, 0]], np.float32))
    np.testing.assert_allclose(d3.get_forces()[0], [2.0, 0, 0], atol=1e-5)


def test_periodic_boundary_pair_and_degenerates():
    cfg = workloads.CONFIGS["parity"]
    p = _params(cfg)
    d = _ctx(cfg)
    # two particles straddling the periodic boundary in x and z
    pos = np.array([[0.1, 4.0, 7.95], [7.9, 4.1, 0.05]], np.float32)
    vel = np.array([[0.3, 0.0, 0.1], [-0.2, 0.1, 0.0]], np.float32)
    d.set_particles(pos, vel)
    F_ref, _, npairs = oracle.forces(p, pos, vel, 0)
    assert npairs == 1
    check_forces(d.get_forces(), F_ref, np.zeros(2))
    # single particle: zero force; N = 0 legal
    d.set_particles(np.array([[1.0, 2.0, 3.0]], np.float32), np.zeros((1, 3), np.float32))
    assert np.all(d.get_forces() == 0)
    d.step(3)
    d.set_particles(np.zeros((0, 3), np.float32), np.zeros((0, 3), np.float32))
    d.step(2)
    assert d.get_count() == 0 and d.get_step() == 2
    # positions outside [0, L) are wrapped (C-10)
    d.set_particles(np.array([[-0.5, 8.0, 17.25]], np.float32), np.zeros((1, 3), np.float32))
    x, _ = d.get_particles()
    np.testing.assert_allclose(x[0], [7.5, 0.0, 1.25], atol=1e-6)


def test_errors_are_reported():
    from paper_1911_04712_b200 import capi
    with pytest.raises(capi.DPDError):
        capi.DPD((2.0, 8.0, 8.0))  # box < 3 rc
    with pytest.raises(capi.DPDError):
        capi.DPD((8.0, 8.0, 8.0), power=1.5)
    d = capi.DPD((8.0, 8.0, 8.0))
    pos = np.array([[1.0, np.nan, 1.0]], np.float32)
    with pytest.raises(capi.DPDError) as e:
        d.set_particles(pos, np.zeros((1, 3), np.float32))
    assert e.value.code == capi.DPD_ERR_NUMERIC


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("body_f", [0.0, 2.0])
def test_per_step_parity_config1(kernel, body_f):
    """100 steps of config 1 (C-13): each step, the oracle is fed the GPU state.  Forces,
    cells, pair words, and the integrator against oracle.kick_drift (C-6), with and
    without the periodic-Poiseuille body force."""
    cfg = workloads.CONFIGS["parity"]
    p = _params(cfg)
    p.body_f = body_f
    eps, eps_img = windows(cfg.box)
    pos0, vel0 = workloads.make_config(cfg)
    d = _ctx(cfg, kernel=kernel)
    if body_f:
        d.set_body_force(body_f)
    d.set_particles(pos0, vel0)
    n = pos0.shape[0]
    box = np.array(cfg.box)
    prev = None
    worst = 0.0
    kick = 0.5 * cfg.dt
    for s in range(cfg.steps + 1):
        pos, u, F, ids = d.get_state()
        assert d.get_step() == s
        assert np.array_equal(np.sort(ids), np.arange(n))
        x_id, u_id, F_id = by_id(ids, pos, u, F)
        # cells / counts / starts: bit-exact against the fp32 definition (C-8)
        cell, count, start = d.debug_cells()
        ocell, ocount, ostart = oracle.cells(p, x_id)
        assert np.array_equal(count, ocount) and np.array_equal(start, ostart)
        assert np.array_equal(cell, ocell)
        # storage order is cell-sorted: cells of consecutive slots are non-decreasing
        assert np.all(np.diff(ocell[ids]) >= 0)
        # forces F_s = F(x_s, u_s, s), per-pair boundary windows (C-12)
        F_ref, allow, _ = oracle.forces(p, x_id, u_id, s, eps=eps, eps_image=eps_img)
        worst = max(worst, check_forces(F_id, F_ref, allow))
        # integrator: the oracle's kick-drift of the previous GPU state (kick dt/2 after set,
        # dt after: the fused second + first half kicks, C-6)
        if prev is not None:
            px, pu, pF, pk = prev
            x_pred, u_pred, _ = oracle.kick_drift(p, px, pu, pF, pk)
            dx = x_id - x_pred
            dx -= box * np.rint(dx / box)
            assert np.abs(dx).max() < 2e-6
            assert np.abs(u_id - u_pred).max() < 1e-5 * (1 + np.abs(u_pred).max())
        # pair set and RNG words, every 20 steps (T3)
        if s % 20 == 0:
            quad = d.debug_pairs()
            oq, oflag = oracle.pairs(p, x_id, s, eps=eps, eps_image=eps_img)
            gset = {tuple(r) for r in quad.tolist()}
            core = {tuple(r) for r, f in zip(oq.tolist(), oflag) if (f & 1) and not (f & 2)}
            boundary = {tuple(r) for r, f in zip(oq.tolist(), oflag) if f & 2}
            assert len(gset) == len(quad)  # no pair visited twice
            assert core <= gset
            assert gset - core <= boundary
        prev = (x_id, u_id, F_id, kick)
        kick = cfg.dt
        if s < cfg.steps:
            d.step(1)
    print(f"worst relative force error {worst:.2e}")


@pytest.mark.parametrize("body_f", [0.0, 2.0])
def test_full_step_velocity_matches_oracle(body_f):
    """Row a6: dpd_get_particles returns the full-step velocity v = u + dt/2 (F + f_body)
    (C-6).  From one initial state, one and three GPU steps against oracle.State's
    GW-VV steps, element by element (fp32 vs fp64; a few steps are far from chaotic
    divergence, C-13)."""
    cfg = workloads.CONFIGS["parity"]
    p = _params(cfg)
    p.body_f = body_f
    eps, eps_img = windows(cfg.box)
    pos0, vel0 = workloads.make_config(cfg)
    box = np.array(cfg.box)
    for k in (1, 3):
        d = _ctx(cfg)
        if body_f:
            d.set_body_force(body_f)
        d.set_particles(pos0, vel0)
        d.step(k)
        x, v = d.get_particles()
        st = oracle.State(p, pos0, vel0).step(k)
        dx = x - st.x
        dx -= box * np.rint(dx / box)
        assert np.abs(dx).max() < 1e-5 * k
        _, allow, _ = oracle.forces(p, st.x, st.u, k, eps=eps, eps_image=eps_img)
        tol = cfg.dt * k * (FORCE_TOL * np.abs(st.F).max() + allow[:, None]) + 1e-5 * (1 + np.abs(st.v))
        err = np.abs(v.astype(np.float64) - st.v)
        assert np.all(err <= tol), (k, err.max(), tol.min())
        # and the velocity really is the full-step one: the half-step u differs by dt/2 F
        assert np.abs(st.v - st.u).max() > 10 * tol.max()


def test_edge_pairs_coincident_cutoff_and_range():
    """Degenerate pairs of the method (P:121-122 strict cutoff, S:191-192 r = 0): coincident
    particles exert no force; a pair at exactly r = r_c does not interact; a pair whose force
    leaves the fixed-point range reports DPD_ERR_NUMERIC instead of a wrong sum."""
    from paper_1911_04712_b200 import capi
    cfg = workloads.CONFIGS["parity"]
    p = _params(cfg)
    d = _ctx(cfg)
    v = np.array([[0.3, -0.2, 0.1], [-0.1, 0.4, 0.0], [0.2, 0.1, -0.3]], np.float32)
    # r = 0: particles 0 and 1 coincide; particle 2 at r = 0.5 from both
    x = np.array([[2.0, 3.0, 4.0], [2.0, 3.0, 4.0], [2.5, 3.0, 4.0]], np.float32)
    d.set_particles(x, v)
    F = d.get_forces()
    F_ref, _, npairs = oracle.forces(p, x, v, 0)
    assert npairs == 2 and np.all(np.isfinite(F))
    check_forces(F, F_ref, np.zeros(3))
    # r = r_c exactly (1.0 in fp32 and fp64): no pair, zero force; and across the periodic x edge
    for x in (np.array([[2.0, 3.0, 4.0], [3.0, 3.0, 4.0]], np.float32),
              np.array([[0.5, 3.0, 4.0], [7.5, 3.0, 4.0]], np.float32)):
        d.set_particles(x, v[:2])
        assert np.all(d.get_forces() == 0.0)
        assert d.debug_pairs().shape[0] == 0
    # just inside r_c interacts
    d.set_particles(np.array([[2.0, 3.0, 4.0], [2.9999, 3.0, 4.0]], np.float32), v[:2])
    assert np.abs(d.get_forces()).max() > 0
    # fixed-point range: a relative speed of 1e4 at r = 0.5 gives |F^D| ~ 1e5, far beyond the
    # scale's bound (a + 6.7 sigma / sqrt(dt) + 20 gamma): reported, never silently wrapped
    fast = np.array([[2.0, 3.0, 4.0], [2.5, 3.0, 4.0]], np.float32)
    with pytest.raises(capi.DPDError) as e:
        d.set_particles(fast, np.array([[1e4, 0, 0], [-1e4, 0, 0]], np.float32))
    assert e.value.code == capi.DPD_ERR_NUMERIC
    # the context stays usable after the error
    d.set_particles(fast, v[:2])
    assert np.all(np.isfinite(d.get_forces()))


@pytest.mark.parametrize("kernel", KERNELS)
def test_dense_cluster_overflow_fallback(kernel):
    """A dense blob (rho ~ 60 locally) overflows the tiled kernel's shared-memory tiles; the
    global-memory fallback must give the same forces (and the reference kernel too)."""
    cfg = workloads.CONFIGS["parity"]
    p = _params(cfg)
    rng = np.random.default_rng(4)
    blob = (rng.random((1500, 3)) * 3.0 + 2.0).astype(np.float32)   # 3^3 volume: rho ~ 56
    fluid = (rng.random((600, 3)) * 8.0).astype(np.float32)
    pos = np.concatenate([blob, fluid])
    vel = rng.normal(size=pos.shape).astype(np.float32)
    d = _ctx(cfg, kernel=kernel)
    d.set_particles(pos, vel)
    F_ref, allow, _ = oracle.forces(p, pos, vel, 0, **window_kw(cfg.box))
    check_forces(d.get_forces(), F_ref, allow)


def test_crowded_cell_full_list_path():
    """One cell holding 40 particles inside a tile that still fits shared memory: the first
    particles of that cell find more partners than a list holds (FT_LCAP), so the tiled
    kernel evaluates the rest in place (stat "full_list_particles"); forces must still be
    the oracle's."""
    from paper_1911_04712_b200 import capi
    cfg = workloads.CONFIGS["parity"]
    p = _params(cfg)
    rng = np.random.default_rng(11)
    crowd = (rng.random((40, 3)) * 0.9 + np.array([3.05, 4.05, 2.05])).astype(np.float32)
    fluid = (rng.random((1500, 3)) * 8.0).astype(np.float32)
    pos = np.concatenate([crowd, fluid])
    vel = rng.normal(size=pos.shape).astype(np.float32)
    d = _ctx(cfg, kernel=0)
    d.set_particles(pos, vel)
    assert capi.dpd_get_stat(d.ctx, "full_list_particles") > 0
    assert capi.dpd_get_stat(d.ctx, "fallback_tiles") == 0
    F_ref, allow, _ = oracle.forces(p, pos, vel, 0, **window_kw(cfg.box))
    check_forces(d.get_forces(), F_ref, allow)


def test_momentum_and_force_sum():
    cfg = workloads.CONFIGS["parity"]
    pos0, vel0 = workloads.make_config(cfg)
    d = _ctx(cfg)
    d.set_particles(pos0, vel0)
    f = d.get_forces().astype(np.float64)
    assert np.abs(f.sum(0)).max() < 1e-5 * np.abs(f).sum()
    _, v0 = d.get_particles()
    P0 = v0.astype(np.float64).sum(0)
    d.step(200)
    _, v = d.get_particles()
    drift = np.abs(v.astype(np.float64).sum(0) - P0).max()
    assert drift < 1e-3 * np.abs(v).sum(1).mean() * np.sqrt(len(v)), drift


def test_temperature_rho8():
    # T = kT within 1% (north_star) from full-step velocities (C-14), 16^3 rho=8
    cfg = workloads.with_box(workloads.CONFIGS["eq64"], (16.0, 16.0, 16.0))
    pos0, vel0 = workloads.make_config(cfg)
    d = _ctx(cfg)
    d.set_particles(pos0, vel0)
    d.step(200)
    Ts = []
    for _ in range(100):
        d.step(10)
        _, v = d.get_particles()
        Ts.append(oracle.temperature(v))
    T = float(np.mean(Ts))
    assert abs(T - cfg.kT) < 0.01 * cfg.kT, T


def test_temperature_config2_full_size_1000_steps():
    """North star: ensemble temperature within 1 % of kT over 1000 steps, at BASELINE config 2
    itself (64^3, rho = 8, 2.1 M particles, Table-2 parameters), full-step velocities (C-14)."""
    cfg = workloads.CONFIGS["eq64"]
    pos0, vel0 = workloads.make_config(cfg)
    d = _ctx(cfg)
    d.set_particles(pos0, vel0)
    d.step(200)
    Ts = []
    for _ in range(50):
        d.step(20)
        _, v = d.get_particles()
        Ts.append(oracle.temperature(v))
    T = float(np.mean(Ts))
    assert abs(T - cfg.kT) < 0.01 * cfg.kT, T


@pytest.mark.parametrize("a", [50.0, 10.0])
def test_groot_warren_pressure_rho8(a):
    """Structure of the GPU-sampled ensemble: p = rho T + W / (3V) with the conservative virial
    W = sum a w(r) r evaluated by the oracle on the GPU's configurations (C-2 item 6) against
    the Groot-Warren EOS p = rho kT + 0.101 a rho^2 within 2 % at rho = 8 (C-15; survey
    measurement +0.5 % / -0.6 % for a = 50 / 10).  8^3 box (4096 particles), Table-2 gamma and
    dt, k = 1/2."""
    cfg = workloads.with_box(workloads.CONFIGS["eq64"], (8.0, 8.0, 8.0))
    d_ = cfg.as_dict()
    d_["a"] = a
    cfg = workloads.Config(**d_)
    p = _params(cfg)
    pos0, vel0 = workloads.make_config(cfg)
    d = _ctx(cfg)
    d.set_particles(pos0, vel0)
    d.step(1000)
    T, W = [], []
    for _ in range(60):
        d.step(20)
        x, v = d.get_particles()
        T.append(oracle.temperature(v))
        W.append(oracle.virial(p, x))
    V = float(np.prod(cfg.box))
    pr = cfg.rho * np.mean(T) + np.mean(W) / (3.0 * V)
    gw = cfg.rho * cfg.kT + 0.101 * a * cfg.rho ** 2
    assert abs(np.mean(T) - cfg.kT) < 0.015 * cfg.kT, np.mean(T)
    assert abs(pr - gw) / gw < 0.02, (pr, gw)


def test_resume_reproduces_rng_words():
    # checkpoint/resume (C-20): set_particles_ex(ids, step0) continues the same RNG stream
    from paper_1911_04712_b200 import capi
    cfg = workloads.CONFIGS["parity"]
    pos0, vel0 = workloads.make_config(cfg)
    d = _ctx(cfg)
    d.set_particles(pos0, vel0)
    d.step(7)
    pos, u, F, ids = d.get_state()
    d2 = _ctx(cfg)
    capi.dpd_set_particles_ex(d2.ctx, pos, u, ids, step0=7)
    F2 = d2.get_forces()
    x_id, F_id = by_id(ids, pos, F)
    np.testing.assert_allclose(F2, F_id, rtol=0, atol=2e-4 * np.abs(F_id).max())


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("name", ["eq64"])
def test_full_size_sampled_parity(name, kernel):
    """BASELINE config at full size, same launch configuration as bench.py: sampled
    particles against the oracle's all-j sums, plus size-independent properties."""
    cfg = workloads.CONFIGS[name]
    p = _params(cfg)
    eps, eps_img = windows(cfg.box)
    pos0, vel0 = workloads.make_config(cfg)
    d = _ctx(cfg, kernel=kernel)
    d.set_particles(pos0, vel0)
    d.step(5)
    pos, u, F, ids = d.get_state()
    n = pos.shape[0]
    assert np.array_equal(np.sort(ids), np.arange(n))
    # >= 4096 particles: 2048 uniform + 384 within r_c of each periodic face
    sel = face_sample(pos, cfg.box, 2048, 384, seed=0)
    assert sel.size >= 4096
    F_ref, allow = oracle.forces_subset(p, pos, u, d.get_step(), sel, ids=ids.astype(np.uint32), eps=eps,
                                        eps_image=eps_img)
    scale = np.abs(F).max()
    err = np.abs(F[sel].astype(np.float64) - F_ref).max(axis=1)
    assert np.all(err <= FORCE_TOL * scale + allow), (err.max(), scale)
    # cell counts bit-exact at full size
    cell, count, start = d.debug_cells()
    _, ocount, ostart = oracle.cells(p, by_id(ids, pos)[0])
    assert np.array_equal(count, ocount) and np.array_equal(start, ostart)
    assert np.abs(F.astype(np.float64).sum(0)).max() < 1e-5 * np.abs(F).sum()


# Boxes whose cell grids leave ragged tiles in every dimension (the tile is 4 x 4 x 2 home
# cells), non-integer cell edges (h = L / floor(L) > r_c), the 3-cell minimum where
# the stencil wraps onto itself, and strongly anisotropic shapes.
RAGGED_BOXES = [(11.3, 9.7, 7.2), (3.0, 3.0, 3.0), (3.5, 17.0, 5.0), (13.0, 4.0, 9.0), (6.0, 5.0, 3.2)]


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("box", RAGGED_BOXES)
@pytest.mark.parametrize("rho", [3.0, 8.0])
def test_per_step_parity_ragged_boxes(box, rho, kernel):
    """10 steps (C-13 protocol) on ragged / minimal / anisotropic boxes: cells bit-exact,
    forces within the bar, every particle accounted for."""
    cfg = workloads.Config("ragged", box, rho, 25.0, 4.5, 1.0, 0.5, 0.01)
    p = _params(cfg)
    eps, eps_img = windows(cfg.box)
    pos0, vel0 = workloads.make_config(cfg)
    d = _ctx(cfg, kernel=kernel)
    d.set_particles(pos0, vel0)
    n = pos0.shape[0]
    for s in range(11):
        pos, u, F, ids = d.get_state()
        assert np.array_equal(np.sort(ids), np.arange(n))
        x_id, u_id, F_id = by_id(ids, pos, u, F)
        cell, count, start = d.debug_cells()
        ocell, ocount, ostart = oracle.cells(p, x_id)
        assert np.array_equal(count, ocount) and np.array_equal(start, ostart) and np.array_equal(cell, ocell)
        F_ref, allow, _ = oracle.forces(p, x_id, u_id, s, eps=eps, eps_image=eps_img)
        check_forces(F_id, F_ref, allow)
        if s < 10:
            d.step(1)


@pytest.mark.parametrize("name", ["pois96", "weak128", "strong256"])
def test_full_size_sampled_parity_other_configs(name):
    """BASELINE configs 3, 4 and 5 at full size (7.1 M / 16.8 M / 134 M particles, the last
    one whole on one GPU) in bench's launch configuration: sampled all-j sums against the
    oracle, cell counts bit-exact, sum F = 0."""
    cfg = workloads.CONFIGS[name]
    p = _params(cfg)
    eps, eps_img = windows(cfg.box)
    pos0, vel0 = workloads.make_config(cfg)
    d = _ctx(cfg)
    if cfg.body_f:
        d.set_body_force(cfg.body_f)
    d.set_particles(pos0, vel0)
    d.step(3)
    pos, u, F, ids = d.get_state()
    n = pos.shape[0]
    assert n == pos0.shape[0]
    # >= 1024 particles: 512 uniform + 96 within r_c of each periodic face
    sel = face_sample(pos, cfg.box, 512, 96, seed=1)
    assert sel.size >= 1024
    F_ref, allow = oracle.forces_subset(p, pos, u, d.get_step(), sel, ids=ids.astype(np.uint32), eps=eps,
                                        eps_image=eps_img)
    scale = np.abs(F).max()
    err = np.abs(F[sel].astype(np.float64) - F_ref).max(axis=1)
    assert np.all(err <= FORCE_TOL * scale + allow), (err.max(), scale)
    _, count, start = d.debug_cells()
    _, ocount, ostart = oracle.cells(p, by_id(ids, pos)[0])
    assert np.array_equal(count, ocount) and np.array_equal(start, ostart)
    assert np.abs(F.astype(np.float64).sum(0)).max() < 1e-5 * np.abs(F).sum()


# Boxes whose x extent leaves a partial last tile (1-3 home cells wide), so segment ends meet
# row ends at every tile width the staging produces (DESIGN §6 step 3: sentinel gaps).
PAIRSET_BOXES = [(11.3, 9.7, 7.2), (17.0, 13.0, 6.0), (9.0, 6.0, 5.0), (8.0, 8.0, 8.0), (3.5, 17.0, 5.0)]


# (box, r_c, rho): r_c = 1 at rho = 8, and cells wider / narrower than one unit (h = L / floor(L / r_c))
PAIRSET_CASES = [(b, 1.0, 8.0) for b in PAIRSET_BOXES] + [((12.0, 9.1, 8.0), 1.3, 3.0), ((7.9, 6.5, 10.0), 0.8, 8.0),
                                                          ((10.0, 9.0, 8.0), 1.0, 0.7)]
# the last case is sparse (rho = 0.7, ~1.5 partners per particle): most lists are shorter than
# the pair walk's phase A, many are empty, and whole warps have nothing to sweep


@pytest.mark.parametrize("box,rc,rho", PAIRSET_CASES)
def test_tiled_pair_set_equals_reference_kernel(box, rc, rho):
    """The tiled kernel's fused sweep tests whole 4-candidate blocks past segment ends and relies
    on geometry (cells two apart are farther than r_c) and per-row sentinels to reject them.
    The pair set it evaluates must equal the reference thread-per-particle kernel's exactly on
    the same state (no duplicate, none missing), up to pairs inside the fp32 cutoff window,
    over 40 steps; no tile may take the global-memory fallback (the sweep itself is under test)."""
    cfg = workloads.Config("pairset", box, rho, 25.0, 4.5, 1.0, 0.5, 0.005, rc=rc)
    pos0, vel0 = workloads.make_config(cfg)
    d = _ctx(cfg, kernel=0)
    d.set_particles(pos0, vel0)
    L = np.array(cfg.box)
    for s in range(41):
        if s % 10 == 0:
            sets = []
            for kern in (0, 1):
                d.set_option("force_kernel", kern)
                q = d.debug_pairs()
                key = q[:, 0].astype(np.int64) * (1 << 32) + q[:, 1].astype(np.int64)
                assert len(np.unique(key)) == len(key), f"kernel {kern}: duplicate pair at step {s}"
                sets.append(key)
            d.set_option("force_kernel", 0)
            diff = np.setxor1d(sets[0], sets[1])
            if diff.size:
                pos, _, _, ids = d.get_state()
                x = np.empty_like(pos, dtype=np.float64)
                x[ids] = pos
                a, b = diff >> 32, diff & 0xFFFFFFFF
                dr = x[a] - x[b]
                dr -= L * np.round(dr / L)
                r2 = (dr * dr).sum(axis=1)
                assert np.all(np.abs(r2 - cfg.rc ** 2) < 1e-4), \
                    f"step {s}: {diff.size} pairs differ away from the cutoff (r2 = {r2[:5]})"
        if s < 40:
            d.step(1)
    from paper_1911_04712_b200 import capi
    assert capi.dpd_get_stat(d.ctx, "fallback_tiles") == 0


def test_crowded_tiles_second_round_pair_set():
    """rho = 9.2: a 4 x 4 x 2 tile holds ~294 home particles (sd 17), so most tiles have more
    than the 9 x 32 = 288 that one round of warp chunks covers and warp 0 sweeps and walks a
    second chunk; ~10 % of the tiles exceed the staging capacity and take the global-memory
    fallback instead.  The pair set must still equal the reference kernel's (no duplicate,
    none missing) and the forces the oracle's, over 20 steps."""
    from paper_1911_04712_b200 import capi
    cfg = workloads.Config("crowded", (8.0, 8.0, 12.0), 9.2, 25.0, 4.5, 1.0, 0.5, 0.005)
    p = _params(cfg)
    pos0, vel0 = workloads.make_config(cfg)
    d = _ctx(cfg, kernel=0)
    d.set_particles(pos0, vel0)
    L = np.array(cfg.box)
    for s in range(21):
        if s % 10 == 0:
            sets = []
            for kern in (0, 1):
                d.set_option("force_kernel", kern)
                q = d.debug_pairs()
                key = q[:, 0].astype(np.int64) * (1 << 32) + q[:, 1].astype(np.int64)
                assert len(np.unique(key)) == len(key), f"kernel {kern}: duplicate pair at step {s}"
                sets.append(key)
            d.set_option("force_kernel", 0)
            diff = np.setxor1d(sets[0], sets[1])
            if diff.size:
                pos, _, _, ids = d.get_state()
                x = np.empty_like(pos, dtype=np.float64)
                x[ids] = pos
                dr = x[diff >> 32] - x[diff & 0xFFFFFFFF]
                dr -= L * np.round(dr / L)
                assert np.all(np.abs((dr * dr).sum(axis=1) - 1.0) < 1e-4)
            x, u, f, ids = d.get_state()
            x_id, u_id, f_id = by_id(ids, x, u, f)
            F_ref, allow, _ = oracle.forces(p, x_id, u_id, s, **window_kw(cfg.box))
            check_forces(f_id, F_ref, allow)
        if s < 20:
            d.step(1)
    ntiles = 2 * 2 * 6
    fb = capi.dpd_get_stat(d.ctx, "fallback_tiles")
    assert fb < 21 * ntiles // 2, "the tiled path must carry most tiles"


def test_kernel_switch_keeps_force_buffers_consistent():
    """The sort's target force buffer is zeroed a step ahead: by the tiled kernel's first wave,
    or by a memset when the reference kernel computes the step.  Alternating the two kernels
    step by step must keep every step's forces at the oracle's (config 1, C-13 protocol)."""
    cfg = workloads.CONFIGS["parity"]
    p = _params(cfg)
    eps, eps_img = windows(cfg.box)
    pos0, vel0 = workloads.make_config(cfg)
    d = _ctx(cfg, kernel=0)
    d.set_particles(pos0, vel0)
    for s in range(9):
        pos, u, F, ids = d.get_state()
        x_id, u_id, F_id = by_id(ids, pos, u, F)
        F_ref, allow, _ = oracle.forces(p, x_id, u_id, s, eps=eps, eps_image=eps_img)
        check_forces(F_id, F_ref, allow)
        d.set_option("force_kernel", (s + 1) % 2)
        d.step(1)
