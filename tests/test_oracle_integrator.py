"""Pins for the oracle's Groot-Warren velocity Verlet (reading C-6; PAPER.md P:47, P:248,
P:97-105 eq. 1), the periodic-Poiseuille body force and the thermostat /
equation of state (P:135 fluctuation-dissipation; Groot & Warren 1997 cited at P:90)."""
import numpy as np
import pytest

import oracle
import workloads


def test_force_free_advection():
    # F = 0 -> x += v dt (wrapped), v unchanged
    p = oracle.DPDParams(box=(8.0, 8.0, 8.0), a=0.0, gamma=0.0, kT=0.0, dt=0.01)
    x, v = workloads.make_particles(p.box, 1.0, 1.0, n=64)
    s = oracle.State(p, x, v)
    s.step(10)
    expect = np.mod(x.astype(np.float64) + 10 * 0.01 * v.astype(np.float64), 8.0)
    d = s.x - expect
    d -= 8.0 * np.rint(d / 8.0)
    assert np.abs(d).max() < 1e-12
    np.testing.assert_array_equal(s.v, v.astype(np.float64))
    assert s.s == 10


def test_zero_temperature_fixed_point():
    # zero-temperature, zero-force fluid at rest stays unchanged
    p = oracle.DPDParams(box=(6.0, 6.0, 6.0), a=0.0, gamma=20.0, kT=0.0, dt=0.01)
    x, _ = workloads.make_particles(p.box, 3.0, 0.0)
    v = np.zeros_like(x)
    s = oracle.State(p, x, v)
    s.step(5)
    np.testing.assert_array_equal(s.x, x.astype(np.float64))
    assert np.all(s.v == 0)


def test_ballistic_single_particle_under_body_force():
    # one particle under the constant body force: x = x0 + v0 t + f t^2 / 2 exactly
    f = 0.05
    p = oracle.DPDParams(box=(16.0, 16.0, 64.0), a=25.0, gamma=4.5, kT=1.0, dt=0.01, body_f=f)
    x0 = np.array([[12.0, 3.0, 20.0]])  # r_x > L/2 -> +f z-hat
    v0 = np.array([[0.0, 0.5, -1.0]])
    s = oracle.State(p, x0, v0)
    s.step(100)
    t = 100 * 0.01
    assert s.v[0, 2] == pytest.approx(-1.0 + f * t, abs=1e-12)
    assert s.x[0, 2] == pytest.approx(20.0 - 1.0 * t + 0.5 * f * t * t, abs=1e-12)
    assert s.x[0, 1] == pytest.approx(3.0 + 0.5 * t, abs=1e-12)


def test_poiseuille_forcing_sign():
    # S:483 [P:366-369]: r_x = L/4 -> -f z-hat; r_x = 3L/4 -> +f z-hat
    f = 0.1
    p = oracle.DPDParams(box=(8.0, 8.0, 8.0), a=0.0, gamma=0.0, kT=0.0, dt=0.01, body_f=f)
    x = np.array([[2.0, 1.0, 1.0], [6.0, 5.0, 5.0], [4.0, 3.0, 7.0]])  # L/4, 3L/4, exactly L/2
    s = oracle.State(p, x, np.zeros_like(x))
    s.step(1)
    np.testing.assert_allclose(s.v[:, 2], [-f * 0.01, f * 0.01, -f * 0.01], atol=1e-15)


def test_momentum_conserved_over_steps():
    # closed periodic system without forcing conserves total momentum
    p = oracle.DPDParams(box=(8.0, 8.0, 8.0), a=25.0, gamma=45.0, kT=1.0, power=0.5, dt=0.01)
    x, v = workloads.make_particles(p.box, 3.0, 1.0)
    s = oracle.State(p, x, v)
    P0 = s.v.sum(axis=0)
    pav = np.abs(s.v).sum(axis=1).mean()
    s.step(200)
    assert np.abs(s.v.sum(axis=0) - P0).max() <= 1e-8 * x.shape[0] * pav


def _equilibrium(p, rho, warm, nsteps, every=5):
    x, v = workloads.make_particles(p.box, rho, p.kT)
    s = oracle.State(p, x, v)
    s.step(warm)
    T, Th, W = [], [], []
    for _ in range(nsteps // every):
        s.step(every)
        T.append(oracle.temperature(s.v))
        Th.append(oracle.temperature(s.u))
        W.append(oracle.virial(p, s.x))
    V = p.box[0] * p.box[1] * p.box[2]
    T, Th, W = map(np.asarray, (T, Th, W))
    return T.mean(), Th.mean(), rho * T.mean() + W.mean() / (3 * V)


@pytest.mark.slow
def test_temperature_and_groot_warren_eos_rho8():
    # Fluctuation-dissipation: <T> = kT within 1% (north_star), full-step v (C-14).
    # Groot-Warren EOS p = rho kT + 0.101 a rho^2 at rho = 8 within 2% (C-15).
    # Table-2 parameters: a=50, gamma=20, kT=1, dt=0.002; k=0.5.
    p = oracle.DPDParams(box=(6.0, 6.0, 6.0), a=50.0, gamma=20.0, kT=1.0, power=0.5, dt=0.002, seed=42)
    T, Th, pr = _equilibrium(p, 8.0, 200, 1000)
    assert abs(T - 1.0) < 0.01, T
    gw = 8.0 * 1.0 + 0.101 * 50.0 * 64.0
    assert abs(pr - gw) / gw < 0.02, (pr, gw)


@pytest.mark.slow
def test_temperature_config1_full_vs_half_step():
    # Config-1 (a=25, gamma=45, dt=0.01): full-step velocities give T ~ kT (1.007, SURVEY
    # Exp-A) while the half-step velocities read ~26% hot -- the reason for reading C-6.
    p = oracle.DPDParams(box=(8.0, 8.0, 8.0), a=25.0, gamma=45.0, kT=1.0, power=0.5, dt=0.01, seed=42)
    T, Th, _ = _equilibrium(p, 3.0, 200, 1000)
    assert abs(T - 1.0) < 0.02, T
    assert Th > 1.15, Th
