"""Pins for the oracle's pair force (eqs. 2-5; readings C-3..C-5, C-11)."""
import math

import numpy as np
import pytest

import oracle
from conftest import read_golden


def P(**kw):
    base = dict(box=(8.0, 8.0, 8.0), rc=1.0, a=0.0, gamma=0.0, kT=0.0, power=1.0, dt=0.01, seed=42)
    base.update(kw)
    return oracle.DPDParams(**base)


def test_conservative_hand_example():
    # S:194 [PAPER eq. 3]: r=0.5, r_c=1, a=10, gamma=0, stationary -> |F|=5.0, repulsive along e_ij
    p = P(a=10.0)
    f, hit, _ = oracle.pair_force(p, [0.5, 0.0, 0.0], [0, 0, 0], 0, 1, 0)
    assert hit
    np.testing.assert_allclose(f, [5.0, 0.0, 0.0], rtol=0, atol=1e-14)
    # direction follows e_ij = r_ij / r for an arbitrary orientation
    d = np.array([0.3, -0.2, 0.1])
    f, hit, _ = oracle.pair_force(p, d, [0, 0, 0], 0, 1, 0)
    r = np.linalg.norm(d)
    np.testing.assert_allclose(f, 10.0 * (1 - r) * d / r, rtol=1e-14)


def test_dissipative_hand_example():
    # r=0.5, k=1, a=0, gamma=4, relative velocity 2 e_ij, xi=0 (kT=0) -> F^D = -2.0 e_ij
    p = P(gamma=4.0, power=1.0, kT=0.0)
    e = np.array([0.0, 0.6, 0.8])
    f, hit, _ = oracle.pair_force(p, 0.5 * e, 2.0 * e, 0, 1, 0)
    assert hit
    np.testing.assert_allclose(f, -2.0 * e, atol=1e-14)
    # approaching particles (v_ij . e < 0) are pushed apart: damping of the relative motion
    f, _, _ = oracle.pair_force(p, 0.5 * e, -2.0 * e, 0, 1, 0)
    np.testing.assert_allclose(f, 2.0 * e, atol=1e-14)
    # w_D = w_R^2 = w^{2k}: at k=0.5 the dissipative weight is w (not w^2)
    p = P(gamma=4.0, power=0.5)
    f, _, _ = oracle.pair_force(p, 0.5 * e, 2.0 * e, 0, 1, 0)
    np.testing.assert_allclose(f, -4.0 * 0.5 * 2.0 * e, atol=1e-14)


def test_cutoff_and_degenerate():
    p = P(a=25.0, gamma=45.0, kT=1.0, power=0.5)
    # r >= r_c -> zero force regardless of other params, strict cutoff (C-11)
    for r in [1.0, 1.0000001, 1.5]:
        f, hit, _ = oracle.pair_force(p, [r, 0, 0], [3, 1, 2], 0, 1, 0)
        assert not hit and np.all(f == 0)
    # r = 0 -> zero force
    f, hit, _ = oracle.pair_force(p, [0, 0, 0], [1, 0, 0], 0, 1, 0)
    assert not hit and np.all(f == 0)
    f, hit, _ = oracle.pair_force(p, [0.9999999, 0, 0], [0, 0, 0], 0, 1, 0)
    assert hit


def test_random_term_scaling_fdt():
    # F^R = sigma xi w_R e / sqrt(dt), sigma = sqrt(2 gamma kT) (C-3)
    # isolate F^R: a = 0, v_ij = 0; quadrupling kT doubles F^R; quartering dt doubles F^R
    e = np.array([1.0, 0.0, 0.0])
    base, _, xi = oracle.pair_force(P(gamma=3.0, kT=1.0, power=0.5), 0.36 * e, [0, 0, 0], 4, 9, 2)
    f_kT, _, _ = oracle.pair_force(P(gamma=3.0, kT=4.0, power=0.5), 0.36 * e, [0, 0, 0], 4, 9, 2)
    f_dt, _, _ = oracle.pair_force(P(gamma=3.0, kT=1.0, power=0.5, dt=0.0025), 0.36 * e, [0, 0, 0], 4, 9, 2)
    np.testing.assert_allclose(f_kT, 2 * base, rtol=1e-14)
    np.testing.assert_allclose(f_dt, 2 * base, rtol=1e-14)
    # magnitude: sqrt(2*3*1) * xi * (1-0.36)^0.5 / sqrt(0.01)
    assert base[0] == pytest.approx(math.sqrt(6.0) * xi * 0.8 / 0.1, rel=1e-14)


@pytest.mark.parametrize("row", read_golden("pair_worked_values.txt"))
def test_worked_values(row):
    idi, idj, step = int(row[0]), int(row[1]), int(row[2])
    w0, w1 = int(row[3], 16), int(row[4], 16)
    xi_ref, fx_ref = float(row[5]), float(row[6])
    # words from the KAT-pinned generator with the C-7 layout (step key pinned in
    # test_oracle_rng.py: fmix32 bijection, injective over 2^24 steps)
    ks = oracle.step_key(42, step)
    w = oracle.philox2x32_10([min(idi, idj), max(idi, idj)], ks)
    assert (int(w[0]), int(w[1])) == (w0, w1)
    assert oracle.pair_words(42, step, idi, idj) == (w0, w1)
    # Box-Muller closed form evaluated independently in Python
    u1, u2 = (w0 + 1) / 2**32, w1 / 2**32
    xi_py = math.sqrt(-2 * math.log(u1)) * math.cos(2 * math.pi * u2)
    assert xi_py == pytest.approx(xi_ref, abs=5e-9)
    assert oracle.xi(w0, w1) == pytest.approx(xi_ref, abs=5e-9)
    # eq. 3-5 for the hand configuration (r=0.5, e=(-1,0,0), at rest): F_x = -(a w + sigma w^k xi / sqrt(dt))
    fx_py = -(25.0 * 0.5 + math.sqrt(2 * 45.0 * 1.0) * math.sqrt(0.5) * xi_py / math.sqrt(0.01))
    assert fx_py == pytest.approx(fx_ref, abs=5e-7)
    p = P(a=25.0, gamma=45.0, kT=1.0, power=0.5, dt=0.01)
    d = oracle.min_image(p, [1.0, 1.0, 1.0], [1.5, 1.0, 1.0])
    f, hit, _ = oracle.pair_force(p, d, [0, 0, 0], idi, idj, step)
    assert hit
    assert f[0] == pytest.approx(fx_ref, abs=5e-8)
    assert f[1] == 0 and f[2] == 0


def test_swap_gives_exact_negation_and_central():
    # Newton's third law: swapping (i, j) negates the force exactly
    p = P(a=25.0, gamma=45.0, kT=1.0, power=0.5, dt=0.01)
    rng = np.random.default_rng(5)
    for _ in range(200):
        xi_, xj_ = rng.random(3) * 8, rng.random(3) * 8
        xj_ = xi_ + rng.normal(size=3) * 0.4
        vi, vj = rng.normal(size=3), rng.normal(size=3)
        ii, jj = rng.integers(0, 10**6, 2)
        d = oracle.min_image(p, xi_, xj_)
        d2 = oracle.min_image(p, xj_, xi_)
        assert np.all(d2 == -d)
        f, hit, _ = oracle.pair_force(p, d, vi - vj, ii, jj, 11)
        g, hit2, _ = oracle.pair_force(p, d2, vj - vi, jj, ii, 11)
        assert hit == hit2
        assert np.all(f == -g)
        # central: f parallel to d
        assert np.linalg.norm(np.cross(f, d)) <= 1e-12 * (np.linalg.norm(f) * np.linalg.norm(d) + 1e-300)


def test_minimum_image_across_boundary():
    p = P()
    d = oracle.min_image(p, [0.1, 7.9, 4.0], [7.9, 0.1, 4.0])
    np.testing.assert_allclose(d, [0.2, -0.2, 0.0], atol=1e-12)
