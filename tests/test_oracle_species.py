"""Pins of the oracle's species interaction matrix.

P:199-202: fluids on both sides of a membrane share density and conservative potential
but may differ in viscosity; across the membrane fluids interact only conservatively and
fluid-membrane pairs only viscously.  The oracle realises this with per-pair (a, gamma)
from symmetric species matrices and sigma = sqrt(2 gamma kT) per pair.  Pins:
  * an all-equal matrix reproduces the single-species sum exactly (same arithmetic);
  * the hand example of S:194 (|F^C| = a w) with the cross entry, not a diagonal one;
  * zero cross entries decouple the system: F(A u B) = F(A) + F(B) (brute force);
  * conservative-only / viscous-only cross terms against the single-species
    term split (a-only and gamma-only runs);
  * symmetric matrices keep Newton-3: sum F = 0 and F_ij = -F_ji.
"""
import numpy as np
import pytest

import oracle

BOX = (6.0, 6.0, 6.0)


def _system(n=400, seed=3):
    rng = np.random.default_rng(seed)
    x = rng.random((n, 3)) * np.array(BOX)
    v = rng.normal(size=(n, 3))
    sp = rng.integers(0, 3, n).astype(np.int32)
    return x, v, sp


def _p(**kw):
    base = dict(box=BOX, rc=1.0, a=25.0, gamma=4.5, kT=1.0, power=0.5, dt=0.01, seed=7)
    base.update(kw)
    return oracle.DPDParams(**base)


def test_uniform_matrix_equals_single_species():
    x, v, sp = _system()
    F1, _, n1 = oracle.forces(_p(), x, v, 5)
    A = np.full((3, 3), 25.0)
    G = np.full((3, 3), 4.5)
    F3, _, n3 = oracle.forces(_p(amat=A, gmat=G, species=sp), x, v, 5)
    assert n1 == n3
    assert np.array_equal(F1, F3)


def test_hand_pair_uses_the_cross_entry():
    # r = 0.5, a = 10 -> |F^C| = a w = 5 along e_ij; the diagonal entries are decoys
    x = np.array([[1.0, 1.0, 1.0], [1.5, 1.0, 1.0]])
    v = np.zeros((2, 3))
    A = np.array([[99.0, 10.0], [10.0, 77.0]])
    G = np.zeros((2, 2))
    F, _, npairs = oracle.forces(_p(kT=0.0, amat=A, gmat=G, species=np.array([0, 1], np.int32)), x, v, 0)
    assert npairs == 1
    assert np.allclose(F[0], [-5.0, 0.0, 0.0], atol=1e-12)
    assert np.allclose(F[1], [5.0, 0.0, 0.0], atol=1e-12)
    # same pair, both species 1: the (1, 1) entry applies
    F, _, _ = oracle.forces(_p(kT=0.0, amat=A, gmat=G, species=np.array([1, 1], np.int32)), x, v, 0)
    assert np.allclose(F[0], [-38.5, 0.0, 0.0], atol=1e-12)


def test_zero_cross_entries_decouple_species():
    x, v, sp = _system(n=300, seed=9)
    sp = (sp > 0).astype(np.int32)  # two species
    A = np.array([[25.0, 0.0], [0.0, 40.0]])
    G = np.array([[4.5, 0.0], [0.0, 9.0]])
    ids = np.arange(len(x), dtype=np.uint32)
    F, _, _ = oracle.forces(_p(amat=A, gmat=G, species=sp), x, v, 3, ids=ids)
    for s, (a, g) in enumerate([(25.0, 4.5), (40.0, 9.0)]):
        m = sp == s
        Fs, _, _ = oracle.forces(_p(a=a, gamma=g), x[m], v[m], 3, ids=ids[m])
        assert np.allclose(F[m], Fs, rtol=0, atol=1e-9)


@pytest.mark.parametrize("mode", ["conservative_only", "viscous_only"])
def test_membrane_style_cross_terms(mode):
    # across the membrane only F^C; fluid-membrane pairs only F^D + F^R.  With
    # every particle of species 0 except one of species 1, the cross pairs of particle k
    # must equal the single-species run with the corresponding term switched off.
    x, v, _ = _system(n=250, seed=5)
    k = 17
    sp = np.zeros(len(x), np.int32)
    sp[k] = 1
    if mode == "conservative_only":
        A = np.array([[25.0, 25.0], [25.0, 25.0]])
        G = np.array([[4.5, 0.0], [0.0, 4.5]])
        ref = _p(gamma=0.0)
    else:
        A = np.array([[25.0, 0.0], [0.0, 25.0]])
        G = np.array([[4.5, 4.5], [4.5, 4.5]])
        ref = _p(a=0.0)
    F, _, _ = oracle.forces(_p(amat=A, gmat=G, species=sp), x, v, 11)
    Fr, _, _ = oracle.forces(ref, x, v, 11)
    assert np.allclose(F[k], Fr[k], rtol=1e-12, atol=1e-12)


def test_symmetric_matrix_newton3():
    x, v, sp = _system(n=350, seed=21)
    rng = np.random.default_rng(2)
    M = rng.random((3, 3)) * 30
    A = (M + M.T) / 2
    N = rng.random((3, 3)) * 8
    G = (N + N.T) / 2
    F, _, _ = oracle.forces(_p(amat=A, gmat=G, species=sp), x, v, 2)
    assert np.abs(F.sum(0)).max() < 1e-10 * np.abs(F).sum()
    # pair antisymmetry: the two-particle system swapped
    i, j = 0, 1
    x2 = np.array([[1.0, 1.0, 1.0], [1.4, 1.3, 0.8]])
    v2 = rng.normal(size=(2, 3))
    s2 = np.array([2, 0], np.int32)
    Fa, _, _ = oracle.forces(_p(amat=A, gmat=G, species=s2), x2, v2, 4, ids=np.array([5, 9], np.uint32))
    Fb, _, _ = oracle.forces(_p(amat=A, gmat=G, species=s2[::-1].copy()), x2[::-1].copy(), v2[::-1].copy(), 4,
                             ids=np.array([9, 5], np.uint32))
    assert np.allclose(Fa[i], Fb[j], atol=1e-12) and np.allclose(Fa[j], Fb[i], atol=1e-12)
    assert np.allclose(Fa[0], -Fa[1], atol=1e-12)
